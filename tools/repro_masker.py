import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2308_15949_b200 import reference as R
a = np.load("tests/golden/maskers.npz")
x, w, s = a["sp0_x"], a["sp0_w"], int(a["sp0_s"])
print(x.shape, s, flush=True)
m = R.spatial_masker_forward(x, w, s)
print("ok", m.coarse.sum(), a["sp0_coarse"].sum(), flush=True)
