import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2308_15949_b200.network import LaudNetwork, random_images
net = LaudNetwork("resnet101", "spatial", "4-2-2-1", 0.5, seed=0)
img = random_images(int(os.environ.get("NB", 256)), seed=1000)
b = net.calibrate(img)
st = net.rate_stats(img)
print(os.environ.get("LAUD_MASKER_IN_CONV1"), [round(r["r"], 3) for r in st])
