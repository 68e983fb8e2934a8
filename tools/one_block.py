"""Run one LAUD-R101 template block (spatial, exact-count mask) for ncu captures.
usage: python tools/one_block.py STAGE [RATIO] [BATCH] [REPS]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2308_15949_b200 import device as D
from paper_2308_15949_b200.network import make_params
stage = int(sys.argv[1]); r = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
n = int(sys.argv[3]) if len(sys.argv) > 3 else 256; reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
plan = (4, 2, 2, 1)
bp = [b for b in make_params("resnet101", 0)["blocks"] if b["stage"] == stage and b["index"] == 1][0]
blk = bp["block"]; s = plan[stage - 1]
ep = D.Epilogue(s1=bp["s1"], b1=bp["b1"], relu1=True, s2=bp["s2"], b2=bp["b2"], relu2=True,
                s3=bp["s3"], b3=bp["b3"], relu_out=True)
db = D.DeviceBlock(blk, bp["w1"], bp["w2"], bp["w3"], None, ep)
h = blk.input_shape.height; o = blk.output_shape; cells = (o.height // s) * (o.width // s)
rng = np.random.default_rng(0)
cz = np.zeros((n, cells), np.uint8)
for i in range(n):
    cz[i, rng.permutation(cells)[: int(round(r * cells))]] = 1
coarse = torch.from_numpy(cz.reshape(-1)).cuda()
x = torch.randn(n, h, h, db.cin_p, device="cuda").relu_().bfloat16()
ws = D.Workspace()
for _ in range(reps):
    db.forward(x, "spatial", s, coarse=coarse, out=x, ws=ws)
torch.cuda.synchronize()
print("done", stage, r, n)
