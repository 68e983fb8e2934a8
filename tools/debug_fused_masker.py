"""Fused conv1 masker vs standalone masker on one block (debug)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2308_15949_b200 import device as D, _lib
from paper_2308_15949_b200.network import make_params
stage, index = int(sys.argv[1]), int(sys.argv[2])
s = int(sys.argv[3]) if len(sys.argv) > 3 else 2
bp = [b for b in make_params("resnet101", 0)["blocks"] if b["stage"] == stage and b["index"] == index][0]
blk = bp["block"]
ep = D.Epilogue(s1=bp["s1"], b1=bp["b1"], relu1=True, s2=bp["s2"], b2=bp["b2"], relu2=True, s3=bp["s3"], b3=bp["b3"], sd=bp["sd"], bd=bp["bd"], relu_out=True)
db = D.DeviceBlock(blk, bp["w1"], bp["w2"], bp["w3"], bp["wd"], ep, masker_w=bp["masker_w"], fold_scale=True)
n, h = int(os.environ.get("NB", 8)), blk.input_shape.height
x = torch.randn(n, h, h, db.cin_p, device="cuda").relu_().bfloat16()
res = {}
for dense in (False, True):
    ws = D.Workspace()
    xx = x.clone()
    out, coarse, cells, counts = db.forward(xx, "spatial", s, ws=ws, conv1_dense=dense)
    torch.cuda.synchronize()
    o = blk.output_shape
    nc = n * (o.height // s) * (o.width // s)
    res[dense] = (coarse[:nc].cpu().numpy().copy(), ws.get("partial", 4).view(torch.float32)[:nc].cpu().numpy().copy())
c0, p0 = res[False]; c1, p1 = res[True]
print("cells", len(c0), "rate std", c0.mean(), "fused", c1.mean(), "agree", (c0 == c1).mean())
print("partial (fused sums) head", p1[:6])
