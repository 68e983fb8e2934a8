"""Kernel times of one LAUD-R101 stage-3 block with the masker fused into a dense
conv1 (torch.profiler kernel durations; env LAUD_PAIR / LAUD_DBG apply).
usage: python tools/conv1_fused_probe.py [STAGE] [BATCH]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import collections
import torch
from paper_2308_15949_b200 import device as D
from paper_2308_15949_b200.network import make_params
stage = int(sys.argv[1]) if len(sys.argv) > 1 else 3
n = int(sys.argv[2]) if len(sys.argv) > 2 else 256
s = (4, 2, 2, 1)[stage - 1]
bp = [b for b in make_params("resnet101", 0)["blocks"] if b["stage"] == stage and b["index"] == 1][0]
blk = bp["block"]
ep = D.Epilogue(s1=bp["s1"], b1=bp["b1"], relu1=True, s2=bp["s2"], b2=bp["b2"], relu2=True,
                s3=bp["s3"], b3=bp["b3"], relu_out=True)
db = D.DeviceBlock(blk, bp["w1"], bp["w2"], bp["w3"], None, ep, masker_w=bp["masker_w"], masker_bias=0.0)
h = blk.input_shape.height
x = torch.randn(n, h, h, db.cin_p, device="cuda").relu_().bfloat16()
ws = D.Workspace()
for _ in range(3):
    db.forward(x.clone(), "spatial", s, ws=ws, conv1_dense=True)
torch.cuda.synchronize()
xs = [x.clone() for _ in range(5)]
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    for xi in xs:
        db.forward(xi, "spatial", s, ws=ws, conv1_dense=True)
    torch.cuda.synchronize()
tot = collections.defaultdict(list)
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA and "laud" in e.name:
        tot[e.name].append(e.device_time)
print(os.environ.get("LAUD_PAIR"), os.environ.get("LAUD_DBG"),
      {k.split("(")[0][-40:]: round(sum(v) / len(v), 1) for k, v in tot.items()})
