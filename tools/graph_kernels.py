"""Per-kernel device time of one network forward replayed as a CUDA graph
(torch.profiler / CUPTI kernel records), aggregated by kernel name.

usage: LAUD_PDL=0 python tools/graph_kernels.py [arch] [paradigm] [batch] [plan]
(with PDL on, a kernel's record starts at its early launch and includes its
griddepcontrol.wait, so run with LAUD_PDL=0 for clean per-kernel times.)"""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2308_15949_b200.network import LaudNetwork  # noqa: E402

arch = sys.argv[1] if len(sys.argv) > 1 else "resnet101"
para = sys.argv[2] if len(sys.argv) > 2 else "spatial"
n = int(sys.argv[3]) if len(sys.argv) > 3 else 256
plan = sys.argv[4] if len(sys.argv) > 4 else ("4-4-2-1" if arch.startswith("regnet") else "4-2-2-1")
net = LaudNetwork(arch, para, plan, 0.5, seed=0)
if para != "static":
    net.calibrate(torch.from_numpy(bench.image_range(100, 164)).cuda())
img = torch.from_numpy(bench.image_range(0, n)).cuda()
g, _ = bench.capture(torch, lambda: net.forward(img), 2)
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    g.replay()
    torch.cuda.synchronize()
agg = collections.defaultdict(lambda: [0, 0.0])
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CUDA and ev.device_time_total > 0:
        name = ev.name.split("(")[0][:80]
        agg[name][0] += 1
        agg[name][1] += ev.device_time_total
tot = sum(v[1] for v in agg.values())
print(f"# {arch} {para} batch {n}: {tot / 1e3:.3f} ms of kernel time in one graph replay")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:30]:
    print(f"{v[1]:10.1f} us {100 * v[1] / tot:5.1f}% {v[0]:4d}  {k}")
