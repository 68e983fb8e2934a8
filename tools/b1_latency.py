"""Batch-1 whole-network latency (CUDA graph, L2 flushed per replay, median of
N): LAUD (masker biases calibrated on held-out images) vs the in-house static
net.  usage: python tools/b1_latency.py [arch] [paradigm] [plan]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2308_15949_b200.network import LaudNetwork  # noqa: E402

arch = sys.argv[1] if len(sys.argv) > 1 else "resnet101"
para = sys.argv[2] if len(sys.argv) > 2 else "spatial"
plan = sys.argv[3] if len(sys.argv) > 3 else "4-2-2-1"
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
img = torch.from_numpy(bench.image_range(0, 1)).cuda()
res = {}
for name, p in (("laud", para), ("static_inhouse", "static")):
    net = LaudNetwork(arch, p, plan, 0.5, seed=0)
    if p != "static":
        net.calibrate(torch.from_numpy(bench.image_range(100, 132)).cuda())
    g, _ = bench.capture(torch, lambda: net.forward(img), 2)
    _, per = bench.timed_graph(torch, g, 30, flush, torch.cuda.current_stream())
    res[name] = round(float(np.median(per)), 4)
    del g, net
print(json.dumps({"arch": arch, "paradigm": para, "plan": plan, "batch1_ms": res,
                  "env": {k: v for k, v in os.environ.items() if k.startswith("LAUD_")}}))
