"""Pipeline timeline of CTA 0 of one conv-engine launch (laud_debug_set_trace).

usage: python tools/engine_trace.py SHAPE   (SHAPE from tools/engine_probe.py)
Prints per-k-block: producer-A issue (empty done), B issue, MMA start (full
done) relative to kernel start, and per tile the epilogue window.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import engine_probe as EP  # noqa: E402
from paper_2308_15949_b200 import _lib  # noqa: E402

TRACE_MMA, TRACE_B, TRACE_A, TRACE_EPI, SLOTS = 0, 4096, 8192, 12288, 16384


def main():
    torch.cuda.set_device(0)
    name = sys.argv[1]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    buf = torch.zeros(SLOTS, dtype=torch.int64, device="cuda")
    lib = _lib.lib()
    spec = EP.shape_defs()[name]
    EP.run(name, spec, flush, reps=2)  # warm
    lib.laud_debug_set_trace(buf.data_ptr())
    print(EP.run(name, spec, flush, reps=1))
    lib.laud_debug_set_trace(None)
    t = buf.cpu().numpy().astype(np.int64)
    nz = t[t > 0]
    t0 = nz.min()
    mma = t[TRACE_MMA:TRACE_MMA + 4096]
    a = t[TRACE_A:TRACE_A + 4096]
    b = t[TRACE_B:TRACE_B + 4096]
    epi = t[TRACE_EPI:TRACE_EPI + 4096].reshape(-1, 4)
    n = int((mma > 0).sum())
    print(f"k-blocks in CTA0: {n}, kernel span seen {(nz.max() - t0) / 1e3:.2f} us")
    d = np.diff(mma[:n])
    print(f"MMA cadence ns: median {np.median(d):.0f} p10 {np.percentile(d, 10):.0f} "
          f"p90 {np.percentile(d, 90):.0f} max {d.max():.0f}")
    lat = mma[:n] - np.maximum(a[:n], b[:n])
    print(f"issue->MMA-ready latency ns: median {np.median(lat):.0f} p90 {np.percentile(lat, 90):.0f}")
    print("first 12 kb (us from start): A-issue / B-issue / MMA-ready")
    for i in range(min(int(os.environ.get("KB", 12)), n)):
        print(f"  kb{i:3d}  {(a[i] - t0) / 1e3:8.2f} {(b[i] - t0) / 1e3:8.2f} {(mma[i] - t0) / 1e3:8.2f}")
    ne = int((epi[:, 0] > 0).sum())
    for i in range(min(ne, 12)):
        print(f"  tile{i:3d} epi acc_full {(epi[i, 0] - t0) / 1e3:8.2f}  tmem->smem {(epi[i, 1] - epi[i, 0]) / 1e3:6.2f}"
              f"  stores {(epi[i, 2] - epi[i, 1]) / 1e3:6.2f} us")


if __name__ == "__main__":
    main()
