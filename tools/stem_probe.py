"""Time the fused stem (laud_stem_pool) alone: CUDA events, L2 flushed per rep.

usage: python tools/stem_probe.py [batch]
Prints one JSON line: us per launch, image+output GB/s, conv TFLOP/s.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2308_15949_b200 import _lib  # noqa: E402
from paper_2308_15949_b200 import device as D  # noqa: E402
from paper_2308_15949_b200.network import IMAGENET_MEAN, IMAGENET_STD  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    img = torch.randint(0, 256, (n, 224, 224, 3), dtype=torch.uint8, device="cuda")
    wf = (torch.randn(64, 256, device="cuda") * 0.1).to(torch.bfloat16).contiguous()
    b = torch.randn(64, device="cuda") * 0.1
    mean = torch.tensor(IMAGENET_MEAN, dtype=torch.float32, device="cuda")
    inv = torch.tensor([1.0 / s for s in IMAGENET_STD], dtype=torch.float32, device="cuda")
    out = torch.empty(n, 56, 56, 64, dtype=torch.bfloat16, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    sh = D.stream_handle()
    stream = torch.cuda.current_stream()

    def run():
        _lib.call("laud_stem_pool", D.ptr(img), n, 224, 224, D.ptr(mean), D.ptr(inv), D.ptr(wf), D.ptr(b),
                  D.ptr(out), sh)

    for _ in range(3):
        run()
    ts = []
    for _ in range(20):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        run()
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    us = ts[len(ts) // 2]
    byts = img.numel() + out.numel() * 2
    flops = 2.0 * n * 112 * 112 * 64 * 147
    print(json.dumps({"kernel": "stem_pool_kernel", "batch": n, "us": round(us, 1),
                      "gbs": round(byts / us / 1e3, 1), "tflops": round(flops / us / 1e6, 1)}))


if __name__ == "__main__":
    main()
