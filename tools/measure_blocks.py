"""Measure LAUD block latencies on the B200 for the predictor recalibration.

usage: python tools/measure_blocks.py OUT.json [--quick]

For ResNet-50/101 stage blocks (first = strided/downsample, template = index 1),
paradigms static / spatial (S from the stage's granularities) / channel (G=1) /
layer, activation ratios and batch sizes: exact-count masks, the block's
device forward replayed as a CUDA graph, L2 flushed (256 MiB) before each
replay, median of REPS CUDA-event timings.  Rows carry what the reference
predictor needs (`latency.predict_block(block, cfg, profile, flags, hw, batch)`)
plus the measured r_dil of spatial masks.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2308_15949_b200 import device as D  # noqa: E402
from paper_2308_15949_b200.network import make_params  # noqa: E402

REPS = 15


def timed(fn, flush):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(2):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    ts = []
    for _ in range(REPS):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    del g
    return float(np.median(ts))


def main():
    out = sys.argv[1]
    quick = "--quick" in sys.argv
    torch.cuda.set_device(0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    rng = np.random.default_rng(0)
    rows = []
    archs = ("resnet101",) if quick else ("resnet50", "resnet101")
    batches = (1, 64) if quick else (1, 16, 64, 256)
    ratios = (0.5,) if quick else (0.25, 0.5, 0.75)
    for arch in archs:
        params = make_params(arch, 0)
        seen = set()
        for bp in params["blocks"]:
            key = (bp["stage"], bp["index"] == 0)
            if bp["index"] > 1 or key in seen:
                continue
            seen.add(key)
            blk = bp["block"]
            ep = D.Epilogue(s1=bp["s1"], b1=bp["b1"], relu1=True, s2=bp["s2"], b2=bp["b2"], relu2=True,
                            s3=bp["s3"], b3=bp["b3"], sd=bp["sd"], bd=bp["bd"], relu_out=True)
            db = D.DeviceBlock(blk, bp["w1"], bp["w2"], bp["w3"], bp["wd"], ep, fold_scale=True)
            ws = D.Workspace()
            h = blk.input_shape.height
            o = blk.output_shape
            s_opts = [s for s in (1, 2, 4, 7) if o.height % s == 0 and s <= o.height]
            for n in batches:
                x = torch.randn(n, h, h, db.cin_p, device="cuda").relu_().bfloat16()
                base = dict(arch=arch, stage=bp["stage"], index=bp["index"], batch=n)

                def add(paradigm, us, **kw):
                    rows.append(dict(base, paradigm=paradigm, us=round(us, 2), **kw))

                # in-place residual for identity-skip blocks, as in the network executor
                out_t = (x if not blk.has_downsample else
                         torch.empty(n, o.height, o.width, db.cout_p, dtype=torch.bfloat16, device="cuda"))
                add("static", timed(lambda: db.forward(x, "static", out=out_t, ws=ws, latency_split=True), flush),
                    r=1.0)
                for s in s_opts:
                    cells = (o.height // s) * (o.width // s)
                    for r in ratios:
                        k = int(round(r * cells))
                        cz = np.zeros((n, cells), np.uint8)
                        for i in range(n):
                            cz[i, rng.permutation(cells)[:k]] = 1
                        coarse = torch.from_numpy(cz.reshape(-1)).cuda()
                        for dense1 in ((False, True) if s <= 2 else (False,)):
                            # latency_split as the network executor runs it (laud.h)
                            us = timed(lambda: db.forward(x, "spatial", s, coarse=coarse, out=out_t, ws=ws,
                                                          conv1_dense=dense1, latency_split=True), flush)
                            add("spatial", us, S=s, r=k / cells, conv1_dense=dense1)
                cm = blk.conv2.out_channels
                for r in ratios:
                    k = int(round(r * cm))
                    mm = np.zeros((n, db.cmid_p), np.uint8)
                    for i in range(n):
                        mm[i, rng.permutation(cm)[:k]] = 1
                    chm = torch.from_numpy(mm.reshape(-1)).cuda()
                    add("channel", timed(lambda: db.forward(x, "channel", out=out_t, ws=ws, chmask=chm), flush),
                        G=1, r=k / cm)
                    kl = int(round(r * n))
                    d = np.zeros(n, np.uint8)
                    d[rng.permutation(n)[:kl]] = 1
                    lm = torch.from_numpy(d).cuda()
                    if n > 1 or kl in (0, 1):
                        add("layer", timed(lambda: db.forward(x, "layer", coarse=lm, out=out_t, ws=ws,
                                                              latency_split=True), flush),
                            r=kl / n)
                print(arch, bp["stage"], bp["index"], n, len(rows), flush=True)
    with open(out, "w") as f:
        json.dump({"device": torch.cuda.get_device_name(0), "reps": REPS,
                   "l2_policy": "256 MiB flush before every replay", "rows": rows}, f, indent=0)


if __name__ == "__main__":
    main()
