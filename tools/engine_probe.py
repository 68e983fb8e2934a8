"""Time the conv engine on isolated shapes (CUDA events, L2 flushed per rep).

usage: python tools/engine_probe.py [name ...]   (env LAUD_BN / LAUD_A_TMA apply)
Prints one JSON line per shape: us, TFLOP/s, compulsory GB/s.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2308_15949_b200 import channel as CH  # noqa: E402


def bf(*shape):
    return (torch.randn(*shape, device="cuda") * 0.5).bfloat16()


def shape_defs():
    d = {}
    # name: (rows/batch geometry, ...) -> dict of conv kwargs and alg flops/bytes
    d["gemm_s3"] = dict(kind="gemm", m=148 * 128 * 2, n=256, k=2304)
    d["gemm_s3_1w"] = dict(kind="gemm", m=148 * 128, n=256, k=2304)
    d["gemm_k256_n1024"] = dict(kind="gemm", m=25088, n=1024, k=256)
    d["gemm_k1024_n256"] = dict(kind="gemm", m=50176, n=256, k=1024)
    d["tiny"] = dict(kind="gemm", m=128, n=256, k=64)
    d["one_wave_k256"] = dict(kind="gemm", m=148 * 128, n=256, k=256)
    d["two_wave_k256"] = dict(kind="gemm", m=2 * 148 * 128, n=256, k=256)
    d["four_wave_k256"] = dict(kind="gemm", m=4 * 148 * 128, n=256, k=256)
    d["conv2_s3"] = dict(kind="conv3x3", n=256, h=14, c=256)
    d["conv2_s3_b1"] = dict(kind="conv3x3", n=1, h=14, c=256)   # batch-1 latency shapes
    d["conv1_s3_b1"] = dict(kind="gemm", m=196, n=256, k=1024)
    d["conv2_s3_r05"] = dict(kind="conv3x3", n=128, h=14, c=256)  # 25088 rows = stage-3 conv2 at r=0.5
    d["conv2_s2"] = dict(kind="conv3x3", n=256, h=28, c=128)
    d["conv2_s1"] = dict(kind="conv3x3", n=256, h=56, c=64)
    d["conv1_s1"] = dict(kind="gemm", m=256 * 56 * 56, n=64, k=256)
    d["conv3_s3"] = dict(kind="conv3", m=25088, n=1024, k=256)
    # patch conv2 over active S x S cells at r = 0.5 (the LAUD schedule's conv2)
    d["pconv_s3"] = dict(kind="patch", n=256, h=14, c=256, s=2)
    d["pconv_s2"] = dict(kind="patch", n=256, h=28, c=128, s=2)
    d["pconv_s1"] = dict(kind="patch", n=256, h=56, c=64, s=4)
    d["pconv_s3_b1"] = dict(kind="patch", n=1, h=14, c=256, s=2)
    # every cell active: the halo kernel as a dense 3x3 conv (vs conv2_s1 / conv2_s2 / conv2_s3)
    d["pconv_s1_all"] = dict(kind="patch", n=256, h=56, c=64, s=4, density=1.0)
    d["pconv_s1_all_s2"] = dict(kind="patch", n=256, h=56, c=64, s=2, density=1.0)
    d["pconv_s2_all"] = dict(kind="patch", n=256, h=28, c=128, s=2, density=1.0)
    d["pconv_s2_all_s4"] = dict(kind="patch", n=256, h=28, c=128, s=4, density=1.0)
    d["pconv_s3_all"] = dict(kind="patch", n=256, h=14, c=256, s=2, density=1.0)
    d["conv3_s1"] = dict(kind="conv3", m=256 * 56 * 56 // 2, n=256, k=64)
    # stage-1 b0 downsample (64 -> 256 over every pixel): a pure output stream
    d["ds_s1"] = dict(kind="gemm", m=256 * 56 * 56, n=256, k=64)
    # RegNetY-1.6GF at batch 1024: the 112x112 stage-1 b0 conv1 (32 -> 48) and a
    # stage-3 1x1 (336 -> 336) — small-K / small-N streaming convs
    d["rg_s1_conv1"] = dict(kind="gemm", m=1024 * 112 * 112, n=48, k=32)
    d["rg_s3_1x1"] = dict(kind="gemm", m=1024 * 196, n=336, k=336)
    # channel skipping at batch 256, stage-3 geometry, k_n = 128 kept channels per sample:
    # conv2 with in-kernel gathered W2[sel] rows (g=1) / plain W2 tiles (g=0, same shape)
    d["chconv2_s3"] = dict(kind="chconv2", n=256, h=14, c=256, k=128, g=1)
    d["chconv2_s3_box"] = dict(kind="chconv2", n=256, h=14, c=256, k=128, g=0)
    d["chconv3_s3"] = dict(kind="chconv3", n=256, h=14, c=256, co=1024, k=128, g=2)
    return d


def run(name, spec, flush, reps=20):
    if spec["kind"] in ("gemm", "conv3"):
        m, n, k = spec["m"], spec["n"], spec["k"]
        a = bf(m, k)
        w = bf(n, 1, k)
        out = torch.empty(m, n, dtype=torch.bfloat16, device="cuda")
        resid = out if spec["kind"] == "conv3" else None
        if resid is not None:
            out.copy_(bf(m, n))
        kw = dict(act=a, in_hw=(m, 1), in_c=k, in_ld=k, weight=w, n_out=n, out=out, out_ld=n,
                  out_hw=(m, 1), batch=1, a_compact=1, resid=resid, resid_ld=n if resid is not None else 0,
                  relu=1)
        flops = 2.0 * m * n * k
        nbytes = 2.0 * (m * k + n * k + m * n * (2 if resid is not None else 1))
    elif spec["kind"] == "patch":
        import numpy as np
        b, h, c, s = spec["n"], spec["h"], spec["c"], spec["s"]
        a = bf(b, h, h, c)
        w = bf(c, 9, c)
        hc = h // s
        keep = int(round(spec.get("density", 0.5) * b * hc * hc))
        cells = np.sort(np.random.default_rng(0).permutation(b * hc * hc)[:keep]).astype(np.int32)
        lst = torch.from_numpy(cells).cuda()
        cnt = torch.tensor([len(cells)], dtype=torch.int32, device="cuda")
        m = len(cells) * s * s
        out = torch.empty(m, c, dtype=torch.bfloat16, device="cuda")
        kw = dict(act=a, in_hw=(h, h), in_c=c, in_ld=c, weight=w, n_out=c, out=out, out_ld=c,
                  out_hw=(h, h), batch=b, ksize=3, pad=1, relu=1, out_mode=CH.OUT_ROW, row_mode=CH.ROWS_PATCH,
                  rows_max=b * h * h, lst=lst, count=cnt, patch=(s, s), cells=(hc, hc))
        flops = 2.0 * m * c * 9 * c
        nbytes = 2.0 * (b * h * h * c + m * c + 9 * c * c)
    elif spec["kind"] in ("chconv2", "chconv3"):
        import numpy as np
        b, h, c, kk = spec["n"], spec["h"], spec["c"], spec["k"]
        sr = (h * h + 127) // 128 * 128
        sel = np.stack([np.sort(np.random.default_rng(i).permutation(c)[:kk]) for i in range(b)]).astype(np.int32)
        selp = np.zeros((b, c), np.int32)
        selp[:, :kk] = sel
        sel_t = torch.from_numpy(selp).cuda()
        cnt = torch.full((b,), kk, dtype=torch.int32, device="cuda")
        if spec["kind"] == "chconv2":
            a = bf(b, h, h, c)
            w = bf(c, 9, c)
            out = torch.empty(b * h * h, c, dtype=torch.bfloat16, device="cuda")
            ex = dict(sample_rows=sr, chan_count=cnt, n_dyn=1, col_index=sel_t, col_index_ld=c)
            if spec["g"]:
                ex.update(b_gather=1, b_index=sel_t, b_index_ld=c, b_rows=c)
            kw = dict(act=a, in_hw=(h, h), in_c=c, in_ld=c, weight=w, n_out=c, out=out, out_ld=c,
                      out_hw=(h, h), batch=b, ksize=3, pad=1, relu=1, out_mode=CH.OUT_ROW, rows_max=b * sr,
                      bias=torch.zeros(c, device="cuda"), **ex)
            flops = 2.0 * b * h * h * kk * 9 * c
            nbytes = 2.0 * (b * h * h * c + b * h * h * kk + 9 * c * c)
        else:
            co = spec["co"]
            a = bf(b * h * h, c)
            w = bf(c, co)
            out = bf(b, h, h, co)
            ex = dict(sample_rows=sr, chan_count=cnt, k_dyn=1, b_gather=2, b_index=sel_t, b_index_ld=c, b_rows=c)
            kw = dict(act=a, in_hw=(h, h), in_c=c, in_ld=c, weight=w, n_out=co, out=out, out_ld=co,
                      out_hw=(h, h), batch=b, a_compact=1, resid=out, resid_ld=co, rows_max=b * sr,
                      bias=torch.zeros(co, device="cuda"), **ex)
            flops = 2.0 * b * h * h * kk * co
            nbytes = 2.0 * (b * h * h * kk + 2 * b * h * h * co + c * co)
    else:
        b, h, c = spec["n"], spec["h"], spec["c"]
        a = bf(b, h, h, c)
        w = bf(c, 9, c)
        out = torch.empty(b * h * h, c, dtype=torch.bfloat16, device="cuda")
        kw = dict(act=a, in_hw=(h, h), in_c=c, in_ld=c, weight=w, n_out=c, out=out, out_ld=c,
                  out_hw=(h, h), batch=b, ksize=3, pad=1, relu=1, out_mode=CH.OUT_ROW)
        m = b * h * h
        flops = 2.0 * m * c * 9 * c
        nbytes = 2.0 * (m * c * 2 + 9 * c * c)
    conv_fn = locals().get("conv_fn", CH.conv)
    for _ in range(3):
        conv_fn(**kw)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        conv_fn(**kw)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    ms = ts[len(ts) // 2]
    return dict(name=name, us=round(ms * 1e3, 2), tflops=round(flops / ms / 1e9, 1),
                gbs=round(nbytes / ms / 1e6, 1), ideal_us_tensor=round(flops / 1.3841e15 * 1e6, 2),
                ideal_us_hbm=round(nbytes / 6.55e12 * 1e6, 2),
                env={k: os.environ.get(k) for k in ("LAUD_BN", "LAUD_A_TMA", "LAUD_CTA2", "LAUD_HALO") if os.environ.get(k)})


def main():
    torch.cuda.set_device(0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    defs = shape_defs()
    names = sys.argv[1:] or list(defs)
    for nm in names:
        print(json.dumps(run(nm, defs[nm], flush)), flush=True)


if __name__ == "__main__":
    main()
