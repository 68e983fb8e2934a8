"""Conv engine (tcgen05 implicit GEMM) and compaction kernels vs PyTorch fp32.

GPU only.  The torch fp32 reference takes the same bf16-rounded inputs and
weights, so the only difference is fp32 accumulation order plus the final
bf16 rounding of the kernel output.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _engine():
    from paper_2308_15949_b200 import channel as CH
    from paper_2308_15949_b200 import device as D
    D.require_cuda()
    return CH, D


def _torch_conv_nhwc(x, w, stride, pad):
    """x (N,H,W,C) bf16, w (Co,Ci,k,k) fp32 -> (N,Ho,Wo,Co) fp32 reference."""
    y = torch.nn.functional.conv2d(x.float().permute(0, 3, 1, 2), w.float(), stride=stride, padding=pad)
    return y.permute(0, 2, 3, 1)


@pytest.mark.parametrize("cin,cout,k,stride,n,h", [
    (64, 64, 1, 1, 2, 8), (128, 256, 1, 1, 1, 16), (256, 512, 1, 2, 2, 14),
    (64, 64, 3, 1, 2, 8), (128, 128, 3, 2, 1, 16), (16, 8, 3, 1, 1, 9), (40, 24, 1, 1, 3, 5),
    (1024, 256, 1, 1, 1, 14), (256, 256, 3, 1, 4, 28),
])
def test_dense_conv_matches_torch(cin, cout, k, stride, n, h):
    CH, D = _engine()
    g = torch.Generator().manual_seed(cin * 7 + cout + k)
    x = torch.randn(n, h, h, cin, generator=g).cuda().to(torch.bfloat16)
    w = (torch.randn(cout, cin, k, k, generator=g) / np.sqrt(cin * k * k)).to(torch.bfloat16).float()
    wp = D.pack_weight(w, cin)
    ho = (h + 2 * (k // 2) - k) // stride + 1
    out = torch.empty(n, ho, ho, cout, dtype=torch.bfloat16, device="cuda")
    CH.conv(act=x, in_hw=(h, h), in_c=cin, in_ld=cin, weight=wp, n_out=cout, out=out, out_ld=cout,
            out_hw=(ho, ho), batch=n, ksize=k, stride=stride, pad=k // 2)
    ref = _torch_conv_nhwc(x, w.cuda(), stride, k // 2)
    err = (out.float() - ref).norm() / ref.norm()
    assert err < 6e-3, float(err)


def test_epilogue_scale_bias_relu_residual():
    CH, D = _engine()
    g = torch.Generator().manual_seed(3)
    n, h, cin, cout = 2, 12, 128, 256
    x = torch.randn(n, h, h, cin, generator=g).cuda().to(torch.bfloat16)
    w = (torch.randn(cout, cin, 1, 1, generator=g) / np.sqrt(cin)).to(torch.bfloat16).float()
    sc = torch.rand(cout, generator=g) + 0.5
    bi = torch.randn(cout, generator=g)
    res = torch.randn(n, h, h, cout, generator=g).cuda().to(torch.bfloat16)
    out = res.clone()
    CH.conv(act=x, in_hw=(h, h), in_c=cin, in_ld=cin, weight=D.pack_weight(w, cin), n_out=cout,
            out=out, out_ld=cout, out_hw=(h, h), batch=n, scale=sc.cuda(), bias=bi.cuda(), relu=1,
            resid=out, resid_ld=cout)
    ref = torch.relu(_torch_conv_nhwc(x, w.cuda(), 1, 0) * sc.cuda() + bi.cuda() + res.float())
    err = (out.float() - ref).norm() / ref.norm()
    assert err < 6e-3, float(err)


def test_patch_rows_gather_scatter():
    """Patch-list rows: 3x3 conv evaluated only on listed S x S patches."""
    CH, D = _engine()
    g = torch.Generator().manual_seed(5)
    n, h, c, s = 2, 16, 64, 4
    x = torch.randn(n, h, h, c, generator=g).cuda().to(torch.bfloat16)
    w = (torch.randn(c, c, 3, 3, generator=g) / np.sqrt(9 * c)).to(torch.bfloat16).float()
    cells = [1, 6, 17, 30]  # linear (n, i, j) cell ids on a 4x4 grid per image
    lst = torch.tensor(cells, dtype=torch.int32, device="cuda")
    cnt = torch.tensor([len(cells)], dtype=torch.int32, device="cuda")
    rows = torch.zeros(len(cells) * s * s, c, dtype=torch.bfloat16, device="cuda")
    CH.conv(act=x, in_hw=(h, h), in_c=c, in_ld=c, weight=D.pack_weight(w, c), n_out=c, out=rows,
            out_ld=c, out_hw=(h, h), batch=n, ksize=3, pad=1, row_mode=CH.ROWS_PATCH,
            rows_max=n * h * h, lst=lst, count=cnt, patch=(s, s), cells=(h // s, h // s),
            out_mode=CH.OUT_ROW)
    ref = _torch_conv_nhwc(x, w.cuda(), 1, 1)
    exp = []
    for cell in cells:
        ni, r = divmod(cell, 16)
        ci, cj = divmod(r, 4)
        exp.append(ref[ni, ci * s:(ci + 1) * s, cj * s:(cj + 1) * s].reshape(s * s, c))
    exp = torch.cat(exp)
    err = (rows.float() - exp).norm() / exp.norm()
    assert err < 6e-3, float(err)


@pytest.mark.parametrize("s,cin,cout,n,h,density", [
    (2, 256, 256, 8, 14, 0.5), (2, 128, 128, 4, 28, 0.5), (4, 64, 64, 4, 56, 0.5), (2, 64, 64, 3, 16, 0.3),
    (4, 128, 128, 2, 28, 0.7), (2, 256, 256, 64, 14, 0.5), (2, 40, 24, 2, 8, 1.0), (4, 64, 64, 1, 8, 0.0),
    (2, 256, 256, 1, 14, 0.5), (2, 512, 256, 2, 14, 0.6), (4, 256, 64, 1, 56, 0.5),
    (2, 256, 256, 256, 14, 0.5), (2, 256, 256, 300, 14, 0.7), (2, 128, 128, 200, 28, 0.5)])
@pytest.mark.parametrize("split", [0, 1])
def test_patch_conv_halo_smem(s, cin, cout, n, h, density, split):
    """3x3 patch conv over active S x S cells (the halo-in-shared-memory kernel for
    S = 2 / 4, stride 1): ragged patch counts (not a multiple of the tile's patch
    count), image-border cells (zero halo), several N tiles, scale/bias/ReLU; with
    latency_split the small grids split K over a cluster (DSMEM reduction) and large
    grids split the last partial wave's tiles over 2-CTA clusters (batch 200-300)."""
    CH, D = _engine()
    g = torch.Generator().manual_seed(s * 1000 + cin + n)
    x = torch.randn(n, h, h, cin, generator=g).cuda().to(torch.bfloat16)
    w = (torch.randn(cout, cin, 3, 3, generator=g) / np.sqrt(9 * cin)).to(torch.bfloat16).float()
    sc = torch.rand(cout, generator=g) + 0.5
    bi = torch.randn(cout, generator=g) * 0.1
    hc = h // s
    rng = np.random.default_rng(n + h)
    cells = np.flatnonzero(rng.random(n * hc * hc) < density).astype(np.int32)
    lst = torch.from_numpy(np.concatenate([cells, np.zeros(4, np.int32)])).cuda()
    cnt = torch.tensor([len(cells)], dtype=torch.int32, device="cuda")
    rows = torch.full((max(len(cells), 1) * s * s, cout), 7.0, dtype=torch.bfloat16, device="cuda")
    CH.conv(act=x, in_hw=(h, h), in_c=cin, in_ld=cin, weight=D.pack_weight(w, cin), n_out=cout, out=rows,
            out_ld=cout, out_hw=(h, h), batch=n, ksize=3, pad=1, row_mode=CH.ROWS_PATCH,
            rows_max=n * h * h, lst=lst, count=cnt, patch=(s, s), cells=(hc, hc),
            out_mode=CH.OUT_ROW, scale=sc.cuda(), bias=bi.cuda(), relu=1, latency_split=split)
    torch.cuda.synchronize()
    if len(cells) == 0:
        assert (rows.float() == 7.0).all()
        return
    ref = torch.relu(_torch_conv_nhwc(x, w.cuda(), 1, 1) * sc.cuda() + bi.cuda())
    idx = torch.from_numpy(cells.astype(np.int64))
    ni, r = idx // (hc * hc), idx % (hc * hc)
    ci, cj = r // hc, r % hc
    exp = torch.stack([ref[a, b * s:(b + 1) * s, c * s:(c + 1) * s].reshape(s * s, cout)
                       for a, b, c in zip(ni.tolist(), ci.tolist(), cj.tolist())]).reshape(-1, cout)
    err = (rows.float() - exp).norm() / exp.norm()
    assert err < 6e-3, float(err)


@pytest.mark.parametrize("kind,cin,cout,k,stride,n,h", [
    ("dense", 2048, 512, 1, 1, 1, 7), ("dense", 1024, 256, 1, 1, 1, 14), ("resid", 128, 512, 1, 1, 1, 7),
    ("dense", 256, 512, 3, 2, 1, 14), ("dense", 128, 128, 3, 2, 2, 28), ("pixels", 512, 512, 3, 1, 1, 7),
    ("pixels", 256, 256, 3, 1, 2, 14), ("dense", 64, 64, 3, 1, 1, 8)])
@pytest.mark.parametrize("split", [0, 1])
def test_engine_cluster_split_k(kind, cin, cout, k, stride, n, h, split):
    """Small-grid cluster split-K of the implicit-GEMM engine (latency_split, plain
    epilogues): the K slices' fp32 partials reduced over distributed shared memory
    then bias [+ residual] + ReLU — dense 1x1 / strided 3x3 rows and an active-pixel
    list (S = 1 patches, the stage-4 LAUD conv2), vs torch fp32; split and unsplit agree."""
    CH, D = _engine()
    g = torch.Generator().manual_seed(cin + cout + k + n + h)
    x = torch.randn(n, h, h, cin, generator=g).cuda().to(torch.bfloat16)
    w = (torch.randn(cout, cin, k, k, generator=g) / np.sqrt(k * k * cin)).to(torch.bfloat16).float()
    bi = torch.randn(cout, generator=g) * 0.1
    pad = k // 2
    ho = (h + 2 * pad - k) // stride + 1
    ref = _torch_conv_nhwc(x, w.cuda(), stride, pad) + bi.cuda()
    kw = dict(act=x, in_hw=(h, h), in_c=cin, in_ld=cin, weight=D.pack_weight(w, cin), n_out=cout, out_ld=cout,
              out_hw=(ho, ho), batch=n, ksize=k, stride=stride, pad=pad, bias=bi.cuda(), relu=1,
              latency_split=split)
    if kind == "pixels":
        rng = np.random.default_rng(h)
        pix = np.flatnonzero(rng.random(n * ho * ho) < 0.5).astype(np.int32)
        lst = torch.from_numpy(np.concatenate([pix, np.zeros(4, np.int32)])).cuda()
        cnt = torch.tensor([len(pix)], dtype=torch.int32, device="cuda")
        out = torch.full((len(pix), cout), 7.0, dtype=torch.bfloat16, device="cuda")
        CH.conv(out=out, row_mode=CH.ROWS_PATCH, rows_max=n * ho * ho, lst=lst, count=cnt, patch=(1, 1),
                cells=(ho, ho), out_mode=CH.OUT_ROW, **kw)
        exp = torch.relu(ref).reshape(-1, cout)[torch.from_numpy(pix.astype(np.int64)).cuda()]
    else:
        out = torch.empty(n, ho, ho, cout, dtype=torch.bfloat16, device="cuda")
        if kind == "resid":
            res = (torch.randn(n, ho, ho, cout, generator=g) * 0.5).cuda().to(torch.bfloat16)
            out.copy_(res)
            CH.conv(out=out, resid=out, resid_ld=cout, **kw)
            exp = torch.relu(ref + res.float())
        else:
            CH.conv(out=out, **kw)
            exp = torch.relu(ref)
    torch.cuda.synchronize()
    err = (out.float() - exp).norm() / exp.norm()
    assert err < 6e-3, float(err)


def test_compaction_matches_argwhere():
    from paper_2308_15949_b200 import reference as R
    rng = np.random.default_rng(0)
    for shape, p in [((3, 7, 7), 0.5), ((256, 14, 14), 0.3), ((1, 1, 1), 1.0), ((5, 3, 2), 0.0),
                     ((64, 56, 56), 0.5)]:
        coarse = rng.random(shape) < p
        plan = R.build_gather_plan(coarse)
        assert plan.indices == tuple(tuple(int(v) for v in r) for r in np.argwhere(coarse))
        assert plan.patch_count == int(coarse.sum())


@pytest.mark.parametrize("c,groups,s,n,h,density", [
    (48, 2, 4, 4, 56, 0.5), (120, 5, 4, 2, 28, 0.5), (336, 14, 2, 8, 14, 0.5), (336, 14, 2, 1, 14, 1.0),
    (120, 5, 2, 3, 28, 0.3)])
def test_grouped_patch_conv_halo(c, groups, s, n, h, density):
    """Grouped 3x3 conv (RegNet conv2, block-diagonal weights) over active S x S
    patches on the halo kernel: each N tile loads only the channel blocks of its
    groups; vs torch's grouped conv at the active cells."""
    CH, D = _engine()
    g = torch.Generator().manual_seed(c + groups + s)
    x = torch.randn(n, h, h, c, generator=g).cuda().to(torch.bfloat16)
    w = (torch.randn(c, c // groups, 3, 3, generator=g) / np.sqrt(9 * c // groups)).to(torch.bfloat16).float()
    hc = h // s
    rng = np.random.default_rng(n + h + c)
    cells = np.flatnonzero(rng.random(n * hc * hc) < density).astype(np.int32)
    lst = torch.from_numpy(np.concatenate([cells, np.zeros(4, np.int32)])).cuda()
    cnt = torch.tensor([len(cells)], dtype=torch.int32, device="cuda")
    rows = torch.empty((len(cells) * s * s, c), dtype=torch.bfloat16, device="cuda")
    CH.conv(act=x, in_hw=(h, h), in_c=c, in_ld=c, weight=D.pack_weight(w, c, groups=groups), n_out=c, out=rows,
            out_ld=c, out_hw=(h, h), batch=n, ksize=3, pad=1, row_mode=CH.ROWS_PATCH, rows_max=n * h * h,
            lst=lst, count=cnt, patch=(s, s), cells=(hc, hc), out_mode=CH.OUT_ROW, groups=groups)
    torch.cuda.synchronize()
    ref = torch.nn.functional.conv2d(x.float().permute(0, 3, 1, 2), w.cuda(), padding=1,
                                     groups=groups).permute(0, 2, 3, 1)
    idx = torch.from_numpy(cells.astype(np.int64))
    ni, r = idx // (hc * hc), idx % (hc * hc)
    ci, cj = r // hc, r % hc
    exp = torch.stack([ref[a, b * s:(b + 1) * s, q * s:(q + 1) * s].reshape(s * s, c)
                       for a, b, q in zip(ni.tolist(), ci.tolist(), cj.tolist())]).reshape(-1, c)
    err = (rows.float() - exp).norm() / exp.norm()
    assert err < 6e-3, float(err)


@pytest.mark.parametrize("c,groups,stride,n,h", [
    (48, 2, 1, 2, 8), (120, 5, 2, 2, 14), (336, 14, 1, 1, 14), (888, 37, 2, 1, 14), (64, 8, 1, 2, 9)])
def test_grouped_conv_matches_torch(c, groups, stride, n, h):
    """Block-diagonal grouped 3x3 conv (RegNet conv2): per-tile K windows."""
    CH, D = _engine()
    g = torch.Generator().manual_seed(c + groups)
    x = torch.randn(n, h, h, c, generator=g).cuda().to(torch.bfloat16)
    w = (torch.randn(c, c // groups, 3, 3, generator=g) / np.sqrt(9 * c // groups)).to(torch.bfloat16).float()
    wp = D.pack_weight(w, c, groups=groups)
    ho = (h + 2 - 3) // stride + 1
    out = torch.empty(n, ho, ho, c, dtype=torch.bfloat16, device="cuda")
    CH.conv(act=x, in_hw=(h, h), in_c=c, in_ld=c, weight=wp, n_out=c, out=out, out_ld=c,
            out_hw=(ho, ho), batch=n, ksize=3, stride=stride, pad=1, groups=groups)
    ref = torch.nn.functional.conv2d(x.float().permute(0, 3, 1, 2), w.cuda(), stride=stride, padding=1,
                                     groups=groups).permute(0, 2, 3, 1)
    err = (out.float() - ref).norm() / ref.norm()
    assert err < 6e-3, float(err)


@pytest.mark.parametrize("cin,cout,k,stride,n,h", [
    (256, 1024, 1, 1, 128, 14), (256, 256, 3, 1, 128, 14), (512, 1024, 1, 2, 64, 28), (128, 512, 1, 1, 32, 28)])
def test_cta_pair_tiles_match_torch(cin, cout, k, stride, n, h):
    """Shapes large enough for the cta_group::2 (M = 256 pair) tiles."""
    CH, D = _engine()
    g = torch.Generator().manual_seed(cin + cout + k + n)
    x = torch.randn(n, h, h, cin, generator=g).cuda().to(torch.bfloat16)
    w = (torch.randn(cout, cin, k, k, generator=g) / np.sqrt(cin * k * k)).to(torch.bfloat16).float()
    b = torch.randn(cout, generator=g).cuda()
    ho = (h + 2 * (k // 2) - k) // stride + 1
    res = torch.randn(n, ho, ho, cout, generator=g).cuda().to(torch.bfloat16)
    out = res.clone()
    CH.conv(act=x, in_hw=(h, h), in_c=cin, in_ld=cin, weight=D.pack_weight(w, cin), n_out=cout, out=out,
            out_ld=cout, out_hw=(ho, ho), batch=n, ksize=k, stride=stride, pad=k // 2, bias=b, relu=1,
            resid=out, resid_ld=cout)
    ref = torch.relu(_torch_conv_nhwc(x, w.cuda(), stride, k // 2) + b + res.float())
    err = (out.float() - ref).norm() / ref.norm()
    assert err < 6e-3, float(err)


def test_cta_pair_patch_rows_scatter():
    """Pair tiles over an active-patch list (S = 2) with scatter-add into the residual."""
    CH, D = _engine()
    g = torch.Generator().manual_seed(11)
    n, h, c, co, s = 128, 14, 256, 1024, 2
    cells_per = (h // s) ** 2
    rng = np.random.default_rng(0)
    cz = rng.random(n * cells_per) < 0.6
    cells = np.flatnonzero(cz).astype(np.int32)
    lst = torch.from_numpy(cells).cuda()
    cnt = torch.tensor([len(cells)], dtype=torch.int32, device="cuda")
    rows = torch.randn(len(cells) * s * s, c, generator=g).cuda().to(torch.bfloat16)
    w = (torch.randn(co, c, 1, 1, generator=g) / np.sqrt(c)).to(torch.bfloat16).float()
    base = torch.randn(n, h, h, co, generator=g).cuda().to(torch.bfloat16)
    out = base.clone()
    CH.conv(act=rows, in_hw=(h, h), in_c=c, in_ld=c, weight=D.pack_weight(w, c), n_out=co, out=out,
            out_ld=co, out_hw=(h, h), batch=n, a_compact=1, row_mode=CH.ROWS_PATCH, rows_max=n * h * h,
            lst=lst, count=cnt, patch=(s, s), cells=(h // s, h // s), resid=out, resid_ld=co)
    y = rows.float() @ w.cuda().reshape(co, c).t()
    exp = base.float().clone()
    for pi, cell in enumerate(cells.tolist()):
        ni, r = divmod(cell, cells_per)
        ci, cj = divmod(r, h // s)
        blk = y[pi * s * s:(pi + 1) * s * s].reshape(s, s, co)
        exp[ni, ci * s:(ci + 1) * s, cj * s:(cj + 1) * s] += blk
    err = (out.float() - exp).norm() / exp.norm()
    assert err < 6e-3, float(err)
    untouched = ~torch.from_numpy(np.repeat(np.repeat(cz.reshape(n, h // s, h // s), s, 1), s, 2)).cuda()
    assert torch.equal(out[untouched], base[untouched])


@pytest.mark.parametrize("n,h,c", [(2, 112, 64), (3, 15, 24), (1, 7, 8)])
def test_maxpool3s2_matches_torch(n, h, c):
    """Network glue: 3x3 / stride 2 / pad 1 max-pool (packed bf16 max) bit-exact vs torch."""
    from paper_2308_15949_b200 import _lib
    from paper_2308_15949_b200 import device as D
    D.require_cuda()
    x = torch.randn(n, h, h, c, device="cuda").bfloat16()
    ho = (h - 1) // 2 + 1
    y = torch.empty(n, ho, ho, c, device="cuda", dtype=torch.bfloat16)
    _lib.call("laud_maxpool3s2", D.ptr(x), n, h, h, c, D.ptr(y), None)
    torch.cuda.synchronize()
    ref = torch.nn.functional.max_pool2d(x.permute(0, 3, 1, 2).float(), 3, 2, 1).permute(0, 2, 3, 1)
    assert torch.equal(y.float(), ref)


@pytest.mark.parametrize("n,h,w,k", [(2, 17, 17, 7), (1, 224, 224, 7), (2, 9, 12, 3)])
def test_stem_im2col_matches_numpy(n, h, w, k):
    """uint8 NHWC images -> normalised bf16 im2col rows (K layout ky * pad8(3k) + kx * 3 + c,
    zero halo), bit-exact vs the same fp32 arithmetic in numpy (interior word loads and the
    border byte path)."""
    from paper_2308_15949_b200 import _lib
    from paper_2308_15949_b200 import device as D
    D.require_cuda()
    rng = np.random.default_rng(h + k)
    img = rng.integers(0, 256, (n, h, w, 3), dtype=np.uint8)
    mean = np.array([123.7, 116.3, 103.5], np.float32)
    inv = (1.0 / np.array([58.4, 57.1, 57.4], np.float32)).astype(np.float32)
    st, pad = 2, k // 2
    ho, wo = (h + 2 * pad - k) // st + 1, (w + 2 * pad - k) // st + 1
    seg = (3 * k + 7) // 8 * 8
    cols = torch.empty(n * ho * wo, k * seg, dtype=torch.bfloat16, device="cuda")
    imgd = torch.from_numpy(img).cuda()
    md, sd = torch.from_numpy(mean).cuda(), torch.from_numpy(inv).cuda()
    _lib.call("laud_stem_im2col", D.ptr(imgd), n, h, w, k, st, pad, D.ptr(md), D.ptr(sd), D.ptr(cols),
              k * seg, None)
    torch.cuda.synchronize()
    norm = (img.astype(np.float32) - mean) * inv  # fp32, same order as the kernel
    padded = np.zeros((n, h + 2 * pad, w + 2 * pad, 3), np.float32)
    padded[:, pad:pad + h, pad:pad + w] = norm
    ref = np.zeros((n, ho, wo, k, seg), np.float32)
    for ky in range(k):
        for kx in range(k):
            ref[..., ky, kx * 3:kx * 3 + 3] = padded[:, ky:ky + st * ho:st, kx:kx + st * wo:st]
    ref_bf = torch.from_numpy(ref.reshape(n * ho * wo, k * seg)).bfloat16()
    assert torch.equal(cols.cpu(), ref_bf)


@pytest.mark.parametrize("n", [1, 3, 40])
def test_fused_stem_pool_matches_unfused(n):
    """laud_stem_pool (7x7/2 conv from uint8 images in one kernel, im2col-free
    tcgen05 MMAs on overlapping core matrices, bias + ReLU + 3x3/2 max-pool) vs
    the im2col + GEMM + max-pool path and a torch fp32 reference."""
    import ctypes as C
    from paper_2308_15949_b200 import _lib
    from paper_2308_15949_b200.network import IMAGENET_MEAN, IMAGENET_STD
    CH, D = _engine()
    g = torch.Generator().manual_seed(n)
    img = torch.randint(0, 256, (n, 224, 224, 3), dtype=torch.uint8, generator=g).cuda()
    w = (torch.randn(64, 3, 7, 7, generator=g) * 0.1).to(torch.bfloat16).float()
    b = (torch.randn(64, generator=g) * 0.1).cuda()
    mean = torch.tensor(IMAGENET_MEAN, dtype=torch.float32).cuda()
    inv = torch.tensor([1.0 / s for s in IMAGENET_STD], dtype=torch.float32).cuda()
    wf = torch.zeros(64, 7, 8, 4)
    wf[:, :, :7, :3] = w.permute(0, 2, 3, 1)
    wf = torch.cat([wf.reshape(64, 224), torch.zeros(64, 32)], 1).to(torch.bfloat16).cuda().contiguous()
    out = torch.empty(n, 56, 56, 64, dtype=torch.bfloat16, device="cuda")
    sh = D.stream_handle()
    _lib.call("laud_stem_pool", D.ptr(img), n, 224, 224, D.ptr(mean), D.ptr(inv), D.ptr(wf), D.ptr(b), D.ptr(out), sh)
    # unfused: im2col (K = 7 * 24) + engine GEMM + max-pool
    cols_ld = 7 * 24
    cols = torch.empty(n * 112 * 112, cols_ld, dtype=torch.bfloat16, device="cuda")
    _lib.call("laud_stem_im2col", D.ptr(img), n, 224, 224, 7, 2, 3, D.ptr(mean), D.ptr(inv), D.ptr(cols), cols_ld, sh)
    wc = torch.zeros(64, 7, 24)
    wc[:, :, :21] = w.permute(0, 2, 3, 1).reshape(64, 7, 21)
    wcol = D.pack_weight(wc.reshape(64, cols_ld, 1, 1), cols_ld)
    conv = torch.empty(n, 112, 112, 64, dtype=torch.bfloat16, device="cuda")
    CH.conv(act=cols, in_hw=(n * 112 * 112, 1), in_c=cols_ld, in_ld=cols_ld, weight=wcol, n_out=64, out=conv,
            out_ld=64, out_hw=(112, 112), batch=n, a_compact=1, bias=b, relu=1)
    ref2 = torch.empty_like(out)
    _lib.call("laud_maxpool3s2", D.ptr(conv), n, 112, 112, 64, D.ptr(ref2), sh)
    torch.cuda.synchronize()
    diff = (out.float() - ref2.float()).abs()
    assert diff.max().item() <= 0.05 * ref2.float().abs().max().item()
    assert (diff > 0).float().mean().item() < 0.02  # accumulation-order rounding only
    # torch fp32 reference of the same bf16-rounded inputs
    x = ((img.float() - mean) * inv).to(torch.bfloat16).float().permute(0, 3, 1, 2)
    y = torch.relu(torch.nn.functional.conv2d(x, w.cuda(), stride=2, padding=3) + b.view(1, -1, 1, 1))
    y = torch.nn.functional.max_pool2d(y.to(torch.bfloat16).float(), 3, 2, 1).permute(0, 2, 3, 1)
    err = (out.float() - y).norm() / y.norm()
    assert err < 4e-3, float(err)


@pytest.mark.parametrize("n", [1, 3, 37])
def test_fused_stem3_matches_torch(n):
    """laud_stem3 (RegNet stem: 3x3/2 conv from uint8 images + bias + ReLU, one
    kernel, im2col-free tcgen05 MMAs on overlapping core matrices) vs a torch fp32
    reference of the same bf16-rounded normalised inputs and bf16 weights."""
    from paper_2308_15949_b200 import _lib
    from paper_2308_15949_b200.network import IMAGENET_MEAN, IMAGENET_STD
    CH, D = _engine()
    g = torch.Generator().manual_seed(100 + n)
    img = torch.randint(0, 256, (n, 224, 224, 3), dtype=torch.uint8, generator=g).cuda()
    w = (torch.randn(32, 3, 3, 3, generator=g) * 0.2).to(torch.bfloat16).float()
    b = (torch.randn(32, generator=g) * 0.1).cuda()
    mean = torch.tensor(IMAGENET_MEAN, dtype=torch.float32).cuda()
    inv = torch.tensor([1.0 / s for s in IMAGENET_STD], dtype=torch.float32).cuda()
    wf = torch.zeros(32, 3, 4, 4)
    wf[:, :, :3, :3] = w.permute(0, 2, 3, 1)
    wf = wf.reshape(32, 48).to(torch.bfloat16).cuda().contiguous()
    out = torch.empty(n, 112, 112, 32, dtype=torch.bfloat16, device="cuda")
    _lib.call("laud_stem3", D.ptr(img), n, 224, 224, D.ptr(mean), D.ptr(inv), D.ptr(wf), D.ptr(b), D.ptr(out),
              D.stream_handle())
    torch.cuda.synchronize()
    x = ((img.float() - mean) * inv).to(torch.bfloat16).float().permute(0, 3, 1, 2)
    y = torch.relu(torch.nn.functional.conv2d(x, w.cuda(), stride=2, padding=1) + b.view(1, -1, 1, 1))
    y = y.permute(0, 2, 3, 1)
    err = (out.float() - y).norm() / y.norm()
    assert err < 4e-3, float(err)
    assert (out.float() - y).abs().max().item() < 0.05 * y.abs().max().item()
