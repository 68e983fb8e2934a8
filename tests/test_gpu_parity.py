"""GPU parity: the drop-in API (CUDA path) vs the CPU oracle and the golden fixtures.

Tolerances (BASELINE north star):
  * masks / gather plans / dilation: bit-exact (near-tie cells excluded and counted);
  * bf16 block outputs: <= 1e-3 norm-relative vs the bf16-emulating oracle
    (same rounding points), and reported vs pure fp64;
  * GPU sparse vs GPU dense-masked: bit-exact (identical rounding points);
  * cells the mask leaves inactive: bitwise equal to the skip path.
"""
import json
from pathlib import Path

import numpy as np
import pytest

from oracle import laud_oracle as O
from paper_2308_15949_b200.core import BlockSpec, ConvLayerSpec, DynamicConfig, Paradigm, TensorShape

pytestmark = pytest.mark.gpu
G = Path(__file__).resolve().parent / "golden"
BF16_TOL = 1e-3


def _R():
    from paper_2308_15949_b200 import reference as R
    from paper_2308_15949_b200 import device as D
    D.require_cuda()
    return R


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def _oracle_mask(R, m):
    if isinstance(m, R.SpatialMask):
        return O.SpatialMask(m.coarse, m.upsampled, m.granularity)
    if isinstance(m, R.LayerMask):
        return O.LayerMask(m.decisions)
    if isinstance(m, R.ChannelMask):
        return O.ChannelMask(m.coarse, m.expanded, m.granularity)
    return m


def test_spatial_masker_decisions_match_oracle():
    R = _R()
    a = np.load(G / "maskers.npz")
    for i in range(4):
        x, w, s = a[f"sp{i}_x"], a[f"sp{i}_w"], int(a[f"sp{i}_s"])
        m = R.spatial_masker_forward(x, w, s)
        ref = a[f"sp{i}_coarse"]
        # near-tie guard: |d| <= 1e-6 * sum |p||w| may legitimately flip in fp32
        n, c, h, ww = x.shape
        pooled = x.reshape(n, c, h // s, s, ww // s, s).mean(axis=(3, 5))
        wd = (w[0] - w[1]).reshape(c)
        d = np.einsum("nchw,c->nhw", pooled, wd)
        scale = np.einsum("nchw,c->nhw", np.abs(pooled), np.abs(wd))
        safe = np.abs(d) > 1e-6 * scale
        assert np.array_equal(m.coarse[safe], ref[safe])
        assert (~safe).sum() == 0
        assert np.array_equal(m.upsampled, a[f"sp{i}_up"])


def test_spatial_masker_train_mode_replays_reference_rng():
    R = _R()
    a = np.load(G / "maskers.npz")
    for i in range(4):
        x, w, s = a[f"sp{i}_x"], a[f"sp{i}_w"], int(a[f"sp{i}_s"])
        mt = R.spatial_masker_forward(x, w, s, mode="train", tau=0.7, rng=np.random.default_rng(99 + i))
        assert np.array_equal(mt.coarse, a[f"sp{i}_train_coarse"])
        np.testing.assert_allclose(mt.soft, a[f"sp{i}_train_soft"], rtol=1e-4, atol=1e-6)


def test_masker_on_block_input_large():
    """fp32 masker at full BASELINE size (R101 s1 block input, batch 8, S=4)."""
    R = _R()
    rng = np.random.default_rng(7)
    x = rng.standard_normal((8, 256, 56, 56)).astype(np.float32).astype(np.float64)
    w = rng.standard_normal((2, 256, 1, 1)) / 16
    m = R.spatial_masker_forward(x, w, 4)
    ref = O.spatial_masker_forward(x, w, 4)
    assert m.coarse.shape == (8, 14, 14)
    assert np.mean(m.coarse == ref.coarse) == 1.0


def test_dilate_and_rates_matches_oracle():
    R = _R()
    a = np.load(G / "maskers.npz")
    for i in range(4):
        coarse, s = a[f"sp{i}_coarse"], int(a[f"sp{i}_s"])
        for k in (1, 3, 5):
            m = R.SpatialMask(coarse, R.upsample_coarse(coarse, s), s)
            r, rd, dil = R.dilate_and_rates(m, k)
            r2, rd2, dil2 = O.dilate_and_rates(O.SpatialMask(coarse, O.upsample_coarse(coarse, s), s), k)
            assert r == r2 and abs(rd - rd2) < 1e-12 and np.array_equal(dil, dil2)
        np.testing.assert_allclose(R.dilate_and_rates(R.SpatialMask(coarse, R.upsample_coarse(coarse, s), s), 3)[:2],
                                   a[f"sp{i}_rates"], atol=1e-12)


def _cases():
    meta = json.loads((G / "equivalence.json").read_text())
    return meta


@pytest.mark.parametrize("m", _cases(), ids=lambda m: m["key"])
def test_block_sparse_matches_oracle(m):
    R = _R()
    case = O.EquivalenceCase(Paradigm(m["paradigm"]), m["channels"], m["height"], m["width"],
                             m["granularity"], m["seed"])
    block, mask, bw, x, cfg = O.case_inputs(case)
    if case.paradigm is Paradigm.SPATIAL:
        rmask = R.SpatialMask(mask.coarse, mask.upsampled, mask.granularity)
    elif case.paradigm is Paradigm.CHANNEL:
        rmask = R.ChannelMask(mask.coarse, mask.expanded, mask.granularity)
    else:
        rmask = R.LayerMask(mask.decisions)
    rbw = R.BlockWeights(bw.w1, bw.w2, bw.w3, bw.w_down)
    y = R.block_forward_sparse(x, rbw, block, cfg, rmask)
    emu = O.block_forward_sparse(x, bw, block, cfg, mask, emulate_bf16=True)
    ref = np.load(G / "equivalence.npz")[m["key"] + "__sparse"]
    assert _rel(y, emu) <= BF16_TOL, _rel(y, emu)
    assert _rel(y, ref) <= 1e-2  # pure fp64 reference, bf16 storage error
    # inactive cells carry the skip path bitwise (bf16 of the skip)
    skip = O.round_bf16(O.skip_path(O.round_bf16(x), block,
                                    O.BlockWeights(*(O.round_bf16(w) if w is not None else None
                                                     for w in (bw.w1, bw.w2, bw.w3, bw.w_down))),
                                    None, O.round_bf16))
    if case.paradigm is Paradigm.SPATIAL:
        inactive = ~mask.upsampled
        if not block.has_downsample:
            np.testing.assert_array_equal(y.transpose(0, 2, 3, 1)[inactive],
                                          skip.transpose(0, 2, 3, 1)[inactive])
        else:
            assert _rel(y.transpose(0, 2, 3, 1)[inactive], skip.transpose(0, 2, 3, 1)[inactive]) < 1e-2


@pytest.mark.parametrize("case", [c for c in O.default_cases(per_paradigm=8)
                                  if c.paradigm is not Paradigm.CHANNEL],
                         ids=lambda c: f"{c.paradigm.value}-{c.channels}-{c.height}-g{c.granularity}-s{c.seed}")
def test_gpu_equivalence_suite_is_exact(case):
    R = _R()
    rc = R.EquivalenceCase(case.paradigm, case.channels, case.height, case.width, case.granularity, case.seed)
    assert R.run_equivalence_case(rc) == 0.0
    block, mask, *_ = O.case_inputs(case)
    if case.paradigm is Paradigm.SPATIAL and mask.coarse.any():
        assert R.run_equivalence_case(rc, inject_fault=True) > 1e-3


def test_config1_block_matches_reference_golden():
    """BASELINE config 1 through the drop-in: R50 s3b1, 14x14x1024, S=2, batch 1."""
    R = _R()
    from paper_2308_15949_b200.zoo import build_network
    a = np.load(G / "config1.npz")
    block = [b.block for b in build_network("resnet50").blocks if b.stage == 3 and b.index == 1][0]
    rng = np.random.default_rng(0)
    bw = R.make_block_weights(block, rng)
    x = rng.standard_normal((1, 1024, 14, 14))
    mw = rng.standard_normal((2, 1024, 1, 1)) / np.sqrt(1024)
    m = R.spatial_masker_forward(x, mw, 2)
    assert np.array_equal(m.coarse, a["coarse"])
    cfg = DynamicConfig(Paradigm.SPATIAL, spatial_granularity=2)
    y = R.block_forward_sparse(x, bw, block, cfg, m)
    obw = O.BlockWeights(bw.w1, bw.w2, bw.w3, bw.w_down)
    emu = O.block_forward_sparse(x, obw, block, cfg, O.SpatialMask(m.coarse, m.upsampled, 2),
                                 emulate_bf16=True)
    assert _rel(y, emu) <= BF16_TOL
    assert _rel(y, a["y"]) <= 3e-3
    me = R.SpatialMask(a["coarse_exact"], R.upsample_coarse(a["coarse_exact"], 2), 2)
    y2 = R.block_forward_sparse(x, bw, block, cfg, me)
    assert _rel(y2, a["y_exact"]) <= 3e-3


def test_full_and_empty_masks_at_scale():
    """R101 s2b1 geometry (28x28x512, S=2), batch 4: all-ones == static, zeros == identity."""
    R = _R()
    blk = BlockSpec(ConvLayerSpec(512, 128, 1), ConvLayerSpec(128, 128, 3), ConvLayerSpec(128, 512, 1),
                    TensorShape(512, 28, 28))
    rng = np.random.default_rng(11)
    bw = R.make_block_weights(blk, rng)
    x = rng.standard_normal((4, 512, 28, 28))
    ones = np.ones((4, 14, 14), bool)
    y1 = R.block_forward_sparse(x, bw, blk, DynamicConfig(Paradigm.SPATIAL, spatial_granularity=2),
                                R.SpatialMask(ones, R.upsample_coarse(ones, 2), 2))
    ys = R.block_forward_sparse(x, bw, blk, DynamicConfig(Paradigm.STATIC), None)
    np.testing.assert_array_equal(y1, ys)
    zeros = np.zeros_like(ones)
    y0 = R.block_forward_sparse(x, bw, blk, DynamicConfig(Paradigm.SPATIAL, spatial_granularity=2),
                                R.SpatialMask(zeros, R.upsample_coarse(zeros, 2), 2))
    np.testing.assert_array_equal(y0, O.round_bf16(x))


def test_channel_masker_matches_reference():
    R = _R()
    a = np.load(G / "maskers.npz")
    for i in range(3):
        x, w1, w2, g = a[f"ch{i}_x"], a[f"ch{i}_w1"], a[f"ch{i}_w2"], int(a[f"ch{i}_g"])
        m = R.channel_masker_forward(x, (w1, w2), g)
        # near-tie guard on the logit gap (fp32 device vs fp64 reference)
        hid = np.maximum(x.mean(axis=(2, 3)) @ w1.T, 0.0)
        lg = (hid @ w2.T).reshape(x.shape[0], -1, 2)
        gap = lg[..., 0] - lg[..., 1]
        scale = np.abs(hid) @ np.abs(w2.T).reshape(hid.shape[1], -1, 2).sum(-1) + 1e-30
        safe = np.abs(gap) > 1e-5 * scale
        assert np.array_equal(m.coarse[safe], a[f"ch{i}_coarse"][safe])
        assert np.array_equal(m.expanded.shape, a[f"ch{i}_exp"].shape)
        mt = R.channel_masker_forward(x, (w1, w2), g, mode="train", tau=0.5,
                                      rng=np.random.default_rng(7 + i))
        assert np.array_equal(mt.coarse[safe], a[f"ch{i}_train_coarse"][safe])
        np.testing.assert_allclose(mt.soft, a[f"ch{i}_train_soft"], rtol=1e-3, atol=1e-5)


@pytest.mark.parametrize("r", [0.0, 0.25, 0.5, 1.0])
def test_channel_block_large(r):
    """R101 s3 geometry (14x14x1024, mid 256), batch 4: exact-count channel masks."""
    R = _R()
    blk = BlockSpec(ConvLayerSpec(1024, 256, 1), ConvLayerSpec(256, 256, 3), ConvLayerSpec(256, 1024, 1),
                    TensorShape(1024, 14, 14))
    rng = np.random.default_rng(5)
    bw = R.make_block_weights(blk, rng)
    x = rng.standard_normal((4, 1024, 14, 14))
    coarse = np.zeros((4, 256), bool)
    for i in range(4):
        coarse[i, rng.permutation(256)[: int(round(r * 256))]] = True
    m = R.ChannelMask(coarse, coarse, 1)
    cfg = DynamicConfig(Paradigm.CHANNEL, channel_granularity=1)
    y = R.block_forward_sparse(x, bw, blk, cfg, m)
    obw = O.BlockWeights(bw.w1, bw.w2, bw.w3, bw.w_down)
    emu = O.block_forward_sparse(x, obw, blk, cfg, O.ChannelMask(coarse, coarse, 1), emulate_bf16=True)
    assert _rel(y, emu) <= BF16_TOL
    yd = R.block_forward_dense_masked(x, bw, blk, cfg, m)
    assert _rel(y, yd) <= BF16_TOL


@pytest.mark.parametrize("n,g,stride", [(16, 1, 1), (16, 2, 1), (64, 1, 1), (16, 1, 2)])
def test_channel_block_throughput_batch(n, g, stride):
    """The channel schedule the benchmark runs (batch >= 8, R101 stage-3 geometry,
    bf16) vs the bf16-emulating oracle at 1e-3: exact-count per-sample masks at
    r = 0.5 plus a sample that keeps no channel and one that keeps all."""
    R = _R()
    cin = 512 if stride == 2 else 1024
    hw = 28 if stride == 2 else 14
    blk = BlockSpec(ConvLayerSpec(cin, 256, 1), ConvLayerSpec(256, 256, 3, stride), ConvLayerSpec(256, 1024, 1),
                    TensorShape(cin, hw, hw), has_downsample=stride > 1)
    rng = np.random.default_rng(50 + n + g)
    bw = R.make_block_weights(blk, rng)
    x = rng.standard_normal((n, cin, hw, hw))
    d = 256 // g
    coarse = np.zeros((n, d), bool)
    for i in range(2, n):
        coarse[i, rng.permutation(d)[: d // 2]] = True
    coarse[1] = True  # sample 0 keeps nothing, sample 1 everything
    exp = np.repeat(coarse, g, axis=1)
    m = R.ChannelMask(coarse, exp, g)
    cfg = DynamicConfig(Paradigm.CHANNEL, channel_granularity=g)
    y = R.block_forward_sparse(x, bw, blk, cfg, m)
    obw = O.BlockWeights(bw.w1, bw.w2, bw.w3, bw.w_down)
    emu = O.block_forward_sparse(x, obw, blk, cfg, O.ChannelMask(coarse, exp, g), emulate_bf16=True)
    assert _rel(y, emu) <= BF16_TOL, _rel(y, emu)
    # the sample that keeps no channel is exactly its (bf16) skip path
    xr = O.round_bf16(x[:1])
    skip = O.skip_path(xr, blk, O.BlockWeights(*(O.round_bf16(w) for w in (bw.w1, bw.w2, bw.w3, bw.w_down))),
                       rnd=O.round_bf16) if stride > 1 else xr
    assert _rel(y[:1], skip) <= BF16_TOL


@pytest.mark.parametrize("gather", [0, 1])
@pytest.mark.parametrize("cin,cmid,hw,n", [(256, 64, 56, 8), (512, 128, 28, 8), (64, 64, 56, 8), (1024, 256, 14, 16)])
def test_channel_block_gathered_weights_stages(cin, cmid, hw, n, gather, monkeypatch):
    """Large-batch channel schedules — dense-masked (default) and the opt-in
    in-kernel weight gathers (LAUD_CH_GATHER=1: conv2 gathers W2[sel] rows,
    N = k_n; conv3 gathers W3^T K rows into an MN-major B tile) — at the R101
    stage-1/2/3 geometries vs the bf16-emulating oracle; per-sample ratios 0 .. 1."""
    monkeypatch.setenv("LAUD_CH_GATHER", str(gather))
    R = _R()
    blk = BlockSpec(ConvLayerSpec(cin, cmid, 1), ConvLayerSpec(cmid, cmid, 3), ConvLayerSpec(cmid, 4 * cmid, 1),
                    TensorShape(cin, hw, hw), has_downsample=cin != 4 * cmid)
    rng = np.random.default_rng(cin + hw)
    bw = R.make_block_weights(blk, rng)
    x = rng.standard_normal((n, cin, hw, hw))
    coarse = np.zeros((n, cmid), bool)
    for i in range(n):
        coarse[i, rng.permutation(cmid)[: (i * cmid) // (n - 1)]] = True
    m = R.ChannelMask(coarse, coarse, 1)
    cfg = DynamicConfig(Paradigm.CHANNEL, channel_granularity=1)
    y = R.block_forward_sparse(x, bw, blk, cfg, m)
    obw = O.BlockWeights(bw.w1, bw.w2, bw.w3, bw.w_down)
    emu = O.block_forward_sparse(x, obw, blk, cfg, O.ChannelMask(coarse, coarse, 1), emulate_bf16=True)
    assert _rel(y, emu) <= BF16_TOL, _rel(y, emu)


@pytest.mark.parametrize("stage,index,paradigm", [(1, 0, "spatial"), (2, 1, "spatial"), (3, 0, "spatial"),
                                                   (3, 1, "spatial"), (4, 1, "spatial"), (3, 1, "layer"),
                                                   (2, 0, "static")])
def test_regnet_grouped_block_matches_oracle(stage, index, paradigm):
    """RegNetY-1.6GF blocks (grouped conv2, group width 24) through the drop-in."""
    R = _R()
    from paper_2308_15949_b200.zoo import build_network
    net = build_network("regnety-1.6gf")
    block = [b.block for b in net.blocks if b.stage == stage and b.index == index][0]
    s = (4, 4, 2, 1)[stage - 1]
    rng = np.random.default_rng(stage * 10 + index)
    bw = R.make_block_weights(block, rng)
    n = 2
    ci = block.input_shape
    x = rng.standard_normal((n, ci.channels, ci.height, ci.width))
    o = block.output_shape
    if paradigm == "spatial":
        coarse = rng.random((n, o.height // s, o.width // s)) < 0.5
        cfg = DynamicConfig(Paradigm.SPATIAL, spatial_granularity=s)
        m, om = R.SpatialMask(coarse, R.upsample_coarse(coarse, s), s), O.SpatialMask(coarse, O.upsample_coarse(coarse, s), s)
    elif paradigm == "layer":
        d = np.array([True, False])
        cfg = DynamicConfig(Paradigm.LAYER)
        m, om = R.LayerMask(d), O.LayerMask(d)
    else:
        cfg = DynamicConfig(Paradigm.STATIC)
        m = om = None
    y = R.block_forward_sparse(x, bw, block, cfg, m)
    obw = O.BlockWeights(bw.w1, bw.w2, bw.w3, bw.w_down)
    emu = O.block_forward_sparse(x, obw, block, cfg, om, emulate_bf16=True)
    ref = O.block_forward_sparse(x, obw, block, cfg, om)
    assert block.conv2.groups > 1
    assert _rel(y, emu) <= BF16_TOL, _rel(y, emu)
    assert _rel(y, ref) <= 1e-2


FP32_TOL = 1e-5


@pytest.fixture
def fp32_mode():
    R = _R()
    R.set_precision("fp32")
    yield R
    R.set_precision("bf16")


@pytest.mark.parametrize("m", _cases(), ids=lambda m: m["key"])
def test_fp32_mode_block_matches_reference(m, fp32_mode):
    """fp32 mode (FFMA engine): <= 1e-5 norm-relative vs the reference's fp64 output."""
    R = fp32_mode
    case = O.EquivalenceCase(Paradigm(m["paradigm"]), m["channels"], m["height"], m["width"],
                             m["granularity"], m["seed"])
    block, mask, bw, x, cfg = O.case_inputs(case)
    if case.paradigm is Paradigm.SPATIAL:
        rmask = R.SpatialMask(mask.coarse, mask.upsampled, mask.granularity)
    elif case.paradigm is Paradigm.CHANNEL:
        rmask = R.ChannelMask(mask.coarse, mask.expanded, mask.granularity)
    else:
        rmask = R.LayerMask(mask.decisions)
    rbw = R.BlockWeights(bw.w1, bw.w2, bw.w3, bw.w_down)
    y = R.block_forward_sparse(x, rbw, block, cfg, rmask)
    ref = np.load(G / "equivalence.npz")[m["key"] + "__sparse"]
    assert _rel(y, ref) <= FP32_TOL, _rel(y, ref)
    yd = R.block_forward_dense_masked(x, rbw, block, cfg, rmask)
    assert _rel(yd, ref) <= FP32_TOL, _rel(yd, ref)


def test_fp32_mode_config1_and_regnet(fp32_mode):
    """BASELINE config 1 block and a grouped RegNetY block in fp32 mode vs fp64."""
    R = fp32_mode
    from paper_2308_15949_b200.zoo import build_network
    a = np.load(G / "config1.npz")
    block = [b.block for b in build_network("resnet50").blocks if b.stage == 3 and b.index == 1][0]
    rng = np.random.default_rng(0)
    bw = R.make_block_weights(block, rng)
    x = rng.standard_normal((1, 1024, 14, 14))
    mw = rng.standard_normal((2, 1024, 1, 1)) / np.sqrt(1024)
    m = R.spatial_masker_forward(x, mw, 2)
    cfg = DynamicConfig(Paradigm.SPATIAL, spatial_granularity=2)
    y = R.block_forward_sparse(x, bw, block, cfg, m)
    assert _rel(y, a["y"]) <= FP32_TOL, _rel(y, a["y"])
    rb = [b.block for b in build_network("regnety-1.6gf").blocks if b.stage == 3 and b.index == 0][0]
    rng = np.random.default_rng(5)
    rbw = R.make_block_weights(rb, rng)
    xi = rng.standard_normal((2, rb.input_shape.channels, rb.input_shape.height, rb.input_shape.width))
    coarse = rng.random((2, 7, 7)) < 0.5
    om = O.SpatialMask(coarse, O.upsample_coarse(coarse, 2), 2)
    yr = R.block_forward_sparse(xi, rbw, rb, cfg, R.SpatialMask(coarse, R.upsample_coarse(coarse, 2), 2))
    ref = O.block_forward_sparse(xi, O.BlockWeights(rbw.w1, rbw.w2, rbw.w3, rbw.w_down), rb, cfg, om)
    assert _rel(yr, ref) <= FP32_TOL, _rel(yr, ref)


@pytest.mark.parametrize("stage,s", [(3, 2), (2, 2), (4, 1), (1, 4)])
def test_dense_conv1_schedule_is_bitwise_identical(stage, s):
    """conv1 on the dense grid (reference.py:385) == conv1 on the dilated pixel list."""
    import torch
    from paper_2308_15949_b200 import device as D
    from paper_2308_15949_b200.network import make_params
    R = _R()
    bp = [b for b in make_params("resnet101", 0)["blocks"] if b["stage"] == stage and b["index"] == 0][0]
    blk = bp["block"]
    ep = D.Epilogue(s1=bp["s1"], b1=bp["b1"], relu1=True, s2=bp["s2"], b2=bp["b2"], relu2=True,
                    s3=bp["s3"], b3=bp["b3"], sd=bp["sd"], bd=bp["bd"], relu_out=True)
    db = D.DeviceBlock(blk, bp["w1"], bp["w2"], bp["w3"], bp["wd"], ep, masker_w=bp["masker_w"], fold_scale=True)
    n, h = 8, blk.input_shape.height
    x = torch.randn(n, h, h, db.cin_p, device="cuda").relu_().bfloat16()
    o = blk.output_shape
    coarse = (torch.rand(n * (o.height // s) * (o.width // s), device="cuda") < 0.5).to(torch.uint8)
    y0, *_ = db.forward(x, "spatial", s, coarse=coarse, conv1_dense=False)
    y1, *_ = db.forward(x, "spatial", s, coarse=coarse, conv1_dense=True)
    torch.cuda.synchronize()
    assert torch.equal(y0, y1)


def test_verify_cli_on_gpu(tmp_path):
    """The reference's `verify` command (cli.py:250-278) against the GPU path:
    the shipped case file passes, the fault hook fails (exit 1)."""
    from paper_2308_15949_b200 import verify
    cases = tmp_path / "cases.txt"  # the golden case set in the reference's case-file format
    cases.write_text("".join(
        f"paradigm={m['paradigm']} channels={m['channels']} height={m['height']} width={m['width']} "
        f"granularity={m['granularity']} seed={m['seed']} tol={m['tol']}\n" for m in _cases()))
    assert verify.main(["--cases", str(cases)]) == 0
    assert verify.main(["--cases", str(cases), "--precision", "fp32"]) == 0
    assert verify.main(["--per-paradigm", "2", "--inject-fault"]) == 1


@pytest.mark.parametrize("stage,index,paradigm", [(2, 1, "spatial"), (3, 0, "spatial"), (4, 1, "spatial"),
                                                   (3, 1, "layer"), (2, 0, "static"), (3, 1, "channel"),
                                                   (2, 0, "channel"), (1, 1, "channel")])
def test_regnet_se_block_matches_oracle_ext(stage, index, paradigm):
    """EXT squeeze-excitation (pool over the sample's active patches) on the device
    vs the oracle EXT, bf16 rounding points emulated."""
    import torch
    from paper_2308_15949_b200 import device as D
    from paper_2308_15949_b200.network import make_params
    _R()
    bp = [b for b in make_params("regnety-1.6gf", 0)["blocks"] if b["stage"] == stage and b["index"] == index][0]
    blk = bp["block"]
    assert "se_w1" in bp
    ep = D.Epilogue(b1=bp["b1"], relu1=True, b2=bp["b2"], relu2=True, b3=bp["b3"], bd=bp["bd"], relu_out=True)
    db = D.DeviceBlock(blk, bp["w1"], bp["w2"], bp["w3"], bp["wd"], ep)
    db.set_se(bp["se_w1"], bp["se_b1"], bp["se_w2"], bp["se_b2"])
    rng = np.random.default_rng(stage)
    n = 3
    ci = blk.input_shape
    x = np.maximum(rng.standard_normal((n, ci.channels, ci.height, ci.width)), 0)
    o = blk.output_shape
    s = (4, 4, 2, 1)[stage - 1]
    oep = O.Epilogues(b1=bp["b1"], relu1=True, b2=bp["b2"], relu2=True, b3=bp["b3"], bd=bp["bd"],
                      relu_out=True, se_w1=bp["se_w1"], se_b1=bp["se_b1"], se_w2=bp["se_w2"], se_b2=bp["se_b2"])
    obw = O.BlockWeights(bp["w1"], bp["w2"], bp["w3"], bp["wd"])
    xd = D.to_device_nhwc(x)
    if paradigm == "spatial":
        coarse = rng.random((n, o.height // s, o.width // s)) < 0.5
        coarse[1] = False  # a sample with no active patch
        y, *_ = db.forward(xd, "spatial", s, coarse=torch.from_numpy(coarse.astype(np.uint8).reshape(-1)).cuda())
        cfg, om = DynamicConfig(Paradigm.SPATIAL, spatial_granularity=s), O.SpatialMask(coarse, O.upsample_coarse(coarse, s), s)
    elif paradigm == "layer":
        d = np.array([True, False, True])
        y, *_ = db.forward(xd, "layer", coarse=torch.from_numpy(d.astype(np.uint8)).cuda())
        cfg, om = DynamicConfig(Paradigm.LAYER), O.LayerMask(d)
    elif paradigm == "channel":  # EXT: grouped conv2 + SE under channel skipping
        db.enable_grouped_channel()
        cm = blk.conv2.out_channels
        cmask = rng.random((n, cm)) < 0.5
        cmask[1] = False  # a sample that keeps no channel
        mm = np.zeros((n, db.cmid_p), np.uint8)
        mm[:, :cm] = cmask
        y, *_ = db.forward(xd, "channel", chmask=torch.from_numpy(mm.reshape(-1)).cuda())
        cfg, om = DynamicConfig(Paradigm.CHANNEL, channel_granularity=1), O.ChannelMask(cmask, cmask, 1)
    else:
        y, *_ = db.forward(xd, "static")
        cfg, om = DynamicConfig(Paradigm.STATIC), None
    torch.cuda.synchronize()
    yg = D.from_device_nhwc(y, o.channels)
    emu = O.block_forward_sparse(x, obw, blk, cfg, om, epilogues=oep, emulate_bf16=True, grouped_channel_ext=True)
    assert _rel(yg, emu) <= 2e-3, _rel(yg, emu)
    no_se = O.block_forward_sparse(x, obw, blk, cfg, om, epilogues=O.Epilogues(
        b1=bp["b1"], relu1=True, b2=bp["b2"], relu2=True, b3=bp["b3"], bd=bp["bd"], relu_out=True), emulate_bf16=True,
        grouped_channel_ext=True)
    assert _rel(yg, no_se) > 1e-2  # the gate is really applied


@pytest.mark.parametrize("stage,index,s,n", [(3, 1, 2, 16), (2, 0, 2, 16), (4, 1, 1, 16), (4, 0, 1, 16),
                                             (3, 1, 2, 128), (1, 1, 4, 8), (2, 1, 2, 32)])
def test_masker_fused_into_conv1_decides_like_standalone(stage, index, s, n):
    """The masker dots accumulated from conv1's A stages (dense conv1, incl. blocks
    whose conv1 has several N tiles; n = 128 at stage 3 runs conv1 on CTA pairs,
    whose readers relay A completion to the leader) decide exactly like the
    standalone masker, with a non-zero calibration bias, and the block outputs
    agree bit for bit where the decisions do."""
    import torch
    from paper_2308_15949_b200 import device as D
    from paper_2308_15949_b200.network import make_params
    _R()
    bp = [b for b in make_params("resnet101", 0)["blocks"] if b["stage"] == stage and b["index"] == index][0]
    blk = bp["block"]
    ep = D.Epilogue(s1=bp["s1"], b1=bp["b1"], relu1=True, s2=bp["s2"], b2=bp["b2"], relu2=True,
                    s3=bp["s3"], b3=bp["b3"], sd=bp["sd"], bd=bp["bd"], relu_out=True)
    db = D.DeviceBlock(blk, bp["w1"], bp["w2"], bp["w3"], bp["wd"], ep, masker_w=bp["masker_w"],
                       masker_bias=0.37, fold_scale=True)
    h = blk.input_shape.height
    x = torch.randn(n, h, h, db.cin_p, device="cuda").relu_().bfloat16()
    o = blk.output_shape
    nc = n * (o.height // s) * (o.width // s)
    got, ys = [], []
    for dense in (False, True):
        y, coarse, _, _ = db.forward(x.clone(), "spatial", s, ws=D.Workspace(), conv1_dense=dense)
        torch.cuda.synchronize()
        got.append(coarse[:nc].cpu().numpy().copy())
        ys.append(y.float().cpu())
    assert 0.0 < got[0].mean() < 1.0
    assert np.mean(got[0] == got[1]) > 0.999
    if (got[0] == got[1]).all():
        assert torch.equal(ys[0], ys[1])


def _grouped_golden(tag):
    d = np.load(G / "grouped_channel.npz")
    cin, cm, g, cout, hw, stride, gran = (int(v) for v in d[f"{tag}_geom"])
    blk = BlockSpec(ConvLayerSpec(cin, cm, 1), ConvLayerSpec(cm, cm, 3, stride, g), ConvLayerSpec(cm, cout, 1),
                    TensorShape(cin, hw, hw), has_downsample=stride > 1 or cin != cout)
    wd = d[f"{tag}_wd"] if f"{tag}_wd" in d else None
    coarse = d[f"{tag}_coarse"]
    return d, blk, (d[f"{tag}_w1"], d[f"{tag}_w2"], d[f"{tag}_w3"], wd), coarse, gran, d[f"{tag}_x"]


@pytest.mark.parametrize("tag", ["a", "b", "c"])
def test_grouped_channel_ext_matches_reference_dense_masked(tag):
    """EXT channel skipping over a grouped conv2 on the GPU (dynamic-width GEMMs over
    the block-diagonal dense kernel) vs the REFERENCE's dense-masked output
    (golden) and the bf16-emulating oracle EXT; off by default like the reference."""
    R = _R()
    from paper_2308_15949_b200.errors import ShapeMismatch
    d, blk, ws, coarse, gran, x = _grouped_golden(tag)
    bw = R.BlockWeights(*ws)
    m = R.ChannelMask(coarse, np.repeat(coarse, gran, axis=1), gran)
    cfg = DynamicConfig(Paradigm.CHANNEL, channel_granularity=gran)
    with pytest.raises(ShapeMismatch):
        R.block_forward_sparse(x, bw, blk, cfg, m)
    y = R.block_forward_sparse(x, bw, blk, cfg, m, grouped_channel_ext=True)
    emu = O.block_forward_sparse(x, O.BlockWeights(*ws), blk, cfg, O.ChannelMask(coarse, m.expanded, gran),
                                 emulate_bf16=True, grouped_channel_ext=True)
    assert _rel(y, emu) <= BF16_TOL, _rel(y, emu)
    assert _rel(y, d[f"{tag}_y_dense"]) <= 1e-2


@pytest.mark.parametrize("tag", ["a", "b"])
def test_grouped_channel_ext_fp32_mode(tag, fp32_mode):
    """fp32 mode: <= 1e-5 vs the reference's fp64 dense-masked output."""
    R = fp32_mode
    d, blk, ws, coarse, gran, x = _grouped_golden(tag)
    m = R.ChannelMask(coarse, np.repeat(coarse, gran, axis=1), gran)
    cfg = DynamicConfig(Paradigm.CHANNEL, channel_granularity=gran)
    y = R.block_forward_sparse(x, R.BlockWeights(*ws), blk, cfg, m, grouped_channel_ext=True)
    assert _rel(y, d[f"{tag}_y_dense"]) <= 1e-5


@pytest.mark.parametrize("stage,r", [(2, 0.5), (3, 0.3), (4, 0.75)])
def test_regnet_grouped_channel_ext_block(stage, r):
    """RegNetY-1.6GF template blocks (group width 24) with exact-count channel masks."""
    R = _R()
    from paper_2308_15949_b200.zoo import build_network
    net = build_network("regnety-1.6gf")
    block = [b.block for b in net.blocks if b.stage == stage and b.index == 1][0]
    rng = np.random.default_rng(40 + stage)
    bw = R.make_block_weights(block, rng)
    n, cm = 2, block.conv2.out_channels
    ci = block.input_shape
    x = rng.standard_normal((n, ci.channels, ci.height, ci.width))
    coarse = np.zeros((n, cm), bool)
    for i in range(n):
        coarse[i, rng.permutation(cm)[: int(round(r * cm))]] = True
    m = R.ChannelMask(coarse, coarse, 1)
    cfg = DynamicConfig(Paradigm.CHANNEL, channel_granularity=1)
    y = R.block_forward_sparse(x, bw, block, cfg, m, grouped_channel_ext=True)
    emu = O.block_forward_sparse(x, O.BlockWeights(bw.w1, bw.w2, bw.w3, bw.w_down), block, cfg,
                                 O.ChannelMask(coarse, coarse, 1), emulate_bf16=True, grouped_channel_ext=True)
    assert _rel(y, emu) <= BF16_TOL, _rel(y, emu)
    yd = O.block_forward_dense_masked(x, O.BlockWeights(bw.w1, bw.w2, bw.w3, bw.w_down), block, cfg,
                                      O.ChannelMask(coarse, coarse, 1))
    assert _rel(y, yd) <= 1e-2


def test_conv2d_direct_matches_reference_golden():
    """conv2d_direct (`reference.py:52-69`) through the drop-in: the reference's own
    outputs (golden, incl. a grouped strided conv), its validation errors, and the
    CUDA-NHWC-in / CUDA-NHWC-out form."""
    import torch
    R = _R()
    from paper_2308_15949_b200.errors import ShapeMismatch
    a = np.load(G / "convs.npz")
    l1 = ConvLayerSpec(16, 8, 1)
    l2 = ConvLayerSpec(8, 8, 3, 2, 2)
    y1 = R.conv2d_direct(a["conv_x"], l1, a["bw_w1"])
    assert _rel(y1, a["conv1_y"]) <= 5e-3  # bf16 storage
    y2 = R.conv2d_direct(a["conv2_x"], l2, a["bw_w2"])
    assert _rel(y2, a["conv2_y"]) <= 5e-3
    with pytest.raises(ShapeMismatch):
        R.conv2d_direct(a["conv_x"][:, :8], l1, a["bw_w1"])
    with pytest.raises(ShapeMismatch):
        R.conv2d_direct(a["conv_x"], l1, a["bw_w1"][:4])
    from paper_2308_15949_b200 import device as D
    xd = D.to_device_nhwc(a["conv_x"])
    yd = R.conv2d_direct(xd, l1, a["bw_w1"])
    assert isinstance(yd, torch.Tensor) and yd.is_cuda and tuple(yd.shape) == (2, 10, 10, 8)
    np.testing.assert_array_equal(D.from_device_nhwc(yd, 8), y1)


def test_conv2d_direct_fp32_mode(fp32_mode):
    R = fp32_mode
    a = np.load(G / "convs.npz")
    assert _rel(R.conv2d_direct(a["conv_x"], ConvLayerSpec(16, 8, 1), a["bw_w1"]), a["conv1_y"]) <= 1e-5
    assert _rel(R.conv2d_direct(a["conv2_x"], ConvLayerSpec(8, 8, 3, 2, 2), a["bw_w2"]), a["conv2_y"]) <= 1e-5


def test_mirror_accepts_cuda_nhwc_tensors():
    """The drop-in's native form: CUDA NHWC tensors in, device
    tensors out, no host round trip; identical to the numpy NCHW form."""
    import torch
    R = _R()
    from paper_2308_15949_b200 import device as D
    from paper_2308_15949_b200.zoo import build_network
    block = [b.block for b in build_network("resnet50").blocks if b.stage == 3 and b.index == 1][0]
    rng = np.random.default_rng(3)
    bw = R.make_block_weights(block, rng)
    x = O.round_bf16(rng.standard_normal((2, 1024, 14, 14)))
    mw = rng.standard_normal((2, 1024, 1, 1)) / 32.0
    xd = D.to_device_nhwc(x)  # bf16 NHWC
    m_np = R.spatial_masker_forward(x, mw, 2)
    m_d = R.spatial_masker_forward(xd, mw, 2)
    assert isinstance(m_d.coarse, torch.Tensor) and m_d.coarse.is_cuda
    np.testing.assert_array_equal(m_d.coarse.cpu().numpy(), m_np.coarse)
    cfg = DynamicConfig(Paradigm.SPATIAL, spatial_granularity=2)
    y_np = R.block_forward_sparse(x, bw, block, cfg, m_np)
    y_d = R.block_forward_sparse(xd, bw, block, cfg, m_d)
    assert isinstance(y_d, torch.Tensor) and y_d.is_cuda and y_d.dtype == torch.bfloat16
    np.testing.assert_array_equal(D.from_device_nhwc(y_d, 1024), y_np)
    yd_np = R.block_forward_dense_masked(x, bw, block, cfg, m_np)
    np.testing.assert_array_equal(D.from_device_nhwc(R.block_forward_dense_masked(xd, bw, block, cfg, m_d), 1024),
                                  yd_np)
    lay = DynamicConfig(Paradigm.LAYER)
    dec = np.array([True, False])
    np.testing.assert_array_equal(
        D.from_device_nhwc(R.block_forward_sparse(xd, bw, block, lay, R.LayerMask(torch.tensor(dec).cuda())), 1024),
        R.block_forward_sparse(x, bw, block, lay, R.LayerMask(dec)))
    # channel masker + channel block on device tensors
    w1 = rng.standard_normal((16, 1024)) / 32.0
    w2 = rng.standard_normal((512, 16)) / 4.0
    cm_np = R.channel_masker_forward(x, (w1, w2), 1)
    cm_d = R.channel_masker_forward(xd, (w1, w2), 1)
    assert isinstance(cm_d.coarse, torch.Tensor)
    dv = (np.maximum(x.mean(axis=(2, 3)) @ w1.T, 0) @ w2.T).reshape(2, -1, 2)
    safe = np.abs(dv[..., 0] - dv[..., 1]) > 1e-4 * np.abs(dv).sum(-1)
    assert np.array_equal(cm_d.coarse.cpu().numpy()[safe], cm_np.coarse[safe])
    ccfg = DynamicConfig(Paradigm.CHANNEL, channel_granularity=1)
    np.testing.assert_array_equal(D.from_device_nhwc(R.block_forward_sparse(xd, bw, block, ccfg, cm_np), 1024),
                                  R.block_forward_sparse(x, bw, block, ccfg, cm_np))
    from paper_2308_15949_b200.errors import ShapeMismatch
    with pytest.raises(ShapeMismatch):
        R.block_forward_sparse(xd[..., :512], bw, block, cfg, m_d)
