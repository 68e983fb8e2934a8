"""Pin the CPU oracle (oracle/laud_oracle.py) to the real reference's outputs.

Fixtures in tests/golden/ were produced by tests/golden/make_golden.py from
/root/reference (dynlat 0.1.0).  No GPU needed.
"""
import json
from pathlib import Path

import numpy as np
import pytest

from oracle import laud_oracle as O
from paper_2308_15949_b200.core import BlockSpec, ConvLayerSpec, DynamicConfig, Paradigm, TensorShape
from paper_2308_15949_b200.errors import GranularityMismatch, MaskShapeMismatch, ShapeMismatch, SpecFileError

G = Path(__file__).resolve().parent / "golden"


def _meta():
    return json.loads((G / "equivalence.json").read_text())


@pytest.mark.parametrize("m", _meta(), ids=lambda m: m["key"])
def test_equivalence_case_matches_reference(m):
    arr = np.load(G / "equivalence.npz")
    case = O.EquivalenceCase(Paradigm(m["paradigm"]), m["channels"], m["height"], m["width"],
                             m["granularity"], m["seed"], m["tol"])
    block, mask, bw, x, cfg = O.case_inputs(case)
    sp = O.block_forward_sparse(x, bw, block, cfg, mask)
    de = O.block_forward_dense_masked(x, bw, block, cfg, mask)
    np.testing.assert_allclose(sp, arr[m["key"] + "__sparse"], rtol=0, atol=1e-11)
    np.testing.assert_allclose(de, arr[m["key"] + "__dense"], rtol=0, atol=1e-11)
    assert O.run_equivalence_case(case) < case.tolerance
    if case.paradigm is Paradigm.SPATIAL and mask.coarse.any():
        # fault hook must be caught, as in the reference (`reference.py:400-401`)
        assert O.run_equivalence_case(case, inject_fault=True) >= case.tolerance
        assert m["delta_fault"] >= case.tolerance


def test_default_cases_file_parses_like_reference():
    text = (G / "equivalence.json").read_text()
    cases = O.parse_cases_text("paradigm=spatial channels=8 height=16 width=16 granularity=4 seed=0 tol=1e-9\n"
                               "# comment\n\nparadigm=layer channels=8 height=8 width=8 seed=3\n")
    assert [c.paradigm for c in cases] == [Paradigm.SPATIAL, Paradigm.LAYER]
    assert cases[1].granularity == 1 and cases[1].tolerance == 1e-9
    with pytest.raises(SpecFileError):
        O.parse_cases_text("paradigm=spatial channels=x")
    assert text


def test_default_cases_suite_passes():
    for c in O.default_cases(per_paradigm=4):
        assert O.run_equivalence_case(c) < c.tolerance


def test_maskers_match_reference():
    a = np.load(G / "maskers.npz")
    for i in range(4):
        x, w, s = a[f"sp{i}_x"], a[f"sp{i}_w"], int(a[f"sp{i}_s"])
        m = O.spatial_masker_forward(x, w, s)
        assert np.array_equal(m.coarse, a[f"sp{i}_coarse"])
        assert np.array_equal(m.upsampled, a[f"sp{i}_up"])
        mt = O.spatial_masker_forward(x, w, s, mode="train", tau=0.7, rng=np.random.default_rng(99 + i))
        assert np.array_equal(mt.coarse, a[f"sp{i}_train_coarse"])
        np.testing.assert_allclose(mt.soft, a[f"sp{i}_train_soft"], rtol=1e-12)
        plan = O.build_gather_plan(m.coarse)
        assert np.array_equal(np.array(plan.indices, dtype=np.int64).reshape(-1, 3), a[f"sp{i}_plan"])
        assert plan.patch_count == int(m.coarse.sum())
        r, rd, dil = O.dilate_and_rates(m, 3)
        np.testing.assert_allclose([r, rd], a[f"sp{i}_rates"], rtol=0, atol=0)
        assert np.array_equal(dil, a[f"sp{i}_dil"])
        np.testing.assert_array_equal(O.fused_masker_weight_identity(w), a[f"sp{i}_fused"])
    x = np.random.default_rng(0).standard_normal((1, 4, 4, 4))
    assert O.spatial_masker_forward(x, np.ones((2, 4, 1, 1)), 2).coarse.all()
    assert a["tie_coarse"].all()
    for i in range(3):
        m = O.channel_masker_forward(a[f"ch{i}_x"], (a[f"ch{i}_w1"], a[f"ch{i}_w2"]), int(a[f"ch{i}_g"]))
        assert np.array_equal(m.coarse, a[f"ch{i}_coarse"])
        assert np.array_equal(m.expanded, a[f"ch{i}_exp"])
        mt = O.channel_masker_forward(a[f"ch{i}_x"], (a[f"ch{i}_w1"], a[f"ch{i}_w2"]), int(a[f"ch{i}_g"]),
                                      mode="train", tau=0.5, rng=np.random.default_rng(7 + i))
        assert np.array_equal(mt.coarse, a[f"ch{i}_train_coarse"])
        np.testing.assert_allclose(mt.soft, a[f"ch{i}_train_soft"], rtol=1e-12)
    np.testing.assert_allclose(O.gumbel_softmax_pair(a["gumbel_logits"], 0.3), a["gumbel_soft"], rtol=1e-13)


def test_weights_and_convs_match_reference():
    a = np.load(G / "convs.npz")
    blk = BlockSpec(conv1=ConvLayerSpec(16, 8, 1), conv2=ConvLayerSpec(8, 8, 3, 2, 2),
                    conv3=ConvLayerSpec(8, 32, 1), input_shape=TensorShape(16, 10, 10),
                    has_downsample=True)
    bw = O.make_block_weights(blk, np.random.default_rng(11))
    for k, v in (("w1", bw.w1), ("w2", bw.w2), ("w3", bw.w3), ("wd", bw.w_down)):
        np.testing.assert_array_equal(v, a["bw_" + k])
    np.testing.assert_allclose(O.conv2d_direct(a["conv_x"], blk.conv1, bw.w1), a["conv1_y"], atol=1e-12)
    np.testing.assert_allclose(O.conv2d_direct(a["conv2_x"], blk.conv2, bw.w2), a["conv2_y"], atol=1e-12)
    with pytest.raises(ShapeMismatch):
        O.conv2d_direct(a["conv_x"][:, :8], blk.conv1, bw.w1)


def test_config1_matches_reference():
    from paper_2308_15949_b200.zoo import build_network
    a = np.load(G / "config1.npz")
    net = build_network("resnet50")
    block = [b.block for b in net.blocks if b.stage == 3 and b.index == 1][0]
    rng = np.random.default_rng(0)
    bw = O.make_block_weights(block, rng)
    x = rng.standard_normal((1, 1024, 14, 14))
    mw = rng.standard_normal((2, 1024, 1, 1)) / np.sqrt(1024)
    m = O.block_spatial_mask(x, mw, block, 2)
    assert np.array_equal(m.coarse, a["coarse"])
    cfg = DynamicConfig(Paradigm.SPATIAL, spatial_granularity=2)
    y = O.block_forward_sparse(x, bw, block, cfg, m)
    np.testing.assert_allclose(y, a["y"], rtol=1e-6, atol=1e-5)


def test_spec_known_answers():
    # 8x8, S=4, only top-left patch, k=3: r=0.25, r_dil=25/64
    coarse = np.zeros((1, 2, 2), bool)
    coarse[0, 0, 0] = True
    m = O.SpatialMask(coarse, O.upsample_coarse(coarse, 4), 4)
    r, rd, _ = O.dilate_and_rates(m, 3)
    assert r == 0.25 and rd == 25 / 64
    # hidden width for C/G=512 -> 32
    assert O.masker_hidden_width(512) == 32 and O.masker_hidden_width(8) == 16
    # dominant logit -> all ones
    x = np.abs(np.random.default_rng(1).standard_normal((1, 3, 4, 4)))
    w = np.zeros((2, 3, 1, 1)); w[0] = 5.0
    assert O.spatial_masker_forward(x, w, 2).coarse.all()
    # equal logits, train, zero noise -> soft 0.5
    sm = O.spatial_masker_forward(x, np.ones((2, 3, 1, 1)), 2, mode="train", tau=0.3)
    np.testing.assert_allclose(sm.soft, 0.5)
    with pytest.raises(GranularityMismatch):
        O.spatial_masker_forward(x, w, 3)


def test_bf16_rounding():
    v = np.array([1.0, 1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8, -2.5, 3.14159265, 1e-30])
    r = O.round_bf16(v)
    assert r[0] == 1.0 and r[1] == 1.0 and r[2] == 1.0 + 2 ** -6 and r[3] == -2.5
    assert abs(r[4] - 3.140625) < 1e-12


def test_dilated_input_pixels_stride1_equals_output_dilation():
    rng = np.random.default_rng(3)
    blk = BlockSpec(conv1=ConvLayerSpec(8, 8, 1), conv2=ConvLayerSpec(8, 8, 3),
                    conv3=ConvLayerSpec(8, 8, 1), input_shape=TensorShape(8, 16, 16))
    coarse = rng.random((2, 4, 4)) < 0.4
    m = O.SpatialMask(coarse, O.upsample_coarse(coarse, 4), 4)
    _, _, dil = O.dilate_and_rates(m, 3)
    assert np.array_equal(O.dilated_input_pixels(coarse, blk, 4), dil)


def test_bf16_and_epilogue_extensions_reduce_to_reference():
    case = O.EquivalenceCase(Paradigm.SPATIAL, 16, 32, 32, 2, seed=1)
    block, mask, bw, x, cfg = O.case_inputs(case)
    ref = O.block_forward_sparse(x, bw, block, cfg, mask)
    ep = O.Epilogues()
    np.testing.assert_allclose(O.block_forward_sparse(x, bw, block, cfg, mask, epilogues=ep), ref, atol=1e-12)
    yb = O.block_forward_sparse(x, bw, block, cfg, mask, emulate_bf16=True)
    assert np.linalg.norm(yb - ref) / np.linalg.norm(ref) < 1e-2


def test_zoo_matches_reference():
    from paper_2308_15949_b200.zoo import build_network, parse_plan
    z = json.loads((G / "zoo.json").read_text())
    for name in ("resnet50", "resnet101", "regnety-400mf", "regnety-800mf"):
        net = build_network(name)
        got = [[b.stage, b.index, b.block.input_shape.channels, b.block.input_shape.height,
                b.block.conv1.out_channels, b.block.conv2.groups, b.block.conv3.out_channels,
                b.block.stride, int(b.block.has_downsample)] for b in net.blocks]
        assert got == z[name]
        if name.startswith("resnet"):
            assert list(parse_plan("4-2-2-1", net, Paradigm.SPATIAL).values) == z[name + "_plan_4-2-2-1"]
    net = build_network("regnety-1.6gf")
    assert [s.depth for s in net.stages] == [2, 6, 17, 2]
    assert [s.block_template.conv3.out_channels for s in net.stages] == [48, 120, 336, 888]
    assert net.blocks[0].block.conv2.groups == 2


def _grouped_case(d, tag):
    cin, cm, g, cout, hw, stride, gran = (int(v) for v in d[f"{tag}_geom"])
    blk = BlockSpec(conv1=ConvLayerSpec(cin, cm, 1), conv2=ConvLayerSpec(cm, cm, 3, stride, g),
                    conv3=ConvLayerSpec(cm, cout, 1), input_shape=TensorShape(cin, hw, hw),
                    has_downsample=stride > 1 or cin != cout)
    wd = d[f"{tag}_wd"] if f"{tag}_wd" in d else None
    bw = O.BlockWeights(d[f"{tag}_w1"], d[f"{tag}_w2"], d[f"{tag}_w3"], wd)
    coarse = d[f"{tag}_coarse"]
    mask = O.ChannelMask(coarse, np.repeat(coarse, gran, axis=1), gran)
    cfg = DynamicConfig(Paradigm.CHANNEL, channel_granularity=gran)
    return blk, bw, mask, cfg, d[f"{tag}_x"]


@pytest.mark.parametrize("tag", ["a", "b", "c"])
def test_grouped_channel_ext_matches_reference_dense_masked(tag):
    """EXT sparse channel skipping over a grouped conv2 reproduces the REFERENCE's
    dense-masked channel forward (fixture from dynlat) to 1e-9; without the EXT
    flag the oracle rejects it exactly like the reference's sparse executor."""
    d = np.load(G / "grouped_channel.npz")
    blk, bw, mask, cfg, x = _grouped_case(d, tag)
    assert bool(d[f"{tag}_sparse_rejected"])
    with pytest.raises(ShapeMismatch):
        O.block_forward_sparse(x, bw, blk, cfg, mask)
    y = O.block_forward_sparse(x, bw, blk, cfg, mask, grouped_channel_ext=True)
    np.testing.assert_allclose(y, d[f"{tag}_y_dense"], rtol=0, atol=1e-9)
    np.testing.assert_allclose(O.block_forward_dense_masked(x, bw, blk, cfg, mask), d[f"{tag}_y_dense"],
                               rtol=0, atol=1e-11)


def test_grouped_to_dense_is_block_diagonal():
    w = np.arange(6 * 2 * 3 * 3, dtype=float).reshape(6, 2, 3, 3) + 1
    dense = O.grouped_to_dense(w, 3)
    assert dense.shape == (6, 6, 3, 3)
    for o in range(6):
        g = o // 2
        np.testing.assert_array_equal(dense[o, 2 * g:2 * g + 2], w[o])
        assert not dense[o, :2 * g].any() and not dense[o, 2 * g + 2:].any()
