"""Host-side roofline accounting vs the oracle's restatement."""
import numpy as np
import pytest

from oracle import laud_oracle as O
from paper_2308_15949_b200 import roofline as RF
from paper_2308_15949_b200.zoo import build_network


@pytest.mark.parametrize("stage,index,s", [(1, 0, 4), (1, 1, 4), (2, 0, 2), (3, 1, 2), (4, 0, 1), (4, 1, 1)])
def test_spatial_block_flops_match_oracle(stage, index, s):
    net = build_network("resnet101")
    blk = [b.block for b in net.blocks if b.stage == stage and b.index == index][0]
    o = blk.output_shape
    rng = np.random.default_rng(stage + 10 * index)
    for r in (0.0, 0.2, 0.5, 1.0):
        coarse = rng.random((3, o.height // s, o.width // s)) < r
        got = RF.block_algorithmic(blk, "spatial", 3, coarse=coarse, s=s)
        ref = O.spatial_block_flops(blk, coarse, s)
        assert got["r_dil_in"] == pytest.approx(ref["r_dil_in"], abs=1e-12)
        assert got["flops"] == pytest.approx(ref["flops"], rel=1e-12)
        assert got["static_flops"] == pytest.approx(ref["static_flops"], rel=1e-12)


def test_channel_and_layer_credit():
    net = build_network("resnet101")
    blk = [b.block for b in net.blocks if b.stage == 3 and b.index == 1][0]
    n, cm = 4, blk.conv1.out_channels
    keep = np.zeros((n, cm), bool)
    keep[:, : cm // 2] = True
    st = RF.block_algorithmic(blk, "static", n)
    ch = RF.block_algorithmic(blk, "channel", n, keep=keep)
    f1, f2, f3, fd, _ = RF._convs(blk, n)
    gap = n * blk.input_shape.height * blk.input_shape.width * blk.input_shape.channels
    assert ch["flops"] == pytest.approx(2 * (0.5 * f1 + 0.25 * f2 + 0.5 * f3 + gap))
    lay = RF.block_algorithmic(blk, "layer", n, decisions=np.array([1, 0, 1, 0], bool))
    assert lay["flops"] == pytest.approx(2 * (0.5 * (f1 + f2 + f3) + gap))
    assert st["flops"] == pytest.approx(2 * (f1 + f2 + f3))


def test_grouped_conv_counts_group_width():
    net = build_network("regnety-1.6gf")
    blk = [b.block for b in net.blocks if b.stage == 3 and b.index == 1][0]
    g = blk.conv2.groups
    assert g > 1
    f1, f2, f3, fd, _ = RF._convs(blk, 1)
    o = blk.output_shape
    assert f2 == o.height * o.width * blk.conv2.out_channels * (blk.conv2.in_channels // g) * 9
