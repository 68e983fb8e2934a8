"""Generate golden fixtures from the REAL reference package (build container only).

Run from the repo root:  ``PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py``

Imports ``dynlat`` from ``/root/reference/pkg/src`` (read-only, never
copied) and records seeded inputs/outputs of every hot-path function into
``tests/golden/*.npz`` / ``*.json``.  The tests compare ``oracle/`` against
these files, so the oracle is pinned to the reference itself; the GPU box
(which has no /root/reference) only ever reads the committed fixtures.
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
OUT = Path(__file__).resolve().parent
sys.path.insert(0, REF)

from dynlat import core as rcore  # noqa: E402
from dynlat import reference as R  # noqa: E402
from dynlat import zoo as rzoo  # noqa: E402


def _case_key(c):
    return f"{c.paradigm.value}_c{c.channels}_h{c.height}_w{c.width}_g{c.granularity}_s{c.seed}"


def equivalence_cases():
    """Per case: sparse + dense outputs (float64) and the reference's max |delta|."""
    text = (Path(REF) / "dynlat/data/verify/default_cases.txt").read_text()
    cases = R.parse_cases_text(text) + R.default_cases(per_paradigm=6)
    arrays, meta = {}, []
    for c in cases:
        rng = np.random.default_rng(c.seed)
        block = R._case_block(c)
        n, mask = R._case_mask(c, block, rng)
        bw = R.make_block_weights(block, rng)
        x = rng.standard_normal((n, c.channels, c.height, c.width))
        if c.paradigm is rcore.Paradigm.SPATIAL:
            cfg = rcore.DynamicConfig(c.paradigm, spatial_granularity=c.granularity)
        elif c.paradigm is rcore.Paradigm.CHANNEL:
            cfg = rcore.DynamicConfig(c.paradigm, channel_granularity=c.granularity)
        else:
            cfg = rcore.DynamicConfig(c.paradigm)
        k = _case_key(c)
        if k in arrays or any(m["key"] == k for m in meta):
            continue
        arrays[k + "__sparse"] = R.block_forward_sparse(x, bw, block, cfg, mask)
        arrays[k + "__dense"] = R.block_forward_dense_masked(x, bw, block, cfg, mask)
        meta.append(dict(key=k, paradigm=c.paradigm.value, channels=c.channels,
                         height=c.height, width=c.width, granularity=c.granularity,
                         seed=c.seed, tol=c.tolerance,
                         delta=R.run_equivalence_case(c),
                         delta_fault=R.run_equivalence_case(c, inject_fault=True)))
    np.savez_compressed(OUT / "equivalence.npz", **arrays)
    (OUT / "equivalence.json").write_text(json.dumps(meta, indent=1))


def maskers():
    """Spatial/channel maskers (inference + seeded train), plans, dilation, identity."""
    rng = np.random.default_rng(1234)
    a = {}
    for i, (n, c, h, w, s) in enumerate([(2, 16, 8, 8, 2), (1, 64, 16, 16, 4),
                                         (3, 32, 12, 12, 3), (2, 8, 14, 14, 7)]):
        x = rng.standard_normal((n, c, h, w))
        wts = rng.standard_normal((2, c, 1, 1)) / np.sqrt(c)
        m = R.spatial_masker_forward(x, wts, s)
        a[f"sp{i}_x"], a[f"sp{i}_w"], a[f"sp{i}_s"] = x, wts, np.array(s)
        a[f"sp{i}_coarse"], a[f"sp{i}_up"] = m.coarse, m.upsampled
        mt = R.spatial_masker_forward(x, wts, s, mode="train", tau=0.7,
                                      rng=np.random.default_rng(99 + i))
        a[f"sp{i}_train_coarse"], a[f"sp{i}_train_soft"] = mt.coarse, mt.soft
        plan = R.build_gather_plan(m.coarse)
        a[f"sp{i}_plan"] = np.array(plan.indices, dtype=np.int64).reshape(-1, 3)
        r, rd, dil = R.dilate_and_rates(m, 3)
        a[f"sp{i}_rates"] = np.array([r, rd])
        a[f"sp{i}_dil"] = dil
        a[f"sp{i}_fused"] = R.fused_masker_weight_identity(wts)
    # tie: identical logit channels -> every cell computes (reference.py:183)
    x = rng.standard_normal((1, 4, 4, 4))
    wt = np.ones((2, 4, 1, 1))
    a["tie_coarse"] = R.spatial_masker_forward(x, wt, 2).coarse
    for i, (n, c, d, g) in enumerate([(2, 32, 8, 2), (3, 64, 16, 1), (1, 128, 32, 4)]):
        x = rng.standard_normal((n, c, 5, 5))
        h = R.masker_hidden_width(d)
        w1 = rng.standard_normal((h, c)) / np.sqrt(c)
        w2 = rng.standard_normal((2 * d, h)) / np.sqrt(h)
        m = R.channel_masker_forward(x, (w1, w2), g)
        a[f"ch{i}_x"], a[f"ch{i}_w1"], a[f"ch{i}_w2"], a[f"ch{i}_g"] = x, w1, w2, np.array(g)
        a[f"ch{i}_coarse"], a[f"ch{i}_exp"] = m.coarse, m.expanded
        mt = R.channel_masker_forward(x, (w1, w2), g, mode="train", tau=0.5,
                                      rng=np.random.default_rng(7 + i))
        a[f"ch{i}_train_coarse"], a[f"ch{i}_train_soft"] = mt.coarse, mt.soft
    lg = rng.standard_normal((5, 3, 2))
    a["gumbel_logits"] = lg
    a["gumbel_soft"] = R.gumbel_softmax_pair(lg, 0.3)
    np.savez_compressed(OUT / "maskers.npz", **a)


def block_weights_and_convs():
    """make_block_weights draw order + conv2d_direct (groups, stride) values."""
    rng = np.random.default_rng(5)
    a = {}
    blk = rcore.BlockSpec(conv1=rcore.ConvLayerSpec(16, 8, 1),
                          conv2=rcore.ConvLayerSpec(8, 8, 3, 2, 2),
                          conv3=rcore.ConvLayerSpec(8, 32, 1),
                          input_shape=rcore.TensorShape(16, 10, 10), has_downsample=True)
    bw = R.make_block_weights(blk, np.random.default_rng(11))
    a["bw_w1"], a["bw_w2"], a["bw_w3"], a["bw_wd"] = bw.w1, bw.w2, bw.w3, bw.w_down
    x = rng.standard_normal((2, 16, 10, 10))
    a["conv_x"] = x
    a["conv1_y"] = R.conv2d_direct(x, blk.conv1, bw.w1)
    h = rng.standard_normal((2, 8, 10, 10))
    a["conv2_x"] = h
    a["conv2_y"] = R.conv2d_direct(h, blk.conv2, bw.w2)
    np.savez_compressed(OUT / "convs.npz", **a)


def config1():
    """BASELINE config 1: R50 stage-3 block 1, 14x14x1024, S=2, batch 1, seed 0.

    Masker-driven mask (W ~ N(0,1)/sqrt(1024), wired on the output grid)
    and an exact-count mask (round(0.5*49) = 24 cells by permutation).
    Outputs stored as float32 (the GPU gate is 1e-3 relative).
    """
    net = rzoo.build_network("resnet50")
    block = [b.block for b in net.blocks if b.stage == 3 and b.index == 1][0]
    rng = np.random.default_rng(0)
    bw = R.make_block_weights(block, rng)
    x = rng.standard_normal((1, 1024, 14, 14))
    mw = rng.standard_normal((2, 1024, 1, 1)) / np.sqrt(1024)
    m = R.spatial_masker_forward(x, mw, 2)
    cfg = rcore.DynamicConfig(rcore.Paradigm.SPATIAL, spatial_granularity=2)
    y = R.block_forward_sparse(x, bw, block, cfg, m)
    perm = np.random.default_rng(1).permutation(49)[:round(0.5 * 49)]
    coarse = np.zeros(49, bool)
    coarse[perm] = True
    coarse = coarse.reshape(1, 7, 7)
    m2 = R.SpatialMask(coarse, R.upsample_coarse(coarse, 2), 2)
    y2 = R.block_forward_sparse(x, bw, block, cfg, m2)
    np.savez_compressed(OUT / "config1.npz", coarse=m.coarse, y=y.astype(np.float32),
                        coarse_exact=coarse, y_exact=y2.astype(np.float32))


def grouped_channel():
    """Channel skipping over a GROUPED conv2 (RegNet-style): the reference's sparse
    executor rejects it (`reference.py:405-406`), its dense-masked executor defines
    it (`reference.py:331-339`: conv2 input and output masked, groups kept).  The
    oracle's EXT sparse path is pinned to these dense-masked outputs."""
    a = {}
    rng = np.random.default_rng(21)
    for tag, (cin, cm, g, cout, hw, stride, gran) in {
            "a": (16, 24, 3, 32, 8, 1, 1), "b": (24, 48, 6, 48, 10, 2, 2), "c": (32, 32, 4, 32, 6, 1, 4)}.items():
        blk = rcore.BlockSpec(conv1=rcore.ConvLayerSpec(cin, cm, 1),
                              conv2=rcore.ConvLayerSpec(cm, cm, 3, stride, g),
                              conv3=rcore.ConvLayerSpec(cm, cout, 1),
                              input_shape=rcore.TensorShape(cin, hw, hw),
                              has_downsample=stride > 1 or cin != cout)
        bw = R.make_block_weights(blk, rng)
        n = 3
        x = rng.standard_normal((n, cin, hw, hw))
        d = cm // gran
        coarse = np.zeros((n, d), bool)
        for i in range(n):
            coarse[i, rng.permutation(d)[: max(1, d // 2 + i - 1)]] = True
        expanded = np.repeat(coarse, gran, axis=1)
        m = R.ChannelMask(coarse, expanded, gran)
        cfg = rcore.DynamicConfig(rcore.Paradigm.CHANNEL, channel_granularity=gran)
        a[f"{tag}_x"], a[f"{tag}_w1"], a[f"{tag}_w2"], a[f"{tag}_w3"] = x, bw.w1, bw.w2, bw.w3
        if bw.w_down is not None:
            a[f"{tag}_wd"] = bw.w_down
        a[f"{tag}_geom"] = np.array([cin, cm, g, cout, hw, stride, gran])
        a[f"{tag}_coarse"] = coarse
        a[f"{tag}_y_dense"] = R.block_forward_dense_masked(x, bw, blk, cfg, m)
        try:
            R.block_forward_sparse(x, bw, blk, cfg, m)
            a[f"{tag}_sparse_rejected"] = np.array(False)
        except Exception as exc:  # the reference's sparse executor refuses groups != 1
            a[f"{tag}_sparse_rejected"] = np.array(type(exc).__name__ == "ShapeMismatch")
    np.savez_compressed(OUT / "grouped_channel.npz", **a)


def zoo_shapes():
    out = {}
    for name in ("resnet50", "resnet101", "regnety-400mf", "regnety-800mf"):
        net = rzoo.build_network(name)
        out[name] = [[b.stage, b.index, b.block.input_shape.channels, b.block.input_shape.height,
                      b.block.conv1.out_channels, b.block.conv2.groups, b.block.conv3.out_channels,
                      b.block.stride, int(b.block.has_downsample)] for b in net.blocks]
        out[name + "_plan_4-2-2-1"] = list(rzoo.parse_plan("4-2-2-1", net, rcore.Paradigm.SPATIAL).values) \
            if name.startswith("resnet") else None
    (OUT / "zoo.json").write_text(json.dumps(out))


if __name__ == "__main__":
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    equivalence_cases()
    maskers()
    block_weights_and_convs()
    config1()
    grouped_channel()
    zoo_shapes()
    print("golden fixtures written to", OUT)
