"""Masker decisions of the PRODUCT path vs the CPU oracle (SURVEY §8(c) protocol).

The network runs the spatial masker fused into the dense conv1 (conv1's idle
producer warps dot every landed A stage with W0 - W1, one dot per input pixel;
the decision pass sums each cell's window in a fixed order) and the layer
masker as the standalone masker with S = H (`SPEC.md:41`).  These tests feed
both real bf16 block inputs and compare the decisions with the oracle's
`block_spatial_mask` (`reference.py:156-186` composed on the output grid)
evaluated in fp64 on the same bf16-rounded inputs:

  * zero flips on every cell with |d_bar + bias| > 1e-6 * sum|p_c||w_c|;
  * the near-tie count (cells inside the guard) is reported and must be tiny;
  * the active-cell list equals ``np.argwhere`` of the decisions;
  * two runs give bit-identical masks (no float atomics on the decision path).
"""
import numpy as np
import pytest

from oracle import laud_oracle as O

pytestmark = pytest.mark.gpu
TIE = 1e-6


def _block(arch, stage, index, bias=0.37):
    from paper_2308_15949_b200 import device as D
    from paper_2308_15949_b200.network import make_params
    D.require_cuda()
    bp = [b for b in make_params(arch, 0)["blocks"] if b["stage"] == stage and b["index"] == index][0]
    ep = D.Epilogue(s1=bp["s1"], b1=bp["b1"], relu1=True, s2=bp["s2"], b2=bp["b2"], relu2=True,
                    s3=bp["s3"], b3=bp["b3"], sd=bp["sd"], bd=bp["bd"], relu_out=True)
    db = D.DeviceBlock(bp["block"], bp["w1"], bp["w2"], bp["w3"], bp["wd"], ep, masker_w=bp["masker_w"],
                       masker_bias=bias, fold_scale=True)
    return bp, db


def _nchw64(x):
    """Device NHWC bf16 activation -> NCHW float64 numpy (exact)."""
    return x.float().cpu().numpy().transpose(0, 3, 1, 2).astype(np.float64)


def check_decisions(x64, masker_w, block, s, bias, got_coarse, tag=""):
    """§8(c) decision protocol; returns the near-tie count."""
    ref = O.block_spatial_mask(x64, masker_w, block, s, bias).coarse
    dbar, scale = O.masker_margin(x64, masker_w, block, s)
    safe = np.abs(dbar + bias) > TIE * scale
    got = np.asarray(got_coarse).reshape(ref.shape).astype(bool)
    flips = int((got[safe] != ref[safe]).sum())
    ties = int((~safe).sum())
    assert flips == 0, f"{tag}: {flips} decision flips outside the near-tie guard"
    assert ties <= max(2, ref.size // 1000), f"{tag}: {ties} near-tie cells"
    return ties


@pytest.mark.parametrize("arch,stage,index,s,n", [
    ("resnet101", 1, 0, 4, 8), ("resnet101", 1, 1, 4, 8), ("resnet101", 2, 0, 2, 16), ("resnet101", 2, 1, 2, 16),
    ("resnet101", 3, 0, 2, 32), ("resnet101", 3, 1, 2, 32), ("resnet101", 4, 0, 1, 32), ("resnet101", 4, 1, 1, 32),
    ("resnet101", 3, 1, 2, 128),
    # RegNetY-1.6GF: input widths 32 / 48 / 120 / 336 (not multiples of 64: zero-padded K tails)
    ("regnety-1.6gf", 1, 0, 4, 8), ("regnety-1.6gf", 2, 1, 4, 16), ("regnety-1.6gf", 3, 1, 2, 32),
    ("regnety-1.6gf", 4, 1, 1, 32)])
def test_conv1_fused_masker_matches_oracle(arch, stage, index, s, n):
    """R101 blocks (S = 4/2/1, strided b0 blocks, a CTA-pair-sized conv1 at n=128):
    the conv1-fused masker's decisions and cell list vs the fp64 oracle on the
    same bf16 input; masks bit-identical across two runs."""
    import torch
    from paper_2308_15949_b200 import device as D
    bp, db = _block(arch, stage, index)
    blk = bp["block"]
    h = blk.input_shape.height
    torch.manual_seed(stage * 100 + index)
    x = torch.randn(n, h, h, db.cin_p, device="cuda").relu_().bfloat16()
    o = blk.output_shape
    nc = n * (o.height // s) * (o.width // s)
    x64 = _nchw64(x)
    if arch != "resnet101":  # a bias that splits this block's cells (the fixed 0.37 suits the R101 blocks)
        dbar, _ = O.masker_margin(x64, bp["masker_w"], blk, s)
        db.masker_bias = float(-np.median(dbar) + 1e-3)
    masks, lists = [], []
    for _ in range(2):
        ws = D.Workspace()
        _, coarse, cells, counts = db.forward(x.clone(), "spatial", s, ws=ws, conv1_dense=True)
        torch.cuda.synchronize()
        masks.append(coarse[:nc].cpu().numpy().copy())
        cnt = int(counts.view(torch.int32)[0].item())
        lists.append(cells.view(torch.int32)[:cnt].cpu().numpy().copy())
    assert np.array_equal(masks[0], masks[1]), "decisions differ between identical runs"
    assert np.array_equal(lists[0], lists[1])
    assert 0.0 < masks[0].mean() < 1.0
    check_decisions(x64, bp["masker_w"], blk, s, db.masker_bias, masks[0], f"s{stage}b{index}")
    np.testing.assert_array_equal(lists[0], np.flatnonzero(masks[0]))


@pytest.mark.parametrize("stage,index,n", [(1, 1, 8), (2, 0, 16), (3, 1, 32), (4, 0, 32)])
def test_layer_masker_matches_oracle(stage, index, n):
    """Layer skipping: the masker with S = H (one cell per sample) on bf16 inputs."""
    import torch
    from paper_2308_15949_b200 import device as D
    bp, db = _block("resnet101", stage, index, bias=0.0)
    blk = bp["block"]
    h = blk.input_shape.height
    torch.manual_seed(7 + stage)
    x = torch.randn(n, h, h, db.cin_p, device="cuda").relu_().bfloat16()
    x64 = _nchw64(x)
    # centre the threshold on this batch so both decisions occur
    dbar, _ = O.masker_margin(x64, bp["masker_w"], blk, blk.output_shape.height)
    db.masker_bias = float(-np.median(dbar)) + 1e-3 * float(np.std(dbar))
    got = []
    for _ in range(2):
        _, coarse, _, _ = db.forward(x.clone(), "layer", 0, ws=D.Workspace())
        torch.cuda.synchronize()
        got.append(coarse[:n].cpu().numpy().copy())
    assert np.array_equal(got[0], got[1])
    assert 0 < got[0].sum() < n
    check_decisions(x64, bp["masker_w"], blk, blk.output_shape.height, db.masker_bias, got[0], "layer")


def _capture_block_inputs(net, images):
    """Run the network once; per dynamic block, its bf16 input and decisions."""
    import torch
    from paper_2308_15949_b200 import device as D
    seen = []
    orig = D.DeviceBlock.forward

    def hooked(db, x, paradigm="spatial", s=1, **kw):
        xin = x.clone()
        out = orig(db, x, paradigm, s, **kw)
        seen.append((db, xin, paradigm, s, out[1]))
        return out

    D.DeviceBlock.forward = hooked
    try:
        rec = []
        net.forward(images, record=rec)
    finally:
        D.DeviceBlock.forward = orig
    torch.cuda.synchronize()
    return seen, rec


@pytest.mark.parametrize("arch,paradigm,plan,n", [("resnet101", "spatial", "4-2-2-1", 8),
                                                  ("resnet50", "spatial", "4-4-2-1", 8),
                                                  ("resnet50", "layer", "4-2-2-1", 16)])
def test_network_decisions_match_oracle(arch, paradigm, plan, n):
    """Every block of the network (default schedule: conv1-fused masker, calibrated
    biases) decides like the oracle masker on that block's actual bf16 input."""
    from paper_2308_15949_b200.network import LaudNetwork, random_images
    net = LaudNetwork(arch, paradigm, plan, 0.5, seed=0)
    net.calibrate(random_images(n, seed=21))  # calibration batch != checked batch
    seen, rec = _capture_block_inputs(net, random_images(n, seed=22))
    assert len(seen) == len(net.slots)
    ties = 0
    for (db, xin, para, s, coarse), slot, (rslot, rcoarse, _) in zip(seen, net.slots, rec):
        blk = db.block
        ss = s if para == "spatial" else blk.output_shape.height
        cells = n * (blk.output_shape.height // ss) * (blk.output_shape.width // ss)
        mw = [b for b in net.params["blocks"] if b["stage"] == slot.stage and b["index"] == slot.index][0]["masker_w"]
        ties += check_decisions(_nchw64(xin), mw, blk, ss, db.masker_bias, rcoarse.cpu().numpy()[:cells],
                                f"s{slot.stage}b{slot.index}")
    print(f"{arch} {paradigm}: near-tie cells {ties}")
