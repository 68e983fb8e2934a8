"""Whole-network parity: CUDA LaudNetwork vs the oracle network composer.

The GPU's own masker decisions are replayed in the oracle (decisions are
checked separately, tie-guarded, in test_gpu_parity), so the comparison
isolates the arithmetic: bf16 storage at the same points, fp32 vs fp64
accumulation.  Tolerance 2e-2 norm-relative on logits after 33 blocks of
bf16 storage (per-block gate is 1e-3; errors compound through depth).
"""
import numpy as np
import pytest

from oracle import laud_oracle as O

pytestmark = pytest.mark.gpu


def _net(arch, paradigm, plan="4-2-2-1", ratio=0.5):
    import torch
    from paper_2308_15949_b200.network import LaudNetwork, random_images
    net = LaudNetwork(arch, paradigm, plan, ratio, seed=0)
    img = random_images(2, seed=3)
    net.calibrate(img)
    rec = []
    logits = net.forward(img, record=rec)
    torch.cuda.synchronize()
    masks = [c.cpu().numpy() for _, c, _ in rec]
    return net, img.cpu().numpy(), logits[:, :1000].double().cpu().numpy(), masks


@pytest.mark.parametrize("arch,paradigm,plan", [
    ("resnet50", "spatial", "4-2-2-1"), ("resnet101", "spatial", "4-2-2-1"),
    ("resnet50", "spatial", "4-4-2-1"),  # BASELINE config 2's plan
    ("resnet50", "layer", "4-2-2-1"), ("resnet50", "static", "4-2-2-1"),
    ("resnet50", "channel", "1-1-1-1"), ("resnet50", "channel", "2-2-2-2"),
    ("regnety-1.6gf", "spatial", "4-4-2-1"), ("regnety-1.6gf", "layer", "4-4-2-1"),
    ("regnety-1.6gf", "static", "4-4-2-1"), ("regnety-400mf", "spatial", "4-4-2-1"),
    ("regnety-1.6gf", "channel", "1-1-1-1"), ("regnety-400mf", "channel", "2-2-2-2")])
def test_network_matches_oracle(arch, paradigm, plan):
    net, img, logits, masks = _net(arch, paradigm, plan)
    plan = tuple(net.plan)
    ref = O.network_forward(net.params, img, paradigm, plan, masks=masks or None, emulate_bf16=True)
    rel = np.linalg.norm(logits - ref) / np.linalg.norm(ref)
    assert rel < 2e-2, rel
    if paradigm in ("spatial", "channel"):
        r = np.mean([m.mean() for m in masks])
        assert 0.3 < r < 0.7


def test_channel_network_decisions_match_oracle_maskers():
    """Channel network: every block's device masker decisions (with its
    calibration bias) equal the oracle masker on the same block input."""
    net, img, logits, masks = _net("resnet50", "channel", "2-2-2-2")
    rec = []
    O.network_forward(net.params, img, "channel", tuple(net.plan), biases=net.masker_biases(),
                      emulate_bf16=True, record=rec)
    agree = np.mean([np.mean(np.asarray(m.coarse).reshape(-1) == g.reshape(-1).astype(bool))
                     for m, g in zip(rec, masks)])
    assert agree > 0.99, agree


def test_masker_conv3_fusion_matches_unfused():
    """The fused (conv3-epilogue dots) masker decides like the standalone one."""
    import torch
    from paper_2308_15949_b200.network import LaudNetwork, random_images
    net = LaudNetwork("resnet101", "spatial", "4-2-2-1", 0.5, seed=0)
    img = random_images(8, seed=4)
    net.calibrate(img)
    outs, masks = [], []
    for fuse in (False, True):
        net.fuse_masker = fuse
        rec = []
        outs.append(net.forward(img, record=rec)[:, :1000].float().cpu().numpy())
        torch.cuda.synchronize()
        masks.append([c.cpu().numpy() for _, c, _ in rec])
    agree = np.mean([np.mean(a == b) for a, b in zip(*masks)])
    assert agree > 0.999, agree
    rel = np.linalg.norm(outs[0] - outs[1]) / np.linalg.norm(outs[0])
    assert rel < 2e-2, rel


def test_pipelined_runner_matches_forward():
    """Streaming e2e path (upload overlapping the previous forward) returns, per
    batch, the same logits as a plain forward of that batch."""
    import torch
    from paper_2308_15949_b200.network import LaudNetwork, PipelinedRunner, random_images
    net = LaudNetwork("resnet50", "spatial", "4-4-2-1", 0.5, seed=0)
    imgs = [random_images(4, seed=s) for s in (11, 12, 13)]
    net.calibrate(imgs[0])
    ref = [net.forward(b)[:, :1000].float().cpu() for b in imgs]
    runner = PipelinedRunner(net, 4)
    host = [b.cpu().pin_memory() for b in imgs]
    out = torch.empty((3, 4, net.n_cls), dtype=torch.float32, pin_memory=True)
    ms = runner.run(host, out)
    assert ms > 0
    for i in range(3):
        assert torch.equal(out[i, :, :1000], ref[i])


@pytest.mark.parametrize("arch,paradigm,plan", [("resnet101", "spatial", "4-2-2-1"),
                                                ("regnety-1.6gf", "spatial", "4-4-2-1"),
                                                ("resnet50", "channel", "2-2-2-2"),
                                                ("regnety-400mf", "channel", "1-1-1-1")])
def test_network_is_bitwise_deterministic(arch, paradigm, plan):
    """No float atomics on any decision or pooling path (conv1-fused masker,
    channel-masker GAP, SE pooling): two forwards of the same images give
    identical logits, and so do two different batch compositions per image."""
    import torch
    from paper_2308_15949_b200.network import LaudNetwork, random_images
    net = LaudNetwork(arch, paradigm, plan, 0.5, seed=0)
    img = random_images(6, seed=9)
    net.calibrate(img)
    a = net.forward(img)[:, :1000].clone()
    b = net.forward(img)[:, :1000].clone()
    c = torch.cat([net.forward(img[:4])[:, :1000].clone(), net.forward(img[4:])[:, :1000].clone()])
    torch.cuda.synchronize()
    assert torch.equal(a, b)
    assert torch.equal(a, c)
