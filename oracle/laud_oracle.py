"""CPU oracle for the LAUDNet mask-and-compute path — TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference's float64 executor
(``dynlat.reference``, `pkg/src/dynlat/reference.py`).  It is the checker
for the CUDA path, never the product: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline / ``--impl
reference`` leg may import it.  The product package never imports it and
fails loudly without its CUDA library.

Parity pinning: ``tests/golden/make_golden.py`` imports the real reference
from ``/root/reference/pkg/src`` (in the build container only) and writes
seeded inputs/outputs to ``tests/golden/*.npz``; ``tests/test_oracle.py``
checks every function here against those fixtures (and against the
reference's own 9-case ``default_cases.txt`` equivalence suite, tolerance
1e-9), so the oracle is pinned to the reference, not just to itself.

Layout follows the reference: NCHW float64, masks as bool arrays.  Every
function cites the reference lines it restates.  Extensions the reference
lacks (flagged EXT) are compositions the GPU path needs a checker for:
bf16 rounding emulation, folded-BN/ReLU epilogues (default off = reference
semantics), masker->block wiring on the output grid, a network composer, and
sparse channel skipping over grouped conv2 (pinned to the reference's own
dense-masked outputs, tests/golden/grouped_channel.npz).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

from paper_2308_15949_b200.core import (BlockSpec, ConvLayerSpec, DynamicConfig,
                                        Paradigm, TensorShape)
from paper_2308_15949_b200.errors import (GranularityMismatch, MaskShapeMismatch,
                                          ShapeMismatch, SpecFileError)

# ---------------------------------------------------------------------------
# numerics helpers
# ---------------------------------------------------------------------------


def round_bf16(a: np.ndarray) -> np.ndarray:
    """EXT: round to the nearest bfloat16 (ties to even), returned as float64.

    Matches ``__float2bfloat16_rn`` on the device: float64 -> float32 (RN),
    then the upper 16 bits with round-to-nearest-even on the dropped half.
    """
    f = np.ascontiguousarray(a, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    u = (u + 0x7FFF + lsb) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


# ---------------------------------------------------------------------------
# convolution (reference.py:32-69)
# ---------------------------------------------------------------------------


def conv_raw(x: np.ndarray, w: np.ndarray, stride: int = 1, pad: int = 0,
             groups: int = 1) -> np.ndarray:
    """Direct convolution, zero padding ``pad`` (restates `reference.py:32-49`).

    Sum over taps of a channel contraction on the strided, shifted input;
    groups split input/output channels into contiguous blocks (`:43-49`).
    """
    n, c, h, wd = x.shape
    co, cig, kh, kw = w.shape
    if c != cig * groups:
        raise ShapeMismatch(f"input has {c} channels, weights expect {cig * groups}")
    if pad:
        x = np.pad(x, ((0, 0), (0, 0), (pad, pad), (pad, pad)))
    ho = (x.shape[2] - kh) // stride + 1
    wo = (x.shape[3] - kw) // stride + 1
    out = np.zeros((n, co, ho, wo), dtype=np.result_type(x, w))
    cog = co // groups
    for g in range(groups):
        xg = x[:, g * cig:(g + 1) * cig]
        wg = w[g * cog:(g + 1) * cog]
        acc = out[:, g * cog:(g + 1) * cog]
        for dy in range(kh):
            for dx in range(kw):
                win = xg[:, :, dy:dy + stride * (ho - 1) + 1:stride,
                         dx:dx + stride * (wo - 1) + 1:stride]
                acc += np.einsum("nchw,oc->nohw", win, wg[:, :, dy, dx], optimize=True)
    return out


def conv2d_direct(x: np.ndarray, layer: ConvLayerSpec, weights: np.ndarray) -> np.ndarray:
    """Validated conv with k//2 padding (restates `reference.py:52-69`)."""
    if x.ndim != 4:
        raise ShapeMismatch("expected (N, C, H, W) input")
    if x.shape[1] != layer.in_channels:
        raise ShapeMismatch(f"input has {x.shape[1]} channels, layer expects "
                            f"{layer.in_channels}")
    want = (layer.out_channels, layer.in_channels // layer.groups, layer.kernel, layer.kernel)
    if weights.shape != want:
        raise ShapeMismatch(f"weights {weights.shape} != expected {want}")
    return conv_raw(x, weights, layer.stride, layer.kernel // 2, layer.groups)


# ---------------------------------------------------------------------------
# masks (reference.py:77-139)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class SpatialMask:
    """coarse (N, H/S, W/S) + S-fold upsampled (N, H, W) (`reference.py:77-93`)."""
    coarse: np.ndarray
    upsampled: np.ndarray
    granularity: int
    soft: Optional[np.ndarray] = None

    @property
    def rate(self) -> float:
        return float(self.upsampled.mean())


@dataclass(frozen=True)
class ChannelMask:
    """coarse (N, D) + G-fold expanded (N, D*G) (`reference.py:96-107`)."""
    coarse: np.ndarray
    expanded: np.ndarray
    granularity: int
    soft: Optional[np.ndarray] = None

    @property
    def rate(self) -> float:
        return float(self.expanded.mean())


@dataclass(frozen=True)
class LayerMask:
    """one decision per sample (`reference.py:110-119`)."""
    decisions: np.ndarray
    soft: Optional[np.ndarray] = None

    @property
    def rate(self) -> float:
        return float(self.decisions.mean())


@dataclass(frozen=True)
class GatherPlan:
    """(n, i, j) of active cells, row-major ascending (`reference.py:122-130`)."""
    indices: tuple

    @property
    def patch_count(self) -> int:
        return len(self.indices)


def build_gather_plan(coarse: np.ndarray) -> GatherPlan:
    """Row-major list of True cells == np.argwhere order (`reference.py:133-135`)."""
    flat = np.flatnonzero(np.asarray(coarse).reshape(-1))
    idx = np.stack(np.unravel_index(flat, coarse.shape), axis=1) if flat.size else \
        np.zeros((0, 3), dtype=np.int64)
    return GatherPlan(tuple((int(a), int(b), int(c)) for a, b, c in idx))


def upsample_coarse(coarse: np.ndarray, s: int) -> np.ndarray:
    """Nearest-neighbour S x S replication (`reference.py:138-139`)."""
    return np.repeat(np.repeat(coarse, s, axis=-2), s, axis=-1)


def gumbel_softmax_pair(logits, tau, noise=None):
    """P(compute) = 1 / (1 + exp((z1 - z0)/tau)) (`reference.py:142-153`)."""
    if tau <= 0:
        raise ValueError("tau must be positive")
    z = logits if noise is None else logits + noise
    return 1.0 / (1.0 + np.exp((z[..., 1] - z[..., 0]) / tau))


def _decide(logits, mode, tau, rng):
    soft = None
    if mode == "train":
        noise = rng.gumbel(size=logits.shape) if rng is not None else None
        soft = gumbel_softmax_pair(logits, tau, noise)
        z = logits if noise is None else logits + noise
        return z[..., 0] >= z[..., 1], soft
    if mode == "inference":
        return logits[..., 0] >= logits[..., 1], soft
    raise ValueError(f"unknown mode {mode!r}")


def spatial_masker_forward(x, weights, s, mode="inference", tau=None, rng=None) -> SpatialMask:
    """Pool S x S, 1x1 conv to 2 logits, compute wins ties (`reference.py:156-186`)."""
    n, c, h, w = x.shape
    if h % s or w % s:
        raise GranularityMismatch(f"S={s} does not divide {h}x{w}")
    pooled = x.reshape(n, c, h // s, s, w // s, s).mean(axis=(3, 5))
    logits = np.einsum("nchw,oc->nhwo", pooled, weights.reshape(2, c))
    coarse, soft = _decide(logits, mode, tau, rng)
    return SpatialMask(coarse, upsample_coarse(coarse, s), s, soft)


def masker_hidden_width(d: int) -> int:
    """max(D // 16, 16) (`reference.py:221-223`)."""
    return max(d // 16, 16)


def channel_masker_forward(x, weights, g, mode="inference", tau=None, rng=None,
                           bias: float = 0.0) -> ChannelMask:
    """GAP -> relu(W1) -> W2 -> interleaved (keep, skip) pairs (`reference.py:189-218`).

    ``bias`` (EXT, default 0 = reference) is added to the keep logit l0, i.e.
    to every gap l0 - l1 (the device masker's calibration bias).
    """
    w1, w2 = weights
    hidden_w, c = w1.shape
    if x.shape[1] != c:
        raise ShapeMismatch(f"input has {x.shape[1]} channels, masker expects {c}")
    if w2.shape[1] != hidden_w or w2.shape[0] % 2:
        raise ShapeMismatch("second MLP layer must map hidden -> 2*D")
    d = w2.shape[0] // 2
    hid = np.maximum(x.mean(axis=(2, 3)) @ w1.T, 0.0)
    logits = (hid @ w2.T).reshape(-1, d, 2)
    if bias:
        logits = logits.copy()
        logits[..., 0] += bias
    coarse, soft = _decide(logits, mode, tau, rng)
    return ChannelMask(coarse, np.repeat(coarse, g, axis=1), g, soft)


def _dilate_square(m: np.ndarray, radius: int) -> np.ndarray:
    """Binary dilation by a (2r+1)^2 square, clipped at borders (scipy semantics)."""
    h, w = m.shape
    p = np.pad(m, radius)
    out = np.zeros_like(m)
    for dy in range(2 * radius + 1):
        for dx in range(2 * radius + 1):
            out |= p[dy:dy + h, dx:dx + w]
    return out


def dilate_and_rates(mask: SpatialMask, kernel: int):
    """(r, r_dil, dilated) on the upsampled output-grid mask (`reference.py:226-241`)."""
    if kernel % 2 == 0:
        raise ValueError("kernel must be odd")
    up = mask.upsampled
    if kernel == 1:
        dil = up.copy()
    else:
        dil = np.stack([_dilate_square(m, (kernel - 1) // 2) for m in up])
    return float(up.mean()), float(dil.mean()), dil


def fused_masker_weight_identity(weights: np.ndarray) -> np.ndarray:
    """W0 - W1 as a single decision channel (`reference.py:244-253`)."""
    if weights.shape[0] != 2 or weights.shape[-2:] != (1, 1):
        raise ShapeMismatch("expected (2, C, 1, 1) masker weights")
    return weights[0:1] - weights[1:2]


# ---------------------------------------------------------------------------
# block weights (reference.py:261-298)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class BlockWeights:
    """Bias-free block weights (`reference.py:261-268`)."""
    w1: np.ndarray
    w2: np.ndarray
    w3: np.ndarray
    w_down: Optional[np.ndarray] = None


def down_layer(block: BlockSpec) -> ConvLayerSpec:
    """1x1 projection at the block stride (`reference.py:289-292`)."""
    return ConvLayerSpec(block.input_shape.channels, block.conv3.out_channels, 1, block.stride)


def make_block_weights(block: BlockSpec, rng: np.random.Generator) -> BlockWeights:
    """N(0,1)/sqrt(fan_in); draw order w_down, w1, w2, w3 (`reference.py:271-286`)."""

    def draw(layer):
        cig = layer.in_channels // layer.groups
        shape = (layer.out_channels, cig, layer.kernel, layer.kernel)
        return rng.standard_normal(shape) / np.sqrt(cig * layer.kernel ** 2)

    w_down = None
    if block.has_downsample:
        d = down_layer(block)
        w_down = rng.standard_normal((d.out_channels, d.in_channels, 1, 1)) / np.sqrt(d.in_channels)
    w1 = draw(block.conv1)
    w2 = draw(block.conv2)
    w3 = draw(block.conv3)
    return BlockWeights(w1, w2, w3, w_down)


# ---------------------------------------------------------------------------
# EXT: folded BN + activation epilogues (default: identity = reference)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class Epilogues:
    """EXT: per-conv folded BN (scale, bias) and ReLU flags.

    ``None`` everywhere reproduces the reference's linear block
    (`reference.py:7-8`).  The GPU kernels apply scale*acc + bias, then ReLU,
    at exactly these points; out-of-image halo pixels stay exact zeros after
    the conv1 epilogue (the oracle pads *after* conv1, `reference.py:385-386`).
    """
    s1: Optional[np.ndarray] = None
    b1: Optional[np.ndarray] = None
    relu1: bool = False
    s2: Optional[np.ndarray] = None
    b2: Optional[np.ndarray] = None
    relu2: bool = False
    s3: Optional[np.ndarray] = None
    b3: Optional[np.ndarray] = None
    sd: Optional[np.ndarray] = None
    bd: Optional[np.ndarray] = None
    relu_out: bool = False
    # EXT squeeze-excitation after conv2 (RegNetY; `core.py:195` se_hidden
    # = C_mid // se_reduction): s = sigmoid(W2 relu(W1 mean(h2) + b1) + b2),
    # h2 *= s per channel.  Under spatial sparsity the mean runs over the
    # sample's active patches only (the pooling `latency.py:428-430` models);
    # the reference executor itself never reads se_reduction.
    se_w1: Optional[np.ndarray] = None  # [se_hidden, C_mid]
    se_b1: Optional[np.ndarray] = None
    se_w2: Optional[np.ndarray] = None  # [C_mid, se_hidden]
    se_b2: Optional[np.ndarray] = None


def _se_scale(pooled, ep):
    """EXT SE gate from pooled h2 (..., C): sigmoid(W2 relu(W1 p + b1) + b2)."""
    hid = np.maximum(pooled @ ep.se_w1.T + ep.se_b1, 0.0)
    return 1.0 / (1.0 + np.exp(-(hid @ ep.se_w2.T + ep.se_b2)))


def _affine(y, s, b, relu):
    if s is not None:
        y = y * s.reshape(1, -1, 1, 1)
    if b is not None:
        y = y + b.reshape(1, -1, 1, 1)
    if relu:
        y = np.maximum(y, 0.0)
    return y


# ---------------------------------------------------------------------------
# block forward (reference.py:295-436)
# ---------------------------------------------------------------------------


def skip_path(x, block, bw, ep: Optional[Epilogues] = None, rnd=None):
    """Identity copy or dense 1x1/stride projection (`reference.py:295-298`)."""
    if block.has_downsample:
        y = conv2d_direct(x, down_layer(block), bw.w_down)
        if ep is not None:
            y = _affine(y, ep.sd, ep.bd, False)
        return rnd(y) if rnd else y
    return x.copy()


def check_spatial_mask(mask: SpatialMask, block: BlockSpec, n: int):
    """Mask lives on the OUTPUT grid (`reference.py:301-310`)."""
    out = block.output_shape
    s = mask.granularity
    if out.height % s or out.width % s:
        raise GranularityMismatch(f"S={s} does not divide {out.height}x{out.width}")
    want = (n, out.height // s, out.width // s)
    if mask.coarse.shape != want:
        raise MaskShapeMismatch(f"coarse mask {mask.coarse.shape} != {want}")
    if mask.upsampled.shape != (n, out.height, out.width):
        raise MaskShapeMismatch("upsampled mask does not match the output feature")


def block_forward_dense_masked(x, bw: BlockWeights, block: BlockSpec, cfg: DynamicConfig,
                               mask) -> np.ndarray:
    """Training-style dense compute times masks (`reference.py:313-353`)."""
    n = x.shape[0]
    skip = skip_path(x, block, bw)
    p = cfg.paradigm
    if p is Paradigm.SPATIAL:
        check_spatial_mask(mask, block, n)
        y = conv2d_direct(conv2d_direct(conv2d_direct(x, block.conv1, bw.w1),
                                        block.conv2, bw.w2), block.conv3, bw.w3)
        return skip + mask.upsampled[:, None].astype(x.dtype) * y
    if p is Paradigm.CHANNEL:
        m = mask.expanded
        if m.shape != (n, block.conv2.out_channels):
            raise MaskShapeMismatch(f"channel mask {m.shape} != {(n, block.conv2.out_channels)}")
        m = m[:, :, None, None].astype(x.dtype)
        y = conv2d_direct(x, block.conv1, bw.w1)
        y = conv2d_direct(y * m, block.conv2, bw.w2)
        y = conv2d_direct(y * m, block.conv3, bw.w3)
        return skip + y
    if p is Paradigm.LAYER:
        d = mask.decisions
        if d.shape != (n,):
            raise MaskShapeMismatch(f"layer mask {d.shape} != {(n,)}")
        y = conv2d_direct(conv2d_direct(conv2d_direct(x, block.conv1, bw.w1),
                                        block.conv2, bw.w2), block.conv3, bw.w3)
        return skip + d[:, None, None, None].astype(x.dtype) * y
    y = conv2d_direct(conv2d_direct(conv2d_direct(x, block.conv1, bw.w1),
                                    block.conv2, bw.w2), block.conv3, bw.w3)
    return skip + y


def _spatial_sparse(x, bw, block, mask, ep, rnd, misplace_first):
    """Gather halos -> conv2 valid -> conv3 -> scatter-add (`reference.py:378-403`).

    The per-patch loop of the reference is vectorised over patches: all halo
    windows are gathered into one stack, convolved together, and scattered
    back in plan order (scatter-adds of distinct cells commute).
    """
    n = x.shape[0]
    out = block.output_shape
    s = mask.granularity
    st = block.stride
    k = block.conv2.kernel
    pad = k // 2
    halo = (s - 1) * st + k
    skip = skip_path(x, block, bw, ep, rnd)
    h1 = conv2d_direct(x, block.conv1, bw.w1)
    if ep is not None:
        h1 = _affine(h1, ep.s1, ep.b1, ep.relu1)
    if rnd:
        h1 = rnd(h1)
    h1p = np.pad(h1, ((0, 0), (0, 0), (pad, pad), (pad, pad)))
    plan = build_gather_plan(mask.coarse)
    result = skip
    if plan.patch_count == 0:
        if ep is not None and ep.relu_out:
            result = np.maximum(result, 0.0)
        return result
    idx = np.array(plan.indices)
    stack = np.stack([h1p[ni, :, ci * s * st:ci * s * st + halo, cj * s * st:cj * s * st + halo]
                      for ni, ci, cj in idx])
    y = conv_raw(stack, bw.w2, stride=st, pad=0, groups=block.conv2.groups)
    if ep is not None:
        y = _affine(y, ep.s2, ep.b2, ep.relu2)
    if rnd:
        y = rnd(y)
    if ep is not None and ep.se_w1 is not None:  # EXT SE over each sample's active patches
        for ni in np.unique(idx[:, 0]):
            sel = idx[:, 0] == ni
            gate = _se_scale(y[sel].transpose(1, 0, 2, 3).reshape(y.shape[1], -1).mean(axis=1), ep)
            y[sel] = y[sel] * gate.reshape(1, -1, 1, 1)
        if rnd:
            y = rnd(y)
    y = conv_raw(y, bw.w3)
    if ep is not None:
        y = _affine(y, ep.s3, ep.b3, False)
    for p_idx, (ni, ci, cj) in enumerate(idx):
        r0, c0 = ci * s, cj * s
        if misplace_first and p_idx == 0:
            r0 = (r0 + s) % out.height
        result[ni, :, r0:r0 + s, c0:c0 + s] += y[p_idx]
    if ep is not None and ep.relu_out:
        result = np.maximum(result, 0.0)
    return result


def grouped_to_dense(w: np.ndarray, groups: int) -> np.ndarray:
    """EXT: [C_out, C_in/g, k, k] grouped kernel -> [C_out, C_in, k, k] block-diagonal
    dense kernel (zeros between groups; group layout of `reference.py:43-49`)."""
    co, cig, kh, kw = w.shape
    cog = co // groups
    out = np.zeros((co, cig * groups, kh, kw), dtype=w.dtype)
    for g in range(groups):
        out[g * cog:(g + 1) * cog, g * cig:(g + 1) * cig] = w[g * cog:(g + 1) * cog]
    return out


def block_forward_sparse(x, bw: BlockWeights, block: BlockSpec, cfg: DynamicConfig, mask,
                         _misplace_first_patch: bool = False,
                         epilogues: Optional[Epilogues] = None,
                         emulate_bf16: bool = False,
                         grouped_channel_ext: bool = False) -> np.ndarray:
    """Inference-style forward computing only what the mask selects.

    Restates `reference.py:356-436`.  ``epilogues`` (EXT) adds folded
    BN/ReLU; ``emulate_bf16`` (EXT) rounds to bf16 at the points where the
    GPU kernels store bf16 (inputs, weights, h1, h2, skip, output), so bf16
    GPU results can be gated tightly.  Both default to reference semantics.
    """
    rnd = round_bf16 if emulate_bf16 else None
    if rnd:
        x = rnd(x)
        bw = BlockWeights(rnd(bw.w1), rnd(bw.w2), rnd(bw.w3),
                          None if bw.w_down is None else rnd(bw.w_down))
    n = x.shape[0]
    p = cfg.paradigm
    if p is Paradigm.SPATIAL:
        check_spatial_mask(mask, block, n)
        r = _spatial_sparse(x, bw, block, mask, epilogues, rnd, _misplace_first_patch)
        return rnd(r) if rnd else r
    if p is Paradigm.CHANNEL:
        w2 = bw.w2
        if block.conv2.groups != 1:
            if not grouped_channel_ext:
                raise ShapeMismatch("sparse channel execution requires groups == 1")
            # EXT: the grouped conv2 as its block-diagonal dense kernel; W2[sel][:, sel]
            # then keeps exactly the kept-input x kept-output links of each group, the
            # sparse form of the reference's dense-masked channel forward
            # (`reference.py:331-339`, which masks conv2's input and output)
            w2 = grouped_to_dense(w2, block.conv2.groups)
        m = mask.expanded
        if m.shape != (n, block.conv2.out_channels):
            raise MaskShapeMismatch(f"channel mask {m.shape} != {(n, block.conv2.out_channels)}")
        result = skip_path(x, block, bw, epilogues, rnd)
        ep = epilogues
        for ni in range(n):
            sel = np.flatnonzero(m[ni])
            if sel.size == 0:
                # `reference.py:415-416` skips the sample; with the EXT epilogue the
                # dense-masked conv path still contributes conv3's bias (conv3 of
                # an all-zero input is 0, + b3), which is what the device computes
                if ep is not None and ep.b3 is not None:
                    result[ni] += ep.b3.reshape(-1, 1, 1)
                continue
            xi = x[ni:ni + 1]
            h1 = conv_raw(xi, bw.w1[sel])
            if ep is not None:
                h1 = _affine(h1, None if ep.s1 is None else ep.s1[sel],
                             None if ep.b1 is None else ep.b1[sel], ep.relu1)
            if rnd:
                h1 = rnd(h1)
            h2 = conv_raw(h1, w2[np.ix_(sel, sel)], stride=block.conv2.stride,
                          pad=block.conv2.kernel // 2)
            if ep is not None:
                h2 = _affine(h2, None if ep.s2 is None else ep.s2[sel],
                             None if ep.b2 is None else ep.b2[sel], ep.relu2)
            if rnd:
                h2 = rnd(h2)
            if ep is not None and ep.se_w1 is not None:
                # EXT SE under channel skipping: the dense-masked h2 is zero on the
                # dropped channels, so the pooled vector is the kept channels' means
                # scattered into C_m zeros; the gate multiplies the kept channels
                pooled = np.zeros(block.conv2.out_channels)
                pooled[sel] = h2[0].mean(axis=(1, 2))
                h2 = h2 * _se_scale(pooled, ep)[sel].reshape(1, -1, 1, 1)
                if rnd:
                    h2 = rnd(h2)
            h3 = conv_raw(h2, bw.w3[:, sel])
            if ep is not None:
                h3 = _affine(h3, ep.s3, ep.b3, False)
            result[ni] += h3[0]
        if epilogues is not None and epilogues.relu_out:
            result = np.maximum(result, 0.0)
        return rnd(result) if rnd else result
    if p is Paradigm.LAYER:
        d = mask.decisions
        if d.shape != (n,):
            raise MaskShapeMismatch(f"layer mask {d.shape} != {(n,)}")
        result = skip_path(x, block, bw, epilogues, rnd)
        ep = epilogues
        for ni in np.flatnonzero(d):
            y = conv2d_direct(x[ni:ni + 1], block.conv1, bw.w1)
            if ep is not None:
                y = _affine(y, ep.s1, ep.b1, ep.relu1)
            if rnd:
                y = rnd(y)
            y = conv2d_direct(y, block.conv2, bw.w2)
            if ep is not None:
                y = _affine(y, ep.s2, ep.b2, ep.relu2)
            if rnd:
                y = rnd(y)
            if ep is not None and ep.se_w1 is not None:  # EXT SE (whole image)
                y = y * _se_scale(y.mean(axis=(2, 3))[0], ep).reshape(1, -1, 1, 1)
                if rnd:
                    y = rnd(y)
            y = conv2d_direct(y, block.conv3, bw.w3)
            if ep is not None:
                y = _affine(y, ep.s3, ep.b3, False)
            result[ni] += y[0]
        if epilogues is not None and epilogues.relu_out:
            result = np.maximum(result, 0.0)
        return rnd(result) if rnd else result
    # STATIC (`reference.py:436`): the dense block; with EXT options it is the
    # spatial path under an all-ones S=1 mask (identical algebra).
    if epilogues is None and rnd is None:
        return block_forward_dense_masked(x, bw, block, cfg, mask)
    out = block.output_shape
    ones = np.ones((n, out.height, out.width), dtype=bool)
    r = _spatial_sparse(x, bw, block, SpatialMask(ones, ones, 1), epilogues, rnd, False)
    return rnd(r) if rnd else r


# ---------------------------------------------------------------------------
# EXT: masker -> block wiring on the output grid
# ---------------------------------------------------------------------------


def block_spatial_mask(x, masker_w, block: BlockSpec, s: int, bias: float = 0.0) -> SpatialMask:
    """EXT: decide cells of the OUTPUT grid from the block input.

    The reference never wires a masker into a block.  The
    composition used by the GPU path: pool the block input over
    (stride*S)^2 windows so the coarse grid is the output grid's H/S x W/S,
    then `spatial_masker_forward`'s 1x1 conv + tie rule (`reference.py:173-183`).
    ``bias`` (EXT, default 0) shifts logit 0 — a masker conv bias.
    """
    st = block.stride
    m = spatial_masker_forward(x, masker_w, s * st)
    if bias:
        n, c, h, w = x.shape
        ss = s * st
        pooled = x.reshape(n, c, h // ss, ss, w // ss, ss).mean(axis=(3, 5))
        logits = np.einsum("nchw,oc->nhwo", pooled, masker_w.reshape(2, c))
        coarse = logits[..., 0] + bias >= logits[..., 1]
        return SpatialMask(coarse, upsample_coarse(coarse, s), s)
    return SpatialMask(m.coarse, upsample_coarse(m.coarse, s), s)


def masker_margin(x, masker_w, block: BlockSpec, s: int) -> np.ndarray:
    """EXT: |d_bar| per cell and the near-tie scale sum|p_c||w_c|."""
    st = block.stride
    n, c, h, w = x.shape
    ss = s * st
    pooled = x.reshape(n, c, h // ss, ss, w // ss, ss).mean(axis=(3, 5))
    wd = (masker_w[0] - masker_w[1]).reshape(c)
    dbar = np.einsum("nchw,c->nhw", pooled, wd)
    scale = np.einsum("nchw,c->nhw", np.abs(pooled), np.abs(wd))
    return dbar, scale


def dilated_input_pixels(coarse: np.ndarray, block: BlockSpec, s: int) -> np.ndarray:
    """EXT: bool (N, H_in, W_in) of conv1 pixels any active patch's halo reads.

    Active cell (i, j) reads input rows [i*s*st - 1, i*s*st + (s-1)*st + 1]
    (conv2's 3x3 window at stride st, `reference.py:384,391-396`), clipped to
    the image; this is the conv1 work set (r_dil_in of SURVEY §8d).
    """
    st = block.stride
    n = coarse.shape[0]
    hi, wi = block.input_shape.height, block.input_shape.width
    out = np.zeros((n, hi, wi), dtype=bool)
    for ni, ci, cj in np.argwhere(coarse):
        r0, c0 = ci * s * st - 1, cj * s * st - 1
        r1, c1 = ci * s * st + (s - 1) * st + 2, cj * s * st + (s - 1) * st + 2
        out[ni, max(r0, 0):min(r1, hi), max(c0, 0):min(c1, wi)] = True
    return out


# ---------------------------------------------------------------------------
# seeded equivalence suite (reference.py:444-567)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class EquivalenceCase:
    """Replayable sparse-vs-dense case (`reference.py:444-454`)."""
    paradigm: Paradigm
    channels: int
    height: int
    width: int
    granularity: int
    seed: int
    tolerance: float = 1e-9


def case_block(case: EquivalenceCase) -> BlockSpec:
    """Case geometry: stride when seed%3==1, widen when seed%4==2 (`reference.py:457-477`)."""
    c = case.channels
    mid = max(2, c // 2)
    strided = case.seed % 3 == 1 and case.height % 2 == 0 and case.width % 2 == 0
    out_c = 2 * c if case.seed % 4 == 2 else c
    stride = 2 if strided else 1
    if case.paradigm is Paradigm.SPATIAL and strided:
        if (case.height // 2) % case.granularity or (case.width // 2) % case.granularity:
            stride, out_c = 1, c
    if case.paradigm is Paradigm.CHANNEL:
        mid = max(case.granularity, mid - mid % case.granularity)
    return BlockSpec(conv1=ConvLayerSpec(c, mid, 1), conv2=ConvLayerSpec(mid, mid, 3, stride),
                     conv3=ConvLayerSpec(mid, out_c, 1),
                     input_shape=TensorShape(c, case.height, case.width),
                     has_downsample=(stride > 1 or out_c != c))


def case_mask(case: EquivalenceCase, block: BlockSpec, rng):
    """Batch 1 + seed%2, rate ~ U(0.1, 0.9), Bernoulli cells (`reference.py:480-496`)."""
    n = 1 + case.seed % 2
    out = block.output_shape
    rate = 0.1 + 0.8 * rng.random()
    if case.paradigm is Paradigm.SPATIAL:
        g = case.granularity
        coarse = rng.random((n, out.height // g, out.width // g)) < rate
        return n, SpatialMask(coarse, upsample_coarse(coarse, g), g)
    if case.paradigm is Paradigm.CHANNEL:
        d = block.conv2.out_channels // case.granularity
        coarse = rng.random((n, d)) < rate
        return n, ChannelMask(coarse, np.repeat(coarse, case.granularity, axis=1),
                              case.granularity)
    if case.paradigm is Paradigm.LAYER:
        return n, LayerMask(rng.random(n) < rate)
    return n, None


def case_config(case: EquivalenceCase) -> DynamicConfig:
    if case.paradigm is Paradigm.SPATIAL:
        return DynamicConfig(Paradigm.SPATIAL, spatial_granularity=case.granularity)
    if case.paradigm is Paradigm.CHANNEL:
        return DynamicConfig(Paradigm.CHANNEL, channel_granularity=case.granularity)
    return DynamicConfig(case.paradigm)


def case_inputs(case: EquivalenceCase):
    """RNG replay order: rate, mask, weights, x (`reference.py:501-505`)."""
    rng = np.random.default_rng(case.seed)
    block = case_block(case)
    n, mask = case_mask(case, block, rng)
    bw = make_block_weights(block, rng)
    x = rng.standard_normal((n, case.channels, case.height, case.width))
    return block, mask, bw, x, case_config(case)


def run_equivalence_case(case: EquivalenceCase, inject_fault: bool = False) -> float:
    """max |sparse - dense_masked| (`reference.py:499-520`)."""
    block, mask, bw, x, cfg = case_inputs(case)
    dense = block_forward_dense_masked(x, bw, block, cfg, mask)
    fault = inject_fault and case.paradigm is Paradigm.SPATIAL and bool(mask.coarse.any())
    sparse = block_forward_sparse(x, bw, block, cfg, mask, _misplace_first_patch=fault)
    return float(np.max(np.abs(sparse - dense)))


def default_cases(per_paradigm: int = 25, max_side: int = 32):
    """Deterministic case spread (`reference.py:523-538`)."""
    shapes = [(8, 16, 16), (16, 32, 32), (4, 8, 8), (8, 24, 24)]
    cases = []
    for para in (Paradigm.SPATIAL, Paradigm.CHANNEL, Paradigm.LAYER):
        for i in range(per_paradigm):
            c, h, w = shapes[i % len(shapes)]
            h, w = min(h, max_side), min(w, max_side)
            g = [1, 2, 4][i % 3] if para is Paradigm.SPATIAL else (
                [1, 2][i % 2] if para is Paradigm.CHANNEL else 1)
            cases.append(EquivalenceCase(para, c, h, w, g, seed=i))
    return cases


def parse_cases_text(text: str, path: str = "<cases>"):
    """``key=value`` case lines, '#' comments (`reference.py:541-567`)."""
    cases = []
    for lineno, raw in enumerate(text.splitlines(), start=1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        kv = dict(tok.split("=", 1) for tok in line.split())
        try:
            cases.append(EquivalenceCase(
                paradigm=Paradigm(kv["paradigm"]), channels=int(kv["channels"]),
                height=int(kv["height"]), width=int(kv["width"]),
                granularity=int(kv.get("granularity", 1)), seed=int(kv["seed"]),
                tolerance=float(kv.get("tol", 1e-9))))
        except (KeyError, ValueError) as exc:
            raise SpecFileError(f"{path}:{lineno}: bad case line ({exc})") from exc
    return cases


# ---------------------------------------------------------------------------
# EXT: algorithmic accounting (flops.py:81-172 restated for the measured mask)
# ---------------------------------------------------------------------------


def spatial_block_flops(block: BlockSpec, coarse: np.ndarray, s: int) -> dict:
    """Algorithmic FLOPs of one spatial block under an exact mask.

    2*(r_dil_in*F1 + r*F2 + r*F3 + F_down + masker); halo recompute not
    credited; conv2 counts C_in/groups per output (`flops.py:81-88`).
    """
    n = coarse.shape[0]
    out = block.output_shape
    cin, hi, wi = block.input_shape.channels, block.input_shape.height, block.input_shape.width
    cm, co = block.conv1.out_channels, block.conv3.out_channels
    g = block.conv2.groups
    r = float(coarse.mean()) if coarse.size else 0.0
    r_dil_in = float(dilated_input_pixels(coarse, block, s).mean())
    f1 = n * hi * wi * cin * cm
    f2 = n * out.height * out.width * cm * (cm // g) * 9
    f3 = n * out.height * out.width * cm * co
    fd = n * out.height * out.width * cin * co if block.has_downsample else 0
    fm = n * hi * wi * cin
    total = 2 * (r_dil_in * f1 + r * f2 + r * f3 + fd + fm)
    static = 2 * (f1 + f2 + f3 + fd)
    return dict(r=r, r_dil_in=r_dil_in, flops=total, static_flops=static)


# ---------------------------------------------------------------------------
# EXT: network composer — stem, max-pool, blocks, GAP, FC
# ---------------------------------------------------------------------------

IMAGENET_MEAN = np.array([123.675, 116.28, 103.53])
IMAGENET_STD = np.array([58.395, 57.12, 57.375])


def maxpool3s2(x):
    """3x3 / stride 2 / pad 1 max-pool, NCHW (padding never wins)."""
    n, c, h, w = x.shape
    ho, wo = (h - 1) // 2 + 1, (w - 1) // 2 + 1
    p = np.pad(x, ((0, 0), (0, 0), (1, 1), (1, 1)), constant_values=-np.inf)
    out = np.full((n, c, ho, wo), -np.inf)
    for dy in range(3):
        for dx in range(3):
            out = np.maximum(out, p[:, :, dy:dy + 2 * (ho - 1) + 1:2, dx:dx + 2 * (wo - 1) + 1:2])
    return out


def network_forward(params: dict, images_u8: np.ndarray, paradigm: str = "spatial",
                    plan=(4, 2, 2, 1), biases=None, masks=None, emulate_bf16: bool = False,
                    record=None) -> np.ndarray:
    """EXT: whole-network forward on the CPU in fp64 (N, H, W, 3) uint8 -> logits.

    The reference has block specs only (`zoo.py:160-241`); this
    composes stem -> max-pool -> blocks (`block_forward_sparse` per block with
    folded-BN/ReLU epilogues) -> GAP -> FC with the parameters produced by
    ``paper_2308_15949_b200.network.make_params``.  ``masks`` (optional list of
    coarse arrays, one per block) overrides the masker decisions, so GPU runs
    can be replayed exactly; ``biases`` are the per-block masker biases.
    """
    rnd = round_bf16 if emulate_bf16 else (lambda a: a)
    net = params["net"]
    x = (images_u8.astype(np.float64) - IMAGENET_MEAN) / IMAGENET_STD
    x = rnd(x.transpose(0, 3, 1, 2))
    st = net.stem
    y = conv_raw(x, rnd(params["stem_w"]), st.stride, st.kernel // 2)
    x = rnd(np.maximum(y + params["stem_b"].reshape(1, -1, 1, 1), 0.0))
    if net.stem_pool:
        x = maxpool3s2(x)
    for i, bp in enumerate(params["blocks"]):
        blk = bp["block"]
        out = blk.output_shape
        # folded BN as the device executor packs it: W' = W * s (rounded once), + b
        fold = lambda w, sc: None if w is None else w * sc.reshape(-1, 1, 1, 1)  # noqa: E731
        ep = Epilogues(b1=bp["b1"], relu1=True, b2=bp["b2"], relu2=True, b3=bp["b3"], bd=bp["bd"],
                       relu_out=True, se_w1=bp.get("se_w1"), se_b1=bp.get("se_b1"),
                       se_w2=bp.get("se_w2"), se_b2=bp.get("se_b2"))
        bw = BlockWeights(fold(bp["w1"], bp["s1"]), fold(bp["w2"], bp["s2"]),
                          fold(bp["w3"], bp["s3"]), fold(bp["wd"], bp["sd"]))
        bias = 0.0 if biases is None else biases[i]
        if paradigm == "static":
            cfg = DynamicConfig(Paradigm.STATIC)
            mask = None
        elif paradigm == "channel":
            g = plan[bp["stage"] - 1]
            cfg = DynamicConfig(Paradigm.CHANNEL, channel_granularity=g)
            if masks is not None:
                c = np.asarray(masks[i]).reshape(x.shape[0], -1).astype(bool)
                mask = ChannelMask(c, np.repeat(c, g, axis=1), g)
            else:
                mask = channel_masker_forward(x, (bp["ch_w1"], bp["ch_w2"]), g, bias=bias)
        elif paradigm == "layer":
            cfg = DynamicConfig(Paradigm.LAYER)
            if masks is not None:
                d = np.asarray(masks[i]).reshape(-1).astype(bool)
            else:
                d = block_spatial_mask(x, bp["masker_w"], blk, out.height, bias).coarse.reshape(-1)
            mask = LayerMask(d)
        else:
            s = plan[bp["stage"] - 1]
            cfg = DynamicConfig(Paradigm.SPATIAL, spatial_granularity=s)
            if masks is not None:
                c = np.asarray(masks[i]).reshape(x.shape[0], out.height // s, out.width // s).astype(bool)
                mask = SpatialMask(c, upsample_coarse(c, s), s)
            else:
                mask = block_spatial_mask(x, bp["masker_w"], blk, s, bias)
        if record is not None:
            record.append(mask)
        x = block_forward_sparse(x, bw, blk, cfg, mask, epilogues=ep, emulate_bf16=emulate_bf16,
                                 grouped_channel_ext=True)
    feat = rnd(x.mean(axis=(2, 3)))
    return feat @ rnd(params["fc_w"]).T + params["fc_b"]
