"""Drop-in for ``dynlat.reference`` (`pkg/src/dynlat/reference.py`) on B200.

Same names, signatures, return types and exceptions as the reference's
mask-and-compute module, but every mask, plan and block forward is computed
by the sm_100a kernels of ``_laud.so``:

=====================================  =======================================
reference (file:line)                  here
=====================================  =======================================
spatial_masker_forward   156-186       K1 masker + compaction (fp32 decisions)
channel_masker_forward   189-218       K5 channel masker (GAP + 2-layer MLP)
build_gather_plan        133-135       K1b stable compaction of a given mask
dilate_and_rates         226-241       dilation kernel (same compaction core)
block_forward_sparse     356-436       gather-conv1 -> patch conv2 -> conv3 +
                                       scatter-add (tcgen05 implicit GEMMs)
block_forward_dense_masked 313-353     dense tcgen05 convs with mask epilogues
run_equivalence_case     499-520       GPU sparse vs GPU dense-masked
=====================================  =======================================

Inputs may be the reference's numpy NCHW float64 arrays (converted to
NHWC on the device: bf16 for the block path, fp32 for masker decisions) —
outputs then come back as numpy like the reference's — or CUDA tensors in
the native NHWC layout (see ``device.py``).  Arithmetic is bf16 with fp32
accumulation; decisions of the maskers are fp32.  There is no CPU fallback:
without a CUDA device or the built library every function raises
``DeviceError``.
"""

from __future__ import annotations

import ctypes as C
import weakref
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _lib
from . import device as D
from .core import BlockSpec, ConvLayerSpec, DynamicConfig, Paradigm, TensorShape
from .errors import GranularityMismatch, MaskShapeMismatch, ShapeMismatch, SpecFileError

# ---------------------------------------------------------------------------
# mask / plan types (reference.py:77-135)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class SpatialMask:
    coarse: np.ndarray
    upsampled: np.ndarray
    granularity: int
    soft: Optional[np.ndarray] = None

    @property
    def rate(self) -> float:
        return float(np.asarray(self.upsampled).mean())


@dataclass(frozen=True)
class ChannelMask:
    coarse: np.ndarray
    expanded: np.ndarray
    granularity: int
    soft: Optional[np.ndarray] = None

    @property
    def rate(self) -> float:
        return float(np.asarray(self.expanded).mean())


@dataclass(frozen=True)
class LayerMask:
    decisions: np.ndarray
    soft: Optional[np.ndarray] = None

    @property
    def rate(self) -> float:
        return float(np.asarray(self.decisions).mean())


@dataclass(frozen=True)
class GatherPlan:
    """(sample, cell-row, cell-col) of every active patch, row-major.

    ``device_list`` / ``device_count`` hold the same plan as produced on the
    GPU (int32 linear cell indices + count) for callers that stay on device.
    """
    indices: tuple
    device_list: Optional[torch.Tensor] = None
    device_count: Optional[torch.Tensor] = None

    @property
    def patch_count(self) -> int:
        return len(self.indices)


def upsample_coarse(coarse, s: int):
    """Nearest S x S replication (`reference.py:138-139`); layout helper."""
    if isinstance(coarse, torch.Tensor):
        return coarse.repeat_interleave(s, dim=-2).repeat_interleave(s, dim=-1)
    return np.repeat(np.repeat(coarse, s, axis=-2), s, axis=-1)


def gumbel_softmax_pair(logits, tau: float, noise=None):
    """Relaxed P(compute) for 2-way logits (`reference.py:142-153`)."""
    if tau <= 0:
        raise ValueError("tau must be positive")
    z = logits if noise is None else logits + noise
    return 1.0 / (1.0 + np.exp((z[..., 1] - z[..., 0]) / tau))


# ---------------------------------------------------------------------------
# helpers
# ---------------------------------------------------------------------------


def _scan(ws: D.Workspace, items: int) -> torch.Tensor:
    return ws.get("scan", _lib.lib().laud_scan_workspace_bytes(max(1, items)), zero=True)


def _dev_in(x, channels: int, dtype):
    """Block/masker input -> (device NHWC tensor, came_from_numpy).

    numpy arrays are the reference's (N, C, H, W) float64 layout and are
    converted on the device; CUDA tensors are the native layout, (N, H, W,
    pad8(C)) in the compute dtype, and are used in place (no host round trip).
    """
    if isinstance(x, torch.Tensor):
        if not x.is_cuda:
            raise ShapeMismatch("torch inputs must be CUDA tensors in NHWC layout")
        if x.ndim != 4:
            raise ShapeMismatch("expected an (N, H, W, C) CUDA tensor")
        if x.shape[-1] != D.pad8(channels):
            raise ShapeMismatch(f"input has {x.shape[-1]} (padded NHWC) channels, expected {D.pad8(channels)}")
        return (x if x.dtype == dtype else x.to(dtype)).contiguous(), False
    xn = np.asarray(x)
    if xn.ndim != 4:
        raise ShapeMismatch("expected (N, C, H, W) input")
    if xn.shape[1] != channels:
        raise ShapeMismatch(f"input has {xn.shape[1]} channels, expected {channels}")
    return D.to_device_nhwc(xn, dtype=dtype), True


def _dev_out(y: torch.Tensor, channels: int, numpy_in: bool):
    """numpy in -> numpy (N, C, H, W) float64 out; CUDA in -> the device NHWC tensor."""
    return D.from_device_nhwc(y, channels) if numpy_in else y


def _decide_train(dbar: np.ndarray, tau, rng):
    """Train-mode decision from the device logit difference d = l0 - l1.

    Same RNG draw as the reference (`rng.gumbel(size=logits.shape)` with the
    pair on the last axis, `reference.py:177-181`), so seeded runs replay.
    """
    noise = rng.gumbel(size=dbar.shape + (2,)) if rng is not None else None
    zd = dbar if noise is None else dbar + noise[..., 0] - noise[..., 1]
    if tau is None or tau <= 0:
        raise ValueError("tau must be positive")
    soft = 1.0 / (1.0 + np.exp(-zd / tau))
    return zd >= 0, soft


def spatial_masker_forward(x, weights, s: int, mode: str = "inference",
                           tau: Optional[float] = None,
                           rng: Optional[np.random.Generator] = None) -> SpatialMask:
    """Pool S x S, 1x1 conv to 2 logits, decide (`reference.py:156-186`).

    Runs the fused-masker identity on the device: d = mean(x) . (W0 - W1) in
    fp32, decision d >= 0 (compute wins ties), stable compaction of the
    active cells.  numpy input -> numpy SpatialMask.
    """
    if mode not in ("inference", "train"):
        raise ValueError(f"unknown mode {mode!r}")
    D.require_cuda()
    c = int(np.prod(np.asarray(weights).shape)) // 2
    if isinstance(x, torch.Tensor):  # native: CUDA NHWC (bf16 or fp32), decided in fp32
        xd, numpy_in = _dev_in(x, c, x.dtype if x.dtype in (torch.bfloat16, torch.float32) else torch.float32)
        n, h, w, _ = xd.shape
    else:
        xd, numpy_in = _dev_in(x, c, torch.float32)
        n, h, w = xd.shape[0], xd.shape[1], xd.shape[2]
    if h % s or w % s:
        raise GranularityMismatch(f"S={s} does not divide {h}x{w}")
    wts = np.asarray(weights, dtype=np.float64).reshape(2, c)
    cp = xd.shape[-1]
    wd = np.zeros(cp, np.float32)
    wd[:c] = (wts[0] - wts[1]).astype(np.float32)
    wdt = torch.from_numpy(wd).cuda()
    ws = D.workspace()
    cells = n * (h // s) * (w // s)
    lib = _lib.lib()
    npart = lib.laud_masker_partial_floats(n, h, w, cp, s, 1)
    part = torch.empty(max(1, npart), dtype=torch.float32, device="cuda")
    coarse = torch.empty(cells, dtype=torch.uint8, device="cuda")
    lst = torch.empty(max(1, cells), dtype=torch.int32, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
    _lib.call("laud_spatial_masker", D.ptr(xd), int(xd.dtype == torch.float32), cp, n, h, w, cp, s, 1,
              D.ptr(wdt), 0.0,
              D.ptr(coarse), D.ptr(lst), D.ptr(cnt), D.ptr(part), D.ptr(_scan(ws, cells)),
              D.stream_handle())
    shape = (n, h // s, w // s)
    soft = None
    if mode == "inference" and not numpy_in:  # stays on the device, no host sync
        cz = coarse.view(shape).bool()
        return SpatialMask(cz, upsample_coarse(cz, s), s, None)
    if mode == "inference":
        cz = coarse.view(shape).bool().cpu().numpy()
    else:
        dbar = part.view(cells, -1).sum(dim=1).double().cpu().numpy().reshape(shape) / (s * s)
        cz, soft = _decide_train(dbar, tau, rng)
    return SpatialMask(cz, upsample_coarse(cz, s), s, soft)


def masker_hidden_width(d: int) -> int:
    """max(D // 16, 16) (`reference.py:221-223`)."""
    return max(d // 16, 16)


def channel_masker_forward(x, weights, g: int, mode: str = "inference",
                           tau: Optional[float] = None,
                           rng: Optional[np.random.Generator] = None) -> ChannelMask:
    """GAP -> relu(W1) -> W2 -> interleaved pairs -> repeat G (`reference.py:189-218`)."""
    from . import channel as CH
    return CH.channel_masker_forward(x, weights, g, mode, tau, rng)


def build_gather_plan(coarse) -> GatherPlan:
    """Row-major active cells == np.argwhere (`reference.py:133-135`), on device."""
    D.require_cuda()
    cz = np.asarray(coarse, dtype=bool) if not isinstance(coarse, torch.Tensor) else coarse
    shape = tuple(cz.shape)
    cells = int(np.prod(shape)) if shape else 1
    cd = (torch.from_numpy(np.ascontiguousarray(cz, dtype=np.uint8)).cuda()
          if not isinstance(cz, torch.Tensor) else cz.to(torch.uint8).contiguous())
    lst = torch.empty(max(1, cells), dtype=torch.int32, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
    ws = D.workspace()
    _lib.call("laud_cells_from_mask", D.ptr(cd), cells, D.ptr(lst), D.ptr(cnt),
              D.ptr(_scan(ws, cells)), D.stream_handle())
    k = int(cnt.item())
    flat = lst[:k].cpu().numpy()
    idx = np.stack(np.unravel_index(flat, shape), axis=1) if k else np.zeros((0, len(shape)), int)
    return GatherPlan(tuple(tuple(int(v) for v in row) for row in idx), lst[:k], cnt)


def dilate_and_rates(mask: SpatialMask, kernel: int):
    """(r, r_dil, dilated) with a k x k square (`reference.py:226-241`), on device."""
    if kernel % 2 == 0:
        raise ValueError("kernel must be odd")
    D.require_cuda()
    coarse = np.asarray(mask.coarse, dtype=bool)
    n, ch, cw = coarse.shape
    s = mask.granularity
    h, w = ch * s, cw * s
    cd = torch.from_numpy(coarse.astype(np.uint8)).cuda()
    pix = n * h * w
    lst = torch.empty(pix, dtype=torch.int32, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
    ws = D.workspace()
    _lib.call("laud_dilate_pixels", D.ptr(cd), n, h, w, s, 1, (kernel - 1) // 2, D.ptr(lst),
              D.ptr(cnt), D.ptr(_scan(ws, pix)), D.stream_handle())
    k = int(cnt.item())
    dil = torch.zeros(pix, dtype=torch.bool, device="cuda")
    dil[lst[:k].long()] = True
    dil = dil.view(n, h, w).cpu().numpy()
    up = np.asarray(mask.upsampled, dtype=bool)
    return float(up.mean()), float(k / pix), dil


def fused_masker_weight_identity(weights: np.ndarray) -> np.ndarray:
    """W0 - W1 (`reference.py:244-253`); the form the device masker consumes."""
    if weights.shape[0] != 2 or tuple(weights.shape[-2:]) != (1, 1):
        raise ShapeMismatch("expected (2, C, 1, 1) masker weights")
    return weights[0:1] - weights[1:2]


# ---------------------------------------------------------------------------
# block weights (reference.py:261-292)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class BlockWeights:
    w1: np.ndarray
    w2: np.ndarray
    w3: np.ndarray
    w_down: Optional[np.ndarray] = None


def _down_layer(block: BlockSpec) -> ConvLayerSpec:
    return ConvLayerSpec(block.input_shape.channels, block.conv3.out_channels, 1, block.stride)


def make_block_weights(block: BlockSpec, rng: np.random.Generator) -> BlockWeights:
    """N(0,1)/sqrt(fan_in), draw order w_down, w1, w2, w3 (`reference.py:271-286`)."""

    def draw(layer):
        cig = layer.in_channels // layer.groups
        return rng.standard_normal((layer.out_channels, cig, layer.kernel, layer.kernel)) / \
            np.sqrt(cig * layer.kernel ** 2)

    wd = None
    if block.has_downsample:
        dl = _down_layer(block)
        wd = rng.standard_normal((dl.out_channels, dl.in_channels, 1, 1)) / np.sqrt(dl.in_channels)
    return BlockWeights(draw(block.conv1), draw(block.conv2), draw(block.conv3), wd)


_DEV_CONVS: dict = {}


def conv2d_direct(x, layer: ConvLayerSpec, weights: np.ndarray):
    """Validated direct convolution, k//2 zero padding, stride, groups, bias-free
    (`reference.py:52-69`), as one tcgen05 implicit GEMM (fp32 FFMA engine in
    fp32 precision mode).  numpy (N, C, H, W) in -> numpy out; a CUDA NHWC
    tensor in -> the NHWC device tensor out (pad8(C_out) channels)."""
    D.require_cuda()
    from . import channel as CH
    w = np.asarray(weights)
    want = (layer.out_channels, layer.in_channels // layer.groups, layer.kernel, layer.kernel)
    if isinstance(x, torch.Tensor):
        if x.ndim != 4:
            raise ShapeMismatch("expected an (N, H, W, C) CUDA tensor")
    elif np.asarray(x).ndim != 4:
        raise ShapeMismatch("expected (N, C, H, W) input")
    elif np.asarray(x).shape[1] != layer.in_channels:
        raise ShapeMismatch(f"input has {np.asarray(x).shape[1]} channels, layer expects {layer.in_channels}")
    if w.shape != want:
        raise ShapeMismatch(f"weights {w.shape} != expected {want}")
    dt = _PRECISION["dtype"]
    g = layer.groups
    if g > 1 and ((layer.in_channels // g) % 8 or (layer.out_channels // g) % 8):
        w, g = D.grouped_to_dense(w, g), 1  # narrow groups: the block-diagonal dense kernel (same sums)
    xd, numpy_in = _dev_in(x, layer.in_channels, dt)
    key = (id(weights), want, dt)
    ent = _DEV_CONVS.get(key)
    if ent is None or ent[0] is not weights:
        ent = (weights, D.pack_weight(w, D.pad8(layer.in_channels), groups=g, dtype=dt), g)
        _DEV_CONVS[key] = ent
    n, h, ww, cp = xd.shape
    k, st = layer.kernel, layer.stride
    ho, wo = (h + 2 * (k // 2) - k) // st + 1, (ww + 2 * (k // 2) - k) // st + 1
    co = D.pad8(layer.out_channels)
    y = torch.empty((n, ho, wo, co), dtype=dt, device=xd.device)
    CH.conv(act=xd, in_hw=(h, ww), in_c=cp, in_ld=cp, weight=ent[1], n_out=co, out=y, out_ld=co,
            out_hw=(ho, wo), batch=n, ksize=k, stride=st, pad=k // 2, groups=ent[2],
            fp32=int(dt == torch.float32))
    return _dev_out(y, layer.out_channels, numpy_in)


_DEV_BLOCKS: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()


class _Key:  # BlockWeights is frozen+eq; key device copies on identity
    pass


_PRECISION = {"dtype": torch.bfloat16}


def set_precision(name: str) -> None:
    """EXT: compute precision of the block executors — "bf16" (default: bf16
    storage, fp32 tcgen05 accumulation; 1e-3 gate) or "fp32" (fp32 storage and
    FFMA; the north star's 1e-5 gate).  Maskers always decide in fp32."""
    if name not in ("bf16", "fp32"):
        raise ValueError(f"precision must be 'bf16' or 'fp32', got {name!r}")
    _PRECISION["dtype"] = torch.float32 if name == "fp32" else torch.bfloat16


def get_precision() -> str:
    return "fp32" if _PRECISION["dtype"] == torch.float32 else "bf16"


def device_block(bw: BlockWeights, block: BlockSpec) -> D.DeviceBlock:
    """Packed device copy of ``bw`` (cached per BlockWeights object and precision)."""
    dt = _PRECISION["dtype"]
    cache = bw.__dict__.get("_laud_dev")
    if cache is not None and cache[0] == block and cache[1].dtype == dt:
        return cache[1]
    db = D.DeviceBlock(block, bw.w1, bw.w2, bw.w3, bw.w_down, dtype=dt)
    object.__setattr__(bw, "_laud_dev", (block, db))
    return db


# ---------------------------------------------------------------------------
# block forward (reference.py:295-436)
# ---------------------------------------------------------------------------


def _check_spatial_mask(mask: SpatialMask, block: BlockSpec, n: int):
    out = block.output_shape
    s = mask.granularity
    if out.height % s or out.width % s:
        raise GranularityMismatch(f"S={s} does not divide {out.height}x{out.width}")
    want = (n, out.height // s, out.width // s)
    if tuple(mask.coarse.shape) != want:
        raise MaskShapeMismatch(f"coarse mask {tuple(mask.coarse.shape)} != {want}")
    if tuple(mask.upsampled.shape) != (n, out.height, out.width):
        raise MaskShapeMismatch("upsampled mask does not match the output feature")


def _check_input(x, block: BlockSpec):
    if x.ndim != 4:
        raise ShapeMismatch("expected (N, C, H, W) input")
    if x.shape[1] != block.input_shape.channels:
        raise ShapeMismatch(f"input has {x.shape[1]} channels, block expects "
                            f"{block.input_shape.channels}")


def _u8(a) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        return a.to(device="cuda", dtype=torch.uint8).reshape(-1).contiguous()
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a), dtype=np.uint8).reshape(-1)).cuda()


def block_forward_sparse(x, bw: BlockWeights, block: BlockSpec, cfg: DynamicConfig, mask,
                         _misplace_first_patch: bool = False, grouped_channel_ext: bool = False):
    """Inference forward computing only what the mask selects (`reference.py:356-436`).

    SPATIAL: gather-conv1 on the halo-dilated pixel set, 3x3 conv over the
    active S x S patches, conv3 fused with the scatter-add into the skip;
    CHANNEL: dynamic-width convs over the kept channels; LAYER: per-sample
    compaction; STATIC: the dense block.  ``_misplace_first_patch`` is the
    reference's fault hook (`reference.py:362, 400-401`), honoured on device.
    ``grouped_channel_ext`` (EXT, default off = the reference's ShapeMismatch)
    runs channel skipping over a grouped conv2 (`channel.channel_block_sparse`).
    """
    D.require_cuda()
    p = cfg.paradigm
    if p is Paradigm.CHANNEL:
        from . import channel as CH
        return CH.channel_block_sparse(x, bw, block, mask, grouped_channel_ext=grouped_channel_ext)
    db = device_block(bw, block)
    xd, numpy_in = _dev_in(x, block.input_shape.channels, db.dtype)
    n = xd.shape[0]
    out = block.output_shape
    if p is Paradigm.SPATIAL:
        _check_spatial_mask(mask, block, n)
        y, *_ = db.forward(xd, "spatial", mask.granularity, coarse=_u8(mask.coarse),
                           misplace_first=_misplace_first_patch)
    elif p is Paradigm.LAYER:
        if tuple(mask.decisions.shape) != (n,):
            raise MaskShapeMismatch(f"layer mask {tuple(mask.decisions.shape)} != {(n,)}")
        y, *_ = db.forward(xd, "layer", out.height, coarse=_u8(mask.decisions))
    else:
        y, *_ = db.forward(xd, "static")
    return _dev_out(y, out.channels, numpy_in)


def block_forward_dense_masked(x, bw: BlockWeights, block: BlockSpec, cfg: DynamicConfig, mask):
    """Training-style: dense convs, masks applied multiplicatively (`reference.py:313-353`).

    Dense tcgen05 convs; the spatial/layer mask multiplies conv3's output in
    its epilogue before the residual add, the channel mask multiplies conv1's
    output (= conv2's input) and conv2's output per sample.
    """
    from . import channel as CH
    D.require_cuda()
    p = cfg.paradigm
    db = device_block(bw, block)
    xd, numpy_in = _dev_in(x, block.input_shape.channels, db.dtype)
    n = xd.shape[0]
    out = block.output_shape
    ymask = None
    chmask = None
    patch = (out.height, out.width)
    if p is Paradigm.SPATIAL:
        _check_spatial_mask(mask, block, n)
        ymask = _u8(mask.coarse)
        patch = (mask.granularity, mask.granularity)
    elif p is Paradigm.CHANNEL:
        chmask = _channel_mask_u8(mask.expanded, n, block.conv2.out_channels, db.cmid_p)
    elif p is Paradigm.LAYER:
        if tuple(mask.decisions.shape) != (n,):
            raise MaskShapeMismatch(f"layer mask {tuple(mask.decisions.shape)} != {(n,)}")
        ymask = _u8(mask.decisions)
    y = CH.dense_block(db, xd, ymask=ymask, patch=patch, chmask=chmask)
    return _dev_out(y, out.channels, numpy_in)


def _channel_mask_u8(m, n: int, cm: int, cmp: int) -> torch.Tensor:
    """(N, C_mid) keep mask (numpy or CUDA tensor) -> device uint8 [N * pad8(C_mid)]."""
    if tuple(m.shape) != (n, cm):
        raise MaskShapeMismatch(f"channel mask {tuple(m.shape)} != {(n, cm)}")
    mm = torch.zeros((n, cmp), dtype=torch.uint8, device="cuda")
    mm[:, :cm] = m.to(device="cuda", dtype=torch.uint8) if isinstance(m, torch.Tensor) else \
        torch.from_numpy(np.ascontiguousarray(np.asarray(m), dtype=np.uint8)).cuda()
    return mm.reshape(-1)


# ---------------------------------------------------------------------------
# seeded equivalence suite (reference.py:444-567)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class EquivalenceCase:
    paradigm: Paradigm
    channels: int
    height: int
    width: int
    granularity: int
    seed: int
    tolerance: float = 1e-9


def _case_block(case: EquivalenceCase) -> BlockSpec:
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
    return BlockSpec(ConvLayerSpec(c, mid, 1), ConvLayerSpec(mid, mid, 3, stride),
                     ConvLayerSpec(mid, out_c, 1), TensorShape(c, case.height, case.width),
                     has_downsample=(stride > 1 or out_c != c))


def _case_mask(case, block, rng):
    n = 1 + case.seed % 2
    out = block.output_shape
    rate = 0.1 + 0.8 * rng.random()
    g = case.granularity
    if case.paradigm is Paradigm.SPATIAL:
        coarse = rng.random((n, out.height // g, out.width // g)) < rate
        return n, SpatialMask(coarse, upsample_coarse(coarse, g), g)
    if case.paradigm is Paradigm.CHANNEL:
        coarse = rng.random((n, block.conv2.out_channels // g)) < rate
        return n, ChannelMask(coarse, np.repeat(coarse, g, axis=1), g)
    if case.paradigm is Paradigm.LAYER:
        return n, LayerMask(rng.random(n) < rate)
    return n, None


def run_equivalence_case(case: EquivalenceCase, inject_fault: bool = False) -> float:
    """max |sparse - dense_masked| of one seeded case, both on the GPU.

    The two GPU paths use identical bf16 rounding points, so on the device
    the deviation is expected to be exactly 0 (the reference's fp64 1e-9
    tolerance therefore still applies); the fault hook must break it.
    """
    rng = np.random.default_rng(case.seed)
    block = _case_block(case)
    n, mask = _case_mask(case, block, rng)
    bw = make_block_weights(block, rng)
    x = rng.standard_normal((n, case.channels, case.height, case.width))
    if case.paradigm is Paradigm.SPATIAL:
        cfg = DynamicConfig(Paradigm.SPATIAL, spatial_granularity=case.granularity)
    elif case.paradigm is Paradigm.CHANNEL:
        cfg = DynamicConfig(Paradigm.CHANNEL, channel_granularity=case.granularity)
    else:
        cfg = DynamicConfig(case.paradigm)
    dense = block_forward_dense_masked(x, bw, block, cfg, mask)
    fault = inject_fault and case.paradigm is Paradigm.SPATIAL and bool(np.any(mask.coarse))
    sparse = block_forward_sparse(x, bw, block, cfg, mask, _misplace_first_patch=fault)
    return float(np.max(np.abs(sparse - dense)))


def default_cases(per_paradigm: int = 25, max_side: int = 32):
    """Deterministic spread of shapes / granularities (`reference.py:523-538`)."""
    shapes = [(8, 16, 16), (16, 32, 32), (4, 8, 8), (8, 24, 24)]
    out = []
    for para in (Paradigm.SPATIAL, Paradigm.CHANNEL, Paradigm.LAYER):
        for i in range(per_paradigm):
            c, h, w = shapes[i % len(shapes)]
            g = {Paradigm.SPATIAL: [1, 2, 4][i % 3], Paradigm.CHANNEL: [1, 2][i % 2]}.get(para, 1)
            out.append(EquivalenceCase(para, c, min(h, max_side), min(w, max_side), g, seed=i))
    return out


def parse_cases_text(text: str, path: str = "<cases>"):
    """One ``key=value`` case per line, '#' comments (`reference.py:541-567`)."""
    out = []
    for lineno, raw in enumerate(text.splitlines(), start=1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        kv = dict(t.split("=", 1) for t in line.split())
        try:
            out.append(EquivalenceCase(Paradigm(kv["paradigm"]), int(kv["channels"]),
                                       int(kv["height"]), int(kv["width"]),
                                       int(kv.get("granularity", 1)), int(kv["seed"]),
                                       float(kv.get("tol", 1e-9))))
        except (KeyError, ValueError) as exc:
            raise SpecFileError(f"{path}:{lineno}: bad case line ({exc})") from exc
    return out
