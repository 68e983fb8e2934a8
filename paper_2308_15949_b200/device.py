"""Device plumbing: layouts, weight packing, workspaces, block launch.

PyTorch is used only for device memory, streams and layout conversion;
every arithmetic op of the path runs in ``_laud.so`` (see ``_lib.py``).

Layouts (DESIGN.md §Data layout):
  activations  NHWC bf16, channels zero-padded to a multiple of 8;
  weights      [c_out][k*k][kpad(c_in)] bf16, kpad = c_in rounded up to 64;
  masks        uint8 per cell of the OUTPUT grid, row-major (n, i, j);
  lists        int32 linear cell / pixel indices plus a device-side count.
"""

from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _lib
from .core import BlockSpec
from .errors import DeviceError


def pad8(c: int) -> int:
    return (c + 7) // 8 * 8


def kpad(c: int) -> int:
    return (c + 63) // 64 * 64


def require_cuda():
    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device: this package has no CPU fallback")
    _lib.lib()


def ptr(t: Optional[torch.Tensor]):
    return None if t is None else C.c_void_p(t.data_ptr())


def stream_handle(stream: Optional[torch.cuda.Stream] = None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


# ---------------------------------------------------------------------------
# layout conversion (host numpy NCHW <-> device NHWC)
# ---------------------------------------------------------------------------


def to_device_nhwc(x: np.ndarray, dtype=torch.bfloat16, device="cuda") -> torch.Tensor:
    """(N, C, H, W) numpy -> (N, H, W, pad8(C)) device tensor, zero padded."""
    n, c, h, w = x.shape
    t = torch.zeros((n, h, w, pad8(c)), dtype=dtype, device=device)
    t[..., :c] = torch.from_numpy(np.ascontiguousarray(x.transpose(0, 2, 3, 1))).to(device, dtype)
    return t


def from_device_nhwc(t: torch.Tensor, c: int) -> np.ndarray:
    """(N, H, W, Cp) device tensor -> (N, C, H, W) float64 numpy."""
    return t[..., :c].permute(0, 3, 1, 2).double().cpu().numpy()


def pack_weight(w, c_in_pad: int, device="cuda", groups: int = 1, dtype=torch.bfloat16) -> torch.Tensor:
    """[c_out, c_in / groups, k, k] (numpy or torch) -> [c_out, k*k, kpad(c_in_pad)] bf16 on device.

    Grouped weights are expanded block-diagonally (zeros outside the group)
    into kpad(c_in_pad) + 64 columns, the layout the engine's per-tile K
    windows read (include/laud.h, laud_conv_args.groups).
    """
    wt = torch.as_tensor(np.asarray(w) if isinstance(w, np.ndarray) else w, dtype=torch.float32)
    co, cig, kh, kw = wt.shape
    if groups > 1:
        ci = cig * groups
        dense = torch.zeros((co, ci, kh, kw), dtype=torch.float32)
        gw_out = co // groups
        for g in range(groups):
            dense[g * gw_out:(g + 1) * gw_out, g * cig:(g + 1) * cig] = wt[g * gw_out:(g + 1) * gw_out]
        wt = dense
    co, ci, kh, kw = wt.shape
    out = torch.zeros((pad8(co), kh * kw, kpad(c_in_pad) + (64 if groups > 1 else 0)), dtype=torch.float32)
    out[:co, :, :ci] = wt.permute(0, 2, 3, 1).reshape(co, kh * kw, ci)
    return out.to(device=device, dtype=dtype).contiguous()


def grouped_to_dense(w, groups: int) -> np.ndarray:
    """[c_out, c_in / groups, k, k] -> [c_out, c_in, k, k] block-diagonal dense kernel."""
    w = np.asarray(w if isinstance(w, np.ndarray) else torch.as_tensor(w).cpu().numpy(), dtype=np.float64)
    co, cig, kh, kw = w.shape
    cog = co // groups
    out = np.zeros((co, cig * groups, kh, kw))
    for g in range(groups):
        out[g * cog:(g + 1) * cog, g * cig:(g + 1) * cig] = w[g * cog:(g + 1) * cog]
    return out


def fvec(v, n: int, fill: float, device="cuda") -> torch.Tensor:
    """Per-channel fp32 vector padded to pad8(n) (padding channels get `fill`)."""
    out = torch.full((pad8(n),), fill, dtype=torch.float32)
    if v is not None:
        out[:n] = torch.as_tensor(np.asarray(v, dtype=np.float32))
    return out.to(device)


# ---------------------------------------------------------------------------
# workspace
# ---------------------------------------------------------------------------


class Workspace:
    """Grow-only device scratch shared by the blocks launched on one stream."""

    def __init__(self, device="cuda"):
        self.device = torch.device(device)
        self._bufs: dict[str, torch.Tensor] = {}
        self._lock = threading.Lock()

    def get(self, name: str, nbytes: int, zero: bool = False) -> torch.Tensor:
        nbytes = max(int(nbytes), 16)
        with self._lock:
            b = self._bufs.get(name)
            if b is None or b.numel() < nbytes:
                b = (torch.zeros if zero else torch.empty)(nbytes, dtype=torch.uint8,
                                                           device=self.device)
                self._bufs[name] = b
            return b


_WS: dict = {}


def workspace(device=None) -> Workspace:
    dev = torch.device(device if device is not None else "cuda")
    idx = dev.index if dev.index is not None else torch.cuda.current_device()
    key = (idx, torch.cuda.current_stream(idx).cuda_stream)
    ws = _WS.get(key)
    if ws is None:
        ws = _WS[key] = Workspace(f"cuda:{idx}")
    return ws


# ---------------------------------------------------------------------------
# a block resident on the device
# ---------------------------------------------------------------------------


@dataclass
class Epilogue:
    """Folded BN scale/bias per conv plus ReLU flags (None = identity)."""
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


def _fold(w, scale):
    """W * scale[:, None, None, None] (numpy), identity when scale is None."""
    if scale is None:
        return w
    return np.asarray(w, dtype=np.float64) * np.asarray(scale, dtype=np.float64).reshape(-1, 1, 1, 1)


class DeviceBlock:
    """Packed weights + epilogue vectors of one bottleneck block."""

    def __init__(self, block: BlockSpec, w1, w2, w3, w_down=None, epilogue: Optional[Epilogue] = None,
                 masker_w=None, masker_bias: float = 0.0, device="cuda", fold_scale: bool = False,
                 dtype=torch.bfloat16, grouped_channel_ext: bool = False):
        require_cuda()
        if dtype not in (torch.bfloat16, torch.float32):
            raise DeviceError("compute dtype must be bf16 (tcgen05) or fp32 (FFMA numerics mode)")
        self.dtype = dtype
        self.block = block
        self.c_in, self.c_mid, self.c_out = (block.conv1.in_channels, block.conv1.out_channels,
                                             block.conv3.out_channels)
        self.cin_p, self.cmid_p, self.cout_p = pad8(self.c_in), pad8(self.c_mid), pad8(self.c_out)
        ep = epilogue or Epilogue()
        if fold_scale:
            # inference BN folding: per-output-channel scale goes into the weights
            w1, w2, w3 = _fold(w1, ep.s1), _fold(w2, ep.s2), _fold(w3, ep.s3)
            w_down = _fold(w_down, ep.sd) if w_down is not None else None
            ep = Epilogue(None, ep.b1, ep.relu1, None, ep.b2, ep.relu2, None, ep.b3, None, ep.bd,
                          ep.relu_out)
        self.w1 = pack_weight(w1, self.cin_p, device, dtype=dtype)
        self.groups = block.conv2.groups
        if self.groups > 1 and self.cmid_p != self.c_mid:
            raise DeviceError("grouped conv2 needs a mid width that is a multiple of 8")
        self.w2 = pack_weight(w2, self.cmid_p, device, groups=self.groups, dtype=dtype)
        # EXT (laud.h w2_dense): channel skipping over a grouped conv2 runs on the
        # block-diagonal dense kernel; without it channel mode keeps the reference's
        # groups == 1 requirement
        self.w2_dense = None
        self._w2_grouped = (w2, device) if self.groups > 1 else None
        if grouped_channel_ext:
            self.enable_grouped_channel()
        self.w3 = pack_weight(w3, self.cmid_p, device, dtype=dtype)
        self.wd = pack_weight(w_down, self.cin_p, device, dtype=dtype) if w_down is not None else None
        self.ep = ep
        self.vec = {}
        for k, n, fill in (("s1", self.c_mid, 1.0), ("b1", self.c_mid, 0.0), ("s2", self.c_mid, 1.0),
                           ("b2", self.c_mid, 0.0), ("s3", self.c_out, 1.0), ("b3", self.c_out, 0.0),
                           ("sd", self.c_out, 1.0), ("bd", self.c_out, 0.0)):
            v = getattr(ep, k)
            self.vec[k] = fvec(v, n, fill, device) if v is not None else None
        self.wdiff = None
        self.masker_bias = float(masker_bias)
        self.conv1_dense = False  # spatial conv1 on the dilated pixel list (see laud.h)
        self.se = None            # EXT squeeze-excitation (set_se)
        if masker_w is not None:
            self.set_masker(masker_w, masker_bias)

    def set_masker(self, masker_w, bias: float = 0.0):
        """Store W0 - W1 (fused-masker identity, `reference.py:244-253`)."""
        mw = np.asarray(masker_w, dtype=np.float64).reshape(2, -1)
        wd = np.zeros(kpad(self.cin_p), dtype=np.float32)  # zero tail: read per 64-channel block
        wd[: mw.shape[1]] = (mw[0] - mw[1]).astype(np.float32)
        self.wdiff = torch.from_numpy(wd).to(self.w1.device)
        self.masker_bias = float(bias)

    def set_se(self, w1, b1, w2, b2):
        """EXT squeeze-excitation after conv2 (include/laud.h, laud_block_args.se_*):
        w1 [hidden, C_mid], b1 [hidden], w2 [C_mid, hidden], b2 [C_mid]."""
        dev = self.w1.device
        f = lambda a: torch.as_tensor(np.asarray(a, dtype=np.float32)).contiguous().to(dev)  # noqa: E731
        w1, w2 = np.asarray(w1), np.asarray(w2)
        if w1.shape[1] != self.c_mid or w2.shape[0] != self.c_mid or self.cmid_p != self.c_mid:
            raise DeviceError("SE needs [hidden, C_mid] / [C_mid, hidden] weights and C_mid % 8 == 0")
        self.se = (f(w1), f(b1), f(w2), f(b2), int(w1.shape[0]))

    def out_hw(self, h: int, w: int):
        return self.block.conv2.out_hw(h, w)

    def set_channel_masker(self, w1, w2, g: int, bias: float = 0.0):
        """Channel masker MLP (`reference.py:189-218`): w1 [h, C_in], w2 [2D, h], G.

        ``bias`` (EXT, default 0 = reference) is added to every logit gap l0 - l1.
        """
        w1 = np.asarray(w1, dtype=np.float32)
        w2 = np.asarray(w2, dtype=np.float32)
        if w1.shape[1] > self.cin_p:
            raise DeviceError("channel masker width exceeds the block input")
        w1p = np.zeros((w1.shape[0], self.cin_p), np.float32)
        w1p[:, : w1.shape[1]] = w1
        dev = self.w1.device
        self.ch_w1 = torch.from_numpy(w1p).to(dev)
        self.ch_w2 = torch.from_numpy(np.ascontiguousarray(w2)).to(dev)
        self.ch_hidden, self.ch_d, self.ch_g = w1.shape[0], w2.shape[0] // 2, int(g)
        self.set_channel_bias(bias)

    def set_channel_bias(self, bias: float):
        self.ch_bias_value = float(bias)
        self.ch_bias = (torch.full((self.ch_d,), float(bias), dtype=torch.float32, device=self.ch_w1.device)
                        if bias != 0.0 else None)

    def _channel_args(self, a, n, ws, chmask):
        cmp = self.cmid_p
        d = getattr(self, "ch_d", 1)
        a.ch_expanded = ptr(chmask) if chmask is not None else ptr(ws.get("ch_exp", n * cmp))
        a.given_chmask = ptr(chmask)
        self._ch_coarse = ws.get("ch_coarse", n * d)
        self._ch_sel = ws.get("ch_sel", n * cmp * 4)
        self._ch_count = ws.get("ch_count", n * 4)
        self._ch_dvals = ws.get("ch_dvals", n * d * 4)
        a.ch_coarse, a.ch_sel, a.ch_count = ptr(self._ch_coarse), ptr(self._ch_sel), ptr(self._ch_count)
        a.ch_dvals = ptr(self._ch_dvals)
        a.wpack = ptr(ws.get("wpack", _lib.lib().laud_channel_pack_bytes(n, self.cin_p, cmp, self.cout_p)))
        if self.groups == 1 and self.dtype == torch.bfloat16:
            if getattr(self, "w3t", None) is None:  # conv3 kernel transposed: [c_mid][c_out] (laud.h w3t)
                self.w3t = self.w3[:, 0, :cmp].t().contiguous()
            a.w3t = ptr(self.w3t)
        if chmask is None:
            if getattr(self, "ch_w1", None) is None:
                raise DeviceError("no channel mask given and no channel masker weights set")
            a.ch_w1, a.ch_w2 = ptr(self.ch_w1), ptr(self.ch_w2)
            a.ch_bias = ptr(getattr(self, "ch_bias", None))
            a.ch_hidden, a.ch_d, a.ch_groups = self.ch_hidden, self.ch_d, self.ch_g

    def enable_grouped_channel(self):
        """EXT: allow channel skipping over this block's grouped conv2 (packs the
        block-diagonal dense kernel once; laud.h w2_dense)."""
        if self._w2_grouped is not None and self.w2_dense is None:
            w2, device = self._w2_grouped
            self.w2_dense = pack_weight(grouped_to_dense(w2, self.groups), self.cmid_p, device, dtype=self.dtype)
        return self

    def forward(self, x: torch.Tensor, paradigm: str = "spatial", s: int = 1,
                coarse: Optional[torch.Tensor] = None, out: Optional[torch.Tensor] = None,
                misplace_first: bool = False, stream=None, ws: Optional[Workspace] = None,
                chmask: Optional[torch.Tensor] = None, coarse_out: Optional[torch.Tensor] = None,
                prev_coarse: Optional[torch.Tensor] = None, dn: Optional[torch.Tensor] = None,
                next_wdiff: Optional[torch.Tensor] = None, conv1_dense: Optional[bool] = None,
                aux_stream=None, latency_split: bool = False):
        """x: (N, H, W, cin_p) bf16 CUDA.  Returns (out, coarse, cell_list, cell_count)."""
        n, h, w, cl = x.shape
        if cl != self.cin_p or x.dtype != self.dtype or not x.is_contiguous():
            raise DeviceError(f"x must be contiguous NHWC {self.dtype} with pad8(C_in) channels")
        esz = 4 if self.dtype == torch.float32 else 2
        ho, wo = self.out_hw(h, w)
        blk = self.block
        if out is None:
            out = torch.empty((n, ho, wo, self.cout_p), dtype=self.dtype, device=x.device)
        ws = ws or workspace(x.device)
        if paradigm == "spatial":
            cells = n * (ho // s) * (wo // s) if s >= 1 and ho % s == 0 and wo % s == 0 else n
        else:
            cells = n
        pix = n * h * w
        i32 = 4
        if coarse is not None:
            coarse_buf = coarse
        elif coarse_out is not None:
            coarse_buf = coarse_out
        else:
            coarse_buf = ws.get("coarse", cells)
        cell_list = ws.get("cell_list", cells * i32)
        counts = ws.get("counts", 16)
        pix_list = ws.get("pix_list", pix * i32)
        h1 = ws.get("h1", pix * self.cmid_p * esz)
        h2 = ws.get("h2", n * ho * wo * self.cmid_p * esz)
        lib = _lib.lib()
        partial_n = 1
        if coarse is None and paradigm in ("spatial", "layer"):
            if self.wdiff is None:
                raise DeviceError("no mask given and no masker weights set")
            ss = s if paradigm == "spatial" else ho
            partial_n = max(1, lib.laud_masker_partial_floats(n, h, w, self.cin_p, ss, blk.stride))
        partial = ws.get("partial", partial_n * 4)
        cell_sums = ws.get("pixel_dots", pix * 4)  # conv1-fused masker: one dot per input pixel (laud.h)
        scan = ws.get("scan", lib.laud_scan_workspace_bytes(max(pix, cells)), zero=True)
        v = self.vec
        a = _lib.BlockArgs(
            paradigm=_lib.PARADIGM[paradigm], n=n, h_in=h, w_in=w, c_in=self.cin_p, x_ld=self.cin_p,
            c_mid=self.cmid_p, c_out=self.cout_p, stride=blk.stride, groups=blk.conv2.groups,
            s=s, has_down=int(blk.has_downsample), x=ptr(x), out=ptr(out), w1=ptr(self.w1),
            w2=ptr(self.w2), w3=ptr(self.w3), wd=ptr(self.wd),
            s1=ptr(v["s1"]), b1=ptr(v["b1"]), s2=ptr(v["s2"]), b2=ptr(v["b2"]),
            s3=ptr(v["s3"]), b3=ptr(v["b3"]), sd=ptr(v["sd"]), bd=ptr(v["bd"]),
            relu1=int(self.ep.relu1), relu2=int(self.ep.relu2), relu_out=int(self.ep.relu_out),
            masker_wdiff=ptr(self.wdiff), masker_bias=self.masker_bias,
            given_coarse=ptr(coarse), coarse_out=ptr(coarse_buf), cell_list=ptr(cell_list),
            cell_count=C.c_void_p(counts.data_ptr()), pix_list=ptr(pix_list),
            pix_count=C.c_void_p(counts.data_ptr() + 4), h1=ptr(h1), h2=ptr(h2),
            partial=ptr(partial), scan=ptr(scan), misplace_first=int(misplace_first),
            fp32=int(self.dtype == torch.float32),
            se_w1=ptr(self.se[0]) if self.se else None, se_b1=ptr(self.se[1]) if self.se else None,
            se_w2=ptr(self.se[2]) if self.se else None, se_b2=ptr(self.se[3]) if self.se else None,
            se_hidden=self.se[4] if self.se else 0,
            conv1_dense=int(self.conv1_dense if conv1_dense is None else conv1_dense),
            cell_sums=ptr(cell_sums))
        if paradigm == "channel":
            self._channel_args(a, n, ws, chmask)
            if self.w2_dense is not None:
                a.w2_dense = ptr(self.w2_dense)
        if dn is not None and paradigm == "spatial":
            a.dn, a.prev_coarse, a.next_wdiff = ptr(dn), ptr(prev_coarse), ptr(next_wdiff)
        if aux_stream is not None:  # small grids: masker forked onto it (laud.h aux_stream)
            a.aux_stream = stream_handle(aux_stream)
        a.latency_split = int(latency_split)  # small grids: conv2 split-K over a cluster
        _lib.check(lib.laud_block_forward(C.byref(a), stream_handle(stream)))
        return out, coarse_buf, cell_list, counts
