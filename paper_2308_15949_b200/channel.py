"""Dense block composition on the conv engine, and the channel paradigm.

``dense_block`` runs a whole bottleneck densely through ``laud_conv`` with
the dense-masked epilogue options (`reference.py:313-353`): a per-cell mask
on conv3's output (spatial / layer) or a per-sample channel mask on conv1's
and conv2's outputs (channel).  It backs ``block_forward_dense_masked``.
"""

from __future__ import annotations

import ctypes as C
from typing import Optional

import torch

from . import _lib
from . import device as D
from .errors import DeviceError

ROWS_DENSE, ROWS_PATCH, ROWS_PIXEL = 0, 1, 2
OUT_PIXEL, OUT_ROW = 0, 1


def conv(*, act, in_hw, in_c, in_ld, weight, n_out, out, out_ld, out_hw, batch, ksize=1, stride=1,
         pad=0, row_mode=ROWS_DENSE, rows_max=None, lst=None, count=None, patch=(1, 1),
         cells=(1, 1), a_compact=0, scale=None, bias=None, relu=0, out_mode=OUT_PIXEL, out_f32=0,
         resid=None, resid_ld=0, relu_inactive=None, ymask_coarse=None, ymask_channel=None,
         misplace_first=0, groups=1, fp32=0, stream=None, **extra):
    """One call of the implicit-GEMM engine (``laud_conv``); ``extra``: further
    ``laud_conv_args`` fields (per-sample / gathered-weight modes), pointers as tensors."""
    a = _lib.ConvArgs(
        row_mode=row_mode, list=D.ptr(lst), count=D.ptr(count),
        rows_max=rows_max if rows_max is not None else batch * out_hw[0] * out_hw[1],
        batch=batch, out_h=out_hw[0], out_w=out_hw[1], patch_h=patch[0], patch_w=patch[1],
        cells_h=cells[0], cells_w=cells[1], act=D.ptr(act), in_h=in_hw[0], in_w=in_hw[1],
        in_c=in_c, in_ld=in_ld, a_compact=a_compact, ksize=ksize, stride=stride, pad=pad,
        weight=D.ptr(weight), n_out=n_out, scale=D.ptr(scale), bias=D.ptr(bias), relu=relu,
        out_mode=out_mode, out=D.ptr(out), out_ld=out_ld, out_f32=out_f32, resid=D.ptr(resid),
        resid_ld=resid_ld, relu_inactive_coarse=D.ptr(relu_inactive),
        ymask_coarse=D.ptr(ymask_coarse), ymask_channel=D.ptr(ymask_channel),
        misplace_first=misplace_first, groups=groups, fp32=fp32)
    for k, v in extra.items():
        setattr(a, k, D.ptr(v) if isinstance(v, torch.Tensor) else v)
    _lib.check(_lib.lib().laud_conv(C.byref(a), D.stream_handle(stream)))


def dense_block(db: D.DeviceBlock, x: torch.Tensor, ymask: Optional[torch.Tensor] = None,
                patch=(1, 1), chmask: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """Dense bottleneck with optional dense-masked epilogues."""
    n, h, w, _ = x.shape
    ho, wo = db.out_hw(h, w)
    blk = db.block
    v = db.vec
    dt = getattr(db, "dtype", torch.bfloat16)
    f32 = int(dt == torch.float32)
    out = torch.empty((n, ho, wo, db.cout_p), dtype=dt, device=x.device)
    h1 = torch.empty((n, h, w, db.cmid_p), dtype=dt, device=x.device)
    h2 = torch.empty((n * ho * wo, db.cmid_p), dtype=dt, device=x.device)
    if blk.has_downsample:
        conv(act=x, in_hw=(h, w), in_c=db.cin_p, in_ld=db.cin_p, weight=db.wd, n_out=db.cout_p,
             out=out, out_ld=db.cout_p, out_hw=(ho, wo), batch=n, stride=blk.stride,
             scale=v["sd"], bias=v["bd"], fp32=f32, stream=stream)
    else:
        out.copy_(x)
    conv(act=x, in_hw=(h, w), in_c=db.cin_p, in_ld=db.cin_p, weight=db.w1, n_out=db.cmid_p,
         out=h1, out_ld=db.cmid_p, out_hw=(h, w), batch=n, scale=v["s1"], bias=v["b1"],
         relu=int(db.ep.relu1), ymask_channel=chmask, fp32=f32, stream=stream)
    conv(act=h1, in_hw=(h, w), in_c=db.cmid_p, in_ld=db.cmid_p, weight=db.w2, n_out=db.cmid_p,
         out=h2, out_ld=db.cmid_p, out_hw=(ho, wo), batch=n, ksize=3, stride=blk.stride, pad=1,
         scale=v["s2"], bias=v["b2"], relu=int(db.ep.relu2), out_mode=OUT_ROW,
         ymask_channel=chmask, groups=getattr(db, "groups", 1), fp32=f32, stream=stream)
    cells = (ho // patch[0], wo // patch[1])
    conv(act=h2, in_hw=(ho, wo), in_c=db.cmid_p, in_ld=db.cmid_p, weight=db.w3, n_out=db.cout_p,
         out=out, out_ld=db.cout_p, out_hw=(ho, wo), batch=n, a_compact=1, scale=v["s3"],
         bias=v["b3"], relu=int(db.ep.relu_out), resid=out, resid_ld=db.cout_p, patch=patch,
         cells=cells, ymask_coarse=ymask, fp32=f32, stream=stream)
    return out


def _rm():
    from . import reference as R
    return R


def channel_masker_forward(x, weights, g, mode="inference", tau=None, rng=None):
    """GAP -> relu(W1 .) -> W2 -> D pairs -> keep iff l0 >= l1 -> repeat G.

    Device version of `reference.py:189-218` (K5 kernel, fp32 math).  Train
    mode replays the reference's Gumbel draw (`rng.gumbel(size=(N, D, 2))`)
    on the device logit gaps.
    """
    import numpy as np
    from .errors import ShapeMismatch
    R = _rm()
    if mode not in ("inference", "train"):
        raise ValueError(f"unknown mode {mode!r}")
    D.require_cuda()
    w1, w2 = (np.asarray(w, dtype=np.float64) for w in weights)
    hd, c = w1.shape
    if w2.shape[1] != hd or w2.shape[0] % 2:
        raise ShapeMismatch("second MLP layer must map hidden -> 2*D")
    d = w2.shape[0] // 2
    xd, numpy_in = R._dev_in(x, c, x.dtype if isinstance(x, torch.Tensor) else torch.float32)
    n, h, w, cp = xd.shape
    cm = d * g
    cmp = D.pad8(cm)
    w1p = np.zeros((hd, cp), np.float32)
    w1p[:, :c] = w1
    t_w1 = torch.from_numpy(w1p).cuda()
    t_w2 = torch.from_numpy(w2.astype(np.float32)).cuda()
    coarse = torch.empty(n * d, dtype=torch.uint8, device="cuda")
    dvals = torch.empty(n * d, dtype=torch.float32, device="cuda")
    exp = torch.empty(n * cmp, dtype=torch.uint8, device="cuda")
    sel = torch.empty(n * cmp, dtype=torch.int32, device="cuda")
    cnt = torch.empty(n, dtype=torch.int32, device="cuda")
    _lib.call("laud_channel_masker", D.ptr(xd), int(xd.dtype == torch.float32), cp, n, h * w, cp, D.ptr(t_w1),
              hd, D.ptr(t_w2),
              d, g, cm, cmp, D.ptr(coarse), D.ptr(dvals), D.ptr(exp), D.ptr(sel), D.ptr(cnt),
              None, D.stream_handle())
    soft = None
    if mode == "inference" and not numpy_in:  # stays on the device
        cz = coarse.view(n, d).bool()
        return R.ChannelMask(cz, cz.repeat_interleave(g, dim=1), g, None)
    if mode == "inference":
        cz = coarse.view(n, d).bool().cpu().numpy()
    else:
        dv = dvals.view(n, d).double().cpu().numpy()
        cz, soft = R._decide_train(dv, tau, rng)
    return R.ChannelMask(cz, np.repeat(cz, g, axis=1), g, soft)


def channel_block_sparse(x, bw, block, mask, grouped_channel_ext: bool = False):
    """Channel-skipping block forward on the device (`reference.py:404-423`).

    ``grouped_channel_ext`` (EXT) lifts the reference's groups == 1 requirement
    (`reference.py:405-406`): a grouped conv2 runs as its block-diagonal dense
    kernel, the sparse form of the reference's dense-masked channel forward."""
    import numpy as np
    from .errors import ShapeMismatch
    R = _rm()
    if block.conv2.groups != 1 and not grouped_channel_ext:
        raise ShapeMismatch("sparse channel execution requires groups == 1")
    db = R.device_block(bw, block)
    if block.conv2.groups != 1:
        db.enable_grouped_channel()
    xd, numpy_in = R._dev_in(x, block.input_shape.channels, db.dtype)
    n = xd.shape[0]
    chm = R._channel_mask_u8(mask.expanded, n, block.conv2.out_channels, db.cmid_p)
    y, *_ = db.forward(xd, "channel", chmask=chm)
    return R._dev_out(y, block.output_shape.channels, numpy_in)
