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
         misplace_first=0, stream=None):
    """One call of the implicit-GEMM engine (``laud_conv``)."""
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
        misplace_first=misplace_first)
    _lib.check(_lib.lib().laud_conv(C.byref(a), D.stream_handle(stream)))


def dense_block(db: D.DeviceBlock, x: torch.Tensor, ymask: Optional[torch.Tensor] = None,
                patch=(1, 1), chmask: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """Dense bottleneck with optional dense-masked epilogues."""
    n, h, w, _ = x.shape
    ho, wo = db.out_hw(h, w)
    blk = db.block
    v = db.vec
    out = torch.empty((n, ho, wo, db.cout_p), dtype=torch.bfloat16, device=x.device)
    h1 = torch.empty((n, h, w, db.cmid_p), dtype=torch.bfloat16, device=x.device)
    h2 = torch.empty((n * ho * wo, db.cmid_p), dtype=torch.bfloat16, device=x.device)
    if blk.has_downsample:
        conv(act=x, in_hw=(h, w), in_c=db.cin_p, in_ld=db.cin_p, weight=db.wd, n_out=db.cout_p,
             out=out, out_ld=db.cout_p, out_hw=(ho, wo), batch=n, stride=blk.stride,
             scale=v["sd"], bias=v["bd"], stream=stream)
    else:
        out.copy_(x)
    conv(act=x, in_hw=(h, w), in_c=db.cin_p, in_ld=db.cin_p, weight=db.w1, n_out=db.cmid_p,
         out=h1, out_ld=db.cmid_p, out_hw=(h, w), batch=n, scale=v["s1"], bias=v["b1"],
         relu=int(db.ep.relu1), ymask_channel=chmask, stream=stream)
    conv(act=h1, in_hw=(h, w), in_c=db.cmid_p, in_ld=db.cmid_p, weight=db.w2, n_out=db.cmid_p,
         out=h2, out_ld=db.cmid_p, out_hw=(ho, wo), batch=n, ksize=3, stride=blk.stride, pad=1,
         scale=v["s2"], bias=v["b2"], relu=int(db.ep.relu2), out_mode=OUT_ROW,
         ymask_channel=chmask, stream=stream)
    cells = (ho // patch[0], wo // patch[1])
    conv(act=h2, in_hw=(ho, wo), in_c=db.cmid_p, in_ld=db.cmid_p, weight=db.w3, n_out=db.cout_p,
         out=out, out_ld=db.cout_p, out_hw=(ho, wo), batch=n, a_compact=1, scale=v["s3"],
         bias=v["b3"], relu=int(db.ep.relu_out), resid=out, resid_ld=db.cout_p, patch=patch,
         cells=cells, ymask_coarse=ymask, stream=stream)
    return out


def channel_masker_forward(x, weights, g, mode="inference", tau=None, rng=None):
    raise DeviceError("channel masker kernel not built yet")


def channel_block_sparse(x, bw, block, mask):
    raise DeviceError("channel-skipping block kernel not built yet")
