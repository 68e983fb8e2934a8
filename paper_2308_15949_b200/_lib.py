"""ctypes binding of the in-tree C-ABI library ``_laud.so`` (include/laud.h).

The library is the only compute path: if it is missing, or there is no CUDA
device, every entry point raises ``DeviceError`` — there is no CPU fallback.
Status codes are re-raised as the reference's exception classes
(`pkg/src/dynlat/errors.py:8-29`).
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from .errors import DeviceError, GranularityMismatch, MaskShapeMismatch, ShapeMismatch

_SO = Path(__file__).resolve().parent / "_laud.so"
if os.environ.get("LAUD_SO_VARIANT"):  # tools/ab.sh: A/B two in-tree builds in one run
    _SO = _SO.with_name(f"_laud_{os.environ['LAUD_SO_VARIANT']}.so")

OK, ERR_GRANULARITY, ERR_MASK_SHAPE, ERR_SHAPE, ERR_UNSUPPORTED, ERR_CUDA, ERR_ARG = range(7)
PARADIGM = {"spatial": 0, "channel": 1, "layer": 2, "static": 3}

_vp, _ip, _fp, _u8p = C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_float), C.POINTER(C.c_uint8)


class ConvArgs(C.Structure):
    """Mirror of ``laud_conv_args`` (include/laud.h)."""
    _fields_ = [
        ("row_mode", C.c_int), ("list", _vp), ("count", _vp), ("rows_max", C.c_int),
        ("batch", C.c_int), ("out_h", C.c_int), ("out_w", C.c_int),
        ("patch_h", C.c_int), ("patch_w", C.c_int), ("cells_h", C.c_int), ("cells_w", C.c_int),
        ("act", _vp), ("in_h", C.c_int), ("in_w", C.c_int), ("in_c", C.c_int), ("in_ld", C.c_int),
        ("a_compact", C.c_int), ("ksize", C.c_int), ("stride", C.c_int), ("pad", C.c_int),
        ("weight", _vp), ("n_out", C.c_int), ("scale", _vp), ("bias", _vp), ("relu", C.c_int),
        ("out_mode", C.c_int), ("out", _vp), ("out_ld", C.c_int), ("out_f32", C.c_int),
        ("resid", _vp), ("resid_ld", C.c_int), ("relu_inactive_coarse", _vp),
        ("ymask_coarse", _vp), ("ymask_channel", _vp), ("sample_rows", C.c_int),
        ("chan_count", _vp), ("n_dyn", C.c_int), ("k_dyn", C.c_int), ("b_batched", C.c_int),
        ("col_index", _vp), ("col_index_ld", C.c_int), ("mdot_w", _vp), ("mdot_out", _vp),
        ("misplace_first", C.c_int), ("groups", C.c_int), ("fp32", C.c_int),
        ("b_gather", C.c_int), ("b_index", _vp), ("b_index_ld", C.c_int), ("b_rows", C.c_int),
        ("latency_split", C.c_int), ("list_expand", C.c_int),
    ]


class BlockArgs(C.Structure):
    """Mirror of ``laud_block_args`` (include/laud.h)."""
    _fields_ = [
        ("paradigm", C.c_int), ("n", C.c_int), ("h_in", C.c_int), ("w_in", C.c_int),
        ("c_in", C.c_int), ("x_ld", C.c_int), ("c_mid", C.c_int), ("c_out", C.c_int),
        ("stride", C.c_int), ("groups", C.c_int), ("s", C.c_int), ("has_down", C.c_int),
        ("x", _vp), ("out", _vp), ("w1", _vp), ("w2", _vp), ("w3", _vp), ("wd", _vp),
        ("s1", _vp), ("b1", _vp), ("s2", _vp), ("b2", _vp), ("s3", _vp), ("b3", _vp),
        ("sd", _vp), ("bd", _vp), ("relu1", C.c_int), ("relu2", C.c_int), ("relu_out", C.c_int),
        ("masker_wdiff", _vp), ("masker_bias", C.c_float), ("given_coarse", _vp),
        ("coarse_out", _vp), ("cell_list", _vp), ("cell_count", _vp), ("pix_list", _vp),
        ("pix_count", _vp), ("h1", _vp), ("h2", _vp), ("partial", _vp), ("scan", _vp),
        ("misplace_first", C.c_int), ("ch_w1", _vp), ("ch_w2", _vp), ("ch_hidden", C.c_int),
        ("ch_d", C.c_int), ("ch_groups", C.c_int), ("given_chmask", _vp), ("ch_coarse", _vp),
        ("ch_expanded", _vp), ("ch_sel", _vp), ("ch_count", _vp), ("ch_dvals", _vp),
        ("wpack", _vp), ("prev_coarse", _vp), ("dn", _vp), ("next_wdiff", _vp), ("ch_bias", _vp), ("fp32", C.c_int),
        ("conv1_dense", C.c_int), ("se_w1", _vp), ("se_b1", _vp), ("se_w2", _vp), ("se_b2", _vp),
        ("se_hidden", C.c_int), ("cell_sums", _vp), ("w2_dense", _vp), ("w3t", _vp), ("aux_stream", _vp), ("latency_split", C.c_int),
    ]


class ProfileRecord(C.Structure):
    """Mirror of ``laud_profile_record`` (include/laud.h)."""
    _fields_ = [("tag", C.c_int), ("ms", C.c_float), ("rows", C.c_longlong),
                ("n_out", C.c_longlong), ("k", C.c_longlong), ("bytes", C.c_longlong),
                ("taps", C.c_int), ("resid", C.c_int)]


_SIGS = {
    "laud_profile_begin": (None, []),
    "laud_debug_set_trace": (None, [_vp]),
    "laud_profile_end": (C.c_int, [C.POINTER(ProfileRecord), C.c_int]),
    "laud_version": (C.c_char_p, []),
    "laud_last_error": (C.c_char_p, []),
    "laud_launch_count": (C.c_uint64, []),
    "laud_scan_workspace_bytes": (C.c_size_t, [C.c_int]),
    "laud_masker_partial_floats": (C.c_size_t, [C.c_int] * 6),
    "laud_channel_pack_bytes": (C.c_size_t, [C.c_int] * 4),
    "laud_channel_masker": (C.c_int, [_vp] + [C.c_int] * 5 + [_vp, C.c_int, _vp] + [C.c_int] * 4
                            + [_vp] * 7),
    "laud_spatial_masker": (C.c_int, [_vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                      C.c_int, _vp, C.c_float, _vp, _vp, _vp, _vp, _vp, _vp]),
    "laud_cells_from_mask": (C.c_int, [_vp, C.c_int, _vp, _vp, _vp, _vp]),
    "laud_dilate_pixels": (C.c_int, [_vp] + [C.c_int] * 6 + [_vp, _vp, _vp, _vp]),
    "laud_conv": (C.c_int, [C.POINTER(ConvArgs), _vp]),
    "laud_block_forward": (C.c_int, [C.POINTER(BlockArgs), _vp]),
    "laud_stem_im2col": (C.c_int, [_vp] + [C.c_int] * 6 + [_vp, _vp, _vp, C.c_int, _vp]),
    "laud_maxpool3s2": (C.c_int, [_vp, C.c_int, C.c_int, C.c_int, C.c_int, _vp, _vp]),
    "laud_stem_pool": (C.c_int, [_vp, C.c_int, C.c_int, C.c_int, _vp, _vp, _vp, _vp, _vp, _vp]),
    "laud_stem3": (C.c_int, [_vp, C.c_int, C.c_int, C.c_int, _vp, _vp, _vp, _vp, _vp, _vp]),
    "laud_global_avgpool": (C.c_int, [_vp, C.c_int, C.c_int, C.c_int, _vp, _vp]),
}

_lib = None


def lib():
    """Load ``_laud.so`` once; raise DeviceError loudly when it cannot run."""
    global _lib
    if _lib is not None:
        return _lib
    if not _SO.exists():
        raise DeviceError(f"CUDA library {_SO} is not built; run "
                          "`python -c 'import __graft_entry__ as g; g.build()'`")
    h = C.CDLL(str(_SO), mode=os.RTLD_LOCAL | getattr(os, "RTLD_NOW", 2))
    for name, (res, args) in _SIGS.items():
        f = getattr(h, name)
        f.restype = res
        f.argtypes = args
    _lib = h
    return h


def exported_symbols():
    return tuple(_SIGS)


def check(rc: int):
    if rc == OK:
        return
    msg = lib().laud_last_error().decode(errors="replace")
    if rc == ERR_GRANULARITY:
        raise GranularityMismatch(msg)
    if rc == ERR_MASK_SHAPE:
        raise MaskShapeMismatch(msg)
    if rc in (ERR_SHAPE, ERR_UNSUPPORTED):
        raise ShapeMismatch(msg)
    if rc == ERR_ARG:
        raise ValueError(msg)
    raise DeviceError(msg)


def call(name: str, *args):
    check(getattr(lib(), name)(*args))
