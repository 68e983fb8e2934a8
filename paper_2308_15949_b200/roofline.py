"""Algorithmic FLOPs / compulsory bytes of the LAUD hot path.

Pure host arithmetic (numpy) used by ``bench.py`` to turn measured times into
roofline fractions.  Only the work the reference algorithm must do is
credited: a spatial block gets ``2·(r_dil_in·F1 + r·F2 + r·F3 + F_down +
masker)`` (halo recompute and the dense-conv1 schedule's extra rows are not
credited), channel skipping ``2·Σ_samples(r_i·F1 + r_i²·F2 + r_i·F3)``
(`flops.py:164-168`), layer skipping ``2·r·ΣF``; grouped convs count
C_in/groups per output (`flops.py:81-88`).  Bytes: |x| once, the output
(``r·|y|`` for in-place stride-1 spatial blocks, whose inactive cells are never
touched), |W| once, 4 bytes per active-cell index.
"""

from __future__ import annotations

import numpy as np

from .core import BlockSpec


def _cover(n_cells: int, s: int, st: int, size: int) -> np.ndarray:
    """[cells, size] bool: input row y is read by cell i's 3x3 halo at stride st."""
    i = np.arange(n_cells)[:, None]
    y = np.arange(size)[None, :]
    lo = i * s * st - 1
    hi = i * s * st + (s - 1) * st + 1
    return (y >= lo) & (y <= hi)


def dilated_input_fraction(coarse: np.ndarray, block: BlockSpec, s: int) -> float:
    """r_dil_in: fraction of conv1's input-grid pixels that any active cell's
    conv2 window reads (the union of halos, clipped to the image)."""
    coarse = np.asarray(coarse).astype(np.float32)
    n, ch, cw = coarse.shape
    st = block.stride
    hi, wi = block.input_shape.height, block.input_shape.width
    ay = _cover(ch, s, st, hi).astype(np.float32)  # [ch, H]
    ax = _cover(cw, s, st, wi).astype(np.float32)  # [cw, W]
    cov = np.einsum("ih,nij,jw->nhw", ay, coarse, ax, optimize=True) > 0
    return float(cov.mean()) if cov.size else 0.0


def _convs(block: BlockSpec, n: int):
    out = block.output_shape
    cin, hi, wi = block.input_shape.channels, block.input_shape.height, block.input_shape.width
    cm, co, g = block.conv1.out_channels, block.conv3.out_channels, block.conv2.groups
    f1 = n * hi * wi * cin * cm
    f2 = n * out.height * out.width * cm * (cm // g) * 9
    f3 = n * out.height * out.width * cm * co
    fd = n * out.height * out.width * cin * co if block.has_downsample else 0
    w = cin * cm + cm * (cm // g) * 9 + cm * co + (cin * co if block.has_downsample else 0)
    return f1, f2, f3, fd, w


def block_algorithmic(block: BlockSpec, paradigm: str, n: int, coarse=None, s: int = 1,
                      keep=None, decisions=None, elt: int = 2) -> dict:
    """Algorithmic FLOPs and compulsory bytes of one block forward over n samples.

    spatial: ``coarse`` [n, H/S, W/S] bool on the output grid; channel: ``keep``
    [n, C_mid] bool (expanded mask); layer: ``decisions`` [n] bool.
    """
    f1, f2, f3, fd, wel = _convs(block, n)
    cin, hi, wi = block.input_shape.channels, block.input_shape.height, block.input_shape.width
    out = block.output_shape
    x_b = n * hi * wi * cin * elt
    y_b = n * out.height * out.width * block.conv3.out_channels * elt
    w_b = wel * elt
    in_place = not block.has_downsample
    d = dict(r=1.0, r_dil_in=1.0, static_flops=2.0 * (f1 + f2 + f3 + fd))
    if paradigm == "spatial":
        coarse = np.asarray(coarse, dtype=bool)
        r = float(coarse.mean()) if coarse.size else 0.0
        rd = dilated_input_fraction(coarse, block, s)
        fm = n * hi * wi * cin
        flops = 2.0 * (rd * f1 + r * f2 + r * f3 + fd + fm)
        nbytes = x_b + (r * y_b if in_place else y_b) + w_b + 4 * int(coarse.sum())
        d.update(r=r, r_dil_in=rd)
    elif paradigm == "channel":
        keep = np.asarray(keep, dtype=bool).reshape(n, -1)[:, : block.conv1.out_channels]
        ri = keep.mean(axis=1) if keep.size else np.zeros(n)
        per = 1.0 / max(n, 1)
        flops = 2.0 * (float(np.sum(ri)) * per * (f1 + f3) + float(np.sum(ri ** 2)) * per * f2 + fd
                       + n * hi * wi * cin)
        nbytes = x_b + y_b + w_b
        d.update(r=float(ri.mean()) if n else 0.0)
    elif paradigm == "layer":
        dec = np.asarray(decisions, dtype=bool).reshape(-1)
        r = float(dec.mean()) if dec.size else 0.0
        flops = 2.0 * (r * (f1 + f2 + f3) + fd + n * hi * wi * cin)
        nbytes = x_b + (r * y_b if in_place else y_b) + w_b
        d.update(r=r)
    else:
        flops = 2.0 * (f1 + f2 + f3 + fd)
        nbytes = x_b + y_b + w_b
    d.update(flops=flops, bytes=float(nbytes))
    return d


def roofline_seconds(flops: float, nbytes: float, peak_tflops: float, peak_gbs: float) -> float:
    """The slower of FLOPs at tensor peak and bytes at HBM bandwidth."""
    return max(flops / (peak_tflops * 1e12), nbytes / (peak_gbs * 1e9))


def stem_fc_algorithmic(net, n: int, elt: int = 2) -> dict:
    """Stem conv (k x k / 2 over 3 channels) + max-pool + GAP + FC of the network."""
    st = net.stem
    h = w = 224
    ho, wo = (h + 2 * (st.kernel // 2) - st.kernel) // st.stride + 1, (w + 2 * (st.kernel // 2) - st.kernel) // st.stride + 1
    f_stem = 2.0 * n * ho * wo * st.out_channels * st.kernel * st.kernel * 3
    f_fc = 2.0 * n * net.classifier_features * net.num_classes
    nbytes = n * h * w * 3 + n * ho * wo * st.out_channels * elt + \
        (st.out_channels * st.kernel ** 2 * 3 + net.classifier_features * net.num_classes) * elt + \
        n * net.num_classes * 4
    return dict(flops=f_stem + f_fc, bytes=float(nbytes))
