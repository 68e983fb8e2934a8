"""B200 block-latency predictor for this executor.

The reference predicts LAUD block latency analytically (`latency.py:559-584`:
per-operator tile search, data + FP32-lane compute terms, a constant per
block).  On the B200 path the operators are this package's kernels, so the
model here follows the executor's own schedule (`csrc/capi.cu`,
`laud_block_forward`): for every kernel the block launches,

    t_k = max(FLOPs_k / (eta_t * P_tensor), bytes_k / (eta_m * BW)) + t_launch

with FLOPs_k / bytes_k the algorithmic counts of that launch,
P_tensor / BW the measured peaks (MEASURED_PEAKS.json), and eta_t, eta_m,
t_launch fitted per kernel class on measured B200 block latencies
(`tools/fit_native_predictor.py`, data `profiles/r01_block_latency_b200.json`,
constants `data/b200_predictor.json`).  The recalibrated reference model is
`data/b200.hw` (loadable by `dynlat.core.load_hardware`).
"""

from __future__ import annotations

import json
from dataclasses import dataclass
from pathlib import Path
from typing import Optional

from .core import BlockSpec, DynamicConfig, Paradigm

DATA = Path(__file__).resolve().parent / "data"
_PEAKS_FALLBACK = {"hbm_gbs": 6551.7, "bf16_tflops_sustained": 1384.1}
CLASSES = ("conv_gather", "conv_dense", "masker", "small")
CHANNEL_DENSE_MIN = 8  # LAUD_CH_DENSE_MIN default: batch from which channel blocks run dense-masked


@dataclass(frozen=True)
class KernelWork:
    cls: str           # one of CLASSES
    flops: float
    bytes: float


def _pad8(c: int) -> int:
    return (c + 7) // 8 * 8


def block_kernels(block: BlockSpec, cfg: DynamicConfig, rate: float, batch: int,
                  conv1_dense: Optional[bool] = None) -> list[KernelWork]:
    """The launches `laud_block_forward` issues for one block, with algorithmic
    FLOPs and compulsory bytes (bf16 storage, 2 B/element)."""
    n = batch
    cin, cm, co = _pad8(block.conv1.in_channels), _pad8(block.conv1.out_channels), _pad8(block.conv3.out_channels)
    h, w = block.input_shape.height, block.input_shape.width
    ho, wo = block.conv2.out_hw(h, w)
    g = block.conv2.groups
    pin, pout = n * h * w, n * ho * wo
    wbytes = 2.0 * (cm * cin + 9 * cm * cm / g + co * cm + (co * cin if block.has_downsample else 0))
    ks: list[KernelWork] = []
    p = cfg.paradigm
    r = 1.0 if p is Paradigm.STATIC else float(rate)

    def conv(rows_in, rows_out, k_in, n_out, taps=1, cls="conv_dense", resid=False, gdiv=1):
        fl = 2.0 * rows_out * n_out * taps * k_in / gdiv
        by = 2.0 * (rows_in * k_in + rows_out * n_out * (2 if resid else 1))
        ks.append(KernelWork(cls, fl, by))

    if p in (Paradigm.SPATIAL, Paradigm.LAYER):
        ks.append(KernelWork("masker", 0.0, 2.0 * pin * cin))
        ks.append(KernelWork("small", 0.0, 5.0 * pout))
    if block.has_downsample:
        conv(pout, pout, cin, co)
    elif p is not Paradigm.STATIC:
        pass  # in-place residual: no skip copy
    if p is Paradigm.CHANNEL:
        ks.append(KernelWork("masker", 0.0, 2.0 * pin * cin))
        if n >= CHANNEL_DENSE_MIN:  # dense-masked schedule (capi.cu channel_forward)
            conv(pin, pin, cin, cm)
            conv(pin, pout, cm, cm, taps=9, cls="conv_gather", gdiv=g)
            conv(pout, pout, cm, co, resid=True)
            return ks
        ks.append(KernelWork("small", 0.0, wbytes * n * r * r))  # per-sample packed weights
        conv(pin, pin, cin, cm * r, cls="conv_dense")
        conv(pin * r, pout, cm * r, cm * r, taps=9, cls="conv_gather")
        conv(pout, pout, cm * r, co, resid=True)
        return ks
    if p is Paradigm.SPATIAL:
        s = cfg.spatial_granularity
        dense1 = (s <= 2) if conv1_dense is None else conv1_dense
        if dense1:
            conv(pin, pin, cin, cm)
        else:
            rdil = min(1.0, r * ((s + 2) / s) ** 2)  # core.py:246-254 one-ring estimate
            ks.append(KernelWork("small", 0.0, 4.0 * pin))
            conv(pin * rdil, pin * rdil, cin, cm, cls="conv_gather")
        conv(pin * r, pout * r, cm, cm, taps=9, cls="conv_gather", gdiv=g)
        conv(pout * r, pout * r, cm, co, resid=True)
        return ks
    # static and layer: whole images of the (active) samples
    conv(pin * r, pin * r, cin, cm)
    conv(pin * r, pout * r, cm, cm, taps=9, cls="conv_gather", gdiv=g)
    conv(pout * r, pout * r, cm, co, resid=True)
    return ks


class B200Predictor:
    """Per-class efficiencies + launch cost fitted on measured B200 blocks."""

    def __init__(self, params: Optional[dict] = None, peaks: Optional[dict] = None):
        if params is None:
            params = json.loads((DATA / "b200_predictor.json").read_text())["params"]
        self.params = params
        pk = peaks or _PEAKS_FALLBACK
        self.tensor = pk.get("bf16_tflops_sustained", 1384.1) * 1e12
        self.bw = pk.get("hbm_gbs", 6551.7) * 1e9

    def kernel_us(self, k: KernelWork) -> float:
        q = self.params[k.cls]
        t_c = k.flops / (q["eta_t"] * self.tensor) if k.flops else 0.0
        t_m = k.bytes / (q["eta_m"] * self.bw) if k.bytes else 0.0
        return max(t_c, t_m) * 1e6 + q["launch_us"]

    def predict_block_us(self, block: BlockSpec, cfg: DynamicConfig, rate: float, batch: int,
                         conv1_dense: Optional[bool] = None) -> float:
        return sum(self.kernel_us(k) for k in block_kernels(block, cfg, rate, batch, conv1_dense))

    def predict_static_us(self, block: BlockSpec, batch: int) -> float:
        return self.predict_block_us(block, DynamicConfig(Paradigm.STATIC), 1.0, batch)
