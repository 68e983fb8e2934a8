"""B200 latency predictor: fitted constants load, predictions
are monotone in the activation rate and track the measured B200 blocks.  CPU only."""
import json
from pathlib import Path

import numpy as np

from paper_2308_15949_b200 import predictor as P
from paper_2308_15949_b200.core import DynamicConfig, Paradigm
from paper_2308_15949_b200.zoo import build_network

ROOT = Path(__file__).resolve().parent.parent


def _block(arch="resnet101", stage=3, index=1):
    return [b.block for b in build_network(arch).blocks if b.stage == stage and b.index == index][0]


def test_fitted_constants_and_monotonicity():
    m = P.B200Predictor()
    blk = _block()
    for para, cfg in ((Paradigm.SPATIAL, DynamicConfig(Paradigm.SPATIAL, spatial_granularity=2)),
                      (Paradigm.CHANNEL, DynamicConfig(Paradigm.CHANNEL, channel_granularity=1)),
                      (Paradigm.LAYER, DynamicConfig(Paradigm.LAYER))):
        ts = [m.predict_block_us(blk, cfg, r, 256) for r in (0.2, 0.5, 0.8)]
        assert ts[0] <= ts[1] <= ts[2], (para, ts)
    assert m.predict_block_us(blk, DynamicConfig(Paradigm.SPATIAL, spatial_granularity=2), 0.5, 256) < \
        m.predict_static_us(blk, 256)


def test_predictor_tracks_measured_b200_blocks():
    data = json.loads((ROOT / "profiles" / "r02m_block_latency_b200.json").read_text())
    m = P.B200Predictor()
    nets = {}
    ape = []
    for r in data["rows"][1::3]:  # held-out rows of the fit
        net = nets.setdefault(r["arch"], build_network(r["arch"]))
        blk = [b.block for b in net.blocks if b.stage == r["stage"] and b.index == r["index"]][0]
        p = Paradigm(r["paradigm"])
        cfg = (DynamicConfig(p, spatial_granularity=r["S"]) if p is Paradigm.SPATIAL else
               DynamicConfig(p, channel_granularity=1) if p is Paradigm.CHANNEL else DynamicConfig(p))
        pred = m.predict_block_us(blk, cfg, r["r"], r["batch"], r.get("conv1_dense"))
        ape.append(abs(pred - r["us"]) / r["us"])
    assert np.median(ape) < 0.2, np.median(ape)


def test_b200_hw_spec_file_format():
    text = (ROOT / "paper_2308_15949_b200" / "data" / "b200.hw").read_text()
    kv = dict(line.split("=", 1) for line in (l.split("#")[0].strip() for l in text.splitlines()) if line)
    kv = {k.strip(): v.strip() for k, v in kv.items()}
    for key in ("name", "pe_count", "fp32_per_pe", "frequency_mhz", "bandwidth_g", "onchip_bandwidth_factor",
                "movement_efficiency", "const_overhead_us"):
        assert key in kv
    assert int(kv["pe_count"]) == 148 and 0 < float(kv["movement_efficiency"]) <= 1


def test_channel_schedule_switch():
    """Channel blocks run dense-masked from CHANNEL_DENSE_MIN samples on (capi.cu
    channel_forward): rate-independent there, rate-dependent per-sample below."""
    m = P.B200Predictor()
    blk = _block()
    cfg = DynamicConfig(Paradigm.CHANNEL, channel_granularity=1)
    big = [m.predict_block_us(blk, cfg, r, 256) for r in (0.2, 0.8)]
    assert abs(big[0] - big[1]) < 1e-9
    small = [m.predict_block_us(blk, cfg, r, 1) for r in (0.2, 0.8)]
    assert small[0] < small[1]
    ks = P.block_kernels(blk, cfg, 0.5, P.CHANNEL_DENSE_MIN)
    assert not any(k.cls == "small" for k in ks)  # no per-sample weight packing


def test_grouped_to_dense_device_matches_oracle():
    from oracle import laud_oracle as O
    from paper_2308_15949_b200 import device as D
    w = np.random.default_rng(0).standard_normal((48, 8, 3, 3))
    np.testing.assert_array_equal(D.grouped_to_dense(w, 6), O.grouped_to_dense(w, 6))
