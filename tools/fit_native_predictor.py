"""Fit the B200 predictor (paper_2308_15949_b200/predictor.py) to measured blocks.

usage: python tools/fit_native_predictor.py profiles/r01_block_latency_b200.json

Least squares on log latency over every third measurement (the rest held
out); per kernel class: tensor efficiency eta_t, memory efficiency eta_m and
a per-launch cost.  Writes paper_2308_15949_b200/data/b200_predictor.json and
profiles/r01_native_predictor_fit.json.
"""
import json
import math
import sys
from pathlib import Path

import numpy as np
from scipy.optimize import least_squares

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2308_15949_b200 import predictor as P  # noqa: E402
from paper_2308_15949_b200.core import DynamicConfig, Paradigm  # noqa: E402
from paper_2308_15949_b200.zoo import build_network  # noqa: E402

CONV = ("conv_gather", "conv_dense")


def unpack(z):
    out, i = {}, 0
    for c in P.CLASSES:
        if c in CONV:
            out[c] = {"eta_t": 1 / (1 + math.exp(-z[i])), "eta_m": 1 / (1 + math.exp(-z[i + 1])),
                      "launch_us": math.exp(z[i + 2])}
            i += 3
        else:
            out[c] = {"eta_t": 1.0, "eta_m": 1 / (1 + math.exp(-z[i])), "launch_us": math.exp(z[i + 1])}
            i += 2
    return out


def main():
    data = json.loads(Path(sys.argv[1]).read_text())
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else None
    nets = {}
    items = []
    for r in data["rows"]:
        net = nets.setdefault(r["arch"], build_network(r["arch"]))
        blk = [b.block for b in net.blocks if b.stage == r["stage"] and b.index == r["index"]][0]
        p = Paradigm(r["paradigm"])
        cfg = (DynamicConfig(p, spatial_granularity=r["S"]) if p is Paradigm.SPATIAL else
               DynamicConfig(p, channel_granularity=r.get("G", 1)) if p is Paradigm.CHANNEL else DynamicConfig(p))
        ks = P.block_kernels(blk, cfg, r["r"], r["batch"], r.get("conv1_dense"))
        items.append((ks, r["us"], r["paradigm"]))
    fit = items[::3]
    hold = [it for i, it in enumerate(items) if i % 3]

    def preds(z, its):
        model = P.B200Predictor(unpack(z), peaks)
        return np.array([sum(model.kernel_us(k) for k in ks) for ks, _, _ in its])

    def resid(z):
        return np.log(preds(z, fit)) - np.log([us for _, us, _ in fit])

    z0 = []
    for c in P.CLASSES:
        z0 += [0.0, 0.0, math.log(3.0)] if c in CONV else [0.0, math.log(3.0)]
    res = least_squares(resid, np.array(z0))
    params = unpack(res.x)

    def stats(its, z):
        pr = preds(z, its)
        ape = np.abs(pr - np.array([us for _, us, _ in its])) / np.array([us for _, us, _ in its])
        return {"mape": float(ape.mean()), "median_ape": float(np.median(ape)),
                "p90_ape": float(np.percentile(ape, 90)), "n": len(its)}

    report = {
        "model": "paper_2308_15949_b200.predictor.B200Predictor (per-launch roofline, fitted efficiencies)",
        "measurements": sys.argv[1],
        "params": params,
        "fit_rows": stats(fit, res.x), "held_out": stats(hold, res.x),
        "by_paradigm_held_out": {p: stats([it for it in hold if it[2] == p], res.x)
                                 for p in ("static", "spatial", "channel", "layer")},
    }
    (ROOT / "paper_2308_15949_b200" / "data").mkdir(exist_ok=True)
    (ROOT / "paper_2308_15949_b200" / "data" / "b200_predictor.json").write_text(
        json.dumps({"params": params, "source": sys.argv[1]}, indent=1) + "\n")
    (ROOT / "profiles" / f"{Path(sys.argv[1]).name.split('_')[0]}_native_predictor_fit.json").write_text(json.dumps(report, indent=1) + "\n")
    print(json.dumps({k: report[k] for k in ("fit_rows", "held_out", "by_paradigm_held_out")}, indent=1))


if __name__ == "__main__":
    main()
