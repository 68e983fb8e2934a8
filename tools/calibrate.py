"""Calibrate the masker biases of benchmark configurations on the GPU and
commit them (paper_2308_15949_b200/data/masker_biases.json).

The bias on each block's masker logit (EXT) stands in for a trained masker's
FLOPs loss: it is set so the block's activation ratio on a HELD-OUT batch
(``bench.calib_images``, disjoint from the timed images) hits the target.
Deterministic (same weights, images and kernels) — this file only lets the
CPU reference arm use exactly the GPU arm's biases.

  python tools/calibrate.py [arch/paradigm/plan/ratio ...]
"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2308_15949_b200.network import LaudNetwork  # noqa: E402

DEFAULT = ["resnet101/spatial/4-2-2-1/0.5", "resnet50/spatial/4-4-2-1/0.5", "resnet101/layer/4-2-2-1/0.5",
           "resnet101/channel/1-1-1-1/0.5", "regnety-1.6gf/spatial/4-4-2-1/0.5"]


def main(keys):
    out = json.loads(bench.BIAS_FILE.read_text()) if bench.BIAS_FILE.exists() else {"configs": {}}
    out["how"] = ("tools/calibrate.py: per block, bias = -(1 - ratio) quantile of the masker decision values "
                  "on bench.calib_images(64) (held out from the timed images), block by block through the network")
    for key in keys:
        arch, para, plan, ratio = key.split("/")
        net = LaudNetwork(arch, para, plan, float(ratio), seed=0)
        net.calibrate(torch.from_numpy(bench.calib_images(64)).cuda())
        out["configs"][key] = {"biases": [float(b) for b in net.masker_biases()], "calib_images": 64}
        print(key, "ok", flush=True)
        del net
        torch.cuda.empty_cache()
    bench.BIAS_FILE.write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main(sys.argv[1:] or DEFAULT)
