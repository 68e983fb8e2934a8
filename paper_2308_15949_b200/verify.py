"""`verify` against the GPU path — the reference's equivalence command
(`cli.py:250-278`, `_cmd_verify`) with the same flags, output and exit codes,
run through this package's CUDA executors.

  python -m paper_2308_15949_b200.verify [--cases FILE] [--per-paradigm N]
                                          [--seed S] [--inject-fault]
                                          [--precision bf16|fp32]

Per case `reference.run_equivalence_case` compares the GPU sparse executor
with the GPU dense-masked executor (`reference.py:499-520`).  Spatial and
layer cases share every rounding point and must agree to the case tolerance
(1e-9, i.e. bit-exact).  Channel cases take different bf16 rounding paths
(ragged per-sample K vs full K with zeroed channels); in bf16 mode their
deviation is judged relative to the output scale at 2e-2 (fp32 mode: the
case tolerance).  Exit 0 on success, 1 on any failure, 2/3 on argument /
validation errors, like the reference CLI (`cli.py:355-365`).
"""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

from . import reference as R
from .core import Paradigm
from .errors import DynlatError

BF16_CHANNEL_REL = 2e-2


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="laud-verify", description="sparse-vs-dense executor equivalence (GPU)")
    ap.add_argument("--cases", default=None, help="case descriptor file")
    ap.add_argument("--per-paradigm", type=int, default=10)
    ap.add_argument("--seed", type=int, default=0, help="offset for case seeds")
    ap.add_argument("--inject-fault", action="store_true",
                    help="test-only: misplace one scatter index, must fail")
    ap.add_argument("--precision", choices=("bf16", "fp32"), default="bf16")
    args = ap.parse_args(argv)
    try:
        R.set_precision(args.precision)
        if args.cases:
            cases = R.parse_cases_text(Path(args.cases).read_text(), args.cases)
        else:
            cases = R.default_cases(per_paradigm=args.per_paradigm)
        if args.seed:
            cases = [R.EquivalenceCase(c.paradigm, c.channels, c.height, c.width, c.granularity,
                                       c.seed + args.seed, c.tolerance) for c in cases]
        if not cases:
            print("verify: 0 cases, nothing to check")
            return 0
        worst: dict[str, float] = {}
        failures = 0
        for i, case in enumerate(cases):
            fault = args.inject_fault and i == 0
            dev = R.run_equivalence_case(case, inject_fault=fault)
            key = case.paradigm.value
            worst[key] = max(worst.get(key, 0.0), dev)
            tol = case.tolerance
            if case.paradigm is Paradigm.CHANNEL and args.precision == "bf16":
                tol = max(tol, BF16_CHANNEL_REL * _channel_scale(case))
            if dev >= tol:
                failures += 1
        for key in sorted(worst):
            print(f"{key}: worst |delta| = {worst[key]:.3e}")
        print(f"{len(cases)} cases, {failures} failures")
        return 1 if failures else 0
    except (DynlatError, ValueError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 3
    finally:
        R.set_precision("bf16")


def _channel_scale(case) -> float:
    """max |output| of the case's dense-masked result (the channel tolerance scale)."""
    import numpy as np
    rng = np.random.default_rng(case.seed)
    block = R._case_block(case)
    n, mask = R._case_mask(case, block, rng)
    bw = R.make_block_weights(block, rng)
    x = rng.standard_normal((n, case.channels, case.height, case.width))
    from .core import DynamicConfig
    cfg = DynamicConfig(Paradigm.CHANNEL, channel_granularity=case.granularity)
    return float(np.max(np.abs(R.block_forward_dense_masked(x, bw, block, cfg, mask))))


if __name__ == "__main__":
    sys.exit(main())
