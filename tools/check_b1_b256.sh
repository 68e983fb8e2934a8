#!/bin/bash
# GPU suite + batch-1 latency (R101, R50) + the b256 / RegNet steps of the current build.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/vec_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/vec_pytest.log
for rep in 1 2; do
  echo "$(timeout 300 python tools/b1_latency.py resnet101 2>&1 | tail -1)"
  echo "$(timeout 300 python tools/b1_latency.py resnet50 spatial 4-4-2-1 2>&1 | tail -1)"
done > gpurun_out/vec_b1.log 2>&1
B="timeout 600 python bench.py --steps 10 --warmup 3 --no-traffic --no-baselines"
$B > gpurun_out/vec_r101.log 2>&1
$B --arch regnety-1.6gf --plan 4-4-2-1 --global-batch 1024 > gpurun_out/vec_rg.log 2>&1
