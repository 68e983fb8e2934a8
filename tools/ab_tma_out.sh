#!/bin/bash
# TMA-store epilogue: GPU suite, isolated shapes and the R101 / RegNet steps, LAUD_TMA_OUT=0 vs 1.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/tma_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/tma_pytest.log
for v in 0 1; do
  LAUD_TMA_OUT=$v timeout 300 python tools/engine_probe.py conv3_s3 conv3_s1 gemm_k256_n1024 gemm_k1024_n256 rg_s3_1x1 > gpurun_out/tma_probe$v.log 2>&1
done
B="timeout 600 python bench.py --steps 10 --warmup 3 --no-traffic --no-baselines"
for i in 1 2; do
  LAUD_TMA_OUT=0 $B > gpurun_out/tma_r101_0_$i.log 2>&1
  LAUD_TMA_OUT=1 $B > gpurun_out/tma_r101_1_$i.log 2>&1
done
LAUD_TMA_OUT=0 $B --arch regnety-1.6gf --plan 4-4-2-1 --global-batch 1024 > gpurun_out/tma_rg_0.log 2>&1
LAUD_TMA_OUT=1 $B --arch regnety-1.6gf --plan 4-4-2-1 --global-batch 1024 > gpurun_out/tma_rg_1.log 2>&1
