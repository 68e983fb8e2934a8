#!/bin/bash
# Pipeline ablation of the 1x1 residual convs (LAUD_DBG bits: 1 no epilogue math,
# 2 no stores, 8/16 no A/B loads, 32 no MMA, 64 no residual loads).
mkdir -p gpurun_out
for d in 0 2 64 66 1 67 24 32 90; do
  LAUD_DBG=$d timeout 300 python tools/engine_probe.py conv3_s3 conv3_s1 gemm_k256_n1024 > gpurun_out/abl_$d.log 2>&1
done
