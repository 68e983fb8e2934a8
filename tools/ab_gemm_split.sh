#!/bin/bash
# Engine cluster split-K for small grids: GPU suite, then batch-1 latency with
# LAUD_GEMM_KSPLIT_MAX=0 (off) vs the default, and the headline step (unaffected path check).
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gks_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/gks_pytest.log
for rep in 1 2; do for v in 0 8; do
  echo "ks=$v $(LAUD_GEMM_KSPLIT_MAX=$v timeout 300 python tools/b1_latency.py resnet101 2>&1 | tail -1)"
  echo "ks=$v $(LAUD_GEMM_KSPLIT_MAX=$v timeout 300 python tools/b1_latency.py resnet50 spatial 4-4-2-1 2>&1 | tail -1)"
done; done > gpurun_out/gks_b1.log 2>&1
LAUD_PDL=0 timeout 300 python tools/graph_kernels.py resnet101 spatial 1 > gpurun_out/gks_gk.txt 2>&1
B="timeout 600 python bench.py --steps 10 --warmup 3 --no-traffic --no-baselines"
LAUD_GEMM_KSPLIT_MAX=0 $B > gpurun_out/gks_r101_0.log 2>&1
$B > gpurun_out/gks_r101_8.log 2>&1
