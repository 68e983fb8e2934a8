#!/bin/bash
# Output-stream-bound 1x1 convs: tile width (LAUD_BN) x store path (LAUD_TMA_OUT).
mkdir -p gpurun_out
for bn in 64 128 256; do for to in 0 1; do
  echo "bn=$bn tma_out=$to $(LAUD_BN=$bn LAUD_TMA_OUT=$to timeout 300 python tools/engine_probe.py ds_s1 conv3_s1 gemm_k256_n1024 | tr '\n' ' ')"
done; done > gpurun_out/probe_ds.log 2>&1
