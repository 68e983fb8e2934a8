#!/bin/bash
# Tile-width A/B on isolated conv shapes (engine_probe under LAUD_BN) + one
# pipeline trace of the stage-3 conv3. usage: bash tools/probe_bn.sh [shapes...]
mkdir -p gpurun_out
S=${@:-conv3_s3 conv3_s1 gemm_k256_n1024 gemm_k1024_n256 rg_s3_1x1}
for bn in 0 128 256; do
  LAUD_BN=$bn timeout 300 python tools/engine_probe.py $S > gpurun_out/probe_bn$bn.log 2>&1
done
timeout 300 python tools/engine_trace.py conv3_s3 > gpurun_out/trace_conv3.log 2>&1
