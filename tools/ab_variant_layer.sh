#!/bin/bash
# Same-box A/B of a _laud_<variant>.so (LAUD_SO_VARIANT) on the channel paradigm + its GPU tests.
V=${1:-oldcm}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "layer or network or masker or spatial" > gpurun_out/ably_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ably_pytest.log
B="timeout 600 python bench.py --steps 10 --warmup 3 --no-traffic --no-baselines --paradigm layer"
for i in 1 2; do
  LAUD_SO_VARIANT=$V $B > gpurun_out/ably_old_$i.log 2>&1
  $B > gpurun_out/ably_new_$i.log 2>&1
done
LAUD_PDL=0 timeout 300 python tools/graph_kernels.py resnet101 layer 256 > gpurun_out/ably_graph.txt 2>&1
