#!/bin/bash
# Same-box A/B of a _laud_<variant>.so (LAUD_SO_VARIANT) on the channel paradigm + its GPU tests.
V=${1:-oldcm}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "channel or network or masker" > gpurun_out/abch_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/abch_pytest.log
B="timeout 600 python bench.py --steps 10 --warmup 3 --no-traffic --no-baselines --paradigm channel"
for i in 1 2; do
  LAUD_SO_VARIANT=$V $B > gpurun_out/abch_old_$i.log 2>&1
  $B > gpurun_out/abch_new_$i.log 2>&1
done
LAUD_PDL=0 timeout 300 python tools/graph_kernels.py resnet101 channel 256 > gpurun_out/abch_graph.txt 2>&1
