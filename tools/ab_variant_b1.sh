#!/bin/bash
# Same-box A/B of _laud_<variant>.so on the batch-1 latency (R101, R50) + the GPU suite.
V=${1:-oldcapi}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/b1ab_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/b1ab_pytest.log
for rep in 1 2; do
  echo "old $(LAUD_SO_VARIANT=$V timeout 300 python tools/b1_latency.py resnet101 2>&1 | tail -1)"
  echo "new $(timeout 300 python tools/b1_latency.py resnet101 2>&1 | tail -1)"
  echo "old $(LAUD_SO_VARIANT=$V timeout 300 python tools/b1_latency.py resnet50 spatial 4-4-2-1 2>&1 | tail -1)"
  echo "new $(timeout 300 python tools/b1_latency.py resnet50 spatial 4-4-2-1 2>&1 | tail -1)"
done > gpurun_out/b1ab.log 2>&1
