#!/bin/bash
# Batch-1 latency vs warps per cell of the one-launch masker (LAUD_MASKER_WPC; 0 = the
# default one-wave rule), its tests, and the headline step (unaffected path check).
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/wpc_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/wpc_pytest.log
for rep in 1 2; do for v in 1 0; do
  echo "wpc=$v $(LAUD_MASKER_WPC=$v timeout 300 python tools/b1_latency.py resnet101 2>&1 | tail -1)"
  echo "wpc=$v $(LAUD_MASKER_WPC=$v timeout 300 python tools/b1_latency.py resnet50 spatial 4-4-2-1 2>&1 | tail -1)"
done; done > gpurun_out/wpc_b1.log 2>&1
