#!/bin/bash
# Same-box A/B of _laud_prek.so (an older BN=256 engine build) on the R101 headline, GPU suite, batch-1 check.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pk_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/pk_pytest.log
B="timeout 600 python bench.py --steps 10 --warmup 3 --no-traffic --no-baselines"
for i in 1 2 3; do LAUD_SO_VARIANT=prek $B > gpurun_out/pk_old_$i.log 2>&1; $B > gpurun_out/pk_new_$i.log 2>&1; done
for rep in 1 2; do echo "$(timeout 300 python tools/b1_latency.py resnet101 2>&1 | tail -1)"; done > gpurun_out/pk_b1.log 2>&1
