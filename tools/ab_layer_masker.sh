#!/bin/bash
# Layer masker kernel A/B (LAUD_CELL_DOT_CONTIG=0: generic cell_dot) on the layer paradigm + tests.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/lm_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/lm_pytest.log
B="timeout 600 python bench.py --steps 10 --warmup 3 --no-traffic --no-baselines --paradigm layer"
for i in 1 2; do LAUD_CELL_DOT_CONTIG=0 $B > gpurun_out/lm_0_$i.log 2>&1; $B > gpurun_out/lm_1_$i.log 2>&1; done
LAUD_PDL=0 timeout 300 python tools/graph_kernels.py resnet101 layer 256 > gpurun_out/lm_gk.txt 2>&1
