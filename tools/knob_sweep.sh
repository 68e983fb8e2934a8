#!/bin/bash
# Re-check the schedule knobs' defaults on the final build (R101 headline step, one run each).
mkdir -p gpurun_out
B="timeout 600 python bench.py --steps 10 --warmup 3 --no-traffic --no-baselines"
for kv in "X=0" "LAUD_TMA_OUT=0" "LAUD_TAIL_SPLIT=0" "LAUD_PAIR=0" "LAUD_PAIR=3" "LAUD_PC_BN=64" "LAUD_MASKER_IN_CONV1=0" "LAUD_SMALL_GRID_BN=0" "X=1"; do
  echo "$kv $(env $kv $B 2>&1 | grep '^{' | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"])')"
done > gpurun_out/knobs.log 2>&1
