#!/bin/bash
# ncu --set full of one kernel launch: tools/ncu_one.sh <name> <kernel-regex> <skip> <command...>
name=$1; kre=$2; skip=$3; shift 3
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:$kre -s $skip -c 1 -o gpurun_out/$name "$@" > gpurun_out/$name.log 2>&1
tail -2 gpurun_out/$name.log
