#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_block.py
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool python tools/sanitize_block.py > gpurun_out/sanitizer_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitizer_$tool.log
done
