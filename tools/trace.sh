mkdir -p gpurun_out
S=/usr/local/cuda/bin/compute-sanitizer
timeout 900 $S --tool memcheck --print-limit 20 python tools/sanitize_block.py > gpurun_out/san_memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/san_memcheck.log
timeout 1200 $S --tool racecheck --print-limit 20 python tools/sanitize_block.py > gpurun_out/san_racecheck.log 2>&1; echo "rc=$?" >> gpurun_out/san_racecheck.log
timeout 900 $S --tool synccheck --print-limit 20 python tools/sanitize_block.py > gpurun_out/san_synccheck.log 2>&1; echo "rc=$?" >> gpurun_out/san_synccheck.log
