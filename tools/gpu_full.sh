#!/bin/bash
# One gpurun call: smoke, GPU parity suite, bench lines (R101 headline with baselines,
# channel, layer, RegNetY-1.6GF), reference arm, ncu launch list, ncu --set full of the
# conv engine (stage-3 shapes).
set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
timeout 900 python bench.py --paradigm channel --steps 10 --warmup 3 --no-baselines > gpurun_out/bench_channel.log 2>&1
timeout 900 python bench.py --paradigm layer --steps 10 --warmup 3 --no-baselines > gpurun_out/bench_layer.log 2>&1
timeout 900 python bench.py --arch regnety-1.6gf --plan 4-4-2-1 --batch 1024 --steps 10 --warmup 3 --cpu-images 1 > gpurun_out/bench_regnet.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-baselines > gpurun_out/launches_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_gemm -s 60 -c 6 \
  -o gpurun_out/prof python tools/profile_step.py resnet101 spatial 256 > gpurun_out/prof.log 2>&1
ls -la gpurun_out
