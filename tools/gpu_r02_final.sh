#!/bin/bash
# Round-2 final measurement pass (one gpurun call): smoke, GPU suite, headline
# bench (R101 spatial b256 with baselines), reference arm, channel / layer /
# R50 / RegNet lines, 2-rank smoke, ncu launch list + --set full of the top
# kernels, in-graph kernel table.
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
B="timeout 600 python bench.py --steps 10 --warmup 3 --no-traffic"
$B --paradigm channel --no-baselines > gpurun_out/bench_channel.log 2>&1
$B --paradigm layer --no-baselines > gpurun_out/bench_layer.log 2>&1
$B --arch resnet50 --plan 4-4-2-1 --batch 128 --no-baselines > gpurun_out/bench_r50.log 2>&1
$B --arch regnety-1.6gf --plan 4-4-2-1 --global-batch 1024 --cpu-images 1 > gpurun_out/bench_regnet.log 2>&1
LAUD_BENCH_SHARE_GPU=1 timeout 600 python bench.py --gpus 2 --global-batch 256 --steps 5 --warmup 3 --no-traffic --no-baselines > gpurun_out/bench_2rank.log 2>&1
LAUD_PDL=0 timeout 300 python tools/graph_kernels.py resnet101 spatial 256 > gpurun_out/graph_kernels_r101.txt 2>&1
LAUD_PDL=0 timeout 300 python tools/graph_kernels.py regnety-1.6gf spatial 1024 > gpurun_out/graph_kernels_regnet.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-baselines --no-traffic > gpurun_out/launches_bench.log 2>&1
bash tools/ncu_r02_convs.sh
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:patch_conv_kernel<\(int\)2' -s 10 -c 1 \
  -o gpurun_out/pconv python tools/profile_step.py resnet101 spatial 256 > gpurun_out/pconv.log 2>&1
ls -la gpurun_out
