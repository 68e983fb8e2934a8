mkdir -p gpurun_out
LAUD_CONV1_DENSE_ALL=0 timeout 600 python bench.py --steps 20 --warmup 5 --no-baselines > gpurun_out/bench_d0.log 2>&1
LAUD_CONV1_DENSE_ALL=1 timeout 600 python bench.py --steps 20 --warmup 5 --no-baselines > gpurun_out/bench_d1.log 2>&1
LAUD_CONV1_DENSE_ALL=1 timeout 600 python bench.py --steps 20 --warmup 5 --no-baselines --arch resnet50 --plan 4-4-2-1 --batch 128 > gpurun_out/bench_r50_d1.log 2>&1
LAUD_CONV1_DENSE_ALL=0 timeout 600 python bench.py --steps 20 --warmup 5 --no-baselines --arch resnet50 --plan 4-4-2-1 --batch 128 > gpurun_out/bench_r50_d0.log 2>&1
timeout 900 python -m pytest tests/test_gpu_network.py -x -q > gpurun_out/pytest_gpu.log 2>&1
