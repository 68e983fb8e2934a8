mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_network.py -x -q -k "pipelined" > gpurun_out/pytest_gpu.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --no-baselines > gpurun_out/bench_quick.log 2>&1
