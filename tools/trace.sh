mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --no-baselines > gpurun_out/bench_quick.log 2>&1
