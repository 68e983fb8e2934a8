mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
timeout 900 python bench.py --paradigm channel --steps 10 --warmup 3 --cpu-images 1 > gpurun_out/bench_channel.log 2>&1
timeout 600 python bench.py --paradigm layer --steps 10 --warmup 3 --no-baselines > gpurun_out/bench_layer.log 2>&1
