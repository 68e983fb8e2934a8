mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
timeout 900 python bench.py --arch regnety-1.6gf --plan 4-4-2-1 --batch 1024 --steps 10 --warmup 3 --cpu-images 1 > gpurun_out/bench_regnet.log 2>&1
