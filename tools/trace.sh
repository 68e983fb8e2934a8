mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
LAUD_STREAMK=0 python tools/engine_probe.py conv2_s3_r05 conv2_s3 gemm_s3_1w > gpurun_out/probe_sk.log 2>&1
python tools/engine_probe.py conv2_s3_r05 conv2_s3 gemm_s3_1w >> gpurun_out/probe_sk.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --no-baselines > gpurun_out/bench_quick.log 2>&1
