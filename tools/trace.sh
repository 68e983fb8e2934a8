mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_gpu.log 2>&1
LAUD_PAIR=1 python tools/engine_probe.py conv3_s3 conv3_s1 gemm_k256_n1024 > gpurun_out/probe_bn.log 2>&1
LAUD_PAIR=3 python tools/engine_probe.py conv3_s3 conv3_s1 gemm_k256_n1024 >> gpurun_out/probe_bn.log 2>&1
LAUD_PAIR=3 timeout 600 python bench.py --steps 20 --warmup 5 --no-baselines > gpurun_out/bench_quick.log 2>&1
