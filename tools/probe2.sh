mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
python tools/engine_probe.py > gpurun_out/probe_epi.log 2>&1
for s in gemm_k256_n1024 conv3_s3 conv2_s1; do python tools/engine_trace.py $s | grep -v "kb " | head -8; done > gpurun_out/trace.log 2>&1
