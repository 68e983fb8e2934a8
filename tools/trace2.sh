mkdir -p gpurun_out
python tools/engine_probe.py stem gemm_k256_n1024 conv3_s3 conv2_s3 > gpurun_out/probe_stem.log 2>&1
