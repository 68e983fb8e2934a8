mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_engine.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_pair.log 2>&1
python tools/engine_probe.py conv2_s3 conv2_s2 conv2_s1 conv1_s1 > gpurun_out/probe_pair.log 2>&1
python tools/engine_probe.py >> gpurun_out/probe_pair.log 2>&1
