mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "masker or block_sparse" > gpurun_out/pytest_gpu.log 2>&1
LAUD_MASKER_V2=0 python tools/profile_step.py resnet101 spatial 256 > gpurun_out/profile_v1.log 2>&1
python tools/profile_step.py resnet101 spatial 256 > gpurun_out/profile_v2.log 2>&1
