mkdir -p gpurun_out
for m in 4096 20000 1000000; do LAUD_MASKER_FUSED_MAX=$m timeout 600 python bench.py --steps 20 --warmup 5 --no-baselines > gpurun_out/bench_m$m.log 2>&1; done
LAUD_MASKER_FUSED_MAX=1000000 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "masker" > gpurun_out/pytest_m.log 2>&1
