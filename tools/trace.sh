mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
LAUD_A_BOX=3 timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_box3.log 2>&1
for b in 0 1 3; do LAUD_A_BOX=$b timeout 600 python bench.py --steps 20 --warmup 5 --no-baselines > gpurun_out/bench_box$b.log 2>&1; done
LAUD_A_BOX=0 python tools/profile_step.py resnet101 spatial 256 > gpurun_out/prof_box0.log 2>&1
LAUD_A_BOX=3 python tools/profile_step.py resnet101 spatial 256 > gpurun_out/prof_box3.log 2>&1
