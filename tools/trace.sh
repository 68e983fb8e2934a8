mkdir -p gpurun_out
python tools/profile_step.py regnety-1.6gf spatial 1024 > gpurun_out/profile_rg.log 2>&1
