mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_rg.csv python tools/profile_step.py regnety-1.6gf spatial 1024 > /dev/null 2>&1
