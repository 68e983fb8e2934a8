mkdir -p gpurun_out
python tools/engine_probe.py tiny one_wave_k256 two_wave_k256 four_wave_k256 > gpurun_out/probe_waves.log 2>&1
LAUD_DBG=59 python tools/engine_probe.py tiny one_wave_k256 two_wave_k256 four_wave_k256 >> gpurun_out/probe_waves.log 2>&1
