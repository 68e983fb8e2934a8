mkdir -p gpurun_out
python tools/engine_probe.py > gpurun_out/probe_default.log 2>&1
LAUD_A_TMA=0 python tools/engine_probe.py > gpurun_out/probe_cpasync.log 2>&1
LAUD_BN=128 python tools/engine_probe.py > gpurun_out/probe_bn128.log 2>&1
ncu --set full --clock-control none -k regex:conv_gemm -s 3 -c 1 -o gpurun_out/p_gemm python tools/engine_probe.py gemm_s3 > /dev/null 2>&1
ncu --set full --clock-control none -k regex:conv_gemm -s 3 -c 1 -o gpurun_out/p_conv2s1 python tools/engine_probe.py conv2_s1 > /dev/null 2>&1
ncu --set full --clock-control none -k regex:conv_gemm -s 3 -c 1 -o gpurun_out/p_conv3s3 python tools/engine_probe.py conv3_s3 > /dev/null 2>&1
