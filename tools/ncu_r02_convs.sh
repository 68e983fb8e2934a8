ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:\(int\)0, \(int\)6>' -s 20 -c 1 -o gpurun_out/conv3 python tools/profile_step.py resnet101 spatial 256 > gpurun_out/conv3.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:\(int\)256.*\(int\)4, \(int\)4>' -s 15 -c 1 -o gpurun_out/conv1m python tools/profile_step.py resnet101 spatial 256 > gpurun_out/conv1m.log 2>&1
tail -n 2 gpurun_out/conv3.log; tail -n 2 gpurun_out/conv1m.log
