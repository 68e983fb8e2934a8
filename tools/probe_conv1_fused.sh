mkdir -p gpurun_out
for st in 1 2 3; do
  echo "== stage $st fused" ; timeout 300 python tools/conv1_fused_probe.py $st 256
  echo "== stage $st unfused" ; LAUD_MASKER_IN_CONV1=0 timeout 300 python tools/conv1_fused_probe.py $st 256
done > gpurun_out/c1p.log 2>&1
