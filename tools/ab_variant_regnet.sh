mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k "se or regnet" > gpurun_out/sefc_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/sefc_pytest.log
B="timeout 600 python bench.py --steps 10 --warmup 3 --no-traffic --no-baselines --arch regnety-1.6gf --plan 4-4-2-1 --global-batch 1024"
for i in 1 2; do
  LAUD_SO_VARIANT=oldfc $B > gpurun_out/sefc_old_$i.log 2>&1
  $B > gpurun_out/sefc_new_$i.log 2>&1
done
LAUD_PDL=0 timeout 300 python tools/graph_kernels.py regnety-1.6gf spatial 1024 > gpurun_out/sefc_graph.txt 2>&1
