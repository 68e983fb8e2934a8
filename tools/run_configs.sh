#!/bin/bash
# BASELINE configs 2, 4, 5 on one B200 (one JSON line each -> gpurun_out/cfg_*.log)
# plus the N>1 bench path smoke (2 ranks sharing the GPU).
mkdir -p gpurun_out
B="timeout 600 python bench.py --steps 10 --warmup 3 --no-traffic"
# config 2: LAUD-R50 S=4-4-2-1 r=0.5 batch 128
$B --arch resnet50 --plan 4-4-2-1 --batch 128 --cpu-images 2 > gpurun_out/cfg2_r50.log 2>&1
# config 4: R101 channel (G=1, G=2) and layer, network ratio sweep
for r in 0.2 0.5 0.8; do
  $B --paradigm layer --ratio $r --no-baselines > gpurun_out/cfg4_layer_$r.log 2>&1
  $B --paradigm channel --plan 1-1-1-1 --ratio $r --no-baselines > gpurun_out/cfg4_ch_g1_$r.log 2>&1
done
$B --paradigm channel --plan 2-2-2-2 --ratio 0.5 --no-baselines > gpurun_out/cfg4_ch_g2_0.5.log 2>&1
$B --paradigm layer --ratio 0.5 --cpu-images 2 > gpurun_out/cfg4_layer_full.log 2>&1
$B --paradigm channel --ratio 0.5 --cpu-images 2 > gpurun_out/cfg4_ch_full.log 2>&1
# config 5: LAUD-RegNetY-1.6GF spatial 4-4-2-1, global batch 1024 and the per-GPU shards of k = 2, 4, 8
for g in 1024 512 256 128; do
  $B --arch regnety-1.6gf --plan 4-4-2-1 --global-batch $g --no-baselines > gpurun_out/cfg5_regnet_$g.log 2>&1
done
$B --arch regnety-1.6gf --plan 4-4-2-1 --global-batch 1024 --cpu-images 1 > gpurun_out/cfg5_regnet_full.log 2>&1
# N>1 path smoke: 2 ranks on the one GPU (gloo checking collectives)
LAUD_BENCH_SHARE_GPU=1 timeout 600 python bench.py --gpus 2 --batch 64 --steps 5 --warmup 3 --no-traffic --no-baselines > gpurun_out/smoke_2rank.log 2>&1
LAUD_BENCH_SHARE_GPU=1 timeout 600 python bench.py --gpus 2 --global-batch 96 --steps 5 --warmup 3 --no-traffic --no-baselines > gpurun_out/smoke_2rank_strong.log 2>&1
ls gpurun_out/cfg* gpurun_out/smoke*
