# A/B: bench under env variants (one line each)
mkdir -p gpurun_out
: > gpurun_out/ab.log
for v in "$@"; do
  echo "== $v" >> gpurun_out/ab.log
  env $v timeout 600 python bench.py --steps 20 --warmup 5 --no-baselines 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['config'].get('measured_ratio_mean'))" >> gpurun_out/ab.log 2>&1
done
