mkdir -p gpurun_out
for cfg in "LAUD_MASKER_IN_CONV1=0" "LAUD_MASKER_IN_CONV1=0 LAUD_PAIR=0" "LAUD_MASKER_IN_CONV1=1"; do echo "== $cfg"; env $cfg python tools/profile_step.py resnet101 spatial 256 | python -c "
import sys, json
rows=[json.loads(l) for l in sys.stdin if l.startswith('{')]
print('conv1s3', round(sum(r['us'] for r in rows if r['tag']==0 and r['n_out']==256 and r['k']==1024)), 'masker', round(sum(r['us'] for r in rows if r['tag']==1)), 'total', round(sum(r['us'] for r in rows)))
"; done > gpurun_out/iso.log 2>&1
