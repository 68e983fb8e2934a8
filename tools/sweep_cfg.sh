#!/bin/bash
timeout 300 python tools/profile_step.py 2>&1 | python -c "
import sys, json, collections
rows=[json.loads(l) for l in sys.stdin if l.startswith('{')]
by=collections.Counter()
for r in rows: by[r['tag']]+=r['us']
print('  total_ms %.3f' % (sum(r['us'] for r in rows)/1e3), {k: round(v/1e3,3) for k,v in sorted(by.items())})
for r in rows[:24]: print('   ', r['i'], r['tag'], r['us'], r['rows'], r['n_out'], r['k'], r['tflops'])
"
