#!/bin/bash
# GPU box: quick headline numbers per workload (1B records, device-timed, no e2e/cpu/parity).
# Usage: tools/ab.sh "c4 c3" [extra bench args]
ws=${1:-c4}; shift
for w in $ws; do
  timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-e2e --no-cpu --no-loader --no-parity --no-object-api "$@" 2>&1 | \
  python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l)
        print('$w', round(d['value'] / 1e9, 2), 'Grec/s frac', round(d['roofline']['frac'], 3), 'kernel_ms',
              round(d['roofline']['kernel_ms'], 3), d['result_check'])
    elif 'Error' in l or 'error' in l:
        print('$w', l.strip()[:300])
"
done
