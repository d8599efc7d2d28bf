#!/bin/bash
# A/B a library variant: tools/variant_bench.sh <variant dir> <mode> <workload>
set -e
cp paper_2110_10401_b200/libcommtrace_b200.so /tmp/lib_main.so
cp $1/libcommtrace_b200.so paper_2110_10401_b200/libcommtrace_b200.so
CT_DEBUG_MODE=$2 timeout 120 python bench.py --workload $3 --records 200000000 --steps 5 --warmup 2 --no-cpu --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 mode $2', d['config']['workload'][:3], round(d['value']/1e9,2), 'Grec/s', round(d['roofline']['frac'],3))"
cp /tmp/lib_main.so paper_2110_10401_b200/libcommtrace_b200.so
