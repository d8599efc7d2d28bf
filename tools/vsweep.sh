#!/bin/bash
# GPU box: throughput of the main library and each _variants/* build on C4/C2/C3/C5 (200M records).
# Usage: tools/vsweep.sh [variant names...]
P=paper_2110_10401_b200
cp $P/libcommtrace_b200.so /tmp/lib_main.so
for v in main ${@}; do
  if [ "$v" = main ]; then cp /tmp/lib_main.so $P/libcommtrace_b200.so; else cp _variants/$v/libcommtrace_b200.so $P/libcommtrace_b200.so; fi
  for w in c4 c2 c3 c5; do
    timeout 120 python bench.py --workload $w --records 200000000 --steps 5 --warmup 3 --no-e2e --no-cpu 2>&1 | python tools/bsum.py $v
  done
done
cp /tmp/lib_main.so $P/libcommtrace_b200.so
