#!/bin/bash
# GPU box: ncu --set full of the fast kernel for a _variants/<name> build on one workload.
# Usage: tools/prof_variant.sh <variant> <workload> <tag>
P=paper_2110_10401_b200
cp $P/libcommtrace_b200.so /tmp/lib_main.so
cp _variants/$1/libcommtrace_b200.so $P/libcommtrace_b200.so
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fast_kernel -s 2 -c 1 \
  -o gpurun_out/$3 -f python bench.py --workload $2 --records 200000000 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/$3.log 2>&1
cp /tmp/lib_main.so $P/libcommtrace_b200.so
