#!/bin/bash
# GPU box: one `ncu --set full` capture of the fast kernel per workload (200M records).
# Usage: tools/prof1.sh <tag> [workloads...]
tag=$1; shift
mkdir -p gpurun_out
for w in ${@:-c4}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fast_kernel|win_kernel" -s 2 -c 1 \
    -o gpurun_out/${tag}_${w} -f python bench.py --workload $w --records 200000000 --steps 1 --warmup 3 --no-e2e --no-cpu \
    > gpurun_out/${tag}_${w}_ncu.log 2>&1
done
