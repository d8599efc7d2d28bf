#!/bin/bash
# GPU box: launch list of the default bench command + one `ncu --set full` capture of the
# fast kernel per workload.  Usage: tools/prof.sh <tag> [workloads...]
tag=$1; shift
ws=${@:-c4}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/${tag}_launches.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/${tag}_launches_bench.log 2>&1
for w in $ws; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fast_kernel|win_kernel" -s 2 -c 1 \
    -o gpurun_out/${tag}_${w} -f python bench.py --workload $w --records 200000000 --steps 1 --warmup 3 --no-e2e --no-cpu \
    > gpurun_out/${tag}_${w}_ncu.log 2>&1
done
