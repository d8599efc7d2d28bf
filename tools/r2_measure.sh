#!/bin/bash
# GPU box: round-2 measurement set -> gpurun_out/<tag>_*  (tools/r2_measure.sh [tag])
t=${1:-r2}
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/${t}_bench_full.json 2> gpurun_out/${t}_bench_full.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/${t}_launches_bench_default.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu --no-parity --no-loader --no-object-api --no-e2e > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/${t}_launches_c4i.csv \
  python bench.py --workload c4i --records 200000000 --steps 2 --warmup 1 --no-cpu --no-parity --no-loader --no-object-api --no-e2e > /dev/null 2>&1
bash tools/prof1.sh ${t} c4 c3
for w in c2 c3 c5 c4i; do
  timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-e2e --no-cpu --no-loader --no-object-api > gpurun_out/${t}_bench_$w.json 2>&1
done
