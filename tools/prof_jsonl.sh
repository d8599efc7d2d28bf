#!/bin/bash
# GPU box: loader rate + launch list + one `ncu --set full` capture of k_parse.  tools/prof_jsonl.sh <tag>
tag=${1:-jl}
mkdir -p gpurun_out
python tools/jsonl_rate.py 20000 200 > gpurun_out/${tag}_rate.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv \
  python tools/jsonl_rate.py 20000 200 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_parse|k_fused" -s 1 -c 1 \
  -o gpurun_out/${tag}_parse -f python tools/jsonl_rate.py 20000 200 > gpurun_out/${tag}_ncu.log 2>&1
