#!/bin/bash
# GPU box: parity tests then a short per-workload throughput sweep (200M records).
# Usage: tools/quick.sh [pytest args...]
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q "$@" 2>&1 | tail -15
for w in c4 c2 c3 c5; do
  timeout 120 python bench.py --workload $w --records 200000000 --steps 5 --warmup 3 --no-e2e --no-cpu 2>&1 | python tools/bsum.py sweep
done
