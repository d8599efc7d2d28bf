#!/bin/bash
# GPU box: parity tests, then window path vs element path (CT_DEBUG_MODE=8) per workload.
# Usage: tools/fw_ab.sh "<workloads>" [pytest -k expr]
ws=${1:-"c4 c2 c3 c5"}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q ${2:+-k "$2"} 2>&1 | tail -15
for w in $ws; do
  bash tools/ab.sh $w
  CT_DEBUG_MODE=8 bash tools/ab.sh $w | sed 's/^/element-path /'
done
