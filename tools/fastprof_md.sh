#!/bin/bash
# Markdown summary of fast-kernel ncu captures: metrics, stalls, top lines, and warp
# instructions per 32-record window by the ``// REGION`` markers of ct_fast.cu.
# Usage: tools/fastprof_md.sh <records> rep1 [rep2 ...]
recs=$1; shift
src=paper_2110_10401_b200/csrc/ct_fast.cu
ranges=$(awk '/\/\/ REGION/{print NR, $NF}' $src | awk 'NR>1{print lo"-"$1-1":"name} {lo=$1; name=$2} END{print lo"-99999:"name}')
for rep in "$@"; do
  echo "## $(basename $rep .ncu-rep)"
  echo '```'
  bash tools/ncusum.sh $rep 12
  python tools/srcrange.py /tmp/_src.csv $recs $ranges
  echo '```'
  echo
done
