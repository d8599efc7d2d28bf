#!/bin/bash
# GPU box: fast-kernel workloads for the main library and each _variants/<name> (alternating).
# Usage: bash tools/fast_ab.sh "<variants>" "<workloads>"
P=paper_2110_10401_b200
vs=$1; ws=${2:-c4}
cp $P/libcommtrace_b200.so /tmp/lib_main.so
for v in main $vs main $vs; do
  if [ $v = main ]; then cp /tmp/lib_main.so $P/libcommtrace_b200.so; else cp _variants/$v/libcommtrace_b200.so $P/libcommtrace_b200.so; fi
  bash tools/ab.sh "$ws" | sed "s/^/$v /"
done
cp /tmp/lib_main.so $P/libcommtrace_b200.so
