#!/bin/bash
# GPU box: device JSONL loader time for the main library and each _variants/<name>.
# Usage: bash tools/jsonl_ab.sh "<variants>" [jsonl_rate args...]
P=paper_2110_10401_b200
vs=$1; shift
cp $P/libcommtrace_b200.so /tmp/lib_main.so
for v in main $vs main $vs; do
  if [ $v = main ]; then cp /tmp/lib_main.so $P/libcommtrace_b200.so; else cp _variants/$v/libcommtrace_b200.so $P/libcommtrace_b200.so; fi
  echo "== $v $(timeout 200 python tools/jsonl_rate.py "$@" | grep 'device parse')"
done
cp /tmp/lib_main.so $P/libcommtrace_b200.so
