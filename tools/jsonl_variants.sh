# GPU box: device JSONL loader time, main library vs _variants/<name> (alternating).
# Usage: bash tools/jsonl_variants.sh <variant> [jsonl_rate args...]
P=paper_2110_10401_b200
v1=$1; shift
cp $P/libcommtrace_b200.so /tmp/lib_main.so
for v in main $v1 main $v1; do
  if [ $v = main ]; then cp /tmp/lib_main.so $P/libcommtrace_b200.so; else cp _variants/$v/libcommtrace_b200.so $P/libcommtrace_b200.so; fi
  echo "== $v $@"; timeout 200 python tools/jsonl_rate.py "$@" | grep device
done
cp /tmp/lib_main.so $P/libcommtrace_b200.so
