P=paper_2110_10401_b200
cp $P/libcommtrace_b200.so /tmp/lib_main.so
for v in main ${@:-split} main ${@:-split}; do
  if [ $v = main ]; then cp /tmp/lib_main.so $P/libcommtrace_b200.so; else cp _variants/$v/libcommtrace_b200.so $P/libcommtrace_b200.so; fi
  echo "== $v"; timeout 200 python tools/jsonl_rate.py 20000 200 | grep device
done
cp /tmp/lib_main.so $P/libcommtrace_b200.so
