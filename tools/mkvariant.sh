#!/bin/bash
# Build a library variant with extra nvcc flags into _variants/<name>/ (reuses the main
# build's objects for sources other than ct_fast.cu / ct_api.cu / ct_jsonl.cu).
# Usage: tools/mkvariant.sh <name> "<nvcc flags>"
set -e
name=$1; extra=$2
P=paper_2110_10401_b200
out=_variants/$name; mkdir -p $out/_obj
F="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr -I include -Xcompiler -fopenmp $extra"
for s in ct_fast ct_api ct_jsonl; do /usr/local/cuda/bin/nvcc $F -c $P/csrc/$s.cu -o $out/_obj/$s.o; done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libcommtrace_b200.so \
  $out/_obj/ct_fast.o $out/_obj/ct_api.o $out/_obj/ct_jsonl.o $P/_obj/ct_exact.o $P/_obj/ct_emit.o $P/_obj/ct_gen.o $P/_obj/ct_canon.o -lcudart -lgomp
