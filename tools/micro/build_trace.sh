#!/bin/bash
# Builds tools/micro/libfwa_trace.so: libfwa with -DFWA_TRACE (clock64 phase stamps of CTA 0
# in the flat kernels; read with tools/micro/flat_trace.py).
set -e
cd "$(dirname "$0")/../../paper_2501_06480_b200/csrc"
OUT=../../tools/micro/trace_obj
mkdir -p $OUT
for f in *.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
       --expt-relaxed-constexpr -DFWA_TRACE -c $f -o $OUT/${f%.cu}.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o ../../tools/micro/libfwa_trace.so $OUT/*.o -lrt -ldl -lpthread
