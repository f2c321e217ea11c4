#!/bin/bash
# Builds tools/micro/libfwa_tconly.so: libfwa with -DFWA_TRACE -DFWA_TC_ONLY (clock64 phase stamps of CTA 0
# in the flat kernels; read with tools/micro/flat_trace.py).
set -e
cd "$(dirname "$0")/../../paper_2501_06480_b200/csrc"
OUT=../../tools/micro/tconly_obj
mkdir -p $OUT
for f in *.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
       --expt-relaxed-constexpr -DFWA_TRACE -DFWA_TC_ONLY -c $f -o $OUT/${f%.cu}.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o ../../tools/micro/libfwa_tconly.so $OUT/*.o -lrt -ldl -lpthread
