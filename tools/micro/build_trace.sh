#!/bin/bash
# Builds tools/micro/libfwa_trace.so: libfwa with -DFWA_TRACE (clock64 phase stamps of CTA 0
# in the flat kernels; read with tools/micro/flat_trace.py / bflat_trace.py).
# EXTRA="-DFWA_TC_ONLY" NAME=tconly builds the MMA-pipeline-only timing variant.
set -e
NAME=${NAME:-trace}
cd "$(dirname "$0")/../../paper_2501_06480_b200/csrc"
OUT=../../tools/micro/${NAME}_obj
mkdir -p $OUT
ls *.cu | xargs -P 6 -I{} sh -c 'nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -DFWA_TRACE '"$EXTRA"' -c {} -o '"$OUT"'/$(basename {} .cu).o 2>/dev/null || { echo "FAILED {}"; exit 255; }'
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o ../../tools/micro/libfwa_${NAME}.so $OUT/*.o -lrt -ldl -lpthread
