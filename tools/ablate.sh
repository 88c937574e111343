#!/bin/bash
# Build ablation variants of the truncated kernels (-DSIGB_ABLATE=k) as separate libraries
# under build/abl/ (developer tool; tools/time_bwd.py loads one via SIGB_LIB_PATH).
set -e
cd "$(dirname "$0")/../paper_2602_24066_b200/csrc"
mkdir -p ../../build/abl
objs=$(ls build/*.o | grep -v sigb_trunc.o)
for k in "$@"; do
  ( nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -DSIGB_ABLATE=$k \
      -c sigb_trunc.cu -o ../../build/abl/trunc_$k.o && \
    nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -lnvrtc -Xlinker -rpath,/usr/local/cuda/lib64 \
      -o ../../build/abl/lib_$k.so $objs ../../build/abl/trunc_$k.o ) &
done
wait
ls -la ../../build/abl/
