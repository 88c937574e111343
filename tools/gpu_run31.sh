#!/bin/bash
mkdir -p gpurun_out
export SIGB_JIT_CACHE=/tmp/sigjit_cache
timeout 2400 python tools/jit_sweep.py 4096 "" "BCAP=64" "BCAP=80" "BCAP=112" "BCAP=64,BCH=6" "BWARPS=8,BPB=1,BCAP=48,BCH=8" > gpurun_out/sweep31.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sigjit_bwd -c 1 \
  -o gpurun_out/prof_c3_jbwd6 python tools/jit_sweep.py 4096 "" > gpurun_out/ncu31b.log 2>&1
echo done
