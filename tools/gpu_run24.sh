#!/bin/bash
mkdir -p gpurun_out
export SIGB_JIT_CACHE=/tmp/sigjit_cache
timeout 2700 python tools/jit_sweep.py 4096 "BCAP=96" "BCAP=80" "BCAP=64" "BCAP=48" "BCAP=64,BCH=5" "BCAP=80,BCH=5" "BCAP=64,BINTER=1" "BCAP=48,BINTER=1" "BCAP=64,BCH=3,BPB=3" > gpurun_out/sweep24.txt 2>&1
echo done
