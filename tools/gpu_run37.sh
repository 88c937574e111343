#!/bin/bash
mkdir -p gpurun_out
export SIGB_JIT_CACHE=/tmp/sigjit_cache
timeout 2700 python tools/jit_sweep.py 4096 "" "FPAIR=1,FCAP=48,BPAIR=1,BCAP=48" "FPAIR=1,FCAP=64,BPAIR=1,BCAP=40" "FPAIR=1,FCAP=40,BPAIR=1,BCAP=56" "FPAIR=1,FCAP=48,FPB=2,BPAIR=1,BCAP=48,BPB=1" > gpurun_out/sweep37.txt 2>&1
timeout 600 python tools/jit_sweep.py 4000 "FPAIR=1,FCAP=48,BPAIR=1,BCAP=48" >> gpurun_out/sweep37.txt 2>&1
echo done
