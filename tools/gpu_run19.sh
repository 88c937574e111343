#!/bin/bash
mkdir -p gpurun_out
export SIGB_JIT_CACHE=/tmp/sigjit_cache
nvidia-smi --query-gpu=clocks.sm,clocks.mem,power.draw,temperature.gpu,clocks_throttle_reasons.active --format=csv -lms 500 > gpurun_out/clk19.csv &
SMI=$!
timeout 1800 python tools/jit_sweep.py 4096 "" "BWARPS=4,BPB=2,BMINB=1" "" "BWARPS=4,BPB=2,BMINB=1" "BWARPS=2" "BWARPS=4,BCH=16,BMINB=1" \
  "BWARPS=4,BPB=2,BMINB=1,BCAP=96" "BWARPS=4,BPB=2,BMINB=1,BCAP=48" "BWARPS=3,BPB=2,BMINB=1" "BWARPS=4,BPB=2,BMINB=1,FCH=16,FMINB=3" > gpurun_out/sweep19.txt 2>&1
kill $SMI
echo done
