#!/bin/bash
mkdir -p gpurun_out
export SIGB_JIT_CACHE=/tmp/sigjit_cache
P="BWARPS=4,BPB=2,BMINB=1"
timeout 2400 python tools/jit_sweep.py 4096 "$P,BCAP=96" "$P,BCAP=128" "$P,BCAP=96,BCH=4" "$P,BCAP=96,BCH=12" "BWARPS=4,BPB=3,BMINB=1,BCH=4,BCAP=64" \
  "BWARPS=4,BPB=3,BMINB=1,BCH=4,BCAP=80" "BWARPS=2,BPB=4,BMINB=1,BCAP=96" \
  "FCH=16,FPB=3,FMINB=1,$P,BCAP=96" "FCH=8,FPB=4,FMINB=1,$P,BCAP=96" "FCH=12,FPB=3,FMINB=1,FCAP=128,$P,BCAP=96" "FCH=16,FMINB=3,FCAP=128,$P,BCAP=96" > gpurun_out/sweep20.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches20.csv \
  python tools/jit_sweep.py 4096 "$P,BCAP=96" > gpurun_out/ncu20l.log 2>&1
echo done
