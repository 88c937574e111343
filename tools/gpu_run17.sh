#!/bin/bash
mkdir -p gpurun_out
export SIGB_JIT_CACHE=/tmp/sigjit_cache
timeout 1200 python tools/jit_sweep.py 4096 "" "BMINB=1" "BCAP=32" "BCAP=32,BMINB=1" "BWARPS=2" "BWARPS=2,BMINB=1" "BCH=16,BMINB=1" > gpurun_out/sweep17.txt 2>&1
for s in "" "BMINB=1" "BCAP=32" "BWARPS=2"; do
  tag=$(echo "x$s" | tr ',=' '__')
  timeout 600 ncu --section WarpStateStats --section SchedulerStats --section Occupancy --clock-control none -k regex:sigjit_bwd -c 1 --csv --page raw \
    python tools/jit_sweep.py 2048 "$s" > gpurun_out/ncu17_$tag.csv 2> gpurun_out/ncu17_$tag.err
done
echo done
