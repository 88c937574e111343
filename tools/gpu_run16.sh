#!/bin/bash
mkdir -p gpurun_out
export SIGB_JIT_CACHE=/tmp/sigjit_cache
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sigjit_bwd -c 1 \
  -o gpurun_out/prof_c3_jbwd3 python tools/jit_sweep.py 4096 "" > gpurun_out/ncu16b.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sigjit_fwd -c 1 \
  -o gpurun_out/prof_c3_jfwd3 python tools/jit_sweep.py 4096 "FCH=16,FMINB=3" > gpurun_out/ncu16f.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches16.csv \
  python tools/jit_sweep.py 4096 "" > gpurun_out/ncu16l.log 2>&1
echo done
