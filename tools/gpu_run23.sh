#!/bin/bash
mkdir -p gpurun_out
export SIGB_JIT_CACHE=/tmp/sigjit_cache
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sigjit_bwd -c 1 \
  -o gpurun_out/prof_c3_jbwd5 python tools/jit_sweep.py 4096 "" > gpurun_out/ncu23b.log 2>&1
echo done
