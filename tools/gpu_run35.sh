#!/bin/bash
mkdir -p gpurun_out
export SIGB_JIT_CACHE=/tmp/sigjit_cache
timeout 2700 python tools/jit_sweep.py 4096 "" "FMAXREG=128" "FMAXREG=144" "FMAXREG=152" "FMAXREG=160" "BMAXREG=176" "BMAXREG=192" > gpurun_out/sweep35.txt 2>&1
echo done
