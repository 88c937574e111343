#!/bin/bash
mkdir -p gpurun_out
export SIGB_JIT_CACHE=/tmp/sigjit_cache
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k "generated or auto" > gpurun_out/pytest_jit.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_jit.txt
timeout 1500 python tools/jit_sweep.py 4096 "" "BCAP=48" "BCAP=96" "BCAP=128,BMINB=1" "BWARPS=8,BMINB=1" "BCH=4,BMINB=3" \
  "FCH=16,FMINB=3" "FWARPS=8,FMINB=2" "FCAP=64" "FCAP=160,FMINB=2" > gpurun_out/sweep15.txt 2>&1
echo done
