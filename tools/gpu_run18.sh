#!/bin/bash
mkdir -p gpurun_out
export SIGB_JIT_CACHE=/tmp/sigjit_cache
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k "generated or auto" > gpurun_out/pytest_jit.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_jit.txt
timeout 1800 python tools/jit_sweep.py 4096 "" "BWARPS=4,BPB=2,BMINB=1" "BWARPS=2,BPB=3,BMINB=1" "BWARPS=2,BPB=4,BMINB=1,BCH=4" "BWARPS=2" \
  "BWARPS=4,BCH=16,BMINB=1" "BWARPS=4,BPB=2,BMINB=1,BCH=4" "BWARPS=8,BMINB=1,BCH=4" "BWARPS=2,BPB=2,BMINB=1,BCH=8,BCAP=96" \
  "FCH=16,FMINB=3" "FPB=2,FMINB=2" "FWARPS=2,FPB=2,FMINB=4" "FCH=16,FPB=2,FMINB=1" > gpurun_out/sweep18.txt 2>&1
echo done
