#!/bin/bash
mkdir -p gpurun_out
export SIGB_JIT_CACHE=/tmp/sigjit_cache
timeout 2400 python tools/jit_sweep.py 4096 "" "BLOCK=1" "FLOCK=1" "BLOCK=1,FLOCK=1,FPB=4,FCAP=128" "BLOCK=1,BCAP=128" > gpurun_out/sweep26.txt 2>&1
timeout 600 python tools/jit_sweep.py 4000 "BLOCK=1,FLOCK=1" >> gpurun_out/sweep26.txt 2>&1
SIGB_JIT_BLOCK=1 SIGB_JIT_FLOCK=1 timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k "generated" > gpurun_out/pytest_jit.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_jit.txt
echo done
