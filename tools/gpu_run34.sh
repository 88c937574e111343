#!/bin/bash
mkdir -p gpurun_out
export SIGB_JIT_CACHE=/tmp/sigjit_cache
timeout 2700 python tools/jit_sweep.py 4096 "NVRTC_OPTS=--maxrregcount=168" "NVRTC_OPTS=--maxrregcount=144" "NVRTC_OPTS=--maxrregcount=128" "NVRTC_OPTS=--maxrregcount=184" "" > gpurun_out/sweep34.txt 2>&1
echo done
