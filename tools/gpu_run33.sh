#!/bin/bash
mkdir -p gpurun_out
export SIGB_JIT_CACHE=/tmp/sigjit_cache
timeout 2700 python tools/jit_sweep.py 4096 "" "NVRTC_OPTS=-Xptxas+-O2" "NVRTC_OPTS=-Xptxas+-O1" "NVRTC_OPTS=--maxrregcount=168" "NVRTC_OPTS=-Xptxas+--allow-expensive-optimizations=false" > gpurun_out/sweep33.txt 2>&1
echo done
