#!/bin/bash
mkdir -p gpurun_out
export SIGB_JIT_CACHE=/tmp/sigjit_cache
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_logsig.py tests/test_surfaces.py -x -q -k "generated or auto or logsig or surfaces or lead or signature or tensor or reverse or reference or errors or backward" > gpurun_out/pytest_jit.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_jit.txt
timeout 2400 python tools/jit_sweep.py 4096 "" "BCH=5" "BCAP=64" "BCH=5,BCAP=64" "BCAP=128" "FCH=8,FPB=4" "FCH=12,FPB=4" "FCH=16,FPB=3" "FCH=8,FPB=3" "FCAP=128,FCH=12,FPB=4" > gpurun_out/sweep22.txt 2>&1
echo done
