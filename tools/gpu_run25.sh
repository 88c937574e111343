#!/bin/bash
mkdir -p gpurun_out
export SIGB_JIT_CACHE=/tmp/sigjit_cache
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "generated" > gpurun_out/pytest_jit.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_jit.txt
timeout 1800 python tools/jit_sweep.py 4096 "" "BCH=6" "FCAP=128,FPB=4" "FCAP=128" > gpurun_out/sweep25.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches25.csv \
  python tools/jit_sweep.py 4096 "" > gpurun_out/ncu25l.log 2>&1
echo done
