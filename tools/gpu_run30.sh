#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:trunc_forward -c 1 \
  -o gpurun_out/prof_c5_fwd2 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --batch 2048 > gpurun_out/ncu30f.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:trunc_backward -c 1 \
  -o gpurun_out/prof_c5_bwd2 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --batch 1024 > gpurun_out/ncu30b.log 2>&1
echo done
