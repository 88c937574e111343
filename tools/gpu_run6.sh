#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 600 python bench.py --config c2 --no-e2e --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 600 python bench.py --config c1 --no-e2e --no-cpu-baseline --steps 20 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:trunc_backward_kernel -c 1 \
  -o gpurun_out/prof_c5_bwd python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --batch 1024 > gpurun_out/ncu_bwd.log 2>&1
echo done
