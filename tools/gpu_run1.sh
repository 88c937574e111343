#!/bin/bash
# First measurement pass on a B200 (run under gpurun from the repo root).
set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia_smi.txt 2>&1
nproc > gpurun_out/nproc.txt; lscpu > gpurun_out/lscpu.txt 2>&1
timeout 120 ./tools/ubench_fma > gpurun_out/ubench_fma.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 600 python bench.py > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
for c in c2 c3 c4; do
  timeout 600 python bench.py --config $c --no-e2e > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
timeout 300 python bench.py --config c1 --no-e2e --steps 10 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --batch 8192 > gpurun_out/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:trunc_backward_kernel -c 1 \
  -o gpurun_out/prof_c5_bwd python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --batch 1024 > gpurun_out/ncu_bwd.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:trunc_forward_kernel -c 1 \
  -o gpurun_out/prof_c5_fwd python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --batch 2048 > gpurun_out/ncu_fwd.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:backward_kernel -c 1 \
  -o gpurun_out/prof_c4_bwd python bench.py --config c4 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --batch 64 > gpurun_out/ncu_c4.log 2>&1
echo done
