#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 900 python bench.py > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
for c in c2 c3 c4; do
  timeout 600 python bench.py --config $c --no-e2e > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
timeout 300 python bench.py --config c1 --no-e2e --steps 20 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
timeout 300 python bench.py --impl reference > gpurun_out/bench_ref_c5.json 2> gpurun_out/bench_ref_c5.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --batch 8192 > gpurun_out/ncu_launch_bench.log 2>&1
echo done
