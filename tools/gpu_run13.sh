#!/bin/bash
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.txt
timeout 1800 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
for c in c3 c4 c2; do
  timeout 600 python bench.py --config $c --no-e2e > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
echo done
