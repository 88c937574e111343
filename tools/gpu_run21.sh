#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.txt
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --config c3 --no-e2e > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sigjit_bwd -c 1 \
  -o gpurun_out/prof_c3_jbwd4 python bench.py --config c3 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu21b.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sigjit_fwd -c 1 \
  -o gpurun_out/prof_c3_jfwd4 python bench.py --config c3 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu21f.log 2>&1
echo done
