#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_kernels.py -x -q > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
for c in c3 c4; do
  timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:frag_backward_kernel -c 1 \
  -o gpurun_out/prof_c4_fbwd python bench.py --config c4 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --batch 256 > gpurun_out/ncu_c4b.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:frag_forward_kernel -c 1 \
  -o gpurun_out/prof_c3_ffwd python bench.py --config c3 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --batch 2048 > gpurun_out/ncu_c3f.log 2>&1
echo done
