#!/bin/bash
# current (persistent) generated kernels on c3: full ncu capture of fwd and bwd at the bench batch
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sigjit_bwd -c 1 \
  -o gpurun_out/prof_c3_jbwd2 python bench.py --config c3 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_c3b.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sigjit_fwd -c 1 \
  -o gpurun_out/prof_c3_jfwd2 python bench.py --config c3 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_c3f.log 2>&1
echo done
