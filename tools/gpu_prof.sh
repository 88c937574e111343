#!/bin/bash
# ncu --set full of one kernel of a bench config: tools/gpu_prof.sh NAME CONFIG PATHS KERNEL_REGEX [extra env]
# writes gpurun_out/prof/NAME.ncu-rep and its raw csv
NAME=$1; CFG=$2; P=$3; K=$4; shift 4
O=gpurun_out/prof; mkdir -p $O
env "$@" timeout 900 ncu --set full --metrics $(python tools/ncu_summary.py --tensor-metrics) --import-source on \
  --clock-control none -k "regex:$K" -c 1 -f -o $O/$NAME \
  python bench.py --config $CFG --batch $P --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $O/$NAME.log 2>&1
ncu -i $O/$NAME.ncu-rep --page raw --csv > $O/$NAME.raw.csv 2>/dev/null
ncu -i $O/$NAME.ncu-rep --page source --csv > $O/$NAME.source.csv 2>/dev/null
ls -la $O
