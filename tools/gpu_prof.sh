#!/bin/bash
# ncu --set full of one kernel of a bench config: tools/gpu_prof.sh NAME CONFIG PATHS KERNEL_REGEX [extra env]
# writes gpurun_out/prof/NAME.raw.csv.gz and NAME.source.csv.gz (the .ncu-rep stays on the box:
# gpurun copies back at most 64 MiB)
NAME=$1; CFG=$2; P=$3; K=$4; shift 4
O=gpurun_out/prof; mkdir -p $O; R=/tmp/ncu_$NAME
env "$@" timeout 900 ncu --set full --metrics $(python tools/ncu_summary.py --tensor-metrics) --import-source on \
  --clock-control none -k "regex:$K" -c 1 -f -o $R \
  python bench.py --config $CFG --batch $P --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $O/$NAME.log 2>&1
ncu -i $R.ncu-rep --page raw --csv 2>/dev/null | gzip > $O/$NAME.raw.csv.gz
ncu -i $R.ncu-rep --page source --csv 2>/dev/null | gzip > $O/$NAME.source.csv.gz
rm -f $R.ncu-rep
ls -la $O
