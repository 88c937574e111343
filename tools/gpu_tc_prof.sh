#!/bin/bash
O=gpurun_out/tcp; mkdir -p $O
SIGB_TRUNC_TC=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:trunc_tc_forward -c 1 \
  -o $O/prof_c5_tcfwd python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --batch 2048 > $O/ncu.log 2>&1
ncu -i $O/prof_c5_tcfwd.ncu-rep --page raw --csv > $O/prof_c5_tcfwd.csv 2>/dev/null
ncu -i $O/prof_c5_tcfwd.ncu-rep --page source --csv --print-source sass > $O/prof_c5_tcfwd_sass.csv 2>/dev/null
gzip -f $O/prof_c5_tcfwd_sass.csv; rm -f $O/prof_c5_tcfwd.ncu-rep
echo done
