#!/bin/bash
mkdir -p gpurun_out/p32
O=gpurun_out/p32
timeout 900 ncu --set full --clock-control none --import-source on -k regex:trunc_backward -c 1 \
  -o $O/prof_c2_bwd python bench.py --config c2 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --batch 512 > $O/ncu_c2b.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:frag_backward -c 1 \
  -o $O/prof_c4_bwd python bench.py --config c4 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --batch 256 > $O/ncu_c4b.log 2>&1
for r in $O/prof_*.ncu-rep; do
  ncu -i $r --page raw --csv > ${r%.ncu-rep}.csv 2>/dev/null
  ncu -i $r --page source --csv --print-source sass > ${r%.ncu-rep}_sass.csv 2>/dev/null
  gzip -f ${r%.ncu-rep}_sass.csv
  rm -f $r
done
echo done
