#!/bin/bash
# clocked bench lines for the named configs: tools/gpu_bench_some.sh c5 c4 ...
O=gpurun_out/bench_all; mkdir -p $O
declare -A ST=([c1]="6000 5" [c2]="140 3" [c3]="300 5" [c4]="12 3" [c5]="5 3" [p1]="2000 5" [p2]="3000 5")
for c in "$@"; do
  set -- ${ST[$c]}
  timeout 900 python bench.py --config $c --steps $1 --warmup $2 > $O/$c.json 2> $O/$c.err
  tail -1 $O/$c.json | cut -c1-160
done
