#!/bin/bash
O=gpurun_out/e2e; mkdir -p $O
for c in c1 c2 c3 p1 p2; do timeout 600 python bench.py --config $c --steps 200 --warmup 5 --no-cpu-baseline > $O/$c.json 2>&1; done
