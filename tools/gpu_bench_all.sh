#!/bin/bash
# one clocked bench line per config (steps sized for >= 10 nvidia-smi samples), the pathsig rows,
# and c5 in float64 (the reference's backward contract)
O=gpurun_out/bench_all; mkdir -p $O
run() { n=$1; shift; timeout 900 python bench.py "$@" > $O/$n.json 2> $O/$n.err; tail -1 $O/$n.json | cut -c1-200; }
run c1 --config c1 --steps 6000 --warmup 5
run c2 --config c2 --steps 140 --warmup 3
run c3 --config c3 --steps 300 --warmup 5
run c4 --config c4 --steps 12 --warmup 3
run p1 --config p1 --steps 2000 --warmup 5
run p2 --config p2 --steps 3000 --warmup 5
run c5 --config c5 --steps 5 --warmup 3
run c5_fp64 --config c5 --precision fp64 --steps 3 --warmup 3 --no-cpu-baseline
