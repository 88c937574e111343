#!/bin/bash
# full default bench line (c5) + c5 launch list
O=gpurun_out/bench; mkdir -p $O
timeout 900 python bench.py > $O/bench_c5.json 2> $O/bench_c5.err
tail -1 $O/bench_c5.json | cut -c1-400
