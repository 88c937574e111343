#!/bin/bash
O=gpurun_out/r2d; mkdir -p $O
timeout 900 python -m pytest tests/test_full_shape.py tests/test_gpu_parity.py -q -x -k "checkpoint or stride" > $O/pytest_ckpt.txt 2>&1; echo "rc=$?" >> $O/pytest_ckpt.txt
for st in 0 5; do timeout 300 python tools/time_bwd.py 8192 c5 $st f64 >> $O/time.txt 2>&1; done
for st in 0 5; do timeout 300 python tools/time_bwd.py 8192 c5 $st f32 >> $O/time.txt 2>&1; done
run() { n=$1; shift; timeout 900 python bench.py "$@" > $O/$n.json 2> $O/$n.err; echo "$n rc=$?" >> $O/rc.txt; }
run c1 --config c1 --steps 6000 --warmup 5
run p1 --config p1 --steps 2000 --warmup 5
run p2 --config p2 --steps 3000 --warmup 5
run c3 --config c3 --steps 300 --warmup 5
