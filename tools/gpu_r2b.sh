#!/bin/bash
# TC backward: parity, then the c5 bench, then an ncu capture of the new kernel
O=gpurun_out/r2b; mkdir -p $O
timeout 600 python -m pytest tests/test_trunc_tc.py -q -x > $O/pytest_tc.txt 2>&1; echo "rc=$?" >> $O/pytest_tc.txt
timeout 900 python -m pytest tests/test_full_shape.py -q -x -s -k "c5 or c2" > $O/pytest_full.txt 2>&1; echo "rc=$?" >> $O/pytest_full.txt
timeout 900 python bench.py --no-cpu-baseline --no-e2e > $O/bench_c5.json 2> $O/bench_c5.err
echo done
