#!/bin/bash
# Tensor-core truncated forward: parity tests, then c5 bench with and without it.
O=gpurun_out/tc; mkdir -p $O
timeout 600 python -m pytest tests/test_trunc_tc.py -q -x > $O/pytest_tc.txt 2>&1; echo "rc=$?" >> $O/pytest_tc.txt
SIGB_TRUNC_TC=1 timeout 600 python bench.py --no-e2e --no-cpu-baseline > $O/bench_c5_tc.json 2> $O/bench_c5_tc.err
echo done
