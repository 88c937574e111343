#!/bin/bash
# round 2: full-shape parity tests, new bench fields, tensor-pipe metric names
O=gpurun_out/r2a; mkdir -p $O
ncu --query-metrics --chip gb100 2>&1 | grep -i -E "tensor|tmem|utc|tc_" > $O/metrics_tensor.txt
timeout 900 python -m pytest tests/test_full_shape.py tests/test_sharding.py -m gpu -q -s > $O/pytest_full.txt 2>&1; echo "rc=$?" >> $O/pytest_full.txt
timeout 900 python bench.py --no-cpu-baseline > $O/bench_c5.json 2> $O/bench_c5.err
timeout 600 python bench.py --config c3 --no-e2e --no-cpu-baseline --steps 200 > $O/bench_c3.json 2> $O/bench_c3.err
echo done
