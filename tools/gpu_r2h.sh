#!/bin/bash
O=gpurun_out/r2h; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "parallel_in_time" > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
for c in c1 p1; do timeout 600 python bench.py --config $c --steps 2000 --warmup 5 --no-cpu-baseline > $O/$c.json 2> $O/$c.err; done
