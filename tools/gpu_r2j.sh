#!/bin/bash
O=gpurun_out/r2j; mkdir -p $O
timeout 900 python -m pytest tests/test_trunc_tc.py tests/test_full_shape.py -q -x > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
timeout 300 python tools/time_bwd.py 1024 c2 >> $O/time.txt 2>&1
SIGB_TRUNC_TC=0 timeout 300 python tools/time_bwd.py 1024 c2 >> $O/time.txt 2>&1
timeout 300 python tools/time_bwd.py 8192 c5 >> $O/time.txt 2>&1
timeout 600 python bench.py --config c2 --steps 60 --warmup 3 > $O/c2.json 2> $O/c2.err
