#!/bin/bash
O=gpurun_out/r2c; mkdir -p $O
timeout 600 python -m pytest tests/test_trunc_tc.py -q -x > $O/pytest_tc.txt 2>&1; echo "rc=$?" >> $O/pytest_tc.txt
for m in 2 1 0; do SIGB_TRUNC_TC_BWD=$m timeout 120 python tools/time_bwd.py 8192 >> $O/time.txt 2>&1; done
timeout 900 python -m pytest tests/test_full_shape.py -q -x -s -k "c5" > $O/pytest_full.txt 2>&1; echo "rc=$?" >> $O/pytest_full.txt
echo done
