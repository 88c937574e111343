#!/bin/bash
O=gpurun_out/r2g; mkdir -p $O
timeout 300 python -m pytest tests/test_trunc_tc.py tests/test_full_shape.py -q -x -k "tc_forward or c5 or include" > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
timeout 300 python tools/time_bwd.py 8192 c5 >> $O/time.txt 2>&1
SIGB_TRUNC_TC=0 timeout 300 python tools/time_bwd.py 8192 c5 >> $O/time.txt 2>&1
