#!/bin/bash
O=gpurun_out/r2i; mkdir -p $O
timeout 900 python -m pytest tests/test_trunc_tc.py tests/test_full_shape.py -q -x > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
for m in 2 0; do SIGB_TRUNC_TC_BWD=$m timeout 300 python tools/time_bwd.py 1024 c2 >> $O/time.txt 2>&1; done
timeout 300 python tools/time_bwd.py 8192 c5 >> $O/time.txt 2>&1
