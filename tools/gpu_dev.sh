#!/bin/bash
# Inner-loop check after a kernel change: tensor-core and full-shape parity, then c5 / c2 timings.
O=gpurun_out/dev; mkdir -p $O
timeout 600 python -m pytest tests/test_trunc_tc.py tests/test_full_shape.py -q -x > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
timeout 300 python tools/time_bwd.py 8192 c5 > $O/time.txt 2>&1
timeout 300 python tools/time_bwd.py 1024 c2 >> $O/time.txt 2>&1
