#!/bin/bash
O=gpurun_out/r2e; mkdir -p $O
timeout 900 python -m pytest tests/test_full_shape.py tests/test_gpu_parity.py tests/test_trunc_tc.py -q -x -k "checkpoint or stride or tc_backward" > $O/pytest_ckpt.txt 2>&1; echo "rc=$?" >> $O/pytest_ckpt.txt
for st in 0 5; do timeout 300 python tools/time_bwd.py 8192 c5 $st f64 >> $O/time.txt 2>&1; done
for st in 5; do timeout 300 python tools/time_bwd.py 8192 c5 $st f32 >> $O/time.txt 2>&1; done
SIGB_TRUNC_TC_BWD=0 timeout 300 python tools/time_bwd.py 8192 c5 0 f32 >> $O/time.txt 2>&1
