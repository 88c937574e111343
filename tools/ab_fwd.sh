#!/bin/bash
# full GPU suite on the in-tree build, then A/B of two builds on c2, c5 (fp32 CUDA-core backward) and p1
O=gpurun_out/ab; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt; tail -2 $O/pytest.txt
for r in 1 2 3; do for L in "$@"; do
  SIGB_LIB_PATH=$L timeout 300 python tools/time_bwd.py 1024 c2
  SIGB_LIB_PATH=$L SIGB_TRUNC_TC=0 SIGB_TRUNC_TC_BWD=0 timeout 300 python tools/time_bwd.py 4096 c5
done; done
