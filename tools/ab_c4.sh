#!/bin/bash
# interleaved A/B of library builds on c4 (fragment kernels): tools/ab_c4.sh LIB...
for r in 1 2 3; do for L in "$@"; do
  SIGB_LIB_PATH=$L timeout 300 python tools/time_bwd.py 1024 c4
done; done
