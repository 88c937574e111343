#!/bin/bash
# A/B timing of alternative builds on one box: tools/ab.sh CONFIG PATHS LIB... (each run 3 times, interleaved)
CFG=$1; P=$2; shift 2
for r in 1 2 3; do for L in "$@"; do SIGB_LIB_PATH=$L timeout 300 python tools/time_bwd.py $P $CFG; done; done
