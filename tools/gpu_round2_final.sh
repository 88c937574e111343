#!/bin/bash
# Fresh round-2 evidence at the current code: the GPU suite, smoke, the default bench line and its
# launch list (tools/gpu_check.sh), ncu --set full of the c5 P/Q backward and tensor-core forward,
# then one clocked bench line per config (tools/gpu_bench_all.sh).
bash tools/gpu_check.sh
bash tools/gpu_prof.sh c5_pq9 c5 1024 trunc_pq_backward
bash tools/gpu_prof.sh c5_tcfwd4 c5 2048 trunc_tc_forward
bash tools/gpu_bench_all.sh
