#!/bin/bash
# Fresh round-2 evidence at the current code: the GPU suite, smoke, the default bench line and its
# launch list (tools/gpu_check.sh), ncu --set full of the c5 P/Q backward, then one clocked bench
# line per config (tools/gpu_bench_all.sh).
bash tools/gpu_check.sh
bash tools/gpu_prof.sh r02g_c5_pq c5 1024 trunc_pq_backward
bash tools/gpu_bench_all.sh
