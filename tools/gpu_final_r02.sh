#!/bin/bash
# end-of-round evidence at the final code: suite, smoke, default bench line + launch list
# (tools/gpu_check.sh), ncu captures of the two c5 kernels, and the c4 / c3 lines
bash tools/gpu_check.sh
bash tools/gpu_prof.sh c5_pq10 c5 1024 trunc_pq_backward >/dev/null
bash tools/gpu_prof.sh c5_tcfwd6 c5 2048 trunc_tc_forward >/dev/null
bash tools/gpu_bench_some.sh c4 c3
