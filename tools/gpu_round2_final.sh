#!/bin/bash
# Fresh round-2 evidence: ncu --set full of the c5 P/Q backward, the c5 tcgen05 forward and the c3
# generated backward/forward at the current code, then one clocked bench line per config.
bash tools/gpu_prof.sh r02f_c5_pq c5 1024 trunc_pq_backward
bash tools/gpu_prof.sh r02f_c5_tcfwd c5 2048 trunc_tc_forward
bash tools/gpu_prof.sh r02f_c3_jbwd c3 4096 sigjit_bwd
bash tools/gpu_prof.sh r02f_c3_jfwd c3 4096 sigjit_fwd
rm -f gpurun_out/prof/*.source.csv.big
bash tools/gpu_bench_all.sh
