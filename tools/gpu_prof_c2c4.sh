#!/bin/bash
# ncu --set full of the config-2 P/Q backward and the config-4 fragment kernels at the current code,
# then their bench lines (which pick the captured DRAM traffic up from profiles/ncu_summary.json)
bash tools/gpu_prof.sh r02g_c2_pq c2 1024 trunc_pq_backward
bash tools/gpu_prof.sh r02g_c4_fbwd c4 256 frag_backward
bash tools/gpu_prof.sh r02g_c4_ffwd c4 512 frag_forward
