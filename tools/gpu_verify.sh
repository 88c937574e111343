#!/bin/bash
# Quick re-verification after a change: smoke, the full GPU suite, the c5/c3 bench lines.
O=gpurun_out/verify; mkdir -p $O
( time timeout 300 python -c "import __graft_entry__ as g; g.smoke()" ) > $O/smoke.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
timeout 900 python bench.py > $O/bench_c5.json 2> $O/bench_c5.err
timeout 600 python bench.py --config c3 --no-e2e > $O/bench_c3.json 2> $O/bench_c3.err
echo done
