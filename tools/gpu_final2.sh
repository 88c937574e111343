#!/bin/bash
# Round-end pass after the tensor-core forward: smoke, full GPU suite, c5 bench line,
# c5 launch list, memcheck of the tensor-core forward.
O=gpurun_out/final2; mkdir -p $O
nvidia-smi > $O/nvidia_smi.txt 2>&1
( time timeout 300 python -c "import __graft_entry__ as g; g.smoke()" ) > $O/smoke.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
timeout 900 python bench.py > $O/bench_c5.json 2> $O/bench_c5.err
timeout 300 python bench.py --config c1 --no-e2e --steps 20 > $O/bench_c1.json 2> $O/bench_c1.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c5.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $O/ncu_launch_bench.log 2>&1
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_trunc_tc.py -q -x > $O/memcheck_tc.txt 2>&1
echo "rc=$?" >> $O/memcheck_tc.txt
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest tests/test_trunc_tc.py -q -x > $O/synccheck_tc.txt 2>&1
echo "rc=$?" >> $O/synccheck_tc.txt
echo done
