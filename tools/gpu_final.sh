#!/bin/bash
# Round-end measurement pass: smoke, full GPU suite, bench lines for every
# config, the reference arm, the ncu launch list of the default command and
# full captures of the dominant kernels (summarised into profiles/ on the CPU side).
mkdir -p gpurun_out/final
O=gpurun_out/final
nvidia-smi > $O/nvidia_smi.txt 2>&1
( time timeout 300 python -c "import __graft_entry__ as g; g.smoke()" ) > $O/smoke.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
timeout 900 python bench.py > $O/bench_c5.json 2> $O/bench_c5.err
for c in c2 c3 c4; do
  timeout 600 python bench.py --config $c --no-e2e > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 300 python bench.py --config c1 --no-e2e --steps 20 > $O/bench_c1.json 2> $O/bench_c1.err
timeout 300 python bench.py --impl reference > $O/bench_ref_c5.json 2> $O/bench_ref_c5.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c5.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $O/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:frag_backward -c 1 \
  -o $O/prof_c4_bwd python bench.py --config c4 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --batch 256 > $O/ncu_c4b.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:frag_forward -c 1 \
  -o $O/prof_c4_fwd python bench.py --config c4 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --batch 512 > $O/ncu_c4f.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sigjit_bwd -c 1 \
  -o $O/prof_c3_bwd python bench.py --config c3 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $O/ncu_c3b.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sigjit_fwd -c 1 \
  -o $O/prof_c3_fwd python bench.py --config c3 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $O/ncu_c3f.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:trunc_backward -c 1 \
  -o $O/prof_c2_bwd python bench.py --config c2 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --batch 512 > $O/ncu_c2b.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:trunc_forward -c 1 \
  -o $O/prof_c2_fwd python bench.py --config c2 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --batch 1024 > $O/ncu_c2f.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:trunc_backward -c 1 \
  -o $O/prof_c5_bwd python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --batch 1024 > $O/ncu_c5b.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:trunc_forward -c 1 \
  -o $O/prof_c5_fwd python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --batch 2048 > $O/ncu_c5f.log 2>&1
for r in $O/prof_*.ncu-rep; do
  ncu -i $r --page raw --csv > ${r%.ncu-rep}.csv 2>/dev/null
  ncu -i $r --page source --csv --print-source sass > ${r%.ncu-rep}_sass.csv 2>/dev/null
  gzip -f ${r%.ncu-rep}_sass.csv
  rm -f $r
done
du -sh $O
echo done
