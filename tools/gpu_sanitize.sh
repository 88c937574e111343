#!/bin/bash
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --num-cuda-barriers 65536 --print-limit 20 python tools/sanitize_workload.py > gpurun_out/sanitize_$tool.txt 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_$tool.txt
done
echo done
