#!/bin/bash
# parity of the in-tree build (tensor-core and full-shape tests), then interleaved A/B timing of
# the given library builds on c5 and c2: tools/gpu_ab.sh LIB...
O=gpurun_out/ab; mkdir -p $O
timeout 600 python -m pytest tests/test_trunc_tc.py tests/test_full_shape.py -q -x > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
tail -2 $O/pytest.txt
bash tools/ab.sh c5 8192 "$@" > $O/ab_c5.txt 2>&1
bash tools/ab.sh c2 1024 "$@" > $O/ab_c2.txt 2>&1
cat $O/ab_c5.txt $O/ab_c2.txt
