#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_dropin.py tests/test_parity_gpu.py tests/test_parity_configs_gpu.py -x -q -m gpu > $OUT/tests_exact.log 2>&1; tail -3 $OUT/tests_exact.log
for n in 32768 131072; do
  OMP_NUM_THREADS=1 timeout 600 oracle/_ref/ref_dropin_bench $n 64 512 > $OUT/dx_ref1_$n.json 2>&1
  timeout 600 oracle/_ref/ref_dropin_bench $n 64 512 > $OUT/dx_ref_$n.json 2>&1
  timeout 600 oracle/_ref/b200_dropin_bench $n 64 512 > $OUT/dx_b200_$n.json 2>&1
  echo "== $n"; cat $OUT/dx_ref_$n.json $OUT/dx_ref1_$n.json $OUT/dx_b200_$n.json
done
