#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_dropin.py -x -q -m gpu > $OUT/tests_exact3.log 2>&1; tail -2 $OUT/tests_exact3.log
for n in 32768 131072; do
  timeout 600 oracle/_ref/b200_dropin_bench $n 64 512 > $OUT/dx_b200_$n.json 2>&1; cat $OUT/dx_b200_$n.json
done
