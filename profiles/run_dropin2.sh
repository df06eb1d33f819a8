#!/bin/bash
OUT=gpurun_out/dropin2; mkdir -p $OUT
timeout 900 python -m pytest tests/test_dropin.py -x -q > $OUT/tests.log 2>&1; tail -2 $OUT/tests.log
for n in 32768 131072; do
  timeout 600 oracle/_ref/b200_dropin_bench $n 64 512 > $OUT/dropin_b200_$n.json 2>&1
done
cat $OUT/dropin_*.json
