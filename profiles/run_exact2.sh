#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_dropin.py tests/test_parity_gpu.py tests/test_parity_configs_gpu.py tests/test_eval_gpu.py -x -q -m gpu > $OUT/tests_exact2.log 2>&1; tail -3 $OUT/tests_exact2.log
TIERKV_DROPIN_PROF=1 timeout 300 oracle/_ref/b200_dropin_bench 131072 16 16 2>&1 | tail -3
for n in 32768 131072; do
  timeout 600 oracle/_ref/b200_dropin_bench $n 64 512 > $OUT/dx_b200_$n.json 2>&1; cat $OUT/dx_b200_$n.json
done
