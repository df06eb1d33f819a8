#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_stream_gpu.py tests/test_parity_gpu.py -x -q > $OUT/tests_q4.log 2>&1; tail -2 $OUT/tests_q4.log
for q in 1 0; do
  export LC_ATT_QUEUE=$q
  timeout 900 python bench.py --mode stream --cpu-baseline 0 > $OUT/q4_c3_$q.json 2>/dev/null; python -c "
import json; d=json.load(open('$OUT/q4_c3_$q.json')); print('c3 q$q', d['value'], d['ms_per_step'], d['roofline']['frac'], d['check']['ok'], d['grafts_applied_on_device'], d['kernels_per_step'])"
done
