#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
timeout 1500 python -m pytest tests -q -m gpu -x > $OUT/tests_q3.log 2>&1; tail -2 $OUT/tests_q3.log
for q in 1 0; do
  export LC_ATT_QUEUE=$q
  timeout 300 python bench.py --cpu-baseline 0 --parity 1 > $OUT/q3_c2_$q.json 2>/dev/null; python -c "
import json; d=json.load(open('$OUT/q3_c2_$q.json')); print('c2 q$q', d['value'], d['ms_per_step'], d['step_roofline']['frac'], 'e2e', d['e2e']['value'], 'lw', d['layerwise']['value'], d['parity']['ok'])"
  timeout 300 python bench.py --config 1 --cpu-baseline 0 --parity 0 > $OUT/q3_c1_$q.json 2>/dev/null; python -c "
import json; d=json.load(open('$OUT/q3_c1_$q.json')); print('c1 q$q', d['value'], d['ms_per_step'])"
  timeout 300 python bench.py --kv-heads 1 --cpu-baseline 0 --parity 0 > $OUT/q3_32_$q.json 2>/dev/null; python -c "
import json; d=json.load(open('$OUT/q3_32_$q.json')); print('32 q$q', d['value'], d['ms_per_step'])"
done
