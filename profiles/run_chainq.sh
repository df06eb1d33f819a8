#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
LC_NO_FUSED=1 timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_stream_gpu.py tests/test_slots_gpu.py tests/test_gather_gpu.py -x -q > $OUT/tests_cq_chain.log 2>&1; tail -2 $OUT/tests_cq_chain.log
timeout 900 python -m pytest tests/test_parity_configs_gpu.py -x -q > $OUT/tests_cq.log 2>&1; tail -2 $OUT/tests_cq.log
for q in 1 0; do
  export LC_ATT_QUEUE=$q
  timeout 900 python bench.py --config 4 --steps 30 --cpu-baseline 0 > $OUT/cq_c4_$q.json 2>/dev/null; python -c "
import json; d=json.load(open('$OUT/cq_c4_$q.json')); print('c4 q$q', d['value'], d['ms_per_step'], d['step_roofline']['frac'], d['parity']['ok'], d['check']['ok'], d['kernels_per_step'])"
done
