#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
LC_ATT_QUEUE=1 timeout 600 python -m pytest tests/test_parity_gpu.py -x -q -k "batched or degenerate or host" > $OUT/tests_q0.log 2>&1; tail -2 $OUT/tests_q0.log
if grep -q " passed" $OUT/tests_q0.log && ! grep -q "failed" $OUT/tests_q0.log; then
LC_ATT_QUEUE=1 timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_parity_configs_gpu.py tests/test_stream_gpu.py tests/test_gather_gpu.py tests/test_slots_gpu.py -x -q > $OUT/tests_q.log 2>&1; tail -2 $OUT/tests_q.log
for qm in 0 1; do
  if [ $qm = 1 ]; then export LC_ATT_QUEUE=1; else unset LC_ATT_QUEUE; fi
  timeout 300 python bench.py --cpu-baseline 0 > $OUT/q_c2_$qm.json 2>/dev/null; python -c "
import json; d=json.load(open('$OUT/q_c2_$qm.json')); print('queue $qm', d['value'], d['ms_per_step'], d['step_roofline']['frac'], 'e2e', d['e2e']['value'], d['parity']['ok'], d['check']['ok'], 'lw', d['layerwise']['value'])"
done
export LC_ATT_QUEUE=1; timeout 300 python bench.py --kv-heads 1 --cpu-baseline 0 --parity 0 > $OUT/q_32.json 2>/dev/null; python -c "
import json; d=json.load(open('$OUT/q_32.json')); print('queue 32 slots', d['value'], d['ms_per_step'])"
fi
