#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
timeout 300 python -m pytest tests/test_parity_gpu.py -x -q -k "batched or degenerate" > $OUT/tests_m0.log 2>&1; tail -2 $OUT/tests_m0.log
if grep -q " passed" $OUT/tests_m0.log && ! grep -q "failed" $OUT/tests_m0.log; then
timeout 1500 python -m pytest tests -q -m gpu -x > $OUT/tests_m.log 2>&1; tail -2 $OUT/tests_m.log
timeout 300 python bench.py --cpu-baseline 0 --parity 1 > $OUT/m_c2.json 2>/dev/null; python -c "
import json; d=json.load(open('$OUT/m_c2.json')); print('c2', d['value'], d['ms_per_step'], d['step_roofline']['frac'], 'e2e', d['e2e']['value'], 'lw', d['layerwise']['value'], d['parity']['ok'], d['check']['ok'], d['kernels_per_step'])"
timeout 300 python bench.py --config 1 --cpu-baseline 0 --parity 0 > $OUT/m_c1.json 2>/dev/null; python -c "
import json; d=json.load(open('$OUT/m_c1.json')); print('c1', d['value'], d['ms_per_step'], 'e2e', d['e2e']['value'])"
timeout 300 python bench.py --kv-heads 1 --cpu-baseline 0 --parity 0 > $OUT/m_32.json 2>/dev/null; python -c "
import json; d=json.load(open('$OUT/m_32.json')); print('32', d['value'], d['ms_per_step'])"
python tools/e2e_probe.py 2>&1 | tail -7
fi
