#!/bin/bash
# HEAD sanity: every GPU test, smoke, the default bench line and the reference arm.
OUT=gpurun_out/head; mkdir -p $OUT
timeout 1500 python -m pytest tests -q -m gpu > $OUT/tests_gpu.log 2>&1; tail -2 $OUT/tests_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
timeout 900 python bench.py > $OUT/c2.json 2> $OUT/c2.err
timeout 900 python bench.py --impl reference > $OUT/c2_ref.json 2> $OUT/c2_ref.err
python - <<'PY'
import json
for f in ['c2', 'c2_ref']:
    d = json.load(open(f'gpurun_out/head/{f}.json')); sr = d.get('step_roofline') or {}; r = d.get('roofline') or {}
    print(f, round(d['value'], 1), d['ms_per_step'], 'katt', r.get('frac'), 'step', sr.get('frac'), sr.get('frac_fp16_fine_width'), 'e2e', (d.get('e2e') or {}).get('value'), 'parity', (d.get('parity') or {}).get('ok'), d.get('clocks'), d.get('gpu_launches'))
PY
