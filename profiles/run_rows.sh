#!/bin/bash
# Row-list writes one warp per span (k_select P4, k_spans): parity, LC_PROF phases, configs 2 and 4.
OUT=gpurun_out/rows; mkdir -p $OUT
timeout 1200 python -m pytest tests -q -m gpu -x > $OUT/tests.log 2>&1; tail -2 $OUT/tests.log
LC_PROF=1 timeout 500 python bench.py --steps 3 --warmup 3 --graph 0 --cpu-baseline 0 --parity 0 > /dev/null 2> $OUT/prof.err; grep -a "per-CTA" $OUT/prof.err | tail -2
timeout 900 python bench.py > $OUT/c2.json 2> $OUT/c2.err
timeout 1500 python bench.py --config 4 --steps 30 > $OUT/c4.json 2> $OUT/c4.err
timeout 600 python bench.py --config 1 > $OUT/c1.json 2> $OUT/c1.err
python - <<'PY'
import json
for f in ['c1','c2','c4']:
    try:
        d = json.load(open(f'gpurun_out/rows/{f}.json'))
        sr = d.get('step_roofline') or {}; r = d.get('roofline') or {}
        print(f, round(d['value'], 1), 'ms', round(d['ms_per_step'], 4), 'katt', r.get('frac'), 'step', sr.get('frac'), sr.get('frac_fp16_fine_width'), 'sel', sr.get('select_ms'), 'e2e', (d.get('e2e') or {}).get('value'), 'parity', (d.get('parity') or {}).get('ok'), d.get('clocks'))
    except Exception as e:
        print(f, 'ERR', e)
PY
