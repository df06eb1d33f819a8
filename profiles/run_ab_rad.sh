#!/bin/bash
# A/B: k_select radius load hoisted before the exact dot chain (working build) vs HEAD (ab/liblychee_old.so)
OUT=gpurun_out/abr; mkdir -p $OUT
timeout 1500 python -m pytest tests/test_parity_gpu.py tests/test_parity_configs_gpu.py tests/test_slots_gpu.py -q -x > $OUT/tests.log 2>&1; tail -2 $OUT/tests.log
B="python bench.py --steps 50 --warmup 5 --cpu-baseline 0 --parity 0"
for r in 1 2; do
  for v in old new; do
    if [ $v = old ]; then export LC_LIB_PATH=$PWD/ab/liblychee_old.so; else unset LC_LIB_PATH; fi
    timeout 600 $B > $OUT/c2_${v}_$r.json 2>/dev/null
    timeout 600 $B --config 1 > $OUT/c1_${v}_$r.json 2>/dev/null
  done
done
unset LC_LIB_PATH
LC_PROF=1 timeout 500 python bench.py --steps 3 --warmup 3 --graph 0 --cpu-baseline 0 --parity 0 > /dev/null 2> $OUT/prof.err; grep -a "per-CTA" $OUT/prof.err | tail -1
python - <<'PY'
import json, glob
for f in sorted(glob.glob('gpurun_out/abr/*.json')):
    try:
        d = json.load(open(f)); sr = d.get('step_roofline') or {}
        print(f.split('/')[-1], round(d['value'], 1), 'sel', sr.get('select_ms'))
    except Exception as e:
        print(f, 'ERR', e)
PY
