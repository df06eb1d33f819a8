#!/bin/bash
# A/B on one box: ab/liblychee_old.so (HEAD) vs the working build, interleaved.
OUT=gpurun_out/ab; mkdir -p $OUT
B="python bench.py --steps 50 --warmup 5 --cpu-baseline 0 --parity 0"
for r in 1 2; do
  for v in old new; do
    if [ $v = old ]; then export LC_LIB_PATH=$PWD/ab/liblychee_old.so; else unset LC_LIB_PATH; fi
    timeout 600 $B > $OUT/c2_${v}_$r.json 2>/dev/null
    timeout 900 $B --config 4 --steps 30 > $OUT/c4_${v}_$r.json 2>/dev/null
    timeout 600 $B --config 1 > $OUT/c1_${v}_$r.json 2>/dev/null
  done
done
unset LC_LIB_PATH
python - <<'PY'
import json, glob
for f in sorted(glob.glob('gpurun_out/ab/*.json')):
    try:
        d = json.load(open(f)); sr = d.get('step_roofline') or {}
        print(f.split('/')[-1], round(d['value'], 1), 'sel', sr.get('select_ms'))
    except Exception as e:
        print(f, 'ERR', e)
PY
