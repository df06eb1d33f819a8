#!/bin/bash
# A/B of k_graft at 128 threads x 5 CTAs/SM (working build) vs 256 x 4 (ab/liblychee_old.so)
OUT=gpurun_out/abg; mkdir -p $OUT
timeout 900 python -m pytest tests/test_stream_gpu.py tests/test_parity_gpu.py -q -x -k "stream or graft or decode" > $OUT/tests.log 2>&1; tail -2 $OUT/tests.log
for r in 1 2; do
  for v in old new; do
    if [ $v = old ]; then export LC_LIB_PATH=$PWD/ab/liblychee_old.so; else unset LC_LIB_PATH; fi
    timeout 900 python bench.py --mode stream --cpu-baseline 0 > $OUT/c3_${v}_$r.json 2>/dev/null
  done
done
unset LC_LIB_PATH
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_graft' --csv --log-file $OUT/graft_new.csv python bench.py --mode stream --graph 0 --steps 30 --warmup 3 --cpu-baseline 0 > /dev/null 2>&1
LC_LIB_PATH=$PWD/ab/liblychee_old.so timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_graft' --csv --log-file $OUT/graft_old.csv python bench.py --mode stream --graph 0 --steps 30 --warmup 3 --cpu-baseline 0 > /dev/null 2>&1
python - <<'PY'
import json, glob, csv
for f in sorted(glob.glob('gpurun_out/abg/*.json')):
    try:
        d = json.load(open(f)); print(f.split('/')[-1], round(d['value'], 1), d['ms_per_step'])
    except Exception as e:
        print(f, 'ERR', e)
for v in ['old', 'new']:
    try:
        t = [float(r[-1].replace(',', '')) for r in csv.reader(open(f'gpurun_out/abg/graft_{v}.csv')) if len(r) > 5 and r[-3] == 'gpu__time_duration.sum']
        print(v, 'k_graft us', [round(x / 1000, 1) for x in t])
    except Exception as e:
        print(v, 'ERR', e)
PY
