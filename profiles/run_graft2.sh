#!/bin/bash
# k_graft staging (coarse tier batched loads) + k_merge prologue under k_attend's drain:
# all GPU tests, configs 1/4 (static partition) and 3 (grafts), k_graft ncu.
OUT=gpurun_out; mkdir -p $OUT
timeout 1500 python -m pytest tests -q -m gpu -x > $OUT/tests_gpu.log 2>&1; tail -3 $OUT/tests_gpu.log
timeout 600 python bench.py --config 1 > $OUT/c1.json 2> $OUT/c1.err; tail -2 $OUT/c1.err
timeout 1200 python bench.py --config 4 --steps 30 > $OUT/c4.json 2> $OUT/c4.err; tail -2 $OUT/c4.err
timeout 900 python bench.py --mode stream > $OUT/c3.json 2> $OUT/c3.err; tail -2 $OUT/c3.err
python - <<'PY'
import json
for f in ['c1','c4','c3']:
    try:
        d = json.load(open(f'gpurun_out/{f}.json'))
        sr = d.get('step_roofline') or {}
        print(f, round(d['value'], 1), 'ms', round(d['ms_per_step'], 4), 'k_attend frac', d['roofline']['frac'], 'step', sr.get('frac'), 'e2e', (d.get('e2e') or {}).get('value'), 'parity', (d.get('parity') or {}).get('ok'))
    except Exception as e:
        print(f, 'ERR', e)
PY
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'k_select|k_attend|k_merge|k_append|k_graft|k_compact' --csv --log-file $OUT/launches_stream.csv python bench.py --mode stream --graph 0 --steps 140 --warmup 3 --cpu-baseline 0 > $OUT/ncu_stream.log 2>&1
python tools/launch_table.py $OUT/launches_stream.csv $OUT/launches_stream.md r02-stream 'k_' | tail -8
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_graft' -c 1 -o $OUT/prof_k_graft python bench.py --mode stream --graph 0 --steps 20 --warmup 3 --cpu-baseline 0 > $OUT/ncu_graft.log 2>&1
ls $OUT
