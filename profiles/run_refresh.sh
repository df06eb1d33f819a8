#!/bin/bash
# Evidence refresh at HEAD: GPU tests, configs 1/2/4 lines, reference arm,
# config-4 chain launch list.
OUT=gpurun_out; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt
timeout 1500 python -m pytest tests -q -m gpu > $OUT/tests_gpu.log 2>&1; tail -5 $OUT/tests_gpu.log
timeout 600 python bench.py > $OUT/c2.json 2> $OUT/c2.err; tail -2 $OUT/c2.err
timeout 600 python bench.py --impl reference > $OUT/c2_ref.json 2> $OUT/c2_ref.err
timeout 600 python bench.py --config 1 > $OUT/c1.json 2> $OUT/c1.err; tail -2 $OUT/c1.err
timeout 1200 python bench.py --config 4 --steps 30 > $OUT/c4.json 2> $OUT/c4.err; tail -2 $OUT/c4.err
python - <<'PY'
import json
for f in ['c1','c2','c4','c2_ref']:
    try:
        d = json.load(open(f'gpurun_out/{f}.json'))
        sr = d.get('step_roofline') or d.get('roofline') or {}
        print(f, round(d['value'], 1), 'ms', round(d['ms_per_step'], 4), 'frac', sr.get('frac'), 'e2e', (d.get('e2e') or {}).get('value'),
              'cpu', (d.get('cpu_baseline') or {}).get('value'), 'parity', (d.get('parity') or {}).get('ok'))
    except Exception as e:
        print(f, 'ERR', e)
PY
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'k_coarse|k_fine|k_pickq|k_spans|k_attend|k_merge' --csv --log-file $OUT/launches_c4.csv python bench.py --config 4 --steps 3 --warmup 3 --graph 0 --cpu-baseline 0 --parity 0 > $OUT/ncu_c4.log 2>&1
python tools/launch_table.py $OUT/launches_c4.csv $OUT/launches_c4.md r02-c4 | tail -8
