#!/bin/bash
# Final round-2 evidence after the k_select member-bitmap change.
OUT=gpurun_out/final3; mkdir -p $OUT
timeout 1500 python -m pytest tests -q -m gpu > $OUT/tests_gpu.log 2>&1; tail -2 $OUT/tests_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
timeout 900 python bench.py > $OUT/c2.json 2> $OUT/c2.err
timeout 900 python bench.py --impl reference > $OUT/c2_ref.json 2> $OUT/c2_ref.err
timeout 600 python bench.py --config 1 > $OUT/c1.json 2> $OUT/c1.err
timeout 900 python bench.py --mode stream > $OUT/c3.json 2> $OUT/c3.err
timeout 900 python bench.py --config 5 --steps 20 > $OUT/c5.json 2> $OUT/c5.err
python - <<'PY'
import json
for f in ['c1', 'c2', 'c3', 'c5', 'c2_ref']:
    try:
        d = json.load(open(f'gpurun_out/final3/{f}.json')); sr = d.get('step_roofline') or {}; r = d.get('roofline') or {}
        print(f, round(d['value'], 1), d['ms_per_step'], 'katt', r.get('frac'), 'step', sr.get('frac'), sr.get('frac_fp16_fine_width'), 'sel', sr.get('select_ms'), 'e2e', (d.get('e2e') or {}).get('value'), 'cpu', (d.get('cpu_baseline') or {}).get('value'), 'parity', (d.get('parity') or {}).get('ok'), d.get('clocks'))
    except Exception as e:
        print(f, 'ERR', e)
PY
BENCH="python bench.py --steps 3 --warmup 3 --graph 0 --cpu-baseline 0 --parity 0"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'k_select|k_attend|k_merge' --csv --log-file $OUT/launches_c2.csv $BENCH > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_select -s 5 -c 1 -o $OUT/prof_k_select $BENCH > /dev/null 2>&1
ls $OUT
