#!/bin/bash
# End-of-round evidence for the decode step (after dropping the early k_merge trigger):
# GPU tests, smoke, configs 1/2/4 + reference arm, config-2 launch list and ncu captures.
OUT=gpurun_out/final2; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv > $OUT/gpu.txt
timeout 1500 python -m pytest tests -q -m gpu > $OUT/tests_gpu.log 2>&1; tail -2 $OUT/tests_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
timeout 900 python bench.py > $OUT/c2.json 2> $OUT/c2.err
timeout 900 python bench.py --impl reference > $OUT/c2_ref.json 2> $OUT/c2_ref.err
timeout 600 python bench.py --config 1 > $OUT/c1.json 2> $OUT/c1.err
timeout 1500 python bench.py --config 4 --steps 30 > $OUT/c4.json 2> $OUT/c4.err
python - <<'PY'
import json
for f in ['c1','c2','c4','c2_ref']:
    try:
        d = json.load(open(f'gpurun_out/final2/{f}.json'))
        sr = d.get('step_roofline') or {}; r = d.get('roofline') or {}
        print(f, round(d['value'], 1), 'ms', round(d['ms_per_step'], 4), 'katt', r.get('frac'), 'step', sr.get('frac'), sr.get('frac_fp16_fine_width'), 'e2e', (d.get('e2e') or {}).get('value'), 'parity', (d.get('parity') or {}).get('ok'), d.get('clocks'))
    except Exception as e:
        print(f, 'ERR', e)
PY
BENCH="python bench.py --steps 3 --warmup 3 --graph 0 --cpu-baseline 0 --parity 0"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'k_select|k_attend|k_merge' --csv --log-file $OUT/launches_c2.csv $BENCH > /dev/null 2>&1
for k in k_select k_attend k_merge; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 5 -c 1 -o $OUT/prof_$k $BENCH > /dev/null 2>&1
done
ls $OUT
