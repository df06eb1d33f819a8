#!/bin/bash
# k_graft shared-memory staging + k_attend event timing: parity tests, config 2
# and config 3 lines, k_graft ncu capture.
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_stream_gpu.py tests/test_dropin.py -x -q > $OUT/tests_graft.log 2>&1; tail -3 $OUT/tests_graft.log
timeout 600 python bench.py > $OUT/c2.json 2> $OUT/c2.err; tail -2 $OUT/c2.err
timeout 900 python bench.py --mode stream > $OUT/c3.json 2> $OUT/c3.err; tail -2 $OUT/c3.err
python - <<'PY'
import json
for f in ['c2','c3']:
    try:
        d = json.load(open(f'gpurun_out/{f}.json'))
        print(f, round(d['value'], 1), 'ms', round(d['ms_per_step'], 4), 'roof', json.dumps(d.get('roofline'))[:300], 'step', (d.get('step_roofline') or {}).get('frac'))
    except Exception as e:
        print(f, 'ERR', e)
PY
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'k_select|k_attend|k_merge|k_append|k_graft|k_compact' --csv --log-file $OUT/launches_stream.csv python bench.py --mode stream --graph 0 --steps 140 --warmup 3 --cpu-baseline 0 > $OUT/ncu_stream.log 2>&1
python tools/launch_table.py $OUT/launches_stream.csv $OUT/launches_stream.md r02-stream 'k_' | tail -8
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_graft' -c 1 -o $OUT/prof_k_graft python bench.py --mode stream --graph 0 --steps 20 --warmup 3 --cpu-baseline 0 > $OUT/ncu_graft.log 2>&1
ls $OUT
