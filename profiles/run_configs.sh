#!/bin/bash
# Round-2 configs run: new GPU tests, config 1/2/4/5 lines, the streaming
# (config 3) line, drop-in per-call latency, stream ncu launch list.
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_stream_gpu.py tests/test_slots_gpu.py -x -q > $OUT/tests_new.log 2>&1; tail -4 $OUT/tests_new.log
timeout 900 python bench.py > $OUT/c2.json 2> $OUT/c2.err; tail -2 $OUT/c2.err
timeout 600 python bench.py --config 1 > $OUT/c1.json 2> $OUT/c1.err; tail -2 $OUT/c1.err
timeout 1200 python bench.py --config 4 --steps 30 > $OUT/c4.json 2> $OUT/c4.err; tail -2 $OUT/c4.err
timeout 900 python bench.py --config 5 --steps 20 > $OUT/c5.json 2> $OUT/c5.err; tail -2 $OUT/c5.err
timeout 900 python bench.py --mode stream > $OUT/c3.json 2> $OUT/c3.err; tail -2 $OUT/c3.err
for n in 32768 131072; do
  timeout 600 oracle/_ref/ref_dropin_bench $n 64 512 > $OUT/dropin_ref_$n.json 2>&1
  timeout 600 oracle/_ref/b200_dropin_bench $n 64 512 > $OUT/dropin_b200_$n.json 2>&1
done
cat $OUT/dropin_*.json
python - <<'PY'
import json
for f in ['c1','c2','c4','c5','c3']:
    try:
        d = json.load(open(f'gpurun_out/{f}.json'))
        sr = d.get('step_roofline') or d.get('roofline') or {}
        print(f, round(d['value'], 1), 'ms', round(d['ms_per_step'], 4), 'frac', sr.get('frac'), 'e2e', (d.get('e2e') or {}).get('value'),
              'cpu', (d.get('cpu_baseline') or {}).get('value'), 'lw', (d.get('layerwise') or {}).get('value'))
    except Exception as e:
        print(f, 'ERR', e)
PY
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'k_select|k_attend|k_merge|k_append|k_graft' --csv --log-file $OUT/launches_stream.csv python bench.py --mode stream --graph 0 --steps 30 --warmup 3 --cpu-baseline 0 > $OUT/ncu_stream.log 2>&1
python tools/launch_table.py $OUT/launches_stream.csv $OUT/launches_stream.md r02-stream 'lc::k_' | tail -7
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_graft' -c 1 -o $OUT/prof_k_graft python bench.py --mode stream --graph 0 --steps 20 --warmup 3 --cpu-baseline 0 > $OUT/ncu_graft.log 2>&1
ls $OUT | head -80
