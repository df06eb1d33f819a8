#!/bin/bash
# GPU tests (full output tail) + one default bench line with the parity field
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests -q -m gpu > $OUT/tests_gpu.log 2>&1; tail -5 $OUT/tests_gpu.log
timeout 600 python bench.py --steps 30 --warmup 3 --cpu-baseline 0 > $OUT/bench_q.json 2> $OUT/bench_q.err; tail -3 $OUT/bench_q.err
python -c "import json;d=json.load(open('$OUT/bench_q.json'));print('steps/s',d['value'],'ms',d['ms_per_step'],'att_frac',d['roofline']['frac'],'sel_ms',d['step_roofline']['select_ms'],'att_ms',d['step_roofline']['attend_ms'],'step_frac',d['step_roofline']['frac']);print('parity',d['parity'])"
