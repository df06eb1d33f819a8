#!/bin/bash
# k_attend with TMA gather4: parity first (bounded), then the bench
OUT=gpurun_out; mkdir -p $OUT
timeout 300 python -m pytest tests/test_parity_gpu.py -x -q -k "batched or degenerate or host" > $OUT/tests_tma0.log 2>&1; tail -3 $OUT/tests_tma0.log
if grep -q "passed" $OUT/tests_tma0.log && ! grep -q "failed" $OUT/tests_tma0.log; then
  timeout 900 python -m pytest tests/test_slots_gpu.py tests/test_parity_gpu.py tests/test_parity_configs_gpu.py tests/test_stream_gpu.py -x -q > $OUT/tests_tma.log 2>&1; tail -3 $OUT/tests_tma.log
  s() { python -c "
import json,sys; d=json.load(open(sys.argv[1])); print(sys.argv[2], round(d['value'],1), 'ms', round(d['ms_per_step'],4), 'sel', round(d['step_roofline']['select_ms'],4), 'att', round(d['step_roofline']['attend_ms'],4), 'attfrac', round(d['roofline']['frac'],3), 'frac', round(d['step_roofline']['frac'],3), 'chk', d['check']['ok'], (d.get('parity') or {}).get('ok'))" $1 "$2"; }
  timeout 300 python bench.py --cpu-baseline 0 > $OUT/t_c2.json 2>/dev/null; s $OUT/t_c2.json c2
  timeout 300 python bench.py --config 1 --cpu-baseline 0 --parity 0 > $OUT/t_c1.json 2>/dev/null; s $OUT/t_c1.json c1
  timeout 300 python bench.py --kv-heads 1 --cpu-baseline 0 --parity 0 > $OUT/t_32.json 2>/dev/null; s $OUT/t_32.json 32slots
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_attend -s 5 -c 1 -o $OUT/prof_k_attend_tma python bench.py --steps 3 --warmup 3 --graph 0 --cpu-baseline 0 --parity 0 > /dev/null 2>&1
fi
