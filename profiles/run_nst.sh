#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_slots_gpu.py tests/test_parity_gpu.py tests/test_parity_configs_gpu.py tests/test_gather_gpu.py -x -q > $OUT/tests_nst.log 2>&1; tail -2 $OUT/tests_nst.log
s() { python -c "
import json,sys; d=json.load(open(sys.argv[1])); print(sys.argv[2], round(d['value'],1), 'ms', round(d['ms_per_step'],4), 'frac', round(d['step_roofline']['frac'],3), 'lw', round(d['layerwise']['value'],1), (d.get('parity') or {}).get('ok'))" $1 "$2"; }
timeout 300 python bench.py --cpu-baseline 0 > $OUT/n_c2.json 2>/dev/null; s $OUT/n_c2.json c2
timeout 300 python bench.py --kv-heads 1 --cpu-baseline 0 > $OUT/n_32.json 2>/dev/null; s $OUT/n_32.json 32slots
LC_FUSED_SHALLOW=1 timeout 300 python bench.py --kv-heads 1 --cpu-baseline 0 --parity 0 > $OUT/n_32s.json 2>/dev/null; s $OUT/n_32s.json 32slots-shallow
timeout 300 python bench.py --config 1 --cpu-baseline 0 > $OUT/n_c1.json 2>/dev/null; s $OUT/n_c1.json c1
LC_PROF=1 timeout 300 python tools/prof_step.py --steps 2 --kv-heads 1 2>&1 | grep "k_select per-CTA" | tail -1
