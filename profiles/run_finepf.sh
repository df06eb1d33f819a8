#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_parity_configs_gpu.py -x -q -k "long_context" > $OUT/tests_pf.log 2>&1; tail -2 $OUT/tests_pf.log
for pf in 0 1; do LC_FINE_PF=$pf timeout 900 python bench.py --config 4 --steps 30 --cpu-baseline 0 --parity 0 > $OUT/pf_$pf.json 2>/dev/null; python -c "
import json; d=json.load(open('$OUT/pf_$pf.json')); print('pf $pf', d['value'], d['ms_per_step'], d['step_roofline']['frac'], d['step_roofline']['select_ms'])"; done
