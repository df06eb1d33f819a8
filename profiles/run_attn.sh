#!/bin/bash
# k_attend (bulk-copy + ldmatrix) check: parity tests, config-2 bench; single-slot diagnostics
OUT=gpurun_out; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_slots_gpu.py tests/test_parity_gpu.py tests/test_parity_configs_gpu.py -x -q > $OUT/tests_attn.log 2>&1; tail -3 $OUT/tests_attn.log
timeout 600 python bench.py --cpu-baseline 0 > $OUT/c2a.json 2> $OUT/c2a.err; tail -2 $OUT/c2a.err
python -c "
import json; d=json.load(open('$OUT/c2a.json')); print('c2', d['value'], d['ms_per_step'], 'att frac', d['roofline']['frac'], 'att ms', d['roofline']['ms_per_launch'], 'step frac', d['step_roofline']['frac'], 'sel', d['step_roofline']['select_ms'], 'e2e', d['e2e']['value'], 'parity', d['parity']['ok'], d['check'])"
for fl in 0 1; do timeout 300 python bench.py --config 1 --kv-heads 1 --l2-flush $fl --cpu-baseline 0 --parity 0 > $OUT/one_$fl.json 2>/dev/null; python -c "
import json; d=json.load(open('$OUT/one_$fl.json')); print('1-slot flush $fl', d['ms_per_step'], d['layerwise']['ms_per_step'], d['step_roofline']['select_ms'], d['step_roofline']['attend_ms'])"; done
LC_PROF=1 timeout 300 python tools/prof_step.py --steps 3 --layers 1 --kv-heads 1 --tokens 32768 2>&1 | tail -6
