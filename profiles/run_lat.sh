#!/bin/bash
# latency experiments: k_select span writer, k_attend min tokens per warp (few-slot launches)
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_slots_gpu.py tests/test_parity_gpu.py tests/test_parity_configs_gpu.py -x -q > $OUT/tests_lat.log 2>&1; tail -2 $OUT/tests_lat.log
s() { python -c "
import json,sys; d=json.load(open(sys.argv[1])); print(sys.argv[2], round(d['value'],1), 'ms', round(d['ms_per_step'],4), 'sel', round(d['step_roofline']['select_ms'],4), 'att', round(d['step_roofline']['attend_ms'],4), 'frac', round(d['step_roofline']['frac'],3), 'lw', round(d['layerwise']['value'],1))" $1 "$2"; }
timeout 300 python bench.py --cpu-baseline 0 --parity 0 > $OUT/l_c2.json 2>/dev/null; s $OUT/l_c2.json c2
for mt in 64 128 256 512; do LC_ATT_MINTOK=$mt timeout 300 python bench.py --kv-heads 1 --cpu-baseline 0 --parity 0 > $OUT/l_32_$mt.json 2>/dev/null; s $OUT/l_32_$mt.json "32slots mintok$mt"; done
for mt in 128 512; do LC_ATT_MINTOK=$mt timeout 300 python bench.py --config 1 --cpu-baseline 0 --parity 0 > $OUT/l_c1_$mt.json 2>/dev/null; s $OUT/l_c1_$mt.json "c1 mintok$mt"; done
LC_PROF=1 timeout 300 python tools/prof_step.py --steps 2 2>&1 | grep "k_select" | tail -2
LC_PROF=1 timeout 300 python tools/prof_step.py --steps 2 --kv-heads 1 2>&1 | tail -4
