#!/bin/bash
# bench sweep over launch knobs (no cpu baseline); prints one summary line each
for cfg in "$@"; do
  timeout 300 python bench.py --steps 30 --warmup 3 --cpu-baseline 0 $cfg > gpurun_out/sw.json 2> gpurun_out/sw.err || tail -3 gpurun_out/sw.err
  python -c "import json,sys;d=json.load(open('gpurun_out/sw.json'));print('$cfg','steps/s %.1f'%d['value'],'ms %.4f'%d['ms_per_step'],'att_frac %.3f'%d['roofline']['frac'],'sel_ms %.4f'%d['step_roofline']['select_ms'],'att_ms %.4f'%d['step_roofline']['attend_ms'],'step_frac %.3f'%d['step_roofline']['frac'])"
done
