#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
timeout 300 python -m pytest tests/test_gather_gpu.py -x -q > $OUT/tests_gather.log 2>&1; tail -3 $OUT/tests_gather.log
timeout 1500 python -m pytest tests -q -m gpu > $OUT/tests_gpu_all.log 2>&1; tail -3 $OUT/tests_gpu_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; tail -2 $OUT/smoke.log
timeout 300 python bench.py --cpu-baseline 0 > $OUT/g_c2.json 2>/dev/null; python -c "
import json; d=json.load(open('$OUT/g_c2.json')); print('c2', d['value'], d['ms_per_step'], d['step_roofline']['frac'], d['roofline']['frac'], d['e2e']['value'], d['parity']['ok'], d['layerwise']['value'])"
