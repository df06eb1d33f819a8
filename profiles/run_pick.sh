#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
LC_NO_FUSED=1 timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_stream_gpu.py -x -q > $OUT/tests_pick_chain.log 2>&1; tail -2 $OUT/tests_pick_chain.log
timeout 900 python -m pytest tests/test_parity_configs_gpu.py tests/test_parity_gpu.py -x -q > $OUT/tests_pick.log 2>&1; tail -2 $OUT/tests_pick.log
timeout 900 python bench.py --config 4 --steps 30 --cpu-baseline 0 > $OUT/p_c4.json 2>/dev/null; python -c "
import json; d=json.load(open('$OUT/p_c4.json')); print('c4', d['value'], d['ms_per_step'], d['step_roofline']['frac'], d['step_roofline']['select_ms'], d['parity']['ok'], d['check']['ok'])"
LC_NO_FUSED=1 timeout 300 python bench.py --cpu-baseline 0 --parity 1 > $OUT/p_c2chain.json 2>/dev/null; python -c "
import json; d=json.load(open('$OUT/p_c2chain.json')); print('c2 chain', d['value'], d['ms_per_step'], d['step_roofline']['frac'], d['step_roofline']['select_ms'], d['parity']['ok'])"
