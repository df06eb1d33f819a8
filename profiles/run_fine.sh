#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
LC_NO_FUSED=1 timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_stream_gpu.py -x -q > $OUT/tests_fine_chain.log 2>&1; tail -2 $OUT/tests_fine_chain.log
timeout 900 python -m pytest tests/test_parity_configs_gpu.py -x -q > $OUT/tests_fine.log 2>&1; tail -2 $OUT/tests_fine.log
timeout 900 python bench.py --config 4 --steps 30 --cpu-baseline 0 > $OUT/f_c4.json 2>/dev/null; python -c "
import json; d=json.load(open('$OUT/f_c4.json')); print('c4', d['value'], d['ms_per_step'], d['step_roofline']['frac'], d['step_roofline']['select_ms'], d['parity']['ok'], d['check']['ok'])"
LC_NO_FUSED=1 timeout 300 python bench.py --cpu-baseline 0 --parity 1 > $OUT/f_c2chain.json 2>/dev/null; python -c "
import json; d=json.load(open('$OUT/f_c2chain.json')); print('c2 chain', d['value'], d['ms_per_step'], d['step_roofline']['frac'], d['step_roofline']['select_ms'], d['parity']['ok'])"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:'k_fine' -c 3 --csv --log-file $OUT/launches_fine.csv python bench.py --config 4 --steps 2 --warmup 3 --graph 0 --cpu-baseline 0 --parity 0 > /dev/null 2>&1
grep -E "gpu__time|dram__bytes" $OUT/launches_fine.csv | head -6
