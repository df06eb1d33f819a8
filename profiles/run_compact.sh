#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_stream_gpu.py tests/test_parity_gpu.py -x -q > $OUT/tests_compact.log 2>&1; tail -3 $OUT/tests_compact.log
timeout 900 python bench.py --mode stream > $OUT/c3b.json 2> $OUT/c3b.err; tail -2 $OUT/c3b.err; python -c "
import json; d=json.load(open('$OUT/c3b.json')); print('c3', d['value'], d['ms_per_step'], d['roofline']['frac'], d['check']['ok'], d['grafts_applied_on_device'], d['cpu_baseline']['value'])"
timeout 900 python bench.py --config 5 --steps 20 > $OUT/c5b.json 2> $OUT/c5b.err; tail -2 $OUT/c5b.err; python -c "
import json; d=json.load(open('$OUT/c5b.json')); print('c5', d['value'], [ (p['batch'],p['context'],p['budget'],round(p['value']),p['parity']) for p in d['sweep'] if p['parity']])"
