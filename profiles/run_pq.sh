#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
L=paper_2603_08453_b200/liblychee_b200.so
for v in pq512 pq256; do cp exp/lib_$v.so $L; timeout 900 python bench.py --config 4 --steps 30 --cpu-baseline 0 --parity 0 > $OUT/pq_$v.json 2>/dev/null; python -c "
import json; d=json.load(open('$OUT/pq_$v.json')); print('$v', d['value'], d['ms_per_step'], d['step_roofline']['frac'], d['step_roofline']['select_ms'])"; done
