#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
timeout 1500 python -m pytest tests -q -m gpu > $OUT/tests_q2.log 2>&1; tail -2 $OUT/tests_q2.log
for qc in 256 512 1024; do
  LC_ATT_QC=$qc timeout 300 python bench.py --cpu-baseline 0 --parity 0 > $OUT/qc_$qc.json 2>/dev/null; python -c "
import json; d=json.load(open('$OUT/qc_$qc.json')); print('qc $qc', d['value'], d['ms_per_step'], d['step_roofline']['frac'], 'e2e', d['e2e']['value'], 'lw', d['layerwise']['value'])"
done
timeout 300 python bench.py --cpu-baseline 0 --parity 1 > $OUT/qc_def.json 2>/dev/null; python -c "
import json; d=json.load(open('$OUT/qc_def.json')); print('default', d['value'], d['ms_per_step'], d['step_roofline']['frac'], 'e2e', d['e2e']['value'], 'lw', d['layerwise']['value'], d['parity']['ok'])"
timeout 300 python bench.py --config 1 --cpu-baseline 0 --parity 0 > $OUT/qc_c1.json 2>/dev/null; python -c "
import json; d=json.load(open('$OUT/qc_c1.json')); print('c1', d['value'], d['ms_per_step'])"
timeout 900 python bench.py --mode stream --cpu-baseline 0 > $OUT/qc_c3.json 2>/dev/null; python -c "
import json; d=json.load(open('$OUT/qc_c3.json')); print('c3', d['value'], d['ms_per_step'], d['check']['ok'])"
