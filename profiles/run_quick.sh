#!/bin/bash
# tests + bench + per-kernel launch times (ncu) in one GPU call
OUT=gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -4
timeout 600 python bench.py --steps 30 --warmup 3 --cpu-baseline 0 > $OUT/bench_q.json 2> $OUT/bench_q.err; tail -3 $OUT/bench_q.err
python -c "import json;d=json.load(open('$OUT/bench_q.json'));print('steps/s',d['value'],'ms',d['ms_per_step'],'att_frac',d['roofline']['frac'],'sel_ms',d['step_roofline']['select_ms'],'att_ms',d['step_roofline']['attend_ms'],'step_frac',d['step_roofline']['frac'])"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:'k_attend|k_coarse|k_fine|k_pick|k_spans|k_select|k_graft|k_append' --csv --log-file $OUT/launches_q.csv python bench.py --steps 3 --warmup 3 --graph 0 --cpu-baseline 0 > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows=list(csv.reader(open('gpurun_out/launches_q.csv')))
hdr=None; data={}
for r in rows:
    if r and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r)); data.setdefault((d['ID'],d['Kernel Name'][:30]),{})[d['Metric Name']]=float(d['Metric Value'].replace(',',''))
agg=collections.defaultdict(list)
for (i,k),m in data.items(): agg[k].append(m)
for k,l in agg.items():
    print(k, len(l), 'us %.1f'%(sum(x['gpu__time_duration.sum'] for x in l)/len(l)/1e3), 'MB %.1f'%(sum(x['dram__bytes_read.sum'] for x in l)/len(l)/1e6))
PY
