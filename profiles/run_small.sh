#!/bin/bash
# few-slot launches: active-warp cap in k_attend, k_select L2 prefetch depth; k_graft rewrite
OUT=gpurun_out; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_slots_gpu.py tests/test_parity_gpu.py tests/test_stream_gpu.py tests/test_parity_configs_gpu.py -x -q > $OUT/tests_small.log 2>&1; tail -3 $OUT/tests_small.log
s() { python -c "
import json,sys; d=json.load(open(sys.argv[1])); print(sys.argv[2], round(d['value'],1), 'ms', round(d['ms_per_step'],4), 'sel', round(d['step_roofline']['select_ms'],4), 'att', round(d['step_roofline']['attend_ms'],4), 'frac', round(d['step_roofline']['frac'],3), 'lw', round(d['layerwise']['value'],1))" $1 "$2"; }
timeout 300 python bench.py --cpu-baseline 0 --parity 0 > $OUT/s_c2.json 2>/dev/null; s $OUT/s_c2.json c2
timeout 300 python bench.py --config 1 --cpu-baseline 0 --parity 0 > $OUT/s_c1.json 2>/dev/null; s $OUT/s_c1.json c1
timeout 300 python bench.py --config 1 --kv-heads 1 --cpu-baseline 0 --parity 0 > $OUT/s_1.json 2>/dev/null; s $OUT/s_1.json one-slot
for pf in 0 2 4 8; do LC_FUSED_PF=$pf timeout 300 python bench.py --kv-heads 1 --cpu-baseline 0 --parity 0 > $OUT/s_32_$pf.json 2>/dev/null; s $OUT/s_32_$pf.json "32slots pf$pf"; done
for pf in 2 4; do LC_FUSED_PF=$pf timeout 300 python bench.py --cpu-baseline 0 --parity 0 > $OUT/s_c2_$pf.json 2>/dev/null; s $OUT/s_c2_$pf.json "c2 pf$pf"; done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'k_graft|k_append' --csv --log-file $OUT/launches_graft.csv python bench.py --mode stream --graph 0 --steps 30 --warmup 3 --cpu-baseline 0 > /dev/null 2>&1
python tools/launch_table.py $OUT/launches_graft.csv $OUT/launches_graft.md graft 'k_(append|graft)' | tail -3
