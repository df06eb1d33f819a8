#!/bin/bash
# Config 3 cross-checks: eager (no graph) timing, and the ncu launch list of a
# few streaming steps (per-kernel duration and DRAM bytes), k_graft / k_append
# --set full captures.
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python bench.py --mode stream --graph 0 --steps 256 --cpu-baseline 0 > $OUT/stream_eager.json 2> $OUT/stream_eager.err; cat $OUT/stream_eager.json | python -c "import json,sys; d=json.load(sys.stdin); print('eager ms', d['ms_per_step'], d['value'])"
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'lc::' --csv --log-file $OUT/launches_stream.csv python bench.py --mode stream --graph 0 --steps 24 --warmup 3 --cpu-baseline 0 > $OUT/ncu_stream.log 2>&1
python tools/launch_table.py $OUT/launches_stream.csv $OUT/launches_stream.md r02-stream 'lc::k_(select|attend|merge|append|graft)'; 
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_graft' -s 1 -c 1 -o $OUT/prof_k_graft python bench.py --mode stream --graph 0 --steps 24 --warmup 3 --cpu-baseline 0 > $OUT/ncu_graft.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_append' -s 4 -c 1 -o $OUT/prof_k_append python bench.py --mode stream --graph 0 --steps 8 --warmup 3 --cpu-baseline 0 > $OUT/ncu_append.log 2>&1
ls $OUT
