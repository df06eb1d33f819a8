#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
for kv in 8 1; do echo "== kv-heads $kv"; LC_PROF=1 timeout 300 python tools/prof_step.py --steps 2 --kv-heads $kv 2>&1 | grep LC_PROF | tail -4; done
echo "== one layer 32K"; LC_PROF=1 timeout 300 python tools/prof_step.py --steps 2 --config 1 2>&1 | grep LC_PROF | tail -4
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_select|k_attend|k_merge' --csv --log-file $OUT/launches_32.csv python bench.py --kv-heads 1 --steps 3 --warmup 3 --graph 0 --cpu-baseline 0 --parity 0 > /dev/null 2>&1
python tools/launch_table.py $OUT/launches_32.csv $OUT/launches_32.md 32slots 'k_(select|attend|merge)' | tail -4
