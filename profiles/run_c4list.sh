#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'k_coarse|k_fine|k_pickq|k_spans|k_attend|k_merge' --csv --log-file $OUT/launches_c4.csv python bench.py --config 4 --steps 2 --warmup 3 --graph 0 --cpu-baseline 0 --parity 0 > /dev/null 2>&1
python tools/launch_table.py $OUT/launches_c4.csv $OUT/launches_c4.md config4 'k_(coarse|fine|pickq|spans|attend|merge)' 29 | tail -7
