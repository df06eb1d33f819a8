#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:'k_fine' -s 1 -c 1 -o $OUT/prof_k_fine_c4 python bench.py --config 4 --steps 2 --warmup 3 --graph 0 --cpu-baseline 0 --parity 0 > $OUT/ncu_fine.log 2>&1
tail -3 $OUT/ncu_fine.log
