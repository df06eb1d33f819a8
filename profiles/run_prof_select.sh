#!/bin/bash
# phase timers (LC_PROF) and one `--set full` capture each of the selection kernels
OUT=gpurun_out
LC_PROF=1 timeout 300 python bench.py --steps 3 --warmup 3 --graph 0 --cpu-baseline 0 2>&1 >/dev/null | grep LC_PROF | tail -3
BENCH="python bench.py --steps 3 --warmup 3 --graph 0 --cpu-baseline 0"
for k in ${KS:-k_pickq k_spans k_coarse}; do
  timeout 400 ncu --set full --clock-control none --import-source on -k regex:$k -s 5 -c 1 -o $OUT/prof_$k -f $BENCH > $OUT/ncu_$k.log 2>&1
done
