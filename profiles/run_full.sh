#!/bin/bash
# one ncu --set full capture per named kernel (args: kernel regexes)
OUT=gpurun_out
BENCH="python bench.py --steps 3 --warmup 3 --graph 0 --cpu-baseline 0"
for k in "$@"; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 4 -c 1 -o $OUT/prof_$k $BENCH > $OUT/ncu_$k.log 2>&1
  tail -2 $OUT/ncu_$k.log
done
