#!/bin/bash
# Run on the GPU box (gpurun): launch list of our decode-step kernels and one
# `--set full` capture of each, for the bench's config-2 workload.
set -x
OUT=${1:-gpurun_out}
mkdir -p $OUT
BENCH="python bench.py --steps 3 --warmup 3 --graph 0 --cpu-baseline 0"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:'k_select|k_compact|k_attend' --csv --log-file $OUT/launches.csv $BENCH > $OUT/ncu_bench.log 2>&1
for k in k_select k_compact k_attend; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 4 -c 1 -o $OUT/prof_$k $BENCH > $OUT/ncu_$k.log 2>&1
done
ls -la $OUT
