#!/bin/bash
# Run on the GPU box (gpurun): launch list of the decode-step kernels of the
# config-2 bench and one `--set full` capture of each.
OUT=${1:-gpurun_out}
mkdir -p $OUT
BENCH="python bench.py --steps 3 --warmup 3 --graph 0 --cpu-baseline 0"
KS='k_coarse|k_fine|k_pickq|k_spans|k_attend|k_graft|k_append'
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"$KS" --csv --log-file $OUT/launches.csv $BENCH > $OUT/ncu_bench.log 2>&1
for k in k_coarse k_fine k_pickq k_spans k_attend; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 5 -c 1 -o $OUT/prof_$k $BENCH > $OUT/ncu_$k.log 2>&1
done
ls $OUT
