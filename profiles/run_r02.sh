#!/bin/bash
# Round-2 evidence in one GPU call: GPU tests, default bench line (with parity
# + cpu_baseline), reference arm, ncu launch list and `--set full` captures of
# the decode-step kernels (k_select, k_attend, k_merge, and the chain kernels
# still used where k_select does not fit).
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt
lscpu | head -20 > $OUT/cpu.txt
timeout 1200 python -m pytest tests -q -m gpu > $OUT/tests_gpu.log 2>&1; tail -5 $OUT/tests_gpu.log
timeout 600 python bench.py > $OUT/bench_full.json 2> $OUT/bench_full.err; cat $OUT/bench_full.json; tail -3 $OUT/bench_full.err
timeout 600 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err; cat $OUT/bench_ref.json
BENCH="python bench.py --steps 3 --warmup 3 --graph 0 --cpu-baseline 0 --parity 0"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file $OUT/launches_r02.csv $BENCH > $OUT/ncu_bench.log 2>&1
python tools/launch_table.py $OUT/launches_r02.csv $OUT/launches_r02.md r02 && tail -12 $OUT/launches_r02.md
for k in k_select k_attend k_merge; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 5 -c 1 -o $OUT/prof_$k $BENCH > $OUT/ncu_$k.log 2>&1
done
ls $OUT
