#!/bin/bash
# Round-2 end-of-session evidence in one GPU call (all outputs under gpurun_out/final/)
OUT=gpurun_out/final; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv > $OUT/gpu.txt; lscpu | grep -E "Model name|^CPU\(s\)" > $OUT/cpu.txt
timeout 1500 python -m pytest tests -q -m gpu > $OUT/tests_gpu.log 2>&1; tail -2 $OUT/tests_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
timeout 900 python bench.py > $OUT/c2.json 2> $OUT/c2.err
timeout 900 python bench.py --impl reference > $OUT/c2_ref.json 2> $OUT/c2_ref.err
timeout 600 python bench.py --config 1 > $OUT/c1.json 2> $OUT/c1.err
timeout 1500 python bench.py --config 4 --steps 30 > $OUT/c4.json 2> $OUT/c4.err
timeout 900 python bench.py --config 5 --steps 20 > $OUT/c5.json 2> $OUT/c5.err
timeout 900 python bench.py --mode stream > $OUT/c3.json 2> $OUT/c3.err
for n in 32768 131072; do
  timeout 600 oracle/_ref/ref_dropin_bench $n 64 512 > $OUT/dropin_ref_$n.json 2>&1
  OMP_NUM_THREADS=1 timeout 600 oracle/_ref/ref_dropin_bench $n 64 512 > $OUT/dropin_ref1_$n.json 2>&1
  timeout 600 oracle/_ref/b200_dropin_bench $n 64 512 > $OUT/dropin_b200_$n.json 2>&1
done
BENCH="python bench.py --steps 3 --warmup 3 --graph 0 --cpu-baseline 0 --parity 0"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'k_select|k_attend|k_merge' --csv --log-file $OUT/launches_c2.csv $BENCH > /dev/null 2>&1
for k in k_select k_attend k_merge; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 5 -c 1 -o $OUT/prof_$k $BENCH > /dev/null 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'k_select|k_attend|k_merge|k_append|k_graft|k_compact' --csv --log-file $OUT/launches_c3.csv python bench.py --mode stream --graph 0 --steps 140 --warmup 3 --cpu-baseline 0 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_graft' -c 1 -o $OUT/prof_k_graft python bench.py --mode stream --graph 0 --steps 20 --warmup 3 --cpu-baseline 0 > /dev/null 2>&1
ls $OUT
