OUT=gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'k_select|k_attend|k_merge' --csv --log-file $OUT/launches_r2.csv python bench.py --steps 3 --warmup 3 --graph 0 --cpu-baseline 0 --parity 0 > /dev/null 2>&1
python tools/launch_table.py $OUT/launches_r2.csv $OUT/launches_r2.md r02 && tail -3 $OUT/launches_r2.md
timeout 300 python bench.py --steps 30 --warmup 3 --cpu-baseline 0 > $OUT/fu_bench.json 2> $OUT/fu_bench.err; tail -3 $OUT/fu_bench.err
python -c "import json;d=json.load(open('$OUT/fu_bench.json'));print('steps/s',d['value'],'ms',d['ms_per_step'],'sel_ms',d['step_roofline']['select_ms'],'att_ms',d['step_roofline']['attend_ms'],'step_frac',d['step_roofline']['frac'],'e2e',d['e2e']['value'], 'launches', d['kernels_per_step']);print('parity',d['parity']['ok'], d['parity']['mismatches'][:5])"
