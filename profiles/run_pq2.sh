#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
LC_NO_FUSED=1 timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_stream_gpu.py -x -q > $OUT/tests_pq2_chain.log 2>&1; tail -2 $OUT/tests_pq2_chain.log
timeout 900 python -m pytest tests/test_parity_configs_gpu.py -x -q > $OUT/tests_pq2.log 2>&1; tail -2 $OUT/tests_pq2.log
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:'k_fine|k_pickq|k_spans' -s 3 -c 3 -o $OUT/prof_c4_chain python bench.py --config 4 --steps 2 --warmup 3 --graph 0 --cpu-baseline 0 --parity 0 > $OUT/ncu_c4chain.log 2>&1; tail -2 $OUT/ncu_c4chain.log
