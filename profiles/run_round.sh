#!/bin/bash
# End-of-round evidence in one GPU call: the GPU tests, the default bench line,
# the reference arm, the streaming (config 3) line, the ncu launch list and one
# `--set full` capture per decode-step kernel.
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests -q -m gpu > $OUT/tests_gpu.log 2>&1; tail -2 $OUT/tests_gpu.log
timeout 600 python bench.py > $OUT/bench_full.json 2> $OUT/bench_full.err; cat $OUT/bench_full.json
timeout 600 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err; cat $OUT/bench_ref.json
timeout 600 python bench.py --mode stream > $OUT/stream.json 2> $OUT/stream.err; cat $OUT/stream.json
timeout 1500 bash profiles/run_ncu.sh $OUT > /dev/null 2>&1
ls $OUT
