#!/bin/bash
# Config 3 evidence: stream GPU tests, the streaming bench line (one CUDA graph
# of 4096 decode steps), ncu of k_graft / k_append.
OUT=gpurun_out; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_stream_gpu.py -x -q > $OUT/tests_stream.log 2>&1; tail -15 $OUT/tests_stream.log
timeout 900 python bench.py --mode stream > $OUT/stream.json 2> $OUT/stream.err; cat $OUT/stream.json; tail -5 $OUT/stream.err
