#!/bin/bash
# Drop-in per-call path with one stream sync (lc_selection_stage / read_staged):
# parity + reference tests through the drop-in, per-call latency vs the reference.
OUT=gpurun_out/dropin; mkdir -p $OUT
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_dropin.py -x -q > $OUT/tests.log 2>&1; tail -2 $OUT/tests.log
for n in 32768 131072; do
  timeout 600 oracle/_ref/b200_dropin_bench $n 64 512 > $OUT/dropin_b200_$n.json 2>&1
  timeout 600 oracle/_ref/ref_dropin_bench $n 64 512 > $OUT/dropin_ref_$n.json 2>&1
  OMP_NUM_THREADS=1 timeout 600 oracle/_ref/ref_dropin_bench $n 64 512 > $OUT/dropin_ref1_$n.json 2>&1
done
TIERKV_DROPIN_PROF=1 timeout 600 oracle/_ref/b200_dropin_bench 131072 16 16 > $OUT/dropin_prof.json 2> $OUT/dropin_prof.err
tail -5 $OUT/dropin_prof.err
cat $OUT/dropin_*.json
