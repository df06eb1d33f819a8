OUT=gpurun_out
export LC_FUSED_DEBUG=1
timeout 600 python -m pytest tests -q -m gpu -x -k "parity or dropin" > $OUT/fu_tests.log 2>&1; tail -30 $OUT/fu_tests.log | grep -E "passed|failed|Error|assert" | head -20
LC_PROF=1 timeout 300 python tools/prof_step.py --steps 2 2>&1 | grep -E "k_select" | tail -3
timeout 300 python bench.py --steps 30 --warmup 3 --cpu-baseline 0 > $OUT/fu_bench.json 2> $OUT/fu_bench.err; tail -3 $OUT/fu_bench.err
python -c "import json;d=json.load(open('$OUT/fu_bench.json'));print('steps/s',d['value'],'ms',d['ms_per_step'],'sel_ms',d['step_roofline']['select_ms'],'att_ms',d['step_roofline']['attend_ms'],'step_frac',d['step_roofline']['frac']);print('parity',d['parity']['ok'], d['parity']['mismatches'][:5])"
