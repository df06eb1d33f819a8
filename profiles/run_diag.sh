OUT=gpurun_out; mkdir -p $OUT
export LC_FUSED_DEBUG=1
LC_PROF=1 timeout 300 python tools/prof_step.py --steps 3 > $OUT/d_prof_c2.log 2>&1
LC_PROF=1 timeout 300 python tools/prof_step.py --steps 3 --kv-heads 1 > $OUT/d_prof_c2_32.log 2>&1
timeout 300 python bench.py --kv-heads 1 --steps 30 --cpu-baseline 0 --parity 0 > $OUT/d_b32.json 2> $OUT/d_b32.err
timeout 600 python bench.py --tokens 1048576 --layers 4 --steps 20 --cpu-baseline 0 --parity 0 > $OUT/d_b1m.json 2> $OUT/d_b1m.err
LC_PROF=1 timeout 600 python tools/prof_step.py --steps 3 --tokens 1048576 --layers 4 > $OUT/d_prof_1m.log 2>&1
tail -n 30 $OUT/d_prof_c2.log $OUT/d_prof_c2_32.log $OUT/d_prof_1m.log $OUT/d_b1m.err $OUT/d_b32.err
python -c "
import json
for f in ['d_b32.json','d_b1m.json']:
    try:
        d=json.load(open('$OUT/'+f)); print(f, d['value'], d['ms_per_step'], d['step_roofline']['frac'], d['step_roofline']['select_ms'], d['step_roofline']['attend_ms'], d['roofline']['frac'], d['kernels_per_step'])
    except Exception as e: print(f, e)
"
