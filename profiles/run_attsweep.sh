#!/bin/bash
# attention work-split knobs: LC_ATT_TAIL_DIV (every slot's tail = 1/x of its tokens
# goes to the claimed pool), LC_ATT_POOL (pool chunks per warp)
for cfg in "$@"; do
  t=${cfg%,*}; pl=${cfg#*,}
  LC_ATT_TAIL_DIV=$t LC_ATT_POOL=$pl timeout 200 python bench.py --steps 30 --warmup 3 --cpu-baseline 0 > gpurun_out/sw.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/sw.json'));print('tail 1/$t pool $pl', 'steps/s %.1f'%d['value'],'att_ms %.4f'%d['step_roofline']['attend_ms'], d['check']['ok'])"
done
