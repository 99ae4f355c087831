#!/bin/bash
# Run short c$CFG benches under a list of environment settings; print realspace/total times.
# Usage: CFG=2 tools/sweep_env.sh "A=1 B=2" "A=0" ...
O=gpurun_out; mkdir -p $O
CFG=${CFG:-2}
for e in "$@"; do
  env $e python bench.py --config $CFG --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/sweep.log 2>&1
  python -c "
import json,sys
l=open('$O/sweep.log').read().strip().splitlines()[-1]
try:
  j=json.loads(l); s=j['stages_ms']; print('c$CFG $e', 'ms/step', round(j['ms_per_step'],2), 'rs', s['realspace_kernel'], 'spread', s['spread_kernel'], 'gather', s['gather(+terms)_kernel'])
except Exception as ex: print('$e FAILED', l[:300])
" | tee -a $O/sweep_summary.log
done
