#!/bin/bash
# B200-balanced split parameter per BASELINE config (bench.py --config K --xi X)
mkdir -p gpurun_out
run() { # cfg xi
  timeout 600 python bench.py --config $1 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-balanced --xi $2 > gpurun_out/xb_$1_$2.json 2> gpurun_out/xb_$1_$2.err
  python -c "
import json; d=json.load(open('gpurun_out/xb_$1_$2.json')); st=d['stages_ms']; c=d['config']
print('c$1 xi=$2', c['M_ext'], c['P'], round(c['rc'],4), 'ms', round(d['ms_per_step'],2), 'rs', round(st['realspace_kernel'],2), 'sp', round(st['spread_kernel'],2), 'ga', round(st['gather(+terms)_kernel'],2), 'fft', round(st['fft+scale+ifft'],2), 'par', '%.1e' % d['parity_vs_fixture']['rel_rms_sampled'] if d.get('parity_vs_fixture') else None)
" 2>&1 | tail -1
}
for x in 33.5 40 47 54 61; do run 3 $x; done
for x in 34 40 46 52 58; do run 4 $x; done
for x in 50 60 68.5 78; do run 5 $x; done
