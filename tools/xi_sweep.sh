mkdir -p gpurun_out
for xi in 37 45 52 60 70 80; do
  timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --xi $xi > gpurun_out/xi_$xi.json 2> gpurun_out/xi_$xi.err
  python -c "
import json; d=json.load(open('gpurun_out/xi_$xi.json'))
print('$xi', d['config']['M_ext'], d['config']['P'], round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['stages_ms'].items()}, d['parity_vs_fixture']['rel_rms_sampled'])
"
done
