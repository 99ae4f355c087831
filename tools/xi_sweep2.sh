mkdir -p gpurun_out
run() { # xi tag env...
  local xi=$1 tag=$2; shift 2
  env "$@" timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --xi $xi > gpurun_out/xs_$tag.json 2> gpurun_out/xs_$tag.err
  python -c "
import json; d=json.load(open('gpurun_out/xs_$tag.json')); st=d['stages_ms']
print('$tag', d['config']['M_ext'][0], round(d['ms_per_step'],2), 'rs', round(st['realspace_kernel'],2), 'sp', round(st['spread_kernel'],2), 'ga', round(st['gather(+terms)_kernel'],2), 'fft', round(st['fft+scale+ifft'],2), 'par', '%.1e' % d['parity_vs_fixture']['rel_rms_sampled'])
"
}
for xi in 56 59 63 66 71; do run $xi xi$xi SEWALD_X=0; done
for ppc in 16 20 40; do run 63 xi63_ppc$ppc SEWALD_RS_PPC=$ppc; done
