#!/bin/bash
# Stage breakdown of every config, then fp64 op counters of all six real-space variants.
set -u
TAG=${1:-p2}
O=gpurun_out
mkdir -p $O
for c in 3 4 5; do
  python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_${TAG}_c$c.log 2>&1 || exit 1
done
python tools/rs_flops.py > $O/rsf_${TAG}_plain.log 2>&1 || exit 1
ncu --clock-control none -k regex:realspace --metrics \
gpu__time_duration.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active \
  --csv --log-file $O/rsf_${TAG}.csv python tools/rs_flops.py > $O/rsf_${TAG}.log 2>&1
