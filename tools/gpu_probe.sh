#!/bin/bash
# One GPU session: CUDA parity suite, c2 bench, then (after those exit 0)
# ncu fp64 instruction counters of the real-space kernels of every config.
# Usage: tools/gpu_probe.sh TAG
set -u
TAG=${1:-probe}
O=gpurun_out
mkdir -p $O
python -m pytest tests -m gpu -x -q > $O/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> $O/pytest_$TAG.log
python bench.py --steps 5 --warmup 3 > $O/bench_$TAG.log 2>&1 || exit 1
for c in 2 3 4 5; do
  ncu --clock-control none -k regex:realspace --metrics \
gpu__time_duration.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active \
    --csv --log-file $O/flops_${TAG}_c$c.csv python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --no-e2e \
    > $O/ncu_${TAG}_c$c.log 2>&1
done
