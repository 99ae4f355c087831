#!/bin/bash
# Algorithmic fp64 flops per accepted pair: ncu op counters of the branchy
# real-space variant (idle lanes do not execute), all six kernel variants.
# Build it first: mkdir -p build/branchy/obj && make -C paper_2210_01255_b200/csrc \
#   OUT=$PWD/build/branchy OBJ=$PWD/build/branchy/obj NVEXTRA=-DSEWALD_SYM_BRANCHFREE=0
set -u
TAG=${1:-p3}
O=gpurun_out
SEWALD_LIB=build/branchy/libsewald_gpu.so python tools/rs_flops.py > $O/rsf_${TAG}_plain.log 2>&1 || exit 1
SEWALD_LIB=build/branchy/libsewald_gpu.so ncu --clock-control none -k regex:realspace --metrics \
gpu__time_duration.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active \
  --csv --log-file $O/rsf_${TAG}.csv python tools/rs_flops.py > $O/rsf_${TAG}.log 2>&1
python tools/rs_flops.py > $O/rsf_${TAG}_bf_plain.log 2>&1
