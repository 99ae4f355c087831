#!/bin/bash
# ncu --set full of the spread and gather tile kernels at the pinned c2 xi and
# at the B200-balanced xi (grid out of L2). Usage: tools/ncu_sg.sh TAG
set -u
TAG=${1:-sg}
O=gpurun_out
mkdir -p $O
for xi in 37 60; do
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --xi $xi > $O/plain_${TAG}_$xi.json 2>&1 || exit 1
  for k in gather_wide_mma spread_tile_mma_cached; do
    ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o $O/full_${TAG}_${k}_xi$xi -f \
      python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --xi $xi > $O/ncu_${TAG}_${k}_xi$xi.log 2>&1
  done
done
