#!/bin/bash
# Full bench line (both arms) + ncu launch list + ncu --set full captures of the
# top kernels of the c2 step. Each ncu pass runs only after the same command
# exited 0 without ncu. Usage: tools/gpu_profile.sh TAG
set -u
TAG=${1:-prof}
O=gpurun_out
mkdir -p $O
python bench.py > $O/bench_$TAG.json 2> $O/bench_$TAG.err || { echo "bench failed"; exit 1; }
python bench.py --impl reference --steps 2 --warmup 1 > $O/ref_$TAG.json 2> $O/ref_$TAG.err || echo "reference arm failed"
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/plain_$TAG.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_$TAG.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_launch_$TAG.log 2>&1
for k in realspace_sym spread_tile_mma gather_tile_mma; do
  ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o $O/full_${TAG}_$k -f \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_full_${TAG}_$k.log 2>&1
done
