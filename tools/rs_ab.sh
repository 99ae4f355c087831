# A/B timing of variant builds (see tools/README.md)
for c in 2 3; do
  python tools/sg_time.py $c 7 "" SPREAD_SORT=0
  SEWALD_LIB=paper_2210_01255_b200/lib/var_base/libsewald_gpu.so python tools/sg_time.py $c 7 ""
done
