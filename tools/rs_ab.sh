# A/B timing of variant builds (see tools/README.md)
for v in MAIN var_c128 MAIN var_c128; do
  if [ $v = MAIN ]; then L=paper_2210_01255_b200/lib/libsewald_gpu.so; else L=paper_2210_01255_b200/lib/$v/libsewald_gpu.so; fi
  echo "c4 $v $(SEWALD_LIB=$L timeout 300 python tools/rs_time.py 4 5 2>&1 | tail -1)"
done
