# A/B timing of variant builds (see tools/README.md)
for c in 4 1; do for v in var_nbt MAIN var_nbt MAIN; do
  if [ $v = MAIN ]; then L=paper_2210_01255_b200/lib/libsewald_gpu.so; else L=paper_2210_01255_b200/lib/$v/libsewald_gpu.so; fi
  echo "c$c $v $(SEWALD_LIB=$L timeout 300 python tools/rs_time.py $c 5 2>&1 | tail -1)"
done; done
