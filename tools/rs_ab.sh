for v in MAIN var_yc1 var_yc4; do
  if [ $v = MAIN ]; then L=paper_2210_01255_b200/lib/libsewald_gpu.so; else L=paper_2210_01255_b200/lib/$v/libsewald_gpu.so; fi
  echo "$v $(SEWALD_LIB=$L SEWALD_D0_YFUSED=1 python bench.py --config 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['stages_ms']['fft+scale+ifft'], d['parity_vs_fixture']['rel_rms_sampled'])")"
done
