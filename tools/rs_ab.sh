git_base=paper_2210_01255_b200/lib/var_base/libsewald_gpu.so
for c in 2 3 4; do python tools/sg_time.py $c 5 ""; SEWALD_LIB=$git_base python tools/sg_time.py $c 5 ""; done
