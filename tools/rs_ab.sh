# A/B timing of variant builds (see tools/README.md)
python tools/sg_time.py 4 7 "" SPREAD_SORT=0
SEWALD_LIB=paper_2210_01255_b200/lib/var_base/libsewald_gpu.so python tools/sg_time.py 4 7 ""
python tools/sg_time.py 2 5 "" SPREAD_ROWSWEEP=1 SPREAD_ROWSWEEP=1,SPREAD_SORT=0
python -m pytest tests -m gpu -x -q -k "spread or gather or family or families or fullsize" 2>&1 | tail -2
