for c in 2 3; do python tools/sg_time.py $c 7 ""; done
