for c in 2 3 5; do echo "c$c $(timeout 300 python tools/rs_time.py $c 5 2>&1 | tail -1)"; done
