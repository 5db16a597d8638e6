for t in 8 48; do echo "== QS_PLAN_TRIALS=$t"; QS_PLAN_TRIALS=$t AUTO=1 LOWS=4 LADDERS=4 CIRCS=rqc timeout 300 python tools/calib_circ.py 2>&1 | tail -1; done
