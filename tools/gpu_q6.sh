for d in 8 6 3 2; do echo "== QS_TILE_DIRECT=$d"; QS_TILE_DIRECT=$d AUTO=1 LOWS=4 LADDERS=4 CIRCS=qft timeout 300 python tools/calib_circ.py 2>&1 | tail -1; done
