export CIRCS=rqc,qft LADDERS=4 PERMS=5 LOWS=4
TILE_B=11 QS_TILE_NBUF=1 QS_TILE_CTAS=4 timeout 300 python tools/calib_circ.py 2>&1 | tail -2
TILE_B=11 QS_TILE_NBUF=1 QS_TILE_CTAS=3 timeout 300 python tools/calib_circ.py 2>&1 | tail -2
TILE_B=11 QS_TILE_NBUF=2 QS_TILE_CTAS=2 timeout 300 python tools/calib_circ.py 2>&1 | tail -2
TILE_B=12 timeout 300 python tools/calib_circ.py 2>&1 | tail -2
