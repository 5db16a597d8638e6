export CIRCS=rqc,qft LADDERS=4 PERMS=5 LOWS=4
QS_TILE_NBUF=1 QS_TILE_CTAS=2 QS_TILE_TPB=128 timeout 300 python tools/calib_circ.py 2>&1 | tail -2
QS_TILE_NBUF=1 QS_TILE_CTAS=3 QS_TILE_TPB=128 timeout 300 python tools/calib_circ.py 2>&1 | tail -2
QS_TILE_NBUF=1 QS_TILE_CTAS=3 QS_TILE_TPB=256 timeout 300 python tools/calib_circ.py 2>&1 | tail -2
QS_TILE_NBUF=2 QS_TILE_CTAS=1 timeout 300 python tools/calib_circ.py 2>&1 | tail -2
