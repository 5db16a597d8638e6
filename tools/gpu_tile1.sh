timeout 900 python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -15
QS_TILE_MINB=2 timeout 600 python tools/calib_tile.py 2>&1 | tail -20
QS_TILE_MINB=1 TILES=12 timeout 600 python tools/calib_tile.py 2>&1 | tail -8
timeout 300 python tools/calib_pair.py
