timeout 900 python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -15
timeout 600 python tools/tile_micro.py 2>&1 | tail -8
TILES=12 timeout 600 python tools/calib_tile.py 2>&1 | tail -6
