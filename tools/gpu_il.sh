timeout 900 python -m pytest tests/test_gpu_parity.py -m "gpu and not slow" -x -q 2>&1 | tail -3
TILES=12 timeout 600 python tools/calib_tile.py 2>&1 | tail -5
timeout 600 python tools/tile_micro.py 2>&1 | tail -6
QS_TILE_IL=0 TILES=12 timeout 600 python tools/calib_tile.py 2>&1 | tail -5
