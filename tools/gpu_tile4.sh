timeout 900 python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -5
QS_TILE_R=3 timeout 900 python -m pytest tests/test_gpu_parity.py -m "gpu and not slow" -x -q -k "fused or config1 or qft or rqc or sharded" 2>&1 | tail -3
TILES=12 timeout 600 python tools/calib_tile.py 2>&1 | tail -6
QS_TILE_R=3 TILES=12 timeout 600 python tools/calib_tile.py 2>&1 | tail -6
timeout 300 python tools/calib.py
