timeout 600 python tools/tile_micro.py 2>&1 | tail -8
QS_TILE_R=3 timeout 600 python tools/tile_micro.py 2>&1 | tail -8
