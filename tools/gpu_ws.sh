export QS_TILE_WS=1
timeout 300 python -m pytest tests/test_gpu_ladder.py tests/test_gpu_parity.py -m gpu -x -q -k "ladder or fused or qft or rqc or jit" 2>&1 | tail -4
echo "---calib"
CIRCS=rqc,qft LADDERS=4 PERMS=5 LOWS=4 timeout 300 python tools/calib_circ.py 2>&1 | tail -2
