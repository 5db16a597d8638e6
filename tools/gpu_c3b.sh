QS_TILE_C3=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "qft or rqc or jit or fused or tile" 2>&1 | tail -1
for c in 0 1; do echo "== QS_TILE_C3=$c"; QS_TILE_C3=$c AUTO=1 LOWS=4 LADDERS=4 CIRCS=rqc,qft timeout 400 python tools/calib_circ.py 2>&1 | tail -2; done
