timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "qft or rqc or jit or fused or tile" 2>&1 | tail -1
for cfg in "TILE_B=12" "TILE_B=12 QS_TILE_CTAS=3 QS_TILE_NBUF=1 QS_TILE_TPB=128" "TILE_B=12 QS_TILE_CTAS=3 QS_TILE_NBUF=1 QS_TILE_TPB=64"; do
  echo "== $cfg"
  env $cfg AUTO=1 LOWS=4 LADDERS=4 CIRCS=rqc,qft timeout 400 python tools/calib_circ.py 2>&1 | tail -2
done
