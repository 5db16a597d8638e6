for cfg in "TILE_B=12" "TILE_B=11" "TILE_B=11 QS_TILE_CTAS=4 QS_TILE_NBUF=1" "TILE_B=11 QS_TILE_CTAS=3 QS_TILE_NBUF=1" "TILE_B=10 QS_TILE_CTAS=4 QS_TILE_NBUF=1"; do
  echo "== $cfg"
  env $cfg AUTO=1 LOWS=4 LADDERS=4 CIRCS=rqc,qft timeout 400 python tools/calib_circ.py 2>&1 | tail -2
done
