for cfg in "QS_TILE_R=4" "QS_TILE_R=3 QS_TILE_NBUF=2 QS_TILE_CTAS=1" "QS_TILE_R=3" "QS_TILE_R=3 QS_TILE_NBUF=1 QS_TILE_CTAS=2 QS_TILE_TPB=256"; do
  echo "== $cfg"
  env $cfg AUTO=1 LOWS=4 LADDERS=4 CIRCS=qft,rqc timeout 400 python tools/calib_circ.py 2>&1 | tail -2
done
