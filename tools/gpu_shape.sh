# tile-pass pipeline shapes on a memory-only pass (5 in-tile SWAPs) and on QFT(32)
for cfg in "" "QS_TILE_NBUF=2 QS_TILE_CTAS=1" "QS_TILE_NBUF=3 QS_TILE_CTAS=1" "QS_TILE_NBUF=3 QS_TILE_CTAS=2 TILE_B=11" "QS_TILE_NBUF=1 QS_TILE_CTAS=2 TILE_B=11" "QS_TILE_NBUF=2 QS_TILE_CTAS=2 TILE_B=11"; do
  echo "== $cfg"
  env $cfg timeout 300 python tools/perm_probe.py 2>&1 | grep near | head -1
  env $cfg AUTO=1 LOWS=4 LADDERS=4 CIRCS=qft timeout 300 python tools/calib_circ.py 2>&1 | tail -1
done
