for cfg in "12 2 1" "12 3 1" "11 2 2" "11 3 2"; do set -- $cfg
  echo "== b=$1 nbuf=$2 ctas=$3"
  QS_TILE_NBUF=$2 QS_TILE_CTAS=$3 TILES=$1 timeout 600 python tools/calib_tile.py 2>&1 | tail -5
done
