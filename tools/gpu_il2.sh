for cfg in "QS_TILE_DYN=1" "QS_TILE_IL=1" ; do
  echo "== $cfg"
  env $cfg AUTO=1 LOWS=4 LADDERS=4 CIRCS=qft,rqc timeout 300 python tools/calib_circ.py 2>&1 | tail -2
done
