export CIRCS=rqc,qft LADDERS=4 PERMS=5 LOWS=4
for S in 0 3000 6000 10000; do QS_TILE_STAGGER_NS=$S timeout 300 python tools/calib_circ.py 2>&1 | tail -2 | sed "s/^/stagger=$S /"; done
