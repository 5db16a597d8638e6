set -x
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -6
CIRCS=rqc,qft LOWS=3,4 LADDERS=4 PERMS=5 timeout 600 python tools/calib_circ.py 2>&1 | tail -4
