set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "permutation or qft or fused" 2>&1 | tail -5
CIRCS=qft LADDERS=4 PERMS=0,4,5,6 timeout 600 python tools/calib_circ.py 2>&1 | tail -8
