set -x
timeout 1500 python -m pytest tests/test_gpu_ladder.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py -m gpu -x -q 2>&1 | tail -15
CIRCS=rqc,qft LADDERS=4 PERMS=5 timeout 600 python tools/calib_circ.py 2>&1 | tail -4
