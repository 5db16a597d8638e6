timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "perm or qft" 2>&1 | tail -1
for d in 0 1; do echo "== QS_PERM_DYN=$d"; QS_PERM_DYN=$d timeout 300 python tools/perm_probe.py 2>&1 | grep '"with_H_fused": 0' | grep -v near; QS_PERM_DYN=$d AUTO=1 LOWS=4 LADDERS=4 CIRCS=qft timeout 300 python tools/calib_circ.py 2>&1 | tail -1; done
