for v in 0 1 2 3 4 5; do QS_PAIR_VARIANT=$v timeout 300 python tools/calib_pair.py 2>&1 | tail -2; done
