timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "permutation or qft" 2>&1 | tail -2
CIRCS=qft LADDERS=4 PERMS=5 LOWS=4 timeout 600 python tools/calib_circ.py 2>&1 | tail -1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"qs_tile_jit|k_perm" --csv --log-file gpurun_out/launches_qft7.csv python tools/prof_circ.py qft 32 1 > gpurun_out/ncu_lq7.log 2>&1; echo ncu_lq=$?
