set -x
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
CIRCS=rqc,qft LADDERS=4 PERMS=5 timeout 600 python tools/calib_circ.py 2>&1 | tail -4
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"qs_tile_jit|k_perm" --csv --log-file gpurun_out/launches_qft2.csv python tools/prof_circ.py qft 32 1 > gpurun_out/ncu_lq2.log 2>&1; echo ncu_lq=$?
