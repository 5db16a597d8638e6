set -x
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
CIRCS=rqc,qft LADDERS=4 PERMS=5 LOWS=4 timeout 600 python tools/calib_circ.py 2>&1 | tail -2
python tools/prof_circ.py rqc 32 2 > gpurun_out/pc_rqc4.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:qs_tile_jit -s 25 -c 1 -o gpurun_out/prof_rqc_tile4 python tools/prof_circ.py rqc 32 2 > gpurun_out/ncu_rqc4.log 2>&1; echo ncu_rqc=$?
