CIRCS=rqc,qft LADDERS=4 PERMS=5 LOWS=4 timeout 600 python tools/calib_circ.py 2>&1 | tail -2
python tools/prof_circ.py qft 32 2 > gpurun_out/pc_qft6.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:qs_tile_jit -s 4 -c 1 -o gpurun_out/prof_qft_ladder6 python tools/prof_circ.py qft 32 2 > gpurun_out/ncu_qft6.log 2>&1; echo ncu_qft=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_perm -s 1 -c 1 -o gpurun_out/prof_perm6 python tools/prof_circ.py qft 32 2 > gpurun_out/ncu_perm6.log 2>&1; echo ncu_perm=$?
