export TILE_B=12
python tools/prof_gate.py tile 30 2 11 > gpurun_out/p_tile.log 2>&1 && \
 ncu --set full --clock-control none --import-source on -k regex:k_tile -s 1 -c 1 -o gpurun_out/prof_tile11 python tools/prof_gate.py tile 30 2 11 > gpurun_out/ncu_tile.log 2>&1
python tools/prof_gate.py qft 30 1 > gpurun_out/p_qft.log 2>&1 && \
 ncu --set full --clock-control none --import-source on -k regex:k_tile -s 0 -c 1 -o gpurun_out/prof_qft python tools/prof_gate.py qft 30 1 > gpurun_out/ncu_qft.log 2>&1
tail -3 gpurun_out/ncu_tile.log gpurun_out/ncu_qft.log
