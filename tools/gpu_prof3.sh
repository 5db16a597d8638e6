export TILE_B=12 QS_TILE_R=4
python tools/prof_gate.py tile 30 2 11 > gpurun_out/p_tile.log 2>&1 && \
 ncu --set full --clock-control none --import-source on -k regex:k_tile -s 1 -c 1 -o gpurun_out/prof_tile_r4 python tools/prof_gate.py tile 30 2 11 > gpurun_out/ncu_tile.log 2>&1
echo done
