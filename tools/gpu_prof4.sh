export CASES=cz_x40 REPS=2
python tools/tile_micro.py > gpurun_out/p_cz.log 2>&1 && \
 ncu --set full --clock-control none --import-source on -k regex:k_tile -s 1 -c 1 -o gpurun_out/prof_cz40 python tools/tile_micro.py > gpurun_out/ncu_cz.log 2>&1
echo done
