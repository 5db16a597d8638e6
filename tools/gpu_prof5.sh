export CASES=h1_x40 REPS=2
python tools/tile_micro.py > gpurun_out/p_h1.log 2>&1 && \
 ncu --set full --clock-control none --import-source on -k regex:qs_tile_jit -s 1 -c 1 -o gpurun_out/prof_jit_h1 python tools/tile_micro.py > gpurun_out/ncu_h1.log 2>&1
echo done
