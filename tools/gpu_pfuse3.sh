# ncu --set full of the fused reversal pass (QFT(32), tile_low 3)
ncu --set full --clock-control none --import-source on -k regex:qs_tile_jit -s 3 -c 1 -o gpurun_out/pf_fused -f python tools/prof_circ.py qft 32 1 tile_low=3,tile_low_auto=0,perm_fuse=1 > gpurun_out/pf3.log 2>&1
tail -3 gpurun_out/pf3.log
python tools/ncu_summary.py gpurun_out/pf_fused.ncu-rep "fused reversal pass" > gpurun_out/pf_fused.txt 2>&1; cat gpurun_out/pf_fused.txt
