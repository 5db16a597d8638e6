# launch lists: QFT(32) at tile_low 3 fused / unfused and tile_low 4
set -x
python tools/prof_circ.py qft 32 1 tile_low=3,tile_low_auto=0,perm_fuse=1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
i=0
for cfg in tile_low=3,tile_low_auto=0,perm_fuse=1 tile_low=3,tile_low_auto=0,perm_fuse=0 tile_low=4,tile_low_auto=0,perm_fuse=0; do
  i=$((i+1))
  ncu --metrics $M --clock-control none --csv --log-file gpurun_out/pf_$i.csv python tools/prof_circ.py qft 32 1 $cfg > /dev/null 2>&1
  python tools/launch_summary.py gpurun_out/pf_$i.csv "$cfg"
done
