AUTO=0 LOWS=3,4 LADDERS=4 PFUSE=0,1 CIRCS=qft timeout 600 python tools/calib_circ.py
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/pf_4.csv python tools/prof_circ.py qft 32 1 tile_low=3,tile_low_auto=0,perm_fuse=1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/pf_4.csv "tile_low 3 fused"
