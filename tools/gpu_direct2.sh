timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ladder.py -x -q -k "qft or rqc or jit or fused or ladder or tile" 2>&1 | tail -1
AUTO=1 LOWS=4 LADDERS=4 CIRCS=qft,rqc timeout 300 python tools/calib_circ.py 2>&1 | tail -2
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --metrics $M --clock-control none -k regex:"qs_tile_jit|k_perm" --csv --log-file gpurun_out/s3_launches_qft.csv python tools/prof_circ.py qft 32 1 > /dev/null 2>&1; echo lq=$?
python tools/launch_summary.py gpurun_out/s3_launches_qft.csv "QFT(32)|x>, session 3"
