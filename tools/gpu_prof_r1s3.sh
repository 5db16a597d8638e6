# session-3 circuit profiles: ncu --set full of an RQC(32) pass and a QFT(32) ladder pass; launch lists
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
python tools/prof_circ.py rqc 32 1 > /dev/null 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:qs_tile_jit -s 19 -c 1 -o gpurun_out/s3_rqc_pass -f python tools/prof_circ.py rqc 32 2 > gpurun_out/s3_ncu_rqc.log 2>&1; echo ncu_rqc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qs_tile_jit -s 5 -c 1 -o gpurun_out/s3_qft_pass -f python tools/prof_circ.py qft 32 2 > gpurun_out/s3_ncu_qft.log 2>&1; echo ncu_qft=$?
timeout 900 ncu --metrics $M --clock-control none -k regex:"qs_tile_jit|k_perm" --csv --log-file gpurun_out/s3_launches_rqc.csv python tools/prof_circ.py rqc 32 1 > /dev/null 2>&1; echo lr=$?
timeout 900 ncu --metrics $M --clock-control none -k regex:"qs_tile_jit|k_perm" --csv --log-file gpurun_out/s3_launches_qft.csv python tools/prof_circ.py qft 32 1 > /dev/null 2>&1; echo lq=$?
python tools/ncu_summary.py gpurun_out/s3_rqc_pass.ncu-rep "grid RQC(32) tile pass (session 3: dynamic tiles, pipelined gather, direct HBM stores)" "ncu --set full --clock-control none --import-source on -k regex:qs_tile_jit -s 19 -c 1 python tools/prof_circ.py rqc 32 2" > gpurun_out/s3_rqc_pass.txt
python tools/ncu_summary.py gpurun_out/s3_qft_pass.ncu-rep "QFT(32) phase-ladder tile pass (session 3: dynamic tiles, direct HBM loads and stores)" "ncu --set full --clock-control none --import-source on -k regex:qs_tile_jit -s 5 -c 1 python tools/prof_circ.py qft 32 2" > gpurun_out/s3_qft_pass.txt
python tools/launch_summary.py gpurun_out/s3_launches_rqc.csv "grid RQC(32), session 3" > gpurun_out/s3_launches_rqc.txt
python tools/launch_summary.py gpurun_out/s3_launches_qft.csv "QFT(32)|x>, session 3" > gpurun_out/s3_launches_qft.txt
cat gpurun_out/s3_rqc_pass.txt gpurun_out/s3_qft_pass.txt; tail -3 gpurun_out/s3_launches_rqc.txt; cat gpurun_out/s3_launches_qft.txt
