set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "fused or jit or qft or hadamard" 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/bench_r01c.json 2> gpurun_out/bench_r01c.err; echo bench_rc=$?
tail -c 1500 gpurun_out/bench_r01c.json
python tools/prof_circ.py qft 32 2 > gpurun_out/pc_qft.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:qs_tile_jit -s 4 -c 1 -o gpurun_out/prof_qft_ladder python tools/prof_circ.py qft 32 2 > gpurun_out/ncu_qft.log 2>&1; echo ncu_qft=$?
python tools/prof_circ.py rqc 32 2 > gpurun_out/pc_rqc.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:qs_tile_jit -s 28 -c 1 -o gpurun_out/prof_rqc_tile python tools/prof_circ.py rqc 32 2 > gpurun_out/ncu_rqc.log 2>&1; echo ncu_rqc=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"qs_tile_jit|k_perm" --csv --log-file gpurun_out/launches_circ.csv python tools/prof_circ.py rqc 32 1 > gpurun_out/ncu_lc.log 2>&1; echo ncu_lc=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"qs_tile_jit|k_perm" --csv --log-file gpurun_out/launches_qft.csv python tools/prof_circ.py qft 32 1 > gpurun_out/ncu_lq.log 2>&1; echo ncu_lq=$?
ls -la gpurun_out
