set -x
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -6
timeout 900 python bench.py > gpurun_out/bench_r01e.json 2> gpurun_out/bench_r01e.err; echo bench_rc=$?
python -c "import json; d=json.loads(open('gpurun_out/bench_r01e.json').read().strip().splitlines()[-1]); print(d['value'], d['circuits'])"
python tools/prof_circ.py rqc 32 2 > gpurun_out/pc_rqc.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:qs_tile_jit -s 25 -c 1 -o gpurun_out/prof_rqc_tile2 python tools/prof_circ.py rqc 32 2 > gpurun_out/ncu_rqc2.log 2>&1; echo ncu_rqc=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"qs_tile_jit|k_perm|k_" --csv --log-file gpurun_out/launches_rqc2.csv python tools/prof_circ.py rqc 32 1 > gpurun_out/ncu_lr2.log 2>&1; echo ncu_lr=$?
