timeout 1200 python bench.py > gpurun_out/bench_s3.json 2> gpurun_out/bench_s3.err; echo bench_rc=$?
tail -3 gpurun_out/bench_s3.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --metrics $M --clock-control none -k regex:"qs_tile_jit|k_perm" --csv --log-file gpurun_out/s3_launches_qft.csv python tools/prof_circ.py qft 32 1 > /dev/null 2>&1; echo lq=$?
python tools/launch_summary.py gpurun_out/s3_launches_qft.csv "QFT(32)|x>, session 3: 4 ladder passes (direct HBM I/O) + the permutation pass (dynamic tiles)" > gpurun_out/s3_launches_qft.txt; cat gpurun_out/s3_launches_qft.txt
python -c "import json; d=json.loads(open('gpurun_out/bench_s3.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['circuits']['qft_n32']['s_min'], d['circuits']['rqc_n32']['s_min'], d['clocks'], d['roofline'])"
