set -x
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 1200 python bench.py > gpurun_out/bench_s3.json 2> gpurun_out/bench_s3.err; echo bench_rc=$?
tail -3 gpurun_out/bench_s3.err
python -c "import json; d=json.loads(open('gpurun_out/bench_s3.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['e2e']['ms_per_step'], d['circuits']['qft_n32']['s_min'], d['circuits']['rqc_n32']['s_min'], d['clocks'])"
python -c "import __graft_entry__ as g; g.smoke()"
