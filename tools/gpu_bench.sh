set -x
timeout 1200 python bench.py > gpurun_out/bench_r01f.json 2> gpurun_out/bench_r01f.err; echo bench_rc=$?
tail -5 gpurun_out/bench_r01f.err
python -c "import json; d=json.loads(open('gpurun_out/bench_r01f.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e'], d['circuits'], d['clocks'])"
