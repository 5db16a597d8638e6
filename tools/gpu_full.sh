set -x
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 1200 python bench.py > gpurun_out/bench_r01g.json 2> gpurun_out/bench_r01g.err; echo bench_rc=$?
tail -3 gpurun_out/bench_r01g.err
python -c "import json; d=json.loads(open('gpurun_out/bench_r01g.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], {k:(v['s_min'], v['first_run_s']) for k,v in d['circuits'].items()}, d['clocks'])"
