set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv; nproc; free -g | head -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -30
timeout 900 python bench.py --steps 3 --warmup 3 --no-circuits --no-cpu > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo bench_rc=$?
tail -c 4000 gpurun_out/bench1.json; tail -20 gpurun_out/bench1.err
