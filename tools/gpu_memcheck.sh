timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -m "gpu and not slow" -x -q -k "every_position or errors or mixed_global or init_random or basis or launch_count or jit" > gpurun_out/memcheck.log 2>&1; echo rc=$?
tail -15 gpurun_out/memcheck.log
