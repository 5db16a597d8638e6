set -x
python tools/calib.py > gpurun_out/calib.json 2> gpurun_out/calib.err; cat gpurun_out/calib.json
timeout 1200 python -m pytest tests -m "gpu and slow" -x -q 2>&1 | tail -5
python tools/prof_gate.py u2 30 3 15 > gpurun_out/prof_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_pair -s 2 -c 1 -o gpurun_out/prof_u2 python tools/prof_gate.py u2 30 3 15 > gpurun_out/ncu_u2.log 2>&1
python tools/prof_gate.py u4 30 3 12 20 > gpurun_out/prof_plain4.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_quad -s 2 -c 1 -o gpurun_out/prof_u4 python tools/prof_gate.py u4 30 3 12 20 > gpurun_out/ncu_u4.log 2>&1
python bench.py --steps 1 --warmup 1 --no-circuits --no-e2e --no-cpu > gpurun_out/b_plain.json 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_(pair|ctrl|quad|diag|swap)" -s 93 -c 93 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-circuits --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1
ls -la gpurun_out
