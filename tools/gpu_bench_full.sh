nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks.mem --format=csv
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo rc=$?
tail -c 1500 gpurun_out/bench_full.err
python tools/prof_gate.py u2 30 3 15 > gpurun_out/prof_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_pair -s 2 -c 1 -o gpurun_out/prof_u2_oneshot python tools/prof_gate.py u2 30 3 15 > gpurun_out/ncu_u2.log 2>&1
python bench.py --steps 1 --warmup 1 --no-circuits --no-e2e --no-cpu > gpurun_out/b_plain.json 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_(pair|ctrl|quad|diag|swap)" -s 93 -c 93 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-circuits --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1
echo done
