set -x
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 1500 python tools/paper_workloads.py > gpurun_out/paper_workloads.jsonl 2> gpurun_out/paper_workloads.err; echo pw=$?
tail -5 gpurun_out/paper_workloads.err
