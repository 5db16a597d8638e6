"""Merge the ncu launch list of one bench gate step (profiles/r01_s3_launches_bench.csv: per launch
gpu__time_duration and dram bytes, serialised, cold cache) into the §8(d) report records
(profiles/r01_s3_sweep_report.jsonl): the step's 93 gate launches run in the report's order (configs[1]
then configs[2]), so record k gets the DRAM bytes and GB/s of gate launch k.

    python tools/merge_ncu_report.py [launches.csv] [report.jsonl]
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GATE_KERNELS = ("k_pair_hi", "k_pair_t0", "k_ctrl", "k_diag", "k_quad", "k_swap")
SCALE = {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "byte": 1,
         "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main():
    csv_path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "r01_s3_launches_bench.csv")
    rep_path = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "profiles", "r01_s3_sweep_report.jsonl")
    rows = [r for r in csv.reader(open(csv_path)) if len(r) > 10]
    h = rows[0]
    ki, mi, vi, ii, ui = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID", "Metric Unit"))
    d = {}
    for r in rows[1:]:
        d.setdefault(int(r[ii]), {"name": r[ki]})[r[mi]] = float(r[vi].replace(",", "")) * SCALE[r[ui]]
    launches = [d[i] for i in sorted(d) if any(k in d[i]["name"] for k in GATE_KERNELS) and "p2p" not in d[i]["name"]]
    recs = [json.loads(l) for l in open(rep_path)]
    gates = [r for r in recs if r["gate"] != "circuit"]
    # the first gate step starts at the first U2 on qubit 0 (k_pair_t0)
    first = next((k for k, L in enumerate(launches) if "k_pair_t0" in L["name"]), None)
    step = launches[first:first + len(gates)] if first is not None else []
    assert len(step) == len(gates), "launch list holds no full gate step"
    for r, L in zip(gates, step):
        t = L["gpu__time_duration.sum"]
        b = L["dram__bytes_read.sum"] + L["dram__bytes_write.sum"]
        r["ncu_kernel"] = L["name"].split("(")[0]
        r["ncu_dram_bytes"] = b
        r["ncu_dram_gbs"] = b / t / 1e9
        r["ncu_note"] = "one serialised, cold-cache launch of the bench step (ncu --clock-control none)"
    with open(rep_path, "w") as f:
        for r in recs:
            f.write(json.dumps(r) + "\n")
    print(json.dumps({"merged": len(step), "report": rep_path}))


if __name__ == "__main__":
    main()
