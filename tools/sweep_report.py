"""SURVEY.md §8(d) report records on one B200: configs[1] (Haar U2 on t = 0..29) and configs[2] (CNOT,
CPhase, Haar U4 on the 21 pairs of {0, 1, 5, 12, 20, 28, 29}) at n = 30, and the circuits of configs[3]/[4]
at n = 32 — one JSON line per measurement, the protocol of §8(d): 1 untimed warm-up + 10 timed reps per
gate (CUDA events on the library stream), min and median, algorithmic and sector-effective bytes, GB/s,
fraction of 8 TB/s and of the measured copy ceiling (MEASURED_PEAKS.json), the unfused 6.4 TB/s model
time, clocks sampled during the sweep, seeds and git revision.  Correctness is the tests' job
(tests/test_gpu_parity.py, incl. the full-size sampled checks); here only the library's own norm is
recorded.  Measurement tool, not part of the library.

    python tools/sweep_report.py [--reps 10] [--out profiles/r01_s3_sweep_report.jsonl]
"""
import argparse
import json
import os
import statistics
import subprocess
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402  (Clocks sampler)
import paper_2506_09198_b200 as qs  # noqa: E402
from qsinputs import circuits as C  # noqa: E402

SEEDS = {"state": 2506, "gates": 9198, "rqc": 20, "qft_x": 35}


def gate_bytes(g, m):
    """(algorithmic, sector-effective) bytes of one gate on 2^m amplitudes."""
    q = g.qubits()
    full = 32 << m
    if g.name in ("U2", "U4"):
        return full, full
    if g.name == "CNOT":
        return full // 2, full if q[0] == 0 else full // 2
    if g.name == "CPhase":
        return full // 4, full // 2 if 0 in q else full // 4
    raise ValueError(g.name)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_sweep_report.jsonl"))
    ap.add_argument("--no-circuits", action="store_true")
    args = ap.parse_args()
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    ceiling = float(peaks.get("hbm_gbs", 0)) * 1e9 or None
    try:
        rev = subprocess.run(["git", "rev-parse", "--short", "HEAD"], cwd=ROOT, capture_output=True, text=True).stdout.strip()
    except Exception:
        rev = None
    rev = rev or os.environ.get("GIT_REV")
    cores = len(os.sched_getaffinity(0))
    recs = []
    n = 30
    with qs.QState(n) as st, bench.Clocks(0) as clk:
        ss = torch.cuda.ExternalStream(st.stream(0))
        st.init_random(SEEDS["state"])
        for cfg, gates in (("configs[1]", C.sweep_1q(n)), ("configs[2]", C.sweep_2q())):
            for g in gates:
                ts = []
                for r in range(args.reps + 1):
                    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record(ss)
                    st.apply(g)
                    e.record(ss)
                    e.synchronize()
                    if r:
                        ts.append(a.elapsed_time(e) / 1e3)
                alg, eff = gate_bytes(g, n)
                atom = bench.gate_bytes_atom(g, n)  # 64-B read atoms, 32-B write sectors
                tmed, tmin = statistics.median(ts), min(ts)
                recs.append({"config": cfg, "gate": g.name, "qubits": list(g.qubits()), "n": n, "P": 1,
                             "reps": args.reps, "t_min_s": tmin, "t_med_s": tmed, "alg_bytes": alg, "eff_bytes": eff,
                             "hbm_gbs": alg / tmed / 1e9, "eff_gbs": eff / tmed / 1e9, "atom_eff_bytes": atom,
                             "atom_eff_gbs": atom / tmed / 1e9,
                             "atom_pct_of_ceiling": 100 * atom / tmed / ceiling if ceiling else None,
                             "pct_of_8TBs": 100 * eff / tmed / 8e12,
                             "pct_of_ceiling": 100 * eff / tmed / ceiling if ceiling else None,
                             "model_s": eff / 6.4e12, "seeds": SEEDS, "host_cores": cores, "git_rev": rev})
        norm = st.norm2()
    for r in recs:
        r["norm_err"] = abs(1 - norm)
        r["clocks"] = clk.summary()
    if not args.no_circuits:
        m = 32
        with qs.QState(m) as st, bench.Clocks(0) as clk:
            ss = torch.cuda.ExternalStream(st.stream(0))
            st.set_option("jit_async", 0)
            for name, circ, init, model in (("configs[4] QFT|x>", C.qft(m), C.qft_x(m), 3.52),
                                            ("configs[3] grid RQC", C.rqc_grid(m), 0, 15.14)):
                ts = []
                for r in range(6):
                    st.init_basis(init)
                    st.sync()
                    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record(ss)
                    st.run(circ)
                    e.record(ss)
                    e.synchronize()
                    if r:
                        ts.append(a.elapsed_time(e) / 1e3)
                passes, exch = st.last_plan()
                floor = passes * (32 << m) / ceiling if ceiling else None
                recs.append({"config": name, "gate": "circuit", "gates": len(circ), "n": m, "P": 1, "reps": 5,
                             "t_min_s": min(ts), "t_med_s": statistics.median(ts), "hbm_passes": passes,
                             "exchange_steps": exch, "pass_floor_s_at_ceiling": floor,
                             "model_s": model, "model": "unfused gate sum at 6.4 TB/s (SURVEY.md §8(d))",
                             "norm_err": abs(1 - st.norm2()), "seeds": SEEDS, "host_cores": cores, "git_rev": rev,
                             "clocks": None})
            cs = clk.summary()
            for r in recs[-2:]:
                r["clocks"] = cs
    with open(args.out, "w") as f:
        for r in recs:
            f.write(json.dumps(r) + "\n")
    worst = min((r for r in recs if r["gate"] in ("U2", "U4")), key=lambda r: r["eff_gbs"])
    print(json.dumps({"records": len(recs), "worst_u2_u4_eff_gbs": worst["eff_gbs"], "worst": worst["qubits"],
                      "out": args.out}))


if __name__ == "__main__":
    main()
