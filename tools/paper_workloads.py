"""The paper's own workloads on one B200 (like-for-like context for the paper's
CPU figures, not a target).  One JSON line per measurement, CUDA events on the library stream.

  fig ben1  : Hadamard on the second qubit (qubit 1) of a random n-qubit state, n = 23..33
              (PAPER.md:L278-L283), per-gate seconds (median of 10 after 1 warm-up), GB/s;
  fig ben3  : H, Pauli-Y and CNOT (control 1 -> target 2; the paper does not name the qubits) at n = 30;
  fig ben2  : QFT iterative (= recursive order), the swaps-first variant and the cache-blocked variants with
              blocking factors 16 and 64 (every H on a qubit < k; reading R22), n = 23..32,
              seconds per circuit, fused;
  fig rqc   : the paper's ring RQC (L = 5 layers of random {H, X, Y, T} then CNOT i -> i+1 mod n,
              PAPER.md:L327), n = 23..32: gates-only seconds and end-to-end seconds (create + init + gate
              generation + run + destroy, as the paper times it).

    python tools/paper_workloads.py [--max-n 33] [--quick]
"""
import argparse
import json
import os
import statistics
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_09198_b200 as qs  # noqa: E402
from qsinputs import circuits as C  # noqa: E402
from qsinputs import gates as G  # noqa: E402


def timed(st, fn, reps):
    ss = torch.cuda.ExternalStream(st.stream(0))
    out = []
    for r in range(reps + 1):
        st.sync()
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(ss)
        fn()
        e.record(ss)
        torch.cuda.synchronize()
        if r:
            out.append(a.elapsed_time(e) / 1e3)
    return out


def emit(d):
    print(json.dumps(d), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--max-n", type=int, default=33)
    ap.add_argument("--quick", action="store_true")
    args = ap.parse_args()
    reps = 3 if args.quick else 10
    # fig ben1: H on qubit 1
    for n in range(23, args.max_n + 1):
        with qs.QState(n) as st:
            st.init_random(2506)
            ts = timed(st, lambda: st.apply_1q(1, G.H), reps)
            med = statistics.median(ts)
            emit({"fig": "ben1", "gate": "H", "target": 1, "n": n, "s_median": med, "s_min": min(ts),
                  "alg_GBps": 32 * 2 ** n / med / 1e9})
    # fig ben3: H, Y, CNOT at n = 30
    with qs.QState(30) as st:
        st.init_random(2506)
        for name, fn, byts in (("H", lambda: st.apply_1q(1, G.H), 32), ("Y", lambda: st.apply_1q(1, G.Y), 32),
                               ("CNOT", lambda: st.apply_ctrl_1q(1, 2, G.X), 16)):
            ts = timed(st, fn, reps)
            med = statistics.median(ts)
            emit({"fig": "ben3", "gate": name, "n": 30, "s_median": med, "s_min": min(ts),
                  "alg_GBps": byts * 2 ** 30 / med / 1e9})
    # fig ben2: QFT variants; fig rqc: ring RQC
    for n in range(23, min(32, args.max_n) + 1):
        with qs.QState(n) as st:
            for name, circ in (("qft_iterative", C.qft(n)), ("qft_swaps_first", C.qft_swaps_first(n)),
                               ("qft_blocked16", C.qft_blocked(n, 16)), ("qft_blocked64", C.qft_blocked(n, 64))):
                x = C.qft_x(n)
                ts = timed(st, lambda: (st.init_basis(x), st.run(circ)), max(2, reps // 3))
                passes, _ = st.last_plan()
                emit({"fig": "ben2", "circuit": name, "n": n, "s_median": statistics.median(ts), "s_min": min(ts),
                      "gates": len(circ), "hbm_passes": passes, "note": "includes init_basis (one memset pass)"})
            ring = C.rqc_ring(n, layers=5)
            ts = timed(st, lambda: (st.init_basis(0), st.run(ring)), max(2, reps // 3))
            passes, _ = st.last_plan()
            emit({"fig": "rqc", "circuit": "ring_L5", "n": n, "s_median": statistics.median(ts), "s_min": min(ts),
                  "gates": len(ring), "hbm_passes": passes, "note": "init_basis + gates"})
        e2e = []
        for r in range(2):  # end to end as the paper times it: create, init, generate, run, destroy
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            with qs.QState(n) as st:
                st.init_basis(0)
                st.run(C.rqc_ring(n, layers=5, seed=20 + r))
                st.sync()
            e2e.append(time.perf_counter() - t0)
        emit({"fig": "rqc", "circuit": "ring_L5_end_to_end", "n": n, "s_first": e2e[0], "s_second": e2e[1],
              "note": "wall clock: qs_create + init + gate generation + run + qs_destroy (second run: JIT cached)"})


if __name__ == "__main__":
    main()
