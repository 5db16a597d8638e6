"""Cold vs warm circuit times of the JIT tile executor.

For grid RQC(n) on one GPU: the first run of seed A (compiles every pass kernel not yet in the cache),
warm repeats of seed A, then a never-seen seed B end to end (gate generation + init + planning + any
compilation + the gates, wall clock), then warm repeats of seed B.  One JSON line.

    QS_JIT_CACHE=/tmp/fresh python tools/jit_cold.py [n] [seedA] [seedB]
"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_09198_b200 as qs  # noqa: E402
from qsinputs import circuits as C  # noqa: E402


def dev_time(st, circ, reps=3):
    """min device time of `reps` warm runs, and the host time of the qs_run_circuit call (enqueue)"""
    ss = torch.cuda.ExternalStream(st.stream(0))
    ts, hs = [], []
    for _ in range(reps):
        st.init_basis(0)
        st.sync()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(ss)
        h0 = time.perf_counter()
        st.run(circ)
        hs.append(time.perf_counter() - h0)
        b.record(ss)
        b.synchronize()
        ts.append(a.elapsed_time(b) / 1e3)
    return min(ts), min(hs)


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
    sa = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    sb = int(sys.argv[3]) if len(sys.argv) > 3 else 21
    out = {"n": n, "family_kernels": os.environ.get("QS_JIT_FAMILY", "1")}
    with qs.QState(n) as st:
        st.set_option("jit_family", int(out["family_kernels"]))  # 0 specialised, 1 hybrid (default), 2 family
        for tag, seed in (("A", sa), ("B", sb)):
            if tag == "B" and os.environ.get("JIT_WAIT", "1") == "1":
                st.set_option("jit_wait", 1)  # the shape's family kernels, queued by A's first run
            c0 = st.jit_stats()["compiled"]
            t0 = time.perf_counter()
            circ = C.rqc_grid(n, seed=seed)
            st.init_basis(0)
            st.run(circ)
            st.sync()
            out[f"first_wall_s_{tag}"] = time.perf_counter() - t0
            out[f"compiled_{tag}"] = st.jit_stats()["compiled"] - c0
            out[f"warm_s_{tag}"], out[f"warm_host_call_s_{tag}"] = dev_time(st, circ)
        out["passes"] = st.last_plan()[0]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
