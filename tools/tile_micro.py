"""Micro-benchmarks of the fused tile pass at n=30 (one pass each): pipeline cost (trivial ops) and
per-op cost (many ops in one batch)."""
import json
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_09198_b200 as qs  # noqa: E402
from qsinputs import circuits as C  # noqa: E402
from qsinputs import gates as G  # noqa: E402


def main():
    n = 30
    rng = np.random.default_rng(0)
    U = G.haar(2, rng)
    cases = {
        "copy_3cz": [C.gc(0, 1, G.Z)] * 3,
        "h1_x40": [C.g1(3, U)] * 40,
        "h4_x40": [C.g1(q, U) for q in (3, 4, 9, 10)] * 10,
        "cz_x40": [C.gc(3, 9, G.Z)] * 40,
        "cphase_fixed_x40": [C.gc(20, 3, G.phase(0.3))] * 40,
        "quad_x20": [C.g2(3, 9, G.haar(4, rng))] * 20,
    }
    only = os.environ.get("CASES")
    if only:
        cases = {k: v for k, v in cases.items() if k in only.split(",")}
    reps = int(os.environ.get("REPS", "4"))
    with qs.QState(n) as st:
        st.init_random(1)
        ss = torch.cuda.ExternalStream(st.stream(0))
        for name, circ in cases.items():
            ts = []
            for r in range(reps):
                a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(ss)
                st.run(circ)
                e.record(ss)
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(e))
            passes, _ = st.last_plan()
            ms = statistics.median(ts[1:] if len(ts) > 1 else ts)
            print(json.dumps({"case": name, "ops": len(circ), "passes": passes, "ms": round(ms, 3),
                              "R": os.environ.get("QS_TILE_R", "4")}), flush=True)


if __name__ == "__main__":
    main()
