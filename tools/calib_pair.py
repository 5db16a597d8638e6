"""U2 throughput at n=30 for a few targets + a bitwise fingerprint at n=22 (round 1 used it with the
QS_PAIR_VARIANT knob to compare gate-kernel variants; the knob and the variants are gone, round 2)."""
import hashlib
import json
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_09198_b200 as qs  # noqa: E402
from qsinputs import gates as G  # noqa: E402


def main():
    out = {}
    rng = np.random.default_rng(0)
    with qs.QState(22) as st:
        st.init_random(3)
        st.set_option("fuse", 0)
        for t in range(22):
            st.apply_1q(t, G.haar(2, rng))
        out["fingerprint"] = hashlib.sha1(st.read().tobytes()).hexdigest()[:16]
    n = 30
    with qs.QState(n) as st:
        st.init_random(1)
        ss = torch.cuda.ExternalStream(st.stream(0))
        U = G.haar(2, rng)
        for t in (0, 1, 4, 9, 10, 15, 29):
            ts = []
            for r in range(8):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(ss)
                st.apply_1q(t, U)
                b.record(ss)
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            ts = ts[2:]
            out[f"t{t}"] = round((32 << n) / statistics.median(ts) / 1e6, 1)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
