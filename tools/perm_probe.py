"""Permutation-pass probe at n = 32: device time of one SWAP run (k_perm) and of the same run fused into
a tile pass (tile_kernel_perm), for permutations of different reach.  One JSON line per case."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_09198_b200 as qs  # noqa: E402
from qsinputs import circuits as C  # noqa: E402
from qsinputs import gates as G  # noqa: E402


def main():
    n = int(os.environ.get("N", "32"))
    cases = {
        "reverse": [(i, n - 1 - i) for i in range(n // 2)],
        "near_0_4<->5_9": [(i, i + 5) for i in range(5)],
        "mid_0_4<->16_20": [(i, i + 16) for i in range(5)],
        "far_0_4<->27_31": [(i, 31 - i) for i in range(5)],
    }
    with qs.QState(n) as st:
        st.set_option("jit_async", 0)
        st.set_option("tile_low_auto", 0)
        st.set_option("tile_low", 3)
        ss = torch.cuda.ExternalStream(st.stream(0))
        st.init_basis(0)
        for name, pairs in cases.items():
            swaps = [C.g2(a, b, G.SWAP) for a, b in pairs]
            lows = sorted({q for p in pairs for q in p if q < 5})
            for fused in (0, 1):
                circ = ([C.g1(q, G.H) for q in lows] if fused else []) + swaps
                st.set_option("perm_fuse", fused)
                ts = []
                for r in range(4):
                    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record(ss)
                    st.run(circ)
                    e.record(ss)
                    torch.cuda.synchronize()
                    ts.append(a.elapsed_time(e))
                print(json.dumps({"perm": name, "with_H_fused": fused, "passes": st.last_plan()[0],
                                  "ms": round(min(ts[1:]), 3)}), flush=True)


if __name__ == "__main__":
    main()
