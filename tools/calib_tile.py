"""Fused-pass timing at n=30: several circuits x tile sizes.  Prints one JSON line per config."""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_09198_b200 as qs  # noqa: E402
from qsinputs import circuits as C  # noqa: E402


def main():
    n = int(os.environ.get("N", "30"))
    tiles = [int(x) for x in os.environ.get("TILES", "11,12").split(",")]
    circs = {
        "sweep1q_low11": C.sweep_1q(11),
        "sweep1q_30": C.sweep_1q(n),
        "sweep2q": C.sweep_2q(),
        "qft": C.qft(n),
        "ring_rqc": C.rqc_ring(n, layers=5),
    }
    with qs.QState(n) as st:
        st.init_random(1)
        ss = torch.cuda.ExternalStream(st.stream(0))
        for b in tiles:
            st.set_option("tile_qubits", b)
            for name, circ in circs.items():
                ts = []
                for r in range(4):
                    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record(ss)
                    st.run(circ)
                    e.record(ss)
                    torch.cuda.synchronize()
                    ts.append(a.elapsed_time(e))
                passes, _ = st.last_plan()
                ms = statistics.median(ts[1:])
                print(json.dumps({"b": b, "circ": name, "gates": len(circ), "passes": passes, "ms": round(ms, 3),
                                  "pass_gbs": round(passes * (32 << n) / ms / 1e6, 1),
                                  "minb": os.environ.get("QS_TILE_MINB", "2")}), flush=True)


if __name__ == "__main__":
    main()
