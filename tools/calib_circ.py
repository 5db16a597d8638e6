"""Circuit timing at n=32 (64 GiB): grid RQC and QFT|x> under tile options.  One JSON line per run."""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_09198_b200 as qs  # noqa: E402
from qsinputs import circuits as C  # noqa: E402


def main():
    n = int(os.environ.get("N", "32"))
    lows = [int(x) for x in os.environ.get("LOWS", "4").split(",")]
    ladders = [int(x) for x in os.environ.get("LADDERS", "0,4").split(",")]
    which = os.environ.get("CIRCS", "rqc,qft").split(",")
    perms = [int(x) for x in os.environ.get("PERMS", "5").split(",")]
    pfuse = [int(x) for x in os.environ.get("PFUSE", "1").split(",")]
    circs = {}
    if "rqc" in which:
        circs["rqc"] = (C.rqc_grid(n), ("basis", 0))
    if "qft" in which:
        circs["qft"] = (C.qft(n), ("basis", C.qft_x(n)))
    with qs.QState(n) as st:
        st.set_option("jit_async", 0)
        if os.environ.get("TILE_B"):
            st.set_option("tile_qubits", int(os.environ["TILE_B"]))
        ss = torch.cuda.ExternalStream(st.stream(0))
        st.set_option("tile_low_auto", int(os.environ.get("AUTO", "1")))
        for low, lad, pl, pf in [(lo, la, p, f) for lo in lows for la in ladders for p in perms for f in pfuse]:
            st.set_option("perm_fuse", pf)
            st.set_option("tile_low", low)
            st.set_option("ladder_min", lad)
            st.set_option("perm_low", pl)
            for name, (circ, init) in circs.items():
                if name not in which:
                    continue
                ts = []
                for r in range(3):
                    st.init_basis(init[1])
                    st.sync()
                    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record(ss)
                    st.run(circ)
                    e.record(ss)
                    torch.cuda.synchronize()
                    ts.append(a.elapsed_time(e) / 1e3)
                passes, _ = st.last_plan()
                print(json.dumps({"circ": name, "n": n, "tile_b": os.environ.get("TILE_B", "12"),
                                  "ctas": os.environ.get("QS_TILE_CTAS", "1"), "R": os.environ.get("QS_TILE_R", "4"), "tile_low": low, "ladder_min": lad, "perm_low": pl, "perm_fuse": pf, "passes": passes, "s": round(min(ts[1:]), 4),
                                  "first_s": round(ts[0], 3), "norm_err": abs(1 - st.norm2())}), flush=True)


if __name__ == "__main__":
    main()
