"""Minimal driver for ncu: n-qubit random state, `reps` applications of one gate kind.

    python tools/prof_gate.py {u2|u4|cnot|cphase|tile} [n] [reps] [args...]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_09198_b200 as qs  # noqa: E402
from qsinputs import circuits as C  # noqa: E402
from qsinputs import gates as G  # noqa: E402


def main():
    kind = sys.argv[1]
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    extra = [int(x) for x in sys.argv[4:]]
    rng = np.random.default_rng(0)
    with qs.QState(n) as st:
        st.init_random(1)
        if os.environ.get("TILE_B"):
            st.set_option("tile_qubits", int(os.environ["TILE_B"]))
        for _ in range(reps):
            if kind == "u2":
                st.apply_1q(extra[0] if extra else 15, G.haar(2, rng))
            elif kind == "u4":
                st.apply_2q(extra[0] if extra else 12, extra[1] if len(extra) > 1 else 20, G.haar(4, rng))
            elif kind == "cnot":
                st.apply_ctrl_1q(extra[0] if extra else 5, extra[1] if len(extra) > 1 else 12, G.X)
            elif kind == "cphase":
                st.apply_ctrl_1q(extra[0] if extra else 5, extra[1] if len(extra) > 1 else 12, G.phase(0.3))
            elif kind == "tile":
                st.run([C.g1(t, G.haar(2, rng)) for t in range(extra[0] if extra else 11)])
            elif kind == "qft":
                st.run(C.qft(n))
        st.sync()
        print("ok", kind, n, reps, st.norm2())


if __name__ == "__main__":
    main()
