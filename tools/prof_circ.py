"""Minimal driver for ncu on a fused circuit: n-qubit state, the circuit run `reps` times (the first run
compiles the JIT tile kernels).

    python tools/prof_circ.py {rqc|qft} [n] [reps] [opt=v,opt=v...]   (qs_set_option keys)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_09198_b200 as qs  # noqa: E402
from qsinputs import circuits as C  # noqa: E402


def main():
    kind = sys.argv[1]
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    circ = C.rqc_grid(n) if kind == "rqc" else C.qft(n)
    opts = dict(kv.split("=") for kv in sys.argv[4].split(",")) if len(sys.argv) > 4 else {}
    with qs.QState(n) as st:
        st.set_option("jit_async", 0)
        for k, v in opts.items():
            st.set_option(k, int(v))  # every pass runs its JIT kernel (stable launch indices for ncu)
        for _ in range(reps):
            st.init_basis(0 if kind == "rqc" else C.qft_x(n))
            st.run(circ)
        st.sync()
        print("ok", kind, n, reps, st.last_plan(), st.norm2())


if __name__ == "__main__":
    main()
