"""HBM calibration on one B200: torch copy_ (read A, write B), torch in-place
mul_ (read+write A), and our gate kernels on the same 16 GiB, CUDA events, best/median of reps.
Prints one JSON line."""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_09198_b200 as qs  # noqa: E402
from qsinputs import circuits as C  # noqa: E402
from qsinputs import gates as G  # noqa: E402


def timeit(fn, stream, reps=8):
    ts = []
    for _ in range(reps + 2):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts = ts[2:]
    return min(ts), statistics.median(ts)


def main():
    n = 30
    nbytes = 16 << n
    out = {}
    s = torch.cuda.current_stream()
    x = torch.empty(nbytes // 8, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    x.fill_(1.0)
    y.fill_(0.0)
    mn, md = timeit(lambda: y.copy_(x), s)
    out["torch_copy"] = {"best_gbs": 2 * nbytes / mn / 1e6, "median_gbs": 2 * nbytes / md / 1e6}
    mn, md = timeit(lambda: x.mul_(1.0000001), s)
    out["torch_inplace_mul"] = {"best_gbs": 2 * nbytes / mn / 1e6, "median_gbs": 2 * nbytes / md / 1e6}
    del x, y
    torch.cuda.empty_cache()
    with qs.QState(n) as st:
        st.init_random(1)
        ss = torch.cuda.ExternalStream(st.stream(0))
        U = G.haar(2, __import__("numpy").random.default_rng(0))
        U4 = G.haar(4, __import__("numpy").random.default_rng(1))
        for name, fn in [("u2_t0", lambda: st.apply_1q(0, U)), ("u2_t1", lambda: st.apply_1q(1, U)),
                         ("u2_t15", lambda: st.apply_1q(15, U)), ("u2_t29", lambda: st.apply_1q(29, U)),
                         ("u4_12_20", lambda: st.apply_2q(12, 20, U4)), ("u4_0_1", lambda: st.apply_2q(0, 1, U4)),
                         ("scale_all_rmw", lambda: st.apply_1q(0, __import__("numpy").diag([1j, -1j]))),
                         ("cnot_5_12", lambda: st.apply_ctrl_1q(5, 12, G.X)),
                         ("cphase_5_12", lambda: st.apply_ctrl_1q(5, 12, G.phase(0.3))),
                         ("tile_pass_11q", lambda: st.run([C.g1(t, U) for t in range(11)]))]:
            mn, md = timeit(fn, ss)
            b = nbytes * 2
            if name.startswith("cnot"):
                b = nbytes
            if name.startswith("cphase"):
                b = nbytes // 2
            out[name] = {"best_gbs": b / mn / 1e6, "median_gbs": b / md / 1e6, "best_ms": mn}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
