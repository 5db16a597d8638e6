"""Clocks and power during repeated runs of one circuit (fused pass vs single-gate kernels)."""
import json
import os
import subprocess
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_09198_b200 as qs  # noqa: E402
from qsinputs import circuits as C  # noqa: E402


def sample(stop, rows):
    p = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active",
                          "--format=csv,noheader,nounits", "-lms", "50"], stdout=subprocess.PIPE, text=True)
    while not stop.is_set():
        line = p.stdout.readline()
        if line:
            rows.append(line.strip())
    p.terminate()


def main():
    n = int(os.environ.get("N", "30"))
    if os.environ.get("CIRCUITS"):  # the benchmark circuits at n = 32: power while they run
        cases = {"qft": (C.qft(n), 1), "rqc": (C.rqc_grid(n), 1), "u2_sweep": (C.sweep_1q(n), 0)}
    else:
        cases = {"fused_sweep11": (C.sweep_1q(11), 1), "unfused_sweep11": (C.sweep_1q(11), 0),
                 "fused_h1_x40": ([C.g1(3, C.sweep_1q(4)[3].m)] * 40, 1)}
    with qs.QState(n) as st:
        st.init_random(1)
        for name, (circ, fuse) in cases.items():
            st.set_option("fuse", fuse)
            st.run(circ)
            st.sync()
            rows, stop = [], threading.Event()
            th = threading.Thread(target=sample, args=(stop, rows))
            th.start()
            time.sleep(0.3)
            t0 = time.time()
            reps = 0
            while time.time() - t0 < 3.0:
                st.run(circ)
                st.sync()
                reps += 1
            dt = (time.time() - t0) / reps
            stop.set()
            th.join()
            sm = [float(r.split(",")[0]) for r in rows[6:] if r]
            pw = [float(r.split(",")[1]) for r in rows[6:] if r]
            print(json.dumps({"case": name, "ms": round(dt * 1e3, 2), "sm_mhz_med": sorted(sm)[len(sm) // 2] if sm else None,
                              "power_w_med": sorted(pw)[len(pw) // 2] if pw else None,
                              "reasons": rows[len(rows) // 2].split(",")[-1] if rows else None}), flush=True)


if __name__ == "__main__":
    main()
