"""Global-qubit U2 on 2 virtual shards of one GPU at n = 30: the fused peer-memory kernel (p2p = 1) vs
the buffered exchange (p2p = 0: chunked copies standing in for NCCL send/recv + the fused update
kernel), by chunk size.  Device time per gate (CUDA events); all traffic is local HBM."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_09198_b200 as qs  # noqa: E402
from qsinputs import circuits as C  # noqa: E402


def main():
    n = 30
    u = C.sweep_1q(n)[n - 1].m
    for p2p, chunk in ((1, 0), (0, 64 << 20), (0, 256 << 20), (0, 1 << 30)):
        with qs.QState(n, 2, virtual=True) as st:
            st.set_option("p2p", p2p)
            if chunk:
                st.set_option("chunk_bytes", chunk)
            st.init_random(2506)
            ss = torch.cuda.ExternalStream(st.stream(0))
            st.apply_1q(n - 1, u)
            st.sync()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(ss)
            for _ in range(5):
                st.apply_1q(n - 1, u)
            st.sync()
            b.record(ss)
            b.synchronize()
            print(json.dumps({"p2p": p2p, "chunk_MiB": chunk >> 20, "ms": a.elapsed_time(b) / 5}), flush=True)


if __name__ == "__main__":
    main()
