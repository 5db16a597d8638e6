"""Randomised GPU parity: random circuits (every gate family, every qubit position incl. global ones)
on random sizes, shard counts and planner / executor options, against the oracle within the
north_star tolerance and bit for bit against the unfused single-GPU path of the same library."""
import numpy as np
import pytest

import paper_2506_09198_b200 as qs
from gpu_util import NORM_TOL, assert_parity
from qsinputs import circuits as C
from qsinputs import gates as G

pytestmark = pytest.mark.gpu


def random_circuit(rng, n, length):
    out = []
    named1 = [G.H, G.X, G.Y, G.Z, G.T, G.SQRT_X, G.SQRT_Y, G.SQRT_W, np.diag([1j, 1]), np.diag([1, -1j])]
    for _ in range(length):
        r = rng.random()
        a, b = (int(x) for x in rng.choice(n, size=2, replace=False)) if n > 1 else (0, 0)
        if r < 0.25 or n == 1:
            m = G.haar(2, rng) if rng.random() < 0.5 else named1[int(rng.integers(len(named1)))]
            out.append(C.g1(int(rng.integers(n)), m))
        elif r < 0.5:
            m = [G.haar(2, rng), G.X, G.Z, G.phase(rng.random() * 6.28), np.diag([1j, -1])][int(rng.integers(5))]
            out.append(C.gc(a, b, m))
        else:
            m = [G.haar(4, rng), G.SWAP, G.CNOT_Q0_CTRL, np.diag(np.exp(1j * rng.random(4))),
                 np.kron(G.haar(2, rng), G.haar(2, rng))][int(rng.integers(5))]
            out.append(C.g2(a, b, m))
    return out


@pytest.mark.parametrize("seed", range(60))
def test_random_circuits(orc, seed):
    rng = np.random.Generator(np.random.PCG64(1000 + seed))
    P = [1, 1, 2, 4, 8][seed % 5]
    k = P.bit_length() - 1
    n = int(rng.integers(max(1, 8 + k if P > 1 else 1), 15))
    circ = random_circuit(rng, n, int(rng.integers(20, 160)))
    if rng.random() < 0.5:  # a trailing run of disjoint SWAPs (permutation pass, possibly fused)
        circ += [C.g2(i, n - 1 - i, G.SWAP) for i in range(n // 2)]
    ref = orc.random_state(n, 77 + seed)
    orc.run(ref, circ)

    with qs.QState(n) as st:  # unfused single-GPU: the bitwise reference of the GPU paths
        st.set_option("fuse", 0)
        st.init_random(77 + seed)
        st.run(circ)
        base = st.read()
    assert_parity(base, ref, len(circ), f"seed {seed} unfused")

    opts = {"fuse": 1, "tile_qubits": int(rng.integers(6, 13)), "jit": int(rng.integers(0, 2)),
            "tile_low": int(rng.integers(1, 7)), "ladder_min": 0, "reorder": 0, "factor": 0,
            "perm_fuse": int(rng.integers(0, 2)), "tile_low_auto": int(rng.integers(0, 2))}
    small_chunks = P > 1 and rng.random() < 0.5
    # exchange transport (fused peer kernels / buffered pipeline with device copies or NCCL self send-recv)
    # and JIT kernel form (specialised / hybrid / family): all bit-for-bit the unfused single-GPU result
    xport = int(rng.integers(0, 3)) if P > 1 else 0
    opts["jit_family"] = int(rng.integers(0, 3))
    with qs.QState(n, P, virtual=P > 1) as st:
        for kk, v in opts.items():
            st.set_option(kk, v)
        if small_chunks:
            st.set_option("chunk_bytes", 4096)
        if xport:
            st.set_option("p2p", 0)
            st.set_option("vtransport", xport - 1)
        st.init_random(77 + seed)
        st.run(circ)
        got = st.read()
        norm = st.norm2()
    assert np.array_equal(got, base), (seed, n, P, opts, xport)
    assert abs(1 - norm) <= NORM_TOL

    # PHASE LADDER merge on (down to single phase ops), commutation-aware reordering, scalar factoring,
    # remapping, permutation passes, peer-memory or buffered exchanges: parity with the oracle
    opts["ladder_min"] = int(rng.integers(1, 5))
    opts["reorder"] = 1
    opts["factor"] = 1
    opts["remap"] = int(rng.integers(0, 2))
    opts["perm_low"] = int(rng.integers(0, 7))
    opts["p2p"] = int(rng.integers(0, 2))
    with qs.QState(n, P, virtual=P > 1) as st:
        for kk, v in opts.items():
            st.set_option(kk, v)
        st.init_random(77 + seed)
        st.run(circ)
        got = st.read()
    assert_parity(got, ref, len(circ), f"seed {seed} ladders")
