"""PHASE LADDER ops of the fused tile pass (reading R21):
runs of consecutive pure-phase gates that share one qubit are applied as one factor per amplitude.
Phase-heavy random circuits — controls in register slots, in sub-cube tile positions, outside the
tile and on global qubits; the shared qubit as a slot, a fixed bit, or absent — against the oracle
within the north_star tolerance and the tight alarm, on every executor and shard count."""
import numpy as np
import pytest

import paper_2506_09198_b200 as qs
from gpu_util import NORM_TOL, assert_parity
from qsinputs import circuits as C
from qsinputs import gates as G

pytestmark = pytest.mark.gpu


def phase_heavy(rng, n, length):
    out = []
    while len(out) < length:
        r = rng.random()
        if r < 0.15:  # a non-diagonal gate breaks runs and moves register slots
            out.append(C.g1(int(rng.integers(n)), G.haar(2, rng)))
        elif r < 0.6:  # ladder on a shared qubit t: controlled phases, CZ, single-qubit phases on t
            t = int(rng.integers(n))
            for _ in range(int(rng.integers(1, 2 * n))):
                c = int(rng.integers(n))
                if c == t or rng.random() < 0.1:
                    out.append(C.g1(t, G.phase(rng.random() * 6.28) if rng.random() < 0.5 else G.T))
                elif rng.random() < 0.2:
                    out.append(C.gc(c, t, G.Z))
                else:
                    out.append(C.gc(c, t, G.phase(rng.random() * 6.28)) if rng.random() < 0.5
                               else C.gc(t, c, G.phase(rng.random() * 6.28)))
        elif r < 0.85:  # single-qubit phases on different qubits (ladder without a shared qubit)
            for _ in range(int(rng.integers(1, n + 1))):
                out.append(C.g1(int(rng.integers(n)), G.phase(rng.random() * 6.28)))
        else:  # a general diagonal (not a phase form) inside a run
            a, b = (int(x) for x in rng.choice(n, size=2, replace=False))
            out.append(C.g2(a, b, np.diag(np.exp(1j * rng.random(4)))))
    return out[:length]


@pytest.mark.parametrize("seed", range(24))
def test_ladder_random_phase_circuits(orc, seed):
    rng = np.random.Generator(np.random.PCG64(5000 + seed))
    P = [1, 1, 2, 4, 8, 1][seed % 6]
    k = P.bit_length() - 1
    n = int(rng.integers(8 + k, 17))
    circ = phase_heavy(rng, n, int(rng.integers(40, 300)))
    ref = orc.random_state(n, 11 + seed)
    orc.run(ref, circ)
    opts = {"fuse": 1, "tile_qubits": int(rng.integers(6, 13)), "jit": int(seed % 3 != 2),
            "tile_low": int(rng.integers(1, 7)), "ladder_min": int([1, 2, 4][seed % 3]), "reorder": seed % 2}
    with qs.QState(n, P, virtual=P > 1) as st:
        for kk, v in opts.items():
            st.set_option(kk, v)
        st.init_random(11 + seed)
        st.run(circ)
        got = st.read()
        norm = st.norm2()
    assert_parity(got, ref, len(circ), f"seed {seed} P={P} {opts}")
    assert abs(1 - norm) <= NORM_TOL


@pytest.mark.parametrize("n", [12, 20])
def test_ladder_qft_vs_closed_form_every_tile(n):
    """QFT|x> with ladders at every tile size and both executors vs the closed form."""
    x = C.qft_x(n)
    y = np.arange(1 << n, dtype=np.uint64)
    kk = (np.uint64(x) * y) % np.uint64(1 << n)
    ang = np.pi * kk.astype(np.float64) / 2.0 ** (n - 1)
    ref = (np.cos(ang) + 1j * np.sin(ang)) * 2.0 ** (-n / 2)
    for b in (6, 8, 10, 12):
        for jit in (0, 1):
            with qs.QState(n) as st:
                st.set_option("tile_qubits", b)
                st.set_option("jit", jit)
                st.init_basis(x)
                st.run(C.qft(n))
                got = st.read()
            assert_parity(got, ref, len(C.qft(n)), f"QFT n={n} b={b} jit={jit}")
