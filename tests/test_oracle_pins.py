"""Pins for the oracle (CPU only, -m "not gpu").  Each test ties oracle/orc.c to something other
than itself: a worked example printed in PAPER.md/SPEC.md or a published vector (tests/golden/),
a closed form, a library routine (numpy kron / fft / scipy.stats), an exact special case, or an
invariant.  SURVEY.md §8(c) c.5 lists which pin covers which part.
"""
import math
import os

import numpy as np
import pytest
from scipy import stats

from dense_ref import dense_run
from qsinputs import circuits as C
from qsinputs import gates as G

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
EPS = 2.0 ** -53


def _golden(name):
    rows = []
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                rows.append([int(x) for x in line.split()])
    return rows


# --------------------------------------------------------------------------------------------
# index arithmetic
# --------------------------------------------------------------------------------------------
def test_alg1_worked_examples(orc):
    for task, t, up, lo in _golden("alg1_index.txt"):
        assert orc.pair_index(task, t) == (up, lo)


@pytest.mark.parametrize("n", [1, 3, 7, 12])
def test_alg1_bijection(orc, n):
    for t in range(n):
        ups, los = set(), set()
        for task in range(1 << (n - 1)):
            up, lo = orc.pair_index(task, t)
            assert (up >> t) & 1 == 0 and lo == up | (1 << t)
            ups.add(up)
            los.add(lo)
        assert ups == {i for i in range(1 << n) if not (i >> t) & 1}
        assert los == {i for i in range(1 << n) if (i >> t) & 1}


def test_alg1_boundary(orc):
    n = 20
    assert orc.pair_index((1 << (n - 1)) - 1, n - 1) == ((1 << (n - 1)) - 1, (1 << n) - 1)


# --------------------------------------------------------------------------------------------
# random state generator (reading R9)
# --------------------------------------------------------------------------------------------
def test_splitmix64_published_vectors(orc):
    for seed, j, val in _golden("splitmix64.txt"):
        assert orc.splitmix64(seed, j) == val


def test_gauss2_distribution(orc):
    """Box-Muller output: re, im iid N(0,1); |z|^2 ~ Exp(mean 2); arg z ~ U(-pi, pi]."""
    N = 1 << 15
    z = np.array([complex(*orc.gauss2(2506, i)) for i in range(N)])
    for comp in (z.real, z.imag):
        assert stats.kstest(comp, "norm").pvalue > 1e-3
    assert stats.kstest(np.abs(z) ** 2, "expon", args=(0, 2.0)).pvalue > 1e-3
    assert stats.kstest(np.angle(z), "uniform", args=(-math.pi, 2 * math.pi)).pvalue > 1e-3
    assert abs(np.corrcoef(z.real, z.imag)[0, 1]) < 4.0 / math.sqrt(N)
    # different seeds give different streams; the same (seed, i) is reproducible
    assert orc.gauss2(2506, 7) == orc.gauss2(2506, 7)
    assert orc.gauss2(2506, 7) != orc.gauss2(2507, 7)


@pytest.mark.parametrize("n", [1, 5, 12, 18])
def test_random_state_normalised(orc, n):
    a = orc.random_state(n, 2506)
    assert abs(1.0 - orc.norm2(a)) <= 1e-12
    assert abs(1.0 - math.fsum((np.abs(a) ** 2).tolist())) <= 1e-12
    # the amplitude i is gauss2(seed, i) scaled by one common positive factor
    raw = np.array([complex(*orc.gauss2(2506, i)) for i in range(min(a.size, 64))])
    ratio = a[: raw.size] / raw
    assert np.allclose(ratio.imag, 0, atol=1e-15) and np.ptp(ratio.real) < 1e-14 * ratio.real[0]
    if n >= 12:  # E[N |a|^2] = 1
        assert abs(a.size * np.mean(np.abs(a) ** 2) - 1.0) < 1e-9


def test_gauss2_range_is_the_unnormalised_random_state(orc):
    """orc_gauss2_range (the chunked samples the n = 32 DFT check uses) is gauss2 index by index, at any
    start offset, and scaling the whole range by 1/sqrt(its pairwise norm) gives orc_init_random bit for bit."""
    n = 12
    g = orc.gauss2_range(2506, 0, 1 << n)
    for i in (0, 1, 777, (1 << n) - 1):
        assert complex(*orc.gauss2(2506, i)) == g[i]
    off = orc.gauss2_range(2506, (1 << 33) + 5, 3)
    assert [complex(*orc.gauss2(2506, (1 << 33) + 5 + k)) for k in range(3)] == list(off)
    inv = 1.0 / math.sqrt(orc.norm2(g))
    a = orc.random_state(n, 2506)
    assert np.array_equal(a.view(np.float64), g.view(np.float64) * inv)


@pytest.mark.parametrize("n,chunk_bits", [(12, 24), (20, 18)])
def test_dft_sample_helper_is_ifft(orc, n, chunk_bits):
    """tests/dft_check.py (the QFT(32) random-state check: chunked DFT sums over the oracle's samples)
    equals numpy.fft.ifft(psi, norm="ortho") of the oracle's whole normalised random state (SURVEY.md
    §8(c) c.5 'QFT of any state'), with several chunks and 2^16-blocks at n = 20."""
    from dft_check import qft_random_state_samples
    rng = np.random.default_rng(n)
    ys = [0, 1, (1 << n) - 1, 1 << (n - 1)] + [int(v) for v in rng.integers(0, 1 << n, size=60)]
    got, s2 = qft_random_state_samples(orc, n, 2506, ys, chunk_bits=chunk_bits)
    ref = np.fft.ifft(orc.random_state(n, 2506), norm="ortho")[ys]
    assert np.max(np.abs(got - ref)) <= 1e-13 * np.max(np.abs(ref))
    assert abs(s2 / (1 << n) - 2.0) < 0.05  # E|g|^2 = 2


# --------------------------------------------------------------------------------------------
# norm
# --------------------------------------------------------------------------------------------
def test_norm_worked_examples(orc):
    a = orc.basis(10, 37)
    assert orc.norm2(a) == 1.0
    b = orc.random_state(10, 11)
    b *= 2.0
    assert abs(orc.norm2(b) - 4.0) <= 1e-12


def test_norm_pairwise_accuracy(orc):
    rng = np.random.default_rng(0)
    a = (rng.standard_normal(1 << 20) + 1j * rng.standard_normal(1 << 20)).astype(np.complex128)
    exact = math.fsum((a.real ** 2).tolist() + (a.imag ** 2).tolist())
    assert abs(orc.norm2(a) - exact) <= 64 * EPS * exact


# --------------------------------------------------------------------------------------------
# gate application vs dense Kronecker products (brute force on tiny inputs)
# --------------------------------------------------------------------------------------------
def _rand_state(n, seed):
    rng = np.random.default_rng(seed)
    v = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
    return v / np.linalg.norm(v)


@pytest.mark.parametrize("n", [1, 2, 3, 5, 7])
def test_1q_vs_dense_all_targets(orc, n):
    rng = np.random.Generator(np.random.PCG64(n))
    for t in range(n):
        U = G.haar(2, rng)
        psi = _rand_state(n, 100 + t)
        ref = dense_run(psi, [C.g1(t, U)])
        a = psi.copy()
        orc.apply_1q(a, t, U)
        assert np.max(np.abs(a - ref)) <= 1e-14


@pytest.mark.parametrize("n", [2, 3, 6])
def test_ctrl_1q_vs_dense_all_pairs(orc, n):
    rng = np.random.Generator(np.random.PCG64(10 + n))
    for c in range(n):
        for t in range(n):
            if c == t:
                continue
            U = G.haar(2, rng)
            psi = _rand_state(n, 7 * c + t)
            ref = dense_run(psi, [C.gc(c, t, U)])
            a = psi.copy()
            orc.apply_ctrl_1q(a, c, t, U)
            assert np.max(np.abs(a - ref)) <= 1e-14


@pytest.mark.parametrize("n", [2, 3, 6])
def test_2q_vs_dense_all_ordered_pairs(orc, n):
    rng = np.random.Generator(np.random.PCG64(20 + n))
    for q0 in range(n):
        for q1 in range(n):
            if q0 == q1:
                continue
            U = G.haar(4, rng)
            psi = _rand_state(n, 11 * q0 + q1)
            ref = dense_run(psi, [C.g2(q0, q1, U)])
            a = psi.copy()
            orc.apply_2q(a, q0, q1, U)
            assert np.max(np.abs(a - ref)) <= 1e-14


def test_randomised_circuits_vs_dense(orc):
    """randomized (gate, qubits, n) cases agree with the dense product."""
    rng = np.random.Generator(np.random.PCG64(4242))
    for case in range(200):
        n = int(rng.integers(2, 9))
        gates = []
        for _ in range(int(rng.integers(1, 6))):
            kind = ["1q", "c1q", "2q"][int(rng.integers(0, 3))]
            if kind == "1q":
                gates.append(C.g1(int(rng.integers(0, n)), G.haar(2, rng)))
            else:
                a, b = rng.choice(n, size=2, replace=False)
                gates.append(C.gc(a, b, G.haar(2, rng)) if kind == "c1q" else C.g2(a, b, G.haar(4, rng)))
        psi = _rand_state(n, case)
        ref = dense_run(psi, gates)
        out = psi.copy()
        orc.run(out, gates)
        assert np.max(np.abs(out - ref)) <= 1e-13, (case, n)


def test_2q_subindex_convention(orc):
    """U4 = kron(A, B) == B on q0 then A on q1 (numpy kron: A acts on the high sub-bit k>>1),
    and the CNOT-as-U4 matrix (k=1 <-> k=3) == ctrl-1q(q0, q1, X); q0 > q1 included."""
    rng = np.random.Generator(np.random.PCG64(5))
    for (q0, q1) in [(0, 1), (2, 0), (1, 3), (4, 2)]:
        A, B = G.haar(2, rng), G.haar(2, rng)
        psi = _rand_state(5, q0 * 5 + q1)
        x = psi.copy()
        orc.apply_2q(x, q0, q1, np.kron(A, B))
        y = psi.copy()
        orc.apply_1q(y, q0, B)
        orc.apply_1q(y, q1, A)
        assert np.max(np.abs(x - y)) <= 1e-14
        x = psi.copy()
        orc.apply_2q(x, q0, q1, G.CNOT_Q0_CTRL)
        y = psi.copy()
        orc.apply_ctrl_1q(y, q0, q1, G.X)
        assert np.array_equal(x, y)


# --------------------------------------------------------------------------------------------
# exact special cases
# --------------------------------------------------------------------------------------------
def test_truth_tables_bitwise(orc):
    n = 4
    for k in range(1 << n):
        for t in range(n):
            a = orc.basis(n, k)
            orc.apply_1q(a, t, G.X)
            assert np.array_equal(a, orc.basis(n, k ^ (1 << t)))
    a = orc.basis(1, 0)
    orc.apply_1q(a, 0, G.Y)
    assert np.array_equal(a, np.array([0, 1j]))
    # CNOT, control=1, target=0: |10> -> |11>, |01> unchanged
    a = orc.basis(2, 2)
    orc.apply_ctrl_1q(a, 1, 0, G.X)
    assert np.array_equal(a, orc.basis(2, 3))
    a = orc.basis(2, 1)
    orc.apply_ctrl_1q(a, 1, 0, G.X)
    assert np.array_equal(a, orc.basis(2, 1))
    # SWAP |01> -> |10>
    a = orc.basis(2, 1)
    orc.apply_2q(a, 0, 1, G.SWAP)
    assert np.array_equal(a, orc.basis(2, 2))
    # SWAP permutes bits of every basis state
    for k in range(1 << n):
        a = orc.basis(n, k)
        orc.apply_2q(a, 0, 3, G.SWAP)
        b0, b3 = k & 1, (k >> 3) & 1
        kk = (k & ~0b1001) | (b3 << 0) | (b0 << 3)
        assert np.array_equal(a, orc.basis(n, kk))


def test_cphase_special_cases(orc):
    psi = _rand_state(5, 3)
    a = psi.copy()
    orc.apply_ctrl_1q(a, 1, 3, G.phase(0.0))
    assert np.array_equal(a, psi)
    u = np.full(4, 0.5, dtype=np.complex128)  # uniform n=2 state
    orc.apply_ctrl_1q(u, 0, 1, G.phase(math.pi))
    assert np.allclose(u, [0.5, 0.5, 0.5, -0.5], atol=1e-16, rtol=0)
    # symmetric in (c, t)
    a = psi.copy()
    b = psi.copy()
    orc.apply_ctrl_1q(a, 1, 3, G.phase(0.7))
    orc.apply_ctrl_1q(b, 3, 1, G.phase(0.7))
    assert np.array_equal(a, b)


def test_hadamard_twice_identity(orc):
    psi = _rand_state(6, 9)
    a = psi.copy()
    orc.apply_1q(a, 3, G.H)
    orc.apply_1q(a, 3, G.H)
    assert np.max(np.abs(a - psi)) <= 1e-15


# --------------------------------------------------------------------------------------------
# closed forms
# --------------------------------------------------------------------------------------------
@pytest.mark.parametrize("n", [1, 2, 8, 16])
def test_hadamard_all_closed_form(orc, n):
    """H^{(x)n}|0> = uniform 2^{-n/2} within n eps 2^{-n/2} (north_star)."""
    a = orc.basis(n, 0)
    for t in range(n):
        orc.apply_1q(a, t, G.H)
    target = 2.0 ** (-n / 2)
    assert np.all(a.imag == 0)
    assert np.max(np.abs(a.real - target)) <= n * EPS * target


def test_qft_gate_counts():
    for n, h, cp, sw, tot in _golden("qft_counts.txt"):
        q = C.qft(n)
        assert len(q) == tot
        assert sum(g.name == "H" for g in q) == h
        assert sum(g.kind == "c1q" for g in q) == cp
        assert sum(g.name == "SWAP" for g in q) == sw


@pytest.mark.parametrize("n", [1, 2, 3, 6, 11])
def test_qft_basis_closed_form(orc, n):
    """QFT|x> = 2^{-n/2} sum_y e^{+2 pi i x y / 2^n}|y>; phase index k = x*y mod 2^n exact."""
    circ = C.qft(n)
    for x in sorted({0, 1, (1 << n) - 1, C.qft_x(n)}):
        a = orc.basis(n, x)
        orc.run(a, circ)
        y = np.arange(1 << n, dtype=np.uint64)
        k = (np.uint64(x) * y) % np.uint64(1 << n)
        ang = np.pi * k.astype(np.float64) / 2.0 ** (n - 1)
        ref = (np.cos(ang) + 1j * np.sin(ang)) * 2.0 ** (-n / 2)
        tol = 32 * len(circ) * EPS * 2.0 ** (-n / 2) + 4 * EPS
        assert np.max(np.abs(a - ref)) <= tol, (n, x)


@pytest.mark.parametrize("n", [4, 9, 14])
def test_qft_random_state_is_ifft(orc, n):
    psi = orc.random_state(n, 2506)
    a = psi.copy()
    orc.run(a, C.qft(n))
    ref = np.fft.ifft(psi, norm="ortho")
    assert np.max(np.abs(a - ref)) <= 1e-13


def test_qft_round_trip(orc):
    n = 12
    psi = orc.random_state(n, 77)
    a = psi.copy()
    q = C.qft(n)
    orc.run(a, q)
    orc.run(a, C.inverse(q))
    assert np.max(np.abs(a - psi)) <= 1e-13


# --------------------------------------------------------------------------------------------
# circuits: invariants and statistics
# --------------------------------------------------------------------------------------------
def test_rqc_grid_structure():
    counts = {32: (14, 12, 14, 12), 34: (16, 12, 16, 12), 20: (8, 8, 10, 5), 25: (10, 10, 10, 10),
              12: (6, 3, 4, 4)}
    totals = {32: 900, 34: 960, 20: 555, 25: 700}
    for n, abcd in counts.items():
        rows, cols, drop = C.grid_for_n(n)
        assert len(C.grid_sites(rows, cols, drop)) == n
        p = C.grid_couplers(rows, cols, drop)
        assert tuple(len(p[k]) for k in "ABCD") == abcd
        if n in totals:
            circ = C.rqc_grid(n)
            assert len(circ) == totals[n]
            prev = {}
            for g in circ:  # never repeats the previous 1q choice on a qubit
                if g.kind == "1q":
                    assert prev.get(g.q0) != g.name
                    prev[g.q0] = g.name


def test_rqc_porter_thomas_and_norm(orc):
    """Depth-20 grid RQC on the 4x5 grid: norm kept to 1e-12; N sum p^2 ~ 2 (Porter-Thomas)."""
    n = 20
    a = orc.basis(n, 0)
    orc.run(a, C.rqc_grid(n))
    p = np.abs(a) ** 2
    assert abs(1.0 - orc.norm2(a)) <= 1e-12
    assert 1.8 < p.size * np.sum(p * p) < 2.2


def test_config1_norm_and_round_trip(orc):
    n = 14
    psi = orc.random_state(n, 2506)
    circ = C.config1(n)
    a = psi.copy()
    orc.run(a, circ)
    assert abs(1.0 - orc.norm2(a)) <= 1e-12
    orc.run(a, C.inverse(circ))
    assert np.max(np.abs(a - psi)) <= 1e-13


def test_haar_unitary():
    rng = np.random.Generator(np.random.PCG64(1))
    for d in (2, 4):
        for _ in range(50):
            U = G.haar(d, rng)
            assert np.max(np.abs(U.conj().T @ U - np.eye(d))) <= 4 * EPS * d
    for m in (G.H, G.X, G.Y, G.Z, G.T, G.SQRT_X, G.SQRT_Y, G.SQRT_W, G.SWAP, G.CNOT_Q0_CTRL):
        assert np.max(np.abs(m.conj().T @ m - np.eye(m.shape[0]))) <= 4 * EPS
    # sqrt(P)^2 = P
    W = (G.X + G.Y) / math.sqrt(2)
    for s, p in ((G.SQRT_X, G.X), (G.SQRT_Y, G.Y), (G.SQRT_W, W)):
        assert np.max(np.abs(s @ s - p)) <= 4 * EPS


def test_qft_blocked_variant_is_the_same_unitary(orc):
    """PAPER.md:L295's cache-blocked QFT (blocking factor k, reading R22): every H acts on a physical qubit
    < k, and the state equals the iterative QFT's (and, on a basis state, the closed form) for k < n and
    k >= n (then it IS qft(n))."""
    for n, k in ((6, 1), (9, 3), (10, 5), (8, 8), (7, 64)):
        circ = C.qft_blocked(n, k)
        assert all(g.q0 < k for g in circ if g.name == "H")
        a = orc.random_state(n, 12)
        b = a.copy()
        orc.run(a, C.qft(n))
        orc.run(b, circ)
        assert np.max(np.abs(a - b)) <= 1e-14, (n, k)
        x = 13 % (1 << n)
        c = orc.basis(n, x)
        orc.run(c, circ)
        y = np.arange(1 << n)
        assert np.max(np.abs(c - np.exp(2j * np.pi * x * y / 2 ** n) / 2 ** (n / 2))) <= 1e-13
    assert len(C.qft_blocked(7, 64)) == len(C.qft(7))


def test_qft_swaps_first_variant_is_the_same_unitary(orc):
    """the QFT "can be cache-blocked without extra gates by shifting its ending SWAP gates
    to the left" — the builder's swaps-first variant gives the same state as the iterative QFT and the
    closed form on a basis state."""
    for n in (3, 6, 9):
        a = orc.random_state(n, 11)
        b = a.copy()
        orc.run(a, C.qft(n))
        orc.run(b, C.qft_swaps_first(n))
        assert np.max(np.abs(a - b)) <= 1e-14
        x = 5 % (1 << n)
        c = orc.basis(n, x)
        orc.run(c, C.qft_swaps_first(n))
        y = np.arange(1 << n)
        ref = np.exp(2j * np.pi * x * y / 2 ** n) / 2 ** (n / 2)
        assert np.max(np.abs(c - ref)) <= 1e-14
