"""GPU parity: the CUDA path (through the C-ABI) vs the oracle on the same seeded inputs.

Bars (BASELINE.json north_star): max|d amplitude| <= 1e-10 and |1 - norm| <= 1e-12, plus the tight
alarm 32 G eps max|psi|.  Integer-like results (X/CNOT/SWAP permutations,
P-invariance, fused vs unfused) are compared bit for bit.
"""
import math

import numpy as np
import pytest

import paper_2506_09198_b200 as qs
from gpu_util import NORM_TOL, assert_parity
from qsinputs import circuits as C
from qsinputs import gates as G

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def lib():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device (no CPU fallback exists)")
    return qs.load_library()


def _gpu_run(n, circ, init=("random", 2506), P=1, virtual=False, fuse=True, tile=None, chunk=None, ladder=None,
             reorder=None, factor=None, p2p=None, vtransport=None):
    with qs.QState(n, P, virtual=virtual) as st:
        if p2p is not None:
            st.set_option("p2p", int(p2p))
        if vtransport is not None:
            st.set_option("vtransport", int(vtransport))
        if reorder is not None:
            st.set_option("reorder", int(reorder))
        if factor is not None:
            st.set_option("factor", int(factor))
        if fuse is not None:
            st.set_option("fuse", int(fuse))
        if ladder is not None:
            st.set_option("ladder_min", ladder)
        if tile:
            st.set_option("tile_qubits", tile)
        if chunk:
            st.set_option("chunk_bytes", chunk)
        if init[0] == "random":
            st.init_random(init[1])
        else:
            st.init_basis(init[1])
        st.run(circ)
        st.sync()
        return st.read(), st.norm2()


def _orc_run(orc, n, circ, init=("random", 2506)):
    a = orc.random_state(n, init[1]) if init[0] == "random" else orc.basis(n, init[1])
    orc.run(a, circ)
    return a


# ------------------------------------------------------------------------------------------------
# single gates, every position, every kernel variant (direct kernels, qs_apply_*)
# ------------------------------------------------------------------------------------------------
@pytest.mark.parametrize("n", [3, 12])
def test_single_gates_every_position(orc, n):
    rng = np.random.Generator(np.random.PCG64(n))
    cases = []
    for t in range(n):
        cases += [C.g1(t, G.haar(2, rng)), C.g1(t, G.T), C.g1(t, G.X), C.g1(t, np.diag([1j, -1]))]
    for c in range(n):
        for t in range(n):
            if c != t:
                cases += [C.gc(c, t, G.haar(2, rng)), C.gc(c, t, G.X), C.gc(c, t, G.phase(rng.random() * 6)),
                          C.gc(c, t, np.diag([1j, -1j]))]
                cases += [C.g2(c, t, G.haar(4, rng)), C.g2(c, t, G.SWAP),
                          C.g2(c, t, np.diag(np.exp(1j * rng.random(4))))]
    psi = orc.random_state(n, 11)
    with qs.QState(n) as st:
        for g in cases:
            st.write(0, psi)
            st.apply(g)
            got = st.read()
            ref = psi.copy()
            orc.run(ref, [g])
            if g.name in ("SWAP",) or np.array_equal(g.m, G.X):
                assert np.array_equal(got, ref), (g.kind, g.q0, g.q1, g.name)
            else:
                assert_parity(got, ref, 1, f"{g.kind}({g.q0},{g.q1}) {g.name}")


def test_single_gates_larger_state(orc):
    """n = 18: several grid-stride iterations and 256-bit vector paths for every target."""
    n = 18
    rng = np.random.Generator(np.random.PCG64(18))
    psi = orc.random_state(n, 5)
    gates = [C.g1(t, G.haar(2, rng)) for t in range(n)]
    gates += [C.gc(c, t, G.haar(2, rng)) for (c, t) in [(0, 17), (17, 0), (5, 6), (9, 1)]]
    gates += [C.g2(a, b, G.haar(4, rng)) for (a, b) in [(0, 1), (1, 0), (0, 17), (16, 17), (3, 11)]]
    with qs.QState(n) as st:
        st.write(0, psi)
        st.set_option("fuse", 0)
        st.run(gates)
        got = st.read()
    ref = psi.copy()
    orc.run(ref, gates)
    assert_parity(got, ref, len(gates), "n=18 gates")


# ------------------------------------------------------------------------------------------------
# BASELINE configs[0]: n = 20, random state, 20 Haar U2 then 19 Haar U4 on (q, q+1)
# ------------------------------------------------------------------------------------------------
@pytest.mark.parametrize("fuse", [False, True])
def test_config1_n20(orc, fuse):
    n = 20
    circ = C.config1(n)
    got, norm = _gpu_run(n, circ, fuse=fuse)
    ref = _orc_run(orc, n, circ)
    assert_parity(got, ref, len(circ), f"config1 fuse={fuse}")
    assert abs(1.0 - norm) <= NORM_TOL


def test_init_random_matches_oracle(orc):
    for n in (1, 2, 13, 20):
        with qs.QState(n) as st:
            st.init_random(2506)
            got = st.read()
            norm = st.norm2()
        ref = orc.random_state(n, 2506)
        assert_parity(got, ref, 1, f"init_random n={n}")
        assert abs(1.0 - norm) <= NORM_TOL


def test_async_copies_are_stream_ordered():
    """qs_write_amps_async / qs_read_amps_async run in stream order with the gates: write, gate, read
    queued back to back give the gate applied to the written state."""
    import torch
    n = 16
    rng = np.random.Generator(np.random.PCG64(4))
    psi = (rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n))
    psi /= np.linalg.norm(psi)
    src = torch.empty((1 << n) * 2, dtype=torch.float64, pin_memory=True).numpy().view(np.complex128)
    dst = torch.empty((1 << n) * 2, dtype=torch.float64, pin_memory=True).numpy().view(np.complex128)
    src[:] = psi
    with qs.QState(n) as st:
        st.init_random(1)
        qs.qs.qs_write_amps_async(st.h, 0, src)
        st.apply_1q(3, G.X)
        qs.qs.qs_read_amps_async(st.h, 0, 1 << n, dst)
        st.sync()
    ref = psi.reshape(-1, 2, 8)[:, ::-1, :].reshape(-1)  # X on qubit 3 swaps the bit-3 halves
    assert np.array_equal(dst, ref)


def test_basis_and_norm_exact():
    with qs.QState(10) as st:
        st.init_basis(777)
        v = st.read()
        assert v[777] == 1.0 and np.count_nonzero(v) == 1
        assert st.norm2() == 1.0
        st.init_random(3)
        v = st.read()
        st.write(0, 2 * v)
        assert abs(st.norm2() - 4.0) <= 4 * NORM_TOL  # SPEC.md:L62 worked example


# ------------------------------------------------------------------------------------------------
# fusion: bitwise identical to the unfused path, for every tile size (PHASE LADDER merge,
# commutation-aware reordering and scalar factoring off); with them on (the defaults) rounding
# differs: parity instead
# ------------------------------------------------------------------------------------------------
@pytest.mark.parametrize("name", ["config1", "qft", "rqc", "sweep2q"])
def test_fused_bitwise_equals_unfused(name):
    n = 20 if name != "sweep2q" else 30 - 10
    circ = {"config1": C.config1(20), "qft": C.qft(20), "rqc": C.rqc_grid(20),
            "sweep2q": C.sweep_2q(qset=(0, 1, 5, 12, 18, 19))}[name]
    base, _ = _gpu_run(n, circ, fuse=False)
    for b in (6, 9, 11, 12):
        got, _ = _gpu_run(n, circ, fuse=True, tile=b, ladder=0, reorder=0, factor=0)
        assert np.array_equal(got, base), (name, b)
        got, norm = _gpu_run(n, circ, fuse=True, tile=b, ladder=1)  # ladders + reordering + factoring
        assert_parity(got, base, len(circ), f"{name} b={b} ladders+reorder")
        assert abs(1 - norm) <= NORM_TOL


@pytest.mark.parametrize("seed", range(8))
def test_permutation_pass_bitwise(seed):
    """Runs of disjoint SWAPs (random involutions of the local qubits, mixed with other gates and, on
    virtual shards, with global qubits) go through the in-place permutation pass (k_perm.cu): pure data
    movement, so the result is bit-for-bit the unfused SWAP-by-SWAP result, for every perm_low."""
    rng = np.random.Generator(np.random.PCG64(700 + seed))
    P = [1, 1, 2, 8][seed % 4]
    n = int(rng.integers(10, 19))
    circ = [C.g1(q, G.haar(2, rng)) for q in range(n)]
    for _ in range(3):
        qs_ = rng.permutation(n)
        k = int(rng.integers(2, n // 2 + 1))
        circ += [C.g2(int(qs_[2 * i]), int(qs_[2 * i + 1]), G.SWAP) for i in range(k)]
        circ += [C.g1(int(rng.integers(n)), G.haar(2, rng)), C.gc(0, n - 1, G.phase(0.3))]
    circ += [C.g2(i, n - 1 - i, G.SWAP) for i in range(n // 2)]
    base, _ = _gpu_run(n, circ, fuse=False)
    for low in (0, 1, 3, 5, 6):
        with qs.QState(n, P, virtual=P > 1) as st:
            st.set_option("perm_low", low)
            st.set_option("reorder", 0)
            st.set_option("factor", 0)
            st.init_random(2506)
            st.run(circ)
            got = st.read()
        assert np.array_equal(got, base), (seed, P, low)


@pytest.mark.parametrize("n,low,P,jit", [(14, 3, 1, 1), (21, 4, 1, 1), (22, 3, 1, 1), (23, 3, 1, 1), (22, 3, 1, 0),
                                          (23, 3, 2, 1), (22, 3, 4, 1)])
def test_fused_permutation_bitwise(orc, n, low, P, jit):
    """The QFT's final reversal fused into the last tile pass (tile_kernel_pair: tile pairs stored onto
    each other's place) is bit for bit the separate permutation pass, one HBM pass fewer on one GPU; the
    interpreter path (jit = 0) falls back to the pass + k_perm; the result matches the oracle."""
    circ = C.qft(n)
    res = {}
    for pf in (0, 1):
        with qs.QState(n, P, virtual=P > 1) as st:
            st.set_option("tile_low", low)
            st.set_option("tile_low_auto", 0)
            st.set_option("perm_fuse", pf)
            st.set_option("jit", jit)
            st.set_option("jit_async", 0)
            st.init_random(2506)
            st.run(circ)
            res[pf] = (st.read(), st.last_plan()[0], st.norm2())
    assert np.array_equal(res[0][0], res[1][0]), (n, low, P, jit)
    if P == 1:
        assert res[1][1] == res[0][1] - 1, (res[0][1], res[1][1])
    assert_parity(res[1][0], _orc_run(orc, n, circ), len(circ), f"QFT({n}) fused reversal")
    assert abs(1 - res[1][2]) <= NORM_TOL


@pytest.mark.parametrize("n,tile,low,P", [(20, 8, 3, 1), (24, 12, 4, 1), (24, 12, 4, 2), (22, 10, 2, 1)])
def test_hoisted_permutation(orc, n, tile, low, P):
    """Permutation hoisting (qs_plan.h hoist_permutation): the QFT's reversal, too wide for the last
    ladder pass, rides on the stores of two earlier tile passes (tile pairs on two-CTA clusters, tile_kernel_pair, up to
    12-qubit tiles) — one HBM pass fewer than with perm_hoist = 0 — and the state matches the oracle
    (n <= 22) and the unhoisted run at the contract bar and the tight alarm."""
    circ = C.qft(n)
    res = {}
    for ph in (0, 1):
        with qs.QState(n, P, virtual=P > 1) as st:
            st.set_option("tile_qubits", tile)
            st.set_option("tile_low", low)
            st.set_option("tile_low_auto", 0)
            st.set_option("perm_hoist", ph)
            st.set_option("jit_async", 0)
            st.init_random(2506)
            st.run(circ)
            res[ph] = (st.read(), st.last_plan()[0], st.norm2())
    if P == 1:
        assert res[1][1] == res[0][1] - 1, (res[0][1], res[1][1])
    assert_parity(res[1][0], res[0][0], len(circ), f"QFT({n}) hoisted vs not")
    if n <= 22:
        assert_parity(res[1][0], _orc_run(orc, n, circ), len(circ), f"QFT({n}) hoisted reversal")
    assert abs(1 - res[1][2]) <= NORM_TOL


def test_hoisted_permutation_random_circuits(orc):
    """Permutation hoisting on random circuits around a run of disjoint SWAPs (qsinputs.circuits.
    random_with_swap_run; small tiles so that no tile closes under the run): every gate kind relabelled,
    tile pairs on two-CTA clusters with and without direct stores, against the oracle; the hoisted runs
    take one HBM pass fewer than perm_hoist = 0 in most cases."""
    fewer = 0
    for seed in range(12):
        n, b = 14 + seed % 4, 6 + seed % 3
        circ = C.random_with_swap_run(n, seed)
        ref = _orc_run(orc, n, circ)
        passes = {}
        for ph in (0, 1):
            with qs.QState(n) as st:
                st.set_option("tile_qubits", b)
                st.set_option("tile_low", 2)
                st.set_option("tile_low_auto", 0)
                st.set_option("perm_hoist", ph)
                st.set_option("jit_async", 0)
                st.init_random(2506)
                st.run(circ)
                got, norm = st.read(), st.norm2()
                passes[ph] = st.last_plan()[0]
            assert_parity(got, ref, len(circ), f"random+SWAP run seed {seed} perm_hoist={ph}")
            assert abs(1 - norm) <= NORM_TOL
        fewer += passes[1] < passes[0]
    assert fewer >= 3, fewer


def test_jit_bitwise_equals_interpreter():
    """The NVRTC straight-line tile kernels and the interpreter kernel give identical bits, and the
    JIT path is the one that ran (qs_jit_stats)."""
    n = 20
    circ = C.qft(n) + C.rqc_grid(20) + C.config1(n) + C.sweep_2q(qset=(0, 1, 5, 12, 18, 19))
    with qs.QState(n) as st:
        st.set_option("jit", 0)
        st.init_random(5)
        st.run(circ)
        ref = st.read()
        before = st.jit_stats()
        st.set_option("jit", 1)
        st.set_option("jit_async", 0)  # compile before running, so every pass runs its JIT kernel
        st.init_random(5)
        st.run(circ)
        got = st.read()
        after = st.jit_stats()
    assert np.array_equal(got, ref)
    assert after["launched"] > before["launched"] and after["failed"] == 0, (before, after)


def test_family_kernels_bitwise_and_seed_independent():
    """Family pass kernels (grid RQC's sqrtX/sqrtY/sqrtW picked per op at run time, option jit_family = 2)
    give the bits of the specialised kernels (jit_family = 0: entry codes compiled in); a second seed of
    the same shape reuses every family kernel (nothing compiled); the default hybrid (1) matches too."""
    n = 20
    res = {}
    with qs.QState(n) as st:
        st.set_option("jit_wait", 1)  # background compilations of earlier tests must not move the counters
    for seed in (20, 31):
        circ = C.rqc_grid(n, seed=seed)
        for mode in (0, 2, 1):
            with qs.QState(n) as st:
                st.set_option("jit_async", 0)
                st.set_option("jit_family", mode)
                st.init_random(7)
                before = st.jit_stats()
                st.run(circ)
                res[seed, mode] = st.read()
                after = st.jit_stats()
                assert after["failed"] == before["failed"]
                if seed == 31 and mode == 2:
                    assert after["compiled"] == before["compiled"], "family kernels recompiled for a new seed"
        assert np.array_equal(res[seed, 0], res[seed, 2]) and np.array_equal(res[seed, 0], res[seed, 1])
    with qs.QState(n) as st:
        st.set_option("jit_wait", 1)  # joins the background compilations the hybrid mode queued


def test_async_jit_mixes_executors_bitwise():
    """jit_async = 1: passes whose kernel is still compiling run in the interpreter; the result is bit
    for bit the all-JIT result (same op templates), before and after jit_wait."""
    n = 18
    circ = C.rqc_grid(12, depth=14) + C.qft(n) + C.sweep_2q(qset=(0, 3, 9, 17))
    with qs.QState(n) as st:
        st.set_option("jit_async", 0)
        st.init_random(8)
        st.run(circ)
        ref = st.read()
    with qs.QState(n) as st:
        st.set_option("jit_async", 1)
        st.set_option("tile_low", 3)  # other pass structures than the run above: new kernels to compile
        st.set_option("tile_low_auto", 0)
        st.init_random(8)
        st.run(circ)
        first = st.read()
        st.set_option("jit_wait", 1)
        st.init_random(8)
        st.run(circ)
        second = st.read()
    assert_parity(first, ref, len(circ), "async first run")
    assert np.array_equal(first, second)


# ------------------------------------------------------------------------------------------------
# circuits (BASELINE configs[3], [4] at sizes the oracle finishes quickly)
# ------------------------------------------------------------------------------------------------
@pytest.mark.parametrize("n", [1, 2, 5, 16])
def test_qft_basis_closed_form(n):
    circ = C.qft(n)
    x = C.qft_x(n)
    got, norm = _gpu_run(n, circ, init=("basis", x))
    y = np.arange(1 << n, dtype=np.uint64)
    k = (np.uint64(x) * y) % np.uint64(1 << n)
    ang = np.pi * k.astype(np.float64) / 2.0 ** (n - 1)
    ref = (np.cos(ang) + 1j * np.sin(ang)) * 2.0 ** (-n / 2)
    assert_parity(got, ref, len(circ), f"QFT|x> n={n}")
    assert abs(1 - norm) <= NORM_TOL


def test_qft_random_state_is_ifft(orc):
    n = 18
    circ = C.qft(n)
    got, _ = _gpu_run(n, circ)
    psi = orc.random_state(n, 2506)
    assert_parity(got, np.fft.ifft(psi, norm="ortho"), len(circ), "QFT random vs ifft")
    ref = _orc_run(orc, n, circ)
    assert_parity(got, ref, len(circ), "QFT random vs oracle")


def test_qft_round_trip():
    n = 20
    q = C.qft(n)
    got, _ = _gpu_run(n, q + C.inverse(q), init=("random", 9))
    with qs.QState(n) as st:
        st.init_random(9)
        psi = st.read()
    assert_parity(got, psi, 2 * len(q), "QFT round trip")


@pytest.mark.parametrize("n", [12, 20])
def test_rqc_grid(orc, n):
    circ = C.rqc_grid(n)
    got, norm = _gpu_run(n, circ, init=("basis", 0))
    ref = _orc_run(orc, n, circ, init=("basis", 0))
    assert_parity(got, ref, len(circ), f"RQC n={n}")
    assert abs(1 - norm) <= NORM_TOL


def test_qft_swaps_first_variant(orc):
    """The paper's cache-blocked QFT ordering (SWAPs shifted to the front): the
    permutation pass runs first, then the relabelled ladder; same state as the oracle, also sharded."""
    n = 18
    circ = C.qft_swaps_first(n)
    ref = _orc_run(orc, n, circ)
    for P in (1, 4):
        got, norm = _gpu_run(n, circ, P=P, virtual=P > 1)
        assert_parity(got, ref, len(circ), f"QFT swaps-first P={P}")
        assert abs(1 - norm) <= NORM_TOL


def test_qft_blocked_variant(orc):
    """The paper's cache-blocked QFT with blocking factor 16 (reading R22) at n = 20: fused
    path and 4 virtual shards against the oracle."""
    n = 20
    circ = C.qft_blocked(n, 16)
    ref = _orc_run(orc, n, circ)
    for P in (1, 4):
        got, norm = _gpu_run(n, circ, P=P, virtual=P > 1)
        assert_parity(got, ref, len(circ), f"QFT blocked(16) P={P}")
        assert abs(1 - norm) <= NORM_TOL


def test_paper_rqc_ring(orc):
    n = 16
    circ = C.rqc_ring(n, layers=5)
    got, _ = _gpu_run(n, circ, init=("basis", 0))
    ref = _orc_run(orc, n, circ, init=("basis", 0))
    assert_parity(got, ref, len(circ), "ring RQC")


def test_hadamard_all_closed_form():
    for n in (1, 7, 20):
        got, _ = _gpu_run(n, [C.g1(t, G.H) for t in range(n)], init=("basis", 0))
        target = 2.0 ** (-n / 2)
        assert np.all(got.imag == 0)
        assert np.max(np.abs(got.real - target)) <= n * 2.0 ** -53 * target


# ------------------------------------------------------------------------------------------------
# sharded path on one GPU (virtual shards: same planner, pack/unpack and fused update kernels as
# the NCCL path; device copies stand in for send/recv)
# ------------------------------------------------------------------------------------------------
@pytest.mark.parametrize("P", [2, 4, 8])
def test_config1_sharded(orc, P):
    n = 20
    circ = C.config1(n)
    single, _ = _gpu_run(n, circ, reorder=0, factor=0)
    got, norm = _gpu_run(n, circ, P=P, virtual=True, reorder=0, factor=0)
    assert np.array_equal(got, single), "P-invariance (bitwise, gate order)"
    ref = _orc_run(orc, n, circ)
    assert_parity(got, ref, len(circ), f"config1 P={P}")
    got, _ = _gpu_run(n, circ, P=P, virtual=True)
    assert_parity(got, ref, len(circ), f"config1 P={P} reordered")
    assert abs(1 - norm) <= NORM_TOL


@pytest.mark.parametrize("P,chunk", [(2, None), (4, 4096), (8, 4096), (8, None)])
def test_mixed_global_gates_sharded(orc, P, chunk):
    """Every routing class on global qubits, fused and unfused, through the fused peer-memory kernels
    (p2p=1, k_p2p.cu) and through the buffered exchange (p2p=0, the NCCL path's pack / update kernels):
    bit for bit the single-GPU result."""
    n = 14
    rng = np.random.Generator(np.random.PCG64(P))
    circ = []
    for q in range(n):
        circ.append(C.g1(q, G.haar(2, rng)))
    for (c, t) in [(n - 1, 2), (2, n - 1), (n - 1, n - 2), (n - 2, n - 1), (0, n - 1), (n - 1, 0), (n - 3, 1)]:
        circ += [C.gc(c, t, G.haar(2, rng)), C.gc(c, t, G.X), C.gc(c, t, G.phase(rng.random() * 6)),
                 C.g2(c, t, G.haar(4, rng)), C.g2(c, t, G.SWAP)]
    circ += [C.g2(n - 1, n - 2, np.diag(np.exp(1j * rng.random(4)))), C.g1(n - 1, G.T)]
    single, _ = _gpu_run(n, circ, reorder=0, factor=0)
    # p2p=0: the buffered pipeline of the NCCL path (comm stream, double buffers, events); vtransport=1
    # moves its chunks with ncclSend/ncclRecv (to self, one-rank communicator) instead of device copies
    for fuse, p2p, vt in ((False, 1, 0), (True, 1, 0), (False, 0, 0), (True, 0, 0), (False, 0, 1), (True, 0, 1)):
        got, norm = _gpu_run(n, circ, P=P, virtual=True, fuse=fuse, chunk=chunk, reorder=0, factor=0, p2p=p2p,
                             vtransport=vt)
        assert np.array_equal(got, single), f"P={P} fuse={fuse} p2p={p2p} vtransport={vt} not bitwise equal to P=1"
    ref = _orc_run(orc, n, circ)
    assert_parity(single, ref, len(circ), "mixed P=1")
    assert abs(1 - norm) <= NORM_TOL


@pytest.mark.parametrize("P,vt", [(2, 0), (2, 1), (8, 0), (8, 1)])
def test_buffered_exchange_long_pipeline(P, vt):
    """The buffered exchange with hundreds of chunks per gate (chunk 4 KiB, shard 8 MiB at n = 20, P = 2):
    receive buffers are reused every second chunk and pack buffers refilled two chunks ahead, so a missing
    event between the comm and compute streams would corrupt amplitudes.  Bitwise equal to P = 1."""
    n = 20
    rng = np.random.Generator(np.random.PCG64(40 + P))
    g = n - 1
    circ = [C.g1(g, G.haar(2, rng)), C.gc(3, g, G.haar(2, rng)), C.g2(5, g, G.SWAP), C.gc(g, 4, G.X),
            C.g2(g - 1, g, G.haar(4, rng)), C.g1(g - 1, G.haar(2, rng)), C.gc(2, g - 1, G.X)]
    single, _ = _gpu_run(n, circ, reorder=0, factor=0, fuse=False)
    got, norm = _gpu_run(n, circ, P=P, virtual=True, fuse=False, chunk=4096, reorder=0, factor=0, p2p=0,
                         vtransport=vt, )
    assert np.array_equal(got, single), f"P={P} vtransport={vt}"
    assert abs(1 - norm) <= NORM_TOL


@pytest.mark.parametrize("P", [2, 4, 8])
def test_global_remap_bitwise_and_fewer_exchanges(orc, P):
    """Global-qubit remapping (swap-to-local + relabelled SWAPs + restoring SWAPs): bit-for-bit the
    gate-by-gate exchange result (same arithmetic on the same amplitude pairs) and no more exchange
    volume (planner's count) for the grid RQC and the QFT; parity with the oracle with every default on."""
    n = 16
    for circ, init in ((C.rqc_grid(12, depth=12) + C.config1(16), ("random", 3)), (C.qft(n), ("basis", C.qft_x(n)))):
        res, ex = {}, {}
        for remap in (0, 1):
            with qs.QState(n, P, virtual=True) as st:
                st.set_option("remap", remap)
                st.set_option("reorder", 0)
                st.set_option("factor", 0)
                st.set_option("ladder_min", 0)
                st.init_random(init[1]) if init[0] == "random" else st.init_basis(init[1])
                st.run(circ)
                res[remap] = st.read()
                ex[remap] = st.last_plan()[1]
        assert np.array_equal(res[0], res[1])
        assert ex[0] > 0 and ex[1] > 0, ex  # steps may grow: half-shard swaps replace full exchanges
        _, (vol0, vol1) = qs.qs.qs_plan_remap(n, n - (P.bit_length() - 1), circ)
        assert vol1 <= vol0
        got, norm = _gpu_run(n, circ, init=init, P=P, virtual=True)
        ref = _orc_run(orc, n, circ, init=init)
        assert_parity(got, ref, len(circ), f"remap P={P}")
        assert abs(1 - norm) <= NORM_TOL


def test_init_random_sharding_invariant():
    n = 20
    with qs.QState(n) as a:
        a.init_random(2506)
        va = a.read()
    for P in (2, 8):
        with qs.QState(n, P, virtual=True) as b:
            b.init_random(2506)
            assert np.array_equal(b.read(), va)
            b.init_basis((1 << n) - 3)
            v = b.read()
            assert v[(1 << n) - 3] == 1 and np.count_nonzero(v) == 1


@pytest.mark.parametrize("P", [4, 8])
def test_qft_rqc_sharded(orc, P):
    n = 16
    for circ, init in ((C.qft(n), ("basis", C.qft_x(n))), (C.rqc_grid(12, depth=10) + C.qft(n), ("random", 1))):
        single, _ = _gpu_run(n, circ, init=init, ladder=0, reorder=0, factor=0)
        got, _ = _gpu_run(n, circ, init=init, P=P, virtual=True, ladder=0, reorder=0, factor=0)
        assert np.array_equal(got, single)
        ref = _orc_run(orc, n, circ, init=init)
        assert_parity(got, ref, len(circ), f"sharded P={P}")
        got, _ = _gpu_run(n, circ, init=init, P=P, virtual=True)  # PHASE LADDERS (default)
        assert_parity(got, ref, len(circ), f"sharded P={P} ladders")


# ------------------------------------------------------------------------------------------------
# boundary conditions and errors
# ------------------------------------------------------------------------------------------------
def test_errors_and_edges():
    with qs.QState(10, 2, virtual=True) as st:  # exchange chunks must divide every exchange
        for bad in (12288, 4095, 0, -4096):
            with pytest.raises(qs.QSError) as e:
                st.set_option("chunk_bytes", bad)
            assert e.value.code == 1
        st.set_option("chunk_bytes", 8192)
    with qs.QState(4) as st:
        with pytest.raises(qs.QSError) as e:
            st.apply_1q(4, G.X)
        assert e.value.code == 1
        with pytest.raises(qs.QSError):
            st.apply_ctrl_1q(1, 1, G.X)
        with pytest.raises(qs.QSError):
            st.apply_2q(2, 2, G.SWAP)
        with pytest.raises(qs.QSError) as e:
            st.init_basis(16)
        assert e.value.code == 2
        with pytest.raises(qs.QSError) as e:
            st.read(10, 7)
        assert e.value.code == 2
        bad = np.array([[1, 1], [0, 1]], dtype=complex)
        with pytest.raises(qs.QSError):
            st.apply_1q(0, bad)
        st.set_option("check_unitary", 0)
        st.apply_1q(0, bad)  # accepted when the check is off
        with pytest.raises(qs.QSError):
            st.set_option("nonsense", 1)
        st.run([])  # empty circuit: no-op
        st.init_basis(5)
        st.run([])
        assert st.read()[5] == 1
    with pytest.raises(qs.QSError):
        qs.QState(0)
    with pytest.raises(qs.QSError):
        qs.QState(7, 2, virtual=True)  # m = 6 < QS_MIN_LOCAL
    with pytest.raises(qs.QSError):
        qs.QState(10, 3, virtual=True)


def test_graph_replay_bitwise():
    """Option "graph": the repeats of a circuit on a single-shard handle replay a captured CUDA graph of the
    run; the states are bit for bit the directly launched runs', the kernel count per run is the same, and
    alternating circuits keep their own graphs."""
    n = 20
    circs = [C.qft(n), C.rqc_grid(20, depth=12), C.config1(n) + C.sweep_2q(qset=(0, 1, 5, 12, 18, 19))]
    res = {}
    for graph in (0, 1):
        with qs.QState(n) as st:
            st.set_option("graph", graph)
            st.set_option("jit_async", 0)
            out = []
            for rep in range(3):
                for ci, c in enumerate(circs):
                    st.init_random(11 + ci)
                    before = st.launches()
                    st.run(c)
                    st.sync()
                    out.append((st.read(), st.launches() - before, st.last_plan()[0]))
            res[graph] = out
    for (a, la, pa), (b, lb, pb) in zip(res[0], res[1]):
        assert np.array_equal(a, b) and la == lb and pa == pb


def test_plain_c_program_uses_the_abi():
    """examples/qs_hello.c (built beside the library): the C-ABI driven from plain C — H on 20 qubits and a
    20-qubit QFT of a basis state through qs_run_circuit, each checked against its closed form in C."""
    import os
    import subprocess
    exe = os.path.join(os.path.dirname(qs.__file__), "qs_hello")
    assert os.path.exists(exe), "build() compiles examples/qs_hello.c"
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "QFT(20)" in r.stdout


def test_launch_count_and_stream():
    with qs.QState(16) as st:
        n0 = st.launches()
        st.run(C.qft(16))
        st.sync()
        assert st.launches() > n0
        assert st.stream(0) != 0
        passes, exch = st.last_plan()
        assert 0 < passes < 20 and exch == 0


# ------------------------------------------------------------------------------------------------
# full BASELINE sizes (n = 30, 16 GiB), the launch configuration bench.py times
# ------------------------------------------------------------------------------------------------
@pytest.mark.slow
def test_n30_sweeps_vs_oracle(orc):
    """configs[1] + configs[2] at n = 30 on one GPU, each gate once, against the oracle on the host
    (needs ~34 GiB of host RAM)."""
    import psutil
    if psutil.virtual_memory().available < 40 * 2 ** 30:
        pytest.skip("host RAM < 40 GiB for the n=30 oracle")
    n = 30
    circ = C.sweep_1q(n) + C.sweep_2q()
    with qs.QState(n) as st:
        st.set_option("fuse", 0)
        st.init_random(2506)
        st.run(circ)
        st.sync()
        norm = st.norm2()
        ref = orc.random_state(n, 2506)
        orc.run(ref, circ)
        worst = 0.0
        step = 1 << 26
        buf = np.empty(step, dtype=np.complex128)
        for s in range(0, 1 << n, step):
            qs.qs_read_amps(st.h, s, step, buf)
            worst = max(worst, float(np.max(np.abs(buf - ref[s:s + step]))))
    assert worst <= 1e-10 and worst <= 32 * len(circ) * 2.0 ** -53 * float(np.max(np.abs(ref)))
    assert abs(1 - norm) <= NORM_TOL


@pytest.mark.slow
def test_n30_qft_basis_sampled():
    """configs[4] shape at n = 30 (fused path): QFT|x> vs the closed form at sampled outputs."""
    n = 30
    x = C.qft_x(n)
    with qs.QState(n) as st:
        st.init_basis(x)
        st.run(C.qft(n))
        norm = st.norm2()
        rng = np.random.default_rng(0)
        starts = list(rng.integers(0, (1 << n) - 65536, size=16)) + [0, (1 << n) - 65536]
        worst = 0.0
        for s in starts:
            got = st.read(int(s), 65536)
            y = np.arange(int(s), int(s) + 65536, dtype=np.uint64)
            k = (np.uint64(x) * y) % np.uint64(1 << n)
            ang = np.pi * k.astype(np.float64) / 2.0 ** (n - 1)
            ref = (np.cos(ang) + 1j * np.sin(ang)) * 2.0 ** (-n / 2)
            worst = max(worst, float(np.max(np.abs(got - ref))))
    assert worst <= 1e-10 and worst <= 32 * len(C.qft(n)) * 2.0 ** -53 * 2.0 ** (-n / 2)
    assert abs(1 - norm) <= NORM_TOL


# ------------------------------------------------------------------------------------------------
# BASELINE configs[3]/[4] sizes on one GPU (n = 32, 64 GiB): properties that hold at any size
# ------------------------------------------------------------------------------------------------
@pytest.mark.slow
def test_n32_qft_basis_sampled_and_sharding_invariance():
    """QFT(32)|x> vs the closed form at sampled outputs (fused + JIT + PHASE LADDER path, the
    configuration bench.py times), and the same circuit on 8 virtual shards (gate-by-gate phases)
    agrees at those samples within the tight alarm."""
    n = 32
    x = C.qft_x(n)
    circ = C.qft(n)
    rng = np.random.default_rng(1)
    # 256 contiguous blocks of 65,536 at seeded offsets (2^24 amplitudes) plus +-4096
    # around every shard boundary of the P = 8 run (8192-amplitude windows centred on d * 2^29)
    ranges = [(int(s), 65536) for s in rng.integers(0, (1 << n) - 65536, size=256)] + [(0, 65536), ((1 << n) - 65536, 65536)]
    ranges += [((d << (n - 3)) - 4096, 8192) for d in range(1, 8)]
    got = {}
    for P in (1, 8):
        with qs.QState(n, P, virtual=P > 1) as st:
            if P > 1:
                st.set_option("ladder_min", 0)  # gate-by-gate phases on the sharded run
            st.init_basis(x)
            st.run(circ)
            got[P] = [st.read(s, c) for s, c in ranges]
            norm = st.norm2()
            assert abs(1 - norm) <= NORM_TOL
    worst = 0.0
    for (s, _), a, b in zip(ranges, got[1], got[8]):
        assert np.max(np.abs(a - b)) <= 32 * len(circ) * 2.0 ** -53 * 2.0 ** (-n / 2)
        y = np.arange(s, s + a.size, dtype=np.uint64)
        k = (np.uint64(x) * y) % np.uint64(1 << n)
        ang = np.pi * k.astype(np.float64) / 2.0 ** (n - 1)
        ref = (np.cos(ang) + 1j * np.sin(ang)) * 2.0 ** (-n / 2)
        worst = max(worst, float(np.max(np.abs(a - ref))))
    assert worst <= 1e-10 and worst <= 32 * len(circ) * 2.0 ** -53 * 2.0 ** (-n / 2)


@pytest.mark.slow
def test_n33_single_gpu_indices_beyond_2_32():
    """The largest single-B200 state (n = 33, 128 GiB, unsharded): indices beyond 2^32 in the gate
    kernels (H on qubit 32 and 0, then CNOT 32 -> 1, one kernel per gate: four amplitudes of 1/2 at
    closed-form positions) and in the fused path (QFT(33)|x> against the closed form at sampled outputs)."""
    n = 33
    with qs.QState(n) as st:
        st.init_basis(0)
        st.apply_1q(32, G.H)
        st.apply_1q(0, G.H)
        st.apply_ctrl_1q(32, 1, G.X)
        for i in (0, 1, (1 << 32) + 2, (1 << 32) + 3):
            assert abs(st.read(i, 1)[0] - 0.5) <= 1e-15, i
        for i in (2, 3, 1 << 32, (1 << 32) + 1, (1 << 33) - 1):
            assert st.read(i, 1)[0] == 0, i
        assert abs(1 - st.norm2()) <= NORM_TOL
        x = C.qft_x(n)
        circ = C.qft(n)
        st.init_basis(x)
        st.run(circ)
        rng = np.random.default_rng(3)
        starts = [int(v) for v in rng.integers(0, (1 << n) - 65536, size=8)] + [(1 << 32) - 32768, (1 << n) - 65536]
        worst = 0.0
        for s0 in starts:
            a = st.read(s0, 65536)
            y = np.arange(s0, s0 + 65536, dtype=np.uint64)
            k = (np.uint64(x) * y) % np.uint64(1 << n)  # uint64 products wrap mod 2^64: exact mod 2^33
            ang = np.pi * k.astype(np.float64) / 2.0 ** (n - 1)
            ref = (np.cos(ang) + 1j * np.sin(ang)) * 2.0 ** (-n / 2)
            worst = max(worst, float(np.max(np.abs(a - ref))))
        assert worst <= 1e-10 and worst <= 32 * len(circ) * 2.0 ** -53 * 2.0 ** (-n / 2)
        assert abs(1 - st.norm2()) <= NORM_TOL


@pytest.mark.slow
def test_n33_qft_sharded_p8_sampled():
    """The sharded path at scale: QFT(33)|x> on 8 virtual shards (128 GiB; global-qubit remapping,
    fused peer-memory exchange kernels, phase ladders with rank-folded controls, the permutation pass
    for the local part of the reversal) against the closed form at sampled outputs, and the norm."""
    import torch
    n, P = 33, 8
    if torch.cuda.get_device_properties(0).total_memory < 150 * 2 ** 30:
        pytest.skip("needs ~140 GiB of device memory")
    x = C.qft_x(n)
    circ = C.qft(n)
    rng = np.random.default_rng(3)
    starts = [int(s) for s in rng.integers(0, (1 << n) - 65536, size=10)] + [0, (1 << n) - 65536,
                                                                             (1 << (n - 3)) * 5 - 32768]
    with qs.QState(n, P, virtual=True) as st:
        st.init_basis(x)
        st.run(circ)
        norm = st.norm2()
        worst = 0.0
        for s0 in starts:
            got = st.read(s0, 65536)
            y = np.arange(s0, s0 + 65536, dtype=np.uint64)
            k = (np.uint64(x) * y) % np.uint64(1 << n)
            ang = np.pi * k.astype(np.float64) / 2.0 ** (n - 1)
            ref = (np.cos(ang) + 1j * np.sin(ang)) * 2.0 ** (-n / 2)
            worst = max(worst, float(np.max(np.abs(got - ref))))
    assert worst <= 1e-10 and worst <= 32 * len(circ) * 2.0 ** -53 * 2.0 ** (-n / 2), worst
    assert abs(1 - norm) <= NORM_TOL


@pytest.mark.slow
def test_n32_rqc_round_trip():
    """Grid RQC(32) (900 gates) then its inverse from |0..0>: amplitude 0 returns to 1, the rest to 0
    (SURVEY.md §8(c) c.5 'Any circuit'), norm kept to 1e-12 after the forward circuit."""
    n = 32
    circ = C.rqc_grid(n)
    with qs.QState(n) as st:
        st.init_basis(0)
        st.run(circ)
        assert abs(1 - st.norm2()) <= NORM_TOL
        st.run(C.inverse(circ))
        assert abs(1 - st.norm2()) <= NORM_TOL  # and after C-dagger (1800 gates)
        head = st.read(0, 1 << 16)
        tail = st.read((1 << n) - (1 << 16), 1 << 16)
    assert abs(head[0] - 1.0) <= 1e-10
    assert np.max(np.abs(head[1:])) <= 1e-10 and np.max(np.abs(tail)) <= 1e-10


def test_canary_guards_all_paths(monkeypatch):
    """Bounds check of our own (compute-sanitizer is closed on this pool): with QS_DEBUG_CANARY=1 every
    shard sits between 1 MiB guard regions that qs_sync verifies.  Exercise every kernel family at the
    edges of the index space (t = 0, 1, m-1; qubit 0 as control / phase bit), the fused tile path, and
    the sharded exchange (global targets, SWAP local<->global, 2q via swap-to-local, 4 KiB chunks)."""
    monkeypatch.setenv("QS_DEBUG_CANARY", "1")
    rng = np.random.Generator(np.random.PCG64(99))
    for n, P in ((3, 1), (8, 1), (14, 1), (12, 4), (14, 8)):
        m = n - (P.bit_length() - 1)
        circ = []
        for t in sorted({0, 1, m - 1, n - 1}):
            circ += [C.g1(t, G.haar(2, rng)), C.g1(t, G.T)]
        for (a, b) in {(0, 1), (1, 0), (0, n - 1), (n - 1, 0), (m - 1, n - 1), (n - 2, n - 1)}:
            if a == b:
                continue
            circ += [C.gc(a, b, G.haar(2, rng)), C.gc(a, b, G.X), C.gc(a, b, G.phase(0.4)),
                     C.g2(a, b, G.haar(4, rng)), C.g2(a, b, G.SWAP)]
        for fuse in (0, 1):
            with qs.QState(n, P, virtual=P > 1) as st:
                if P > 1:
                    st.set_option("chunk_bytes", 4096)
                st.set_option("fuse", fuse)
                st.init_random(3)
                st.run(circ)
                for g in circ[:6]:
                    st.apply(g)
                st.sync()  # raises if a guard byte changed
                assert abs(1 - st.norm2()) <= NORM_TOL


def test_rank_mode_world1_equals_single():
    """qs_create_rank (the one-process-per-GPU entry point bench.py uses under torchrun) at world 1."""
    n = 16
    circ = C.config1(n) + C.qft(n)
    uid = qs.qs_get_unique_id()
    assert len(uid) == 128
    with qs.QState.rank(n, 1, 0, 0, uid) as st:
        st.init_random(7)
        st.run(circ)
        a = st.read()
        na = st.norm2()
        with pytest.raises(qs.QSError):
            qs.qs_read_amps(st.h, (1 << n) - 1, 2)  # outside the shard / state
    with qs.QState(n) as st:
        st.init_random(7)
        st.run(circ)
        b = st.read()
        nb = st.norm2()
    assert np.array_equal(a, b) and na == nb
