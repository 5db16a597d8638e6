"""GPU parity at the TIMED sizes (BASELINE configs[3]/[4], n = 32, 64 GiB).

bench.py times grid RQC(32) and QFT(32) through the default fused path (tile passes, JIT, phase ladders,
scalar factoring, commutation-aware scheduling).  These tests check the states those runs produce:

  * RQC(32) from |0..0>, default options, against the same circuit through the per-gate kernels
    (fuse = 0, gate order) — the kernels tests/test_gpu_parity.py::test_n30_sweeps_vs_oracle pins to
    the oracle element by element — over ALL 2^32 amplitudes, at the contract bar 1e-10 and the tight
    alarm 32 G eps max|psi|; and against the same circuit on 8 virtual shards
    (global-qubit remapping; fused peer-memory exchange kernels, and the buffered NCCL exchange pipeline),
    again over all 2^32 amplitudes;
  * QFT(32) of the normalised random state gauss2(2506) (configs[4]'s second input) against DFT sums
    at 32 sampled outputs, formed on the host from the ORACLE's samples (tests/dft_check.py, pinned
    against numpy ifft by tests/test_oracle_pins.py).

PAPER.md:L295 (QFT), L327 (RQC).
"""
import numpy as np
import pytest
import torch

import paper_2506_09198_b200 as qs
from gpu_util import ABS_TOL, EPS, NORM_TOL
from qsinputs import circuits as C

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module", autouse=True)
def lib():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device (no CPU fallback exists)")
    return qs.load_library()


def _compare_all(a, b, n, chunk_bits=26):
    """max |a - b| (complex modulus) and max |a| over all 2^n amplitudes, read back chunk by chunk."""
    step = 1 << chunk_bits
    ba = np.empty(step, dtype=np.complex128)
    bb = np.empty(step, dtype=np.complex128)
    worst, amax = 0.0, 0.0
    for s in range(0, 1 << n, step):
        qs.qs_read_amps(a.h, s, step, ba)
        qs.qs_read_amps(b.h, s, step, bb)
        ta, tb = torch.from_numpy(ba), torch.from_numpy(bb)
        worst = max(worst, float((ta - tb).abs().max()))
        amax = max(amax, float(tb.abs().max()))
    return worst, amax


def test_n32_rqc_fused_vs_pergate_and_sharded_all_amplitudes():
    n = 32
    circ = C.rqc_grid(n)
    G = len(circ)
    if torch.cuda.get_device_properties(0).total_memory < 150 * 2 ** 30:
        pytest.skip("needs two 64-GiB states on one device")
    with qs.QState(n) as fused:
        fused.init_basis(0)
        fused.run(circ)
        norm = fused.norm2()
        assert abs(1 - norm) <= NORM_TOL
        with qs.QState(n) as ref:
            ref.set_option("fuse", 0)
            ref.set_option("reorder", 0)
            ref.init_basis(0)
            ref.run(circ)
            assert ref.last_plan()[0] == G  # one kernel per gate
            worst, amax = _compare_all(fused, ref, n)
        tight = 32 * G * EPS * amax
        assert worst <= ABS_TOL and worst <= tight, f"fused vs per-gate: max|d| {worst:.3e}, tight {tight:.3e}"
        assert amax > 0
        # 8 virtual shards twice: the fused peer-memory exchange kernels (default), and the buffered
        # exchange pipeline of the multi-GPU path with its chunks moved by ncclSend/ncclRecv (to self, one-rank
        # communicator: vtransport 1) in 256-MiB chunks — every exchange of the remapped circuit at full size
        for p2p, vt in ((1, 0), (0, 1)):
            with qs.QState(n, 8, virtual=True) as sh:
                sh.set_option("p2p", p2p)
                sh.set_option("vtransport", vt)
                sh.init_basis(0)
                sh.run(circ)
                assert sh.last_plan()[1] > 0  # exchange steps ran
                assert abs(1 - sh.norm2()) <= NORM_TOL
                worst8, _ = _compare_all(sh, fused, n)
            assert worst8 <= ABS_TOL and worst8 <= tight, f"P=8 (p2p={p2p}) vs P=1: max|d| {worst8:.3e}, tight {tight:.3e}"


def test_n32_qft_random_state_vs_dft_sums(orc):
    from dft_check import qft_random_state_samples
    n = 32
    circ = C.qft(n)
    rng = np.random.default_rng(2532)
    ys = [0, 1, 2, (1 << n) - 1, 1 << (n - 1), (1 << 29) - 1, 1 << 29] + [int(v) for v in rng.integers(0, 1 << n, size=25)]
    with qs.QState(n) as st:
        st.init_random(2506)
        st.run(circ)
        norm = st.norm2()
        got = np.array([st.read(y, 1)[0] for y in ys])
    ref, s2 = qft_random_state_samples(orc, n, 2506, ys)
    err = float(np.max(np.abs(got - ref)))
    tight = 32 * len(circ) * EPS * float(np.max(np.abs(ref)))
    assert err <= ABS_TOL and err <= tight, f"max|d| {err:.3e}, tight {tight:.3e}"
    assert abs(1 - norm) <= NORM_TOL
    assert abs(s2 / (1 << n) - 2.0) < 1e-3  # E|g|^2 = 2 over 2^32 samples
