"""Mutation check of the oracle's pins (CPU): copies of oracle/orc.c with one plausible mistake each — a
sign in the complex product, a transposed gate matrix, the control semantics, the 2q sub-index
convention, a dropped term, the Box–Muller radius or angle, the Alg. 1 index arithmetic, the norm —
are compiled and run through a battery of the pins' checks (dense numpy Kronecker products, closed
forms, distribution moments, worked examples).  Every mutant must fail the battery and the unmodified
source must pass it, so a mistake of these kinds in the oracle could not hide behind its own pins.
"""
import subprocess

import numpy as np
import pytest

from dense_ref import dense_run
from oracle import Oracle
from oracle.orc import CFLAGS, SRC
from qsinputs import circuits as C
from qsinputs import gates as G

MUTANTS = {
    "cmul_real_sign": ("*cr = ur * xr - ui * xi;", "*cr = ur * xr + ui * xi;"),
    "cmul_imag_sign": ("*ci = ur * xi + ui * xr;", "*ci = ur * xi - ui * xr;"),
    "1q_matrix_transposed": ("cmul(u[2], u[3], yr, yi, &p1r, &p1i);\n    cmul(u[4], u[5], xr, xi, &p2r, &p2i);",
                             "cmul(u[4], u[5], yr, yi, &p1r, &p1i);\n    cmul(u[2], u[3], xr, xi, &p2r, &p2i);"),
    "1q_update_dropped_term": ("a[2 * up] = p0r + p1r;", "a[2 * up] = p0r;"),
    "control_on_zero": ("if (((ui >> c) & 1) == 1 && ((ui >> t) & 1) == 0)", "if (((ui >> c) & 1) == 0 && ((ui >> t) & 1) == 0)"),
    "2q_q0_q1_swapped": ("((uint64_t)(s & 1) << q0) | ((uint64_t)(s >> 1) << q1)",
                         "((uint64_t)(s & 1) << q1) | ((uint64_t)(s >> 1) << q0)"),
    "2q_accumulate_sign": ("accr = accr + pr;", "accr = accr - pr;"),
    "box_muller_radius": ("sqrt(-2.0 * log(u1))", "sqrt(-1.0 * log(u1))"),
    "box_muller_angle": ("double ang = 2.0 * M_PI * u2;", "double ang = M_PI * u2;"),
    "alg1_block_stride": ("*indexUp = thisBlock * sizeBlock + (thisTask % sizeHalfBlock);",
                          "*indexUp = thisBlock * sizeHalfBlock + (thisTask % sizeHalfBlock);"),
    "norm_drops_imag": ("s = s + (re * re + im * im);", "s = s + (re * re);"),
}


def _build(tmp_path, name, repl):
    src = open(SRC).read()
    if repl is not None:
        old, new = repl
        assert src.count(old) == 1, name  # the mutation site exists exactly once
        src = src.replace(old, new)
    c = tmp_path / f"{name}.c"
    c.write_text(src)
    so = tmp_path / f"lib{name}.so"
    subprocess.check_call(["gcc", *CFLAGS, str(c), "-o", str(so), "-lm"])
    return Oracle.from_library(str(so))


def _battery(o):
    """The pins' kinds of checks, small sizes; raises AssertionError on the first failure."""
    rng = np.random.Generator(np.random.PCG64(5))
    # Alg. 1 worked example (tests/golden/alg1_index.txt: task 5, t = 2 -> (9, 13))
    # and the bijection at t = 2
    assert o.pair_index(5, 2) == (9, 13)
    seen = sorted(i for k in range(16) for i in o.pair_index(k, 2))
    assert seen == list(range(32))
    # norm of a known vector vs numpy
    v = rng.normal(size=64) + 1j * rng.normal(size=64)
    assert abs(o.norm2(v) - float(np.sum(np.abs(v) ** 2))) <= 1e-12 * float(np.sum(np.abs(v) ** 2))
    # Box–Muller moments: E[re^2 + im^2] = 2, E[re] = E[im] = 0, E[re im] = 0 (20000 samples)
    s = np.array([o.gauss2(2506, i) for i in range(20000)])
    assert abs(np.mean(s[:, 0] ** 2 + s[:, 1] ** 2) - 2.0) < 0.1
    assert abs(np.mean(s[:, 0])) < 0.05 and abs(np.mean(s[:, 1])) < 0.05
    assert abs(np.mean(np.arctan2(s[:, 1], s[:, 0]) > 0) - 0.5) < 0.03  # angle uniform on the circle
    # dense Kronecker products: every gate kind on random positions of a random 5-qubit state
    n = 5
    a = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    circ = []
    for _ in range(12):
        q = [int(x) for x in rng.choice(n, size=2, replace=False)]
        circ += [C.g1(q[0], G.haar(2, rng)), C.gc(q[0], q[1], G.haar(2, rng)), C.g2(q[0], q[1], G.haar(4, rng))]
    ref = dense_run(a, circ)
    got = a.copy()
    o.run(got, circ)
    assert np.max(np.abs(got - ref)) <= 1e-12 * np.max(np.abs(ref))
    # H^n |0> = uniform
    b = o.basis(n, 0)
    o.run(b, [C.g1(t, G.H) for t in range(n)])
    assert np.max(np.abs(b - 2.0 ** (-n / 2))) <= 1e-15


def test_unmutated_oracle_passes_battery(tmp_path):
    _battery(_build(tmp_path, "original", None))


@pytest.mark.parametrize("name", sorted(MUTANTS))
def test_every_mutant_is_caught(tmp_path, name):
    o = _build(tmp_path, name, MUTANTS[name])
    with pytest.raises(AssertionError):
        _battery(o)
