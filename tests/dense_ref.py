"""Dense 2^n x 2^n embedding of a gate via numpy.kron (test-side pin for the oracle, n <= 9).

Independent of the oracle's index arithmetic: a gate acting on qubit set Q is written as a sum
of tensor products of single-qubit operators and expanded with np.kron, the most significant
factor being qubit n-1 (qubit t = bit t).  SURVEY.md §8(c) c.2 O10 / c.5.
"""
import numpy as np

P0 = np.array([[1, 0], [0, 0]], dtype=np.complex128)
P1 = np.array([[0, 0], [0, 1]], dtype=np.complex128)
I2 = np.eye(2, dtype=np.complex128)


def E(a, b):
    """|a><b| on one qubit."""
    m = np.zeros((2, 2), dtype=np.complex128)
    m[a, b] = 1.0
    return m


def kron_chain(n, ops):
    """ops: dict qubit -> 2x2; identity elsewhere; qubit n-1 is the leftmost factor."""
    out = np.ones((1, 1), dtype=np.complex128)
    for q in range(n - 1, -1, -1):
        out = np.kron(out, ops.get(q, I2))
    return out


def dense_1q(n, t, U):
    return kron_chain(n, {t: np.asarray(U)})


def dense_ctrl_1q(n, c, t, U):
    return kron_chain(n, {c: P0}) + kron_chain(n, {c: P1, t: np.asarray(U)})


def dense_2q(n, q0, q1, U4):
    """U4 indexed by k = bit_q0 + 2 bit_q1:  sum_{r,s} U4[r,s] |r><s| with |k> = |bit_q1>|bit_q0>."""
    U4 = np.asarray(U4)
    M = np.zeros((1 << n, 1 << n), dtype=np.complex128)
    for r in range(4):
        for s in range(4):
            if U4[r, s] == 0:
                continue
            M += U4[r, s] * kron_chain(n, {q0: E(r & 1, s & 1), q1: E(r >> 1, s >> 1)})
    return M


def dense_gate(n, g):
    if g.kind == "1q":
        return dense_1q(n, g.q0, g.m)
    if g.kind == "c1q":
        return dense_ctrl_1q(n, g.q0, g.q1, g.m)
    return dense_2q(n, g.q0, g.q1, g.m)


def dense_run(psi, gates):
    n = int(psi.size).bit_length() - 1
    out = psi.copy()
    for g in gates:
        out = dense_gate(n, g) @ out
    return out
