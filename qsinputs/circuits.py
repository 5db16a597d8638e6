"""Gate-list builders for the BASELINE.json workloads.

A circuit is a list of ``Gate``:
- kind "1q" : q0 = target,            m = 2x2
- kind "c1q": q0 = control, q1 = target, m = 2x2 applied to the target where the control bit is 1
- kind "2q" : (q0, q1),                m = 4x4 indexed by k = bit_q0 + 2*bit_q1
"""
from dataclasses import dataclass, field
from math import pi
from typing import List

import numpy as np

from . import gates as G
from .rng import SplitMix64Stream, splitmix64


@dataclass
class Gate:
    kind: str
    q0: int
    q1: int = -1
    m: np.ndarray = field(default_factory=lambda: np.eye(2, dtype=np.complex128))
    name: str = ""

    def qubits(self):
        return (self.q0,) if self.kind == "1q" else (self.q0, self.q1)


def g1(t, m, name=""):
    return Gate("1q", int(t), -1, np.asarray(m, dtype=np.complex128), name)


def gc(c, t, m, name=""):
    return Gate("c1q", int(c), int(t), np.asarray(m, dtype=np.complex128), name)


def g2(q0, q1, m, name=""):
    return Gate("2q", int(q0), int(q1), np.asarray(m, dtype=np.complex128), name)


def inverse(circ: List[Gate]) -> List[Gate]:
    """C^dagger: reversed order, each matrix conjugate-transposed (QFT: theta -> -theta)."""
    return [Gate(g.kind, g.q0, g.q1, g.m.conj().T.copy(), g.name + "^dag") for g in reversed(circ)]


# ---------------------------------------------------------------------------------------------
# QFT (BASELINE configs[4]; "Hadamard gate followed by controlled phase shifts")
# ---------------------------------------------------------------------------------------------
def qft(n: int) -> List[Gate]:
    """Iterative ladder (SURVEY.md §8(c) c.3 "QFT(n) gate list", reading R5):
    for t = n-1 .. 0: H(t); for c = t-1 .. 0: CPhase(c, t, pi/2^(t-c)); then SWAP(i, n-1-i).
    Output: QFT|x> = 2^(-n/2) sum_y e^{+2 pi i x y / 2^n} |y>."""
    out = []
    for t in range(n - 1, -1, -1):
        out.append(g1(t, G.H, "H"))
        for c in range(t - 1, -1, -1):
            out.append(gc(c, t, G.phase(pi / 2.0 ** (t - c)), f"R{t - c + 1}"))
    for i in range(n // 2):
        out.append(g2(i, n - 1 - i, G.SWAP, "SWAP"))
    return out


def qft_swaps_first(n: int) -> List[Gate]:
    """The QFT with its final qubit reversal shifted to the front ("cache-blocked without
    extra gates by shifting its ending SWAP gates to the left"; Adamski 2023): the reversal SWAPs, then
    the ladder on reversed labels — the same unitary as qft(n) (R = reversal: QFT = R L = (R L R) R)."""
    out = [g2(i, n - 1 - i, G.SWAP, "SWAP") for i in range(n // 2)]
    for g in qft(n)[: len(qft(n)) - n // 2]:
        r = lambda q: n - 1 - q
        out.append(Gate(g.kind, r(g.q0), r(g.q1) if g.q1 >= 0 else -1, g.m, g.name))
    return out


def qft_blocked(n: int, k: int) -> List[Gate]:
    """Cache-blocked QFT with blocking factor k ("cache-blocked ... ensuring that all
    Hadamard gates operate on local qubits", blocking factors 16 and 64; Adamski 2023; reading R22): the
    iterative ladder of qft(n) on a relabelled register in which every H acts on a physical qubit < k.
    Before the H of logical target t whose physical qubit is >= k, a SWAP brings it into the block, evicting
    the block's logical qubit needed furthest in the future (one already finished as a target, else the
    lowest: targets run n-1 .. 0); controlled phases follow their qubits' current positions; the final
    SWAPs realise the QFT's qubit reversal on top of the accumulated relabelling.  For k >= n this is
    qft(n).  Same unitary as qft(n)."""
    if k >= n:
        return qft(n)
    pos, at = list(range(n)), list(range(n))  # logical -> physical, physical -> logical
    out = []

    def swap(p, q):
        out.append(g2(p, q, G.SWAP, "SWAP"))
        a, b = at[p], at[q]
        at[p], at[q] = b, a
        pos[a], pos[b] = q, p

    for t in range(n - 1, -1, -1):
        if pos[t] >= k:
            done = [p for p in range(k) if at[p] > t]
            p = done[0] if done else min(range(k), key=lambda x: at[x])
            swap(p, pos[t])
        out.append(g1(pos[t], G.H, "H"))
        for c in range(t - 1, -1, -1):
            out.append(gc(pos[c], pos[t], G.phase(pi / 2.0 ** (t - c)), f"R{t - c + 1}"))
    # the reversal: logical q must end at physical n-1-q
    for q in range(n):
        want = n - 1 - q
        if pos[q] != want:
            swap(pos[q], want)
    return out


def qft_x(n: int, seed: int = 35) -> int:
    """The seeded basis input of config 5: x = SM(seed, 0) mod 2^n."""
    return splitmix64(seed, 0) % (1 << n)


# ---------------------------------------------------------------------------------------------
# Sycamore-style grid RQC (BASELINE configs[3]; reading R12)
# ---------------------------------------------------------------------------------------------
def grid_sites(rows: int, cols: int, drop=()):
    drop = set(drop)
    return [(r, c) for r in range(rows) for c in range(cols) if (r, c) not in drop]


def grid_for_n(n: int):
    """(rows, cols, dropped sites) for the grids SURVEY.md §8(c) c.3 names."""
    table = {
        34: (6, 6, [(5, 0), (5, 5)]),
        32: (6, 6, [(0, 0), (0, 5), (5, 0), (5, 5)]),
        12: (3, 4, []),
        20: (4, 5, []),
        25: (5, 5, []),
        36: (6, 6, []),
    }
    if n not in table:
        raise ValueError(f"no grid defined for n={n}")
    return table[n]


def grid_couplers(rows: int, cols: int, drop=()):
    """Patterns A/B (horizontal, c even/odd) and C/D (vertical, r even/odd), row-major edge
    order, edges touching a dropped site omitted.  Returns dict pattern -> [(qa, qb)]."""
    sites = grid_sites(rows, cols, drop)
    index = {s: i for i, s in enumerate(sites)}
    pats = {"A": [], "B": [], "C": [], "D": []}
    for r in range(rows):
        for c in range(cols):
            if (r, c) not in index:
                continue
            if c + 1 < cols and (r, c + 1) in index:
                pats["A" if c % 2 == 0 else "B"].append((index[(r, c)], index[(r, c + 1)]))
            if r + 1 < rows and (r + 1, c) in index:
                pats["C" if r % 2 == 0 else "D"].append((index[(r, c)], index[(r + 1, c)]))
    return pats


def rqc_grid(n: int, depth: int = 20, seed: int = 20) -> List[Gate]:
    """Grid RQC from |0..0>: cycle m applies to every qubit q (ascending) a pick from
    {sqrtX, sqrtY, sqrtW} (m=0: r mod 3; m>0: the (r mod 2)-th of the two gates != prev[q]),
    then CZ on every edge of pattern "ABCD"[m mod 4].  No final 1q layer."""
    rows, cols, drop = grid_for_n(n)
    pats = grid_couplers(rows, cols, drop)
    names = ["sqrtX", "sqrtY", "sqrtW"]
    mats = [G.SQRT_X, G.SQRT_Y, G.SQRT_W]
    s = SplitMix64Stream(seed)
    prev = [-1] * n
    out = []
    for m in range(depth):
        for q in range(n):
            r = s.next()
            if m == 0:
                k = r % 3
            else:
                choices = [i for i in range(3) if i != prev[q]]
                k = choices[r % 2]
            prev[q] = k
            out.append(g1(q, mats[k], names[k]))
        for (a, b) in pats["ABCD"[m % 4]]:
            out.append(gc(a, b, G.cz_target(), "CZ"))
    return out


def rqc_ring(n: int, layers: int = 5, seed: int = 20) -> List[Gate]:
    """The paper's RQC: L layers of a random 1q gate on every qubit, then
    CNOT(i -> (i+1) mod n).  Gate set {H, X, Y, T} (SPEC.md reading; the paper leaves it
    unstated).  SURVEY.md §8(f) rank 4."""
    mats = [G.H, G.X, G.Y, G.T]
    names = ["H", "X", "Y", "T"]
    s = SplitMix64Stream(seed)
    out = []
    for _ in range(layers):
        for q in range(n):
            k = s.next() % 4
            out.append(g1(q, mats[k], names[k]))
        for q in range(n):
            out.append(gc(q, (q + 1) % n, G.X, "CNOT"))
    return out


# ---------------------------------------------------------------------------------------------
# BASELINE configs 1-3
# ---------------------------------------------------------------------------------------------
def config1(n: int = 20, seed_gates: int = 9198) -> List[Gate]:
    """configs[0]: one Haar U2 on each target 0..n-1 in order, then one Haar U4 on each (q, q+1)."""
    rng = np.random.Generator(np.random.PCG64(seed_gates))
    out = [g1(t, G.haar(2, rng), "U2") for t in range(n)]
    out += [g2(q, q + 1, G.haar(4, rng), "U4") for q in range(n - 1)]
    return out


def sweep_1q(n: int = 30, seed_gates: int = 9198) -> List[Gate]:
    """configs[1]: one Haar U2 per target t = 0..n-1 (seeded per t)."""
    return [g1(t, G.haar(2, np.random.Generator(np.random.PCG64([seed_gates, t]))), "U2")
            for t in range(n)]


SWEEP_2Q_QUBITS = (0, 1, 5, 12, 20, 28, 29)


def sweep_2q(qset=SWEEP_2Q_QUBITS, seed_gates: int = 9198) -> List[Gate]:
    """configs[2]: for every pair q0 < q1 of ``qset``: CNOT(q0 -> q1), CPhase(q0, q1, theta),
    Haar U4(q0, q1); theta = 2 pi U[0,1) (reading R11, R13)."""
    rng = np.random.Generator(np.random.PCG64([seed_gates, 2]))
    out = []
    qs = sorted(qset)
    for i in range(len(qs)):
        for j in range(i + 1, len(qs)):
            q0, q1 = qs[i], qs[j]
            theta = 2 * pi * rng.random()
            out.append(gc(q0, q1, G.X, "CNOT"))
            out.append(gc(q0, q1, G.phase(theta), "CPhase"))
            out.append(g2(q0, q1, G.haar(4, rng), "U4"))
    return out


# ---------------------------------------------------------------------------------------------
# test workload for permutation hoisting: random gates, a run of disjoint SWAPs over
# (nearly) all qubits — a permutation pass no tile closes under — then more random gates
# ---------------------------------------------------------------------------------------------
def random_with_swap_run(n: int, seed: int, npre: int = 40, npost: int = 20) -> List[Gate]:
    rng = np.random.default_rng([seed, 6])

    def one():
        k = int(rng.integers(0, 5))
        a, b = (int(x) for x in rng.choice(n, 2, replace=False))
        if k == 0:
            return g1(a, G.haar(2, rng), "U2")
        if k == 1:
            return gc(a, b, G.X, "CNOT")
        if k == 2:
            return gc(a, b, G.phase(float(rng.uniform(0, 2 * pi))), "CPhase")
        if k == 3:
            return g2(a, b, G.haar(4, rng), "U4")
        return g1(a, G.H, "H")

    out = [one() for _ in range(npre)]
    perm = rng.permutation(n)
    for i in range(n // 2 - int(rng.integers(0, 2))):
        a, b = int(perm[2 * i]), int(perm[2 * i + 1])
        out.append(g2(min(a, b), max(a, b), G.SWAP, "SWAP"))
    out += [one() for _ in range(npost)]
    return out
