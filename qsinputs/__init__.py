"""Seeded, synthetic inputs shared by the oracle tests, the CUDA-path tests and bench.py.

This package holds NONE of the method's arithmetic (no gate application, no
state update, no norm, no random-state generator): only the gate matrices the
method consumes and the gate lists of the workloads.
Both sides of every parity test receive the identical doubles produced here.

Contents
- ``gates``    : named 1q/2q matrices (H, X, Y, Z, CNOT, CZ, CPhase, SWAP, sqrt-X/Y/W)
                 and Haar-random U(2)/U(4) generators.
- ``circuits`` : gate-list builders for BASELINE.json configs 1-5 (QFT ladder,
                 Sycamore-style grid RQC, the paper's CNOT-ring RQC, the 1q/2q sweeps).
- ``rng``      : SplitMix64 stream used to draw circuit choices (RQC gate picks, QFT |x>).
"""
from . import rng, gates, circuits  # noqa: F401
from .circuits import Gate  # noqa: F401

SEED_STATE = 2506   # gauss2 random-state seed (SURVEY.md §8(c) c.3 "Seeds")
SEED_GATES = 9198   # PCG64 seed for Haar matrices and random angles
SEED_RQC = 20       # SplitMix64 seed for RQC gate picks
SEED_QFT_X = 35     # x = SM(35, 0) mod 2^n for the QFT basis input
