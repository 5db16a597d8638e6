"""Shared helpers for the GPU parity tests (tolerances from BASELINE.json north_star + SURVEY.md §8(c) c.6)."""
import numpy as np

EPS = 2.0 ** -53
ABS_TOL = 1e-10   # north_star: max |delta amplitude| <= 1e-10
NORM_TOL = 1e-12  # north_star: |1 - norm| <= 1e-12


def tight_tol(ref: np.ndarray, n_gates: int) -> float:
    """SURVEY.md §8(c) c.6 tight alarm: 32 G eps max|psi| (catches fp32 leaks / dropped terms that
    the 1e-10 absolute bar would miss at large n)."""
    return 32.0 * max(n_gates, 1) * EPS * float(np.max(np.abs(ref))) + 1e-300


def assert_parity(got: np.ndarray, ref: np.ndarray, n_gates: int, what: str = ""):
    err = float(np.max(np.abs(got - ref)))
    assert err <= ABS_TOL, f"{what}: max|d| = {err:.3e} > 1e-10"
    tt = tight_tol(ref, n_gates)
    assert err <= tt, f"{what}: max|d| = {err:.3e} > tight {tt:.3e}"
    return err
