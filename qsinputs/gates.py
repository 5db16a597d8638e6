"""Gate matrices (inputs to the method), SURVEY.md §8(c) c.3 "Named gates" / "Haar U(d)".

Conventions (SURVEY.md §8(b) "Matrix layout", reading R2):
- a 1q matrix U acts on (a0, a1) where a0 has the target bit 0;
- a 2q matrix U4 is indexed by the sub-index k = bit_q0 + 2*bit_q1 (q0 is the low sub-bit);
- the flat form is row-major, complex interleaved: [re00, im00, re01, im01, ...].
"""
import struct

import numpy as np

# 1/sqrt(2) correctly rounded: 0x3FE6A09E667F3BCD (= M_SQRT1_2).  Alg. 1 "recRoot2".
H_COEF = struct.unpack("<d", struct.pack("<Q", 0x3FE6A09E667F3BCD))[0]

I2 = np.eye(2, dtype=np.complex128)
H = H_COEF * np.array([[1, 1], [1, -1]], dtype=np.complex128)
X = np.array([[0, 1], [1, 0]], dtype=np.complex128)
Y = np.array([[0, -1j], [1j, 0]], dtype=np.complex128)
Z = np.array([[1, 0], [0, -1]], dtype=np.complex128)
T = np.array([[1, 0], [0, complex(H_COEF, H_COEF)]], dtype=np.complex128)

# sqrt(P) = ((1+i)/2) I + ((1-i)/2) P for P in {X, Y, W}, W = (X+Y)/sqrt(2).
SQRT_X = 0.5 * np.array([[1 + 1j, 1 - 1j], [1 - 1j, 1 + 1j]], dtype=np.complex128)
SQRT_Y = 0.5 * np.array([[1 + 1j, -1 - 1j], [1 + 1j, 1 + 1j]], dtype=np.complex128)
SQRT_W = np.array([[0.5 + 0.5j, -1j * H_COEF], [H_COEF + 0j, 0.5 + 0.5j]], dtype=np.complex128)

# SWAP as a 4x4 in the k = bit_q0 + 2*bit_q1 basis: exchanges k=1 <-> k=2.
SWAP = np.array([[1, 0, 0, 0], [0, 0, 1, 0], [0, 1, 0, 0], [0, 0, 0, 1]], dtype=np.complex128)
# CNOT with control q0, target q1 as a 4x4: maps k=1 (q0=1,q1=0) <-> k=3 (q0=1,q1=1).
CNOT_Q0_CTRL = np.array([[1, 0, 0, 0], [0, 0, 0, 1], [0, 0, 1, 0], [0, 1, 0, 0]], dtype=np.complex128)


def phase(theta: float) -> np.ndarray:
    """diag(1, e^{i theta}); used as the target matrix of CPhase = ctrl-1q(c, t, phase(theta))."""
    return np.array([[1, 0], [0, complex(np.cos(theta), np.sin(theta))]], dtype=np.complex128)


def cz_target() -> np.ndarray:
    """CZ = ctrl-1q(c, t, diag(1, -1))."""
    return Z.copy()


def haar(d: int, rng: np.random.Generator, polish: bool = True) -> np.ndarray:
    """Haar-random U(d) (Mezzadri): Z = (X + iY)/sqrt(2), Q,R = qr(Z), U = Q diag(R_jj/|R_jj|).

    ``polish`` applies one Newton-Schulz step U <- U (3I - U^H U)/2 in long double so that
    ||U^H U - I|| is at the ulp level (keeps the norm within 1e-12 over hundreds of gates).
    """
    zr = rng.standard_normal((d, d))
    zi = rng.standard_normal((d, d))
    zm = (zr + 1j * zi) / np.sqrt(2.0)
    q, r = np.linalg.qr(zm)
    dg = np.diag(r)
    u = q * (dg / np.abs(dg))[None, :]
    if polish:
        ul = u.astype(np.clongdouble)
        eye = np.eye(d, dtype=np.clongdouble)
        ul = ul @ (3 * eye - ul.conj().T @ ul) / 2
        u = ul.astype(np.complex128)
    return u


def flat(m: np.ndarray) -> np.ndarray:
    """Row-major, complex-interleaved float64 copy of a 2x2 or 4x4 matrix."""
    m = np.ascontiguousarray(m, dtype=np.complex128)
    return m.reshape(-1).view(np.float64).copy()
