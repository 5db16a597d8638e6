"""Host-side DFT sums of a random state too large for host memory (test infrastructure).

QFT|psi> = 2^(-n/2) sum_x psi[x] e^{+2 pi i x y / 2^n} |y>   (reading R5)

For sampled outputs y the sum over all 2^n inputs is formed chunk by chunk from the ORACLE's samples
gauss2(seed, x) (orc_gauss2_range), never from the CUDA path: x = base + h 2^16 + j, so

    sum_x g[x] w^{xy} = sum_chunks sum_h w^{(base + h 2^16) y} (sum_j g[base + h 2^16 + j] w^{j y})

with w = e^{2 pi i / 2^n}; the inner sums over j are one complex matrix product per chunk (a library
primitive), every exponent is reduced mod 2^n in exact integer arithmetic.  The state is normalised by
the pairwise sum of |g|^2 over the same chunks (the normalisation of orc_init_random).  Pinned against
numpy.fft.ifft of the oracle's whole random state at small n (tests/test_oracle_pins.py).
"""
import numpy as np

J_BITS = 16


def _phase(k: np.ndarray, n: int) -> np.ndarray:
    """e^{2 pi i k / 2^n} for integer k already reduced mod 2^n (exact in float64 for n <= 52)."""
    ang = (2.0 * np.pi / float(1 << n)) * k.astype(np.float64)
    return np.cos(ang) + 1j * np.sin(ang)


def qft_random_state_samples(orc, n: int, seed: int, ys, chunk_bits: int = 24):
    """(QFT psi)[y] for y in ys, psi = gauss2(seed, .) normalised; returns (values, sum |g|^2)."""
    N = 1 << n
    mask = np.uint64(N - 1)
    y = np.asarray(ys, dtype=np.uint64)
    jb = min(J_BITS, n)
    cb = max(min(chunk_bits, n), jb)
    J, chunk = 1 << jb, 1 << cb
    H = chunk // J
    j = np.arange(J, dtype=np.uint64)
    lo = _phase((j[:, None] * y[None, :]) & mask, n)  # (J, K); j y < 2^(16 + n) fits uint64 for n <= 48
    acc = np.zeros(y.size, dtype=np.complex128)
    s2 = 0.0
    buf = np.empty(chunk, dtype=np.complex128)
    for c in range(N // chunk):
        base = c * chunk
        orc.gauss2_range(seed, base, chunk, out=buf)
        s2 += float(np.sum(buf.real * buf.real + buf.imag * buf.imag))
        inner = buf.reshape(H, J) @ lo  # (H, K)
        h = np.uint64(base) + np.arange(H, dtype=np.uint64) * np.uint64(J)
        hi = _phase((h[:, None] * y[None, :]) & mask, n)  # products wrap mod 2^64: exact mod 2^n
        acc += np.sum(inner * hi, axis=0)
    return acc / np.sqrt(s2) * 2.0 ** (-n / 2), s2
