"""SplitMix64 counter stream for *circuit choices* (SURVEY.md §8(c) c.3).

Element j of the stream seeded with ``seed`` is
    mix(seed + (j+1) * 0x9E3779B97F4A7C15  mod 2^64)
with mix(z): z = (z ^ z>>30) * 0xBF58476D1CE4E5B9; z = (z ^ z>>27) * 0x94D049BB133111EB;
return z ^ z>>31.

Used here only to draw RQC gate picks and the QFT basis index.  The
random *state* generator (gauss2) is part of the method and is implemented
independently by the oracle (oracle/orc.c) and by the CUDA path.
"""
M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15


def _mix(z: int) -> int:
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def splitmix64(seed: int, j: int) -> int:
    """Element j (0-based) of the SplitMix64 stream seeded with ``seed``."""
    return _mix((seed + (j + 1) * GOLDEN) & M64)


class SplitMix64Stream:
    """Sequential reader over the counter stream."""

    def __init__(self, seed: int):
        self.seed = seed & M64
        self.j = 0

    def next(self) -> int:
        v = splitmix64(self.seed, self.j)
        self.j += 1
        return v
