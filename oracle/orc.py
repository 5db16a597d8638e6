"""ctypes wrapper around oracle/liborc.so (ORACLE — test infrastructure only).

The state is a numpy complex128 array of length 2^n (AoS: re, im interleaved in memory,
PAPER.md:L114), passed to C as double*.
"""
import ctypes
import os
import subprocess
from typing import Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "orc.c")
LIB_PATH = os.path.join(HERE, "liborc.so")
CFLAGS = ["-O2", "-std=gnu11", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared"]


def build_oracle(force: bool = False) -> str:
    """Compile orc.c with gcc (plain C, no intrinsics, no FP contraction)."""
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(SRC):
        tmp = LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, SRC, "-o", tmp, "-lm"])
        os.replace(tmp, LIB_PATH)
    return LIB_PATH


_dp = ctypes.POINTER(ctypes.c_double)
_u64 = ctypes.c_uint64


def _ptr(a: np.ndarray):
    assert a.dtype == np.complex128 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def _mat(m) -> np.ndarray:
    m = np.ascontiguousarray(np.asarray(m, dtype=np.complex128))
    return m.reshape(-1).view(np.float64).copy()


def _configure(lib):
    """ctypes signatures of liborc.so's entry points (shared by the library and its test mutants)."""
    lib.orc_pair_index.argtypes = [_u64, ctypes.c_int, ctypes.POINTER(_u64), ctypes.POINTER(_u64)]
    lib.orc_init_basis.argtypes = [_dp, ctypes.c_int, _u64]
    lib.orc_norm2.argtypes = [_dp, ctypes.c_int]
    lib.orc_norm2.restype = ctypes.c_double
    lib.orc_norm2_count.argtypes = [_dp, _u64]
    lib.orc_norm2_count.restype = ctypes.c_double
    lib.orc_splitmix64.argtypes = [_u64, _u64]
    lib.orc_splitmix64.restype = _u64
    lib.orc_gauss2.argtypes = [_u64, _u64, _dp, _dp]
    lib.orc_init_random.argtypes = [_dp, ctypes.c_int, _u64]
    if hasattr(lib, "orc_gauss2_range"):
        lib.orc_gauss2_range.argtypes = [_dp, _u64, _u64, _u64]
    lib.orc_apply_1q.argtypes = [_dp, ctypes.c_int, ctypes.c_int, _dp]
    lib.orc_apply_ctrl_1q.argtypes = [_dp, ctypes.c_int, ctypes.c_int, ctypes.c_int, _dp]
    lib.orc_apply_2q.argtypes = [_dp, ctypes.c_int, ctypes.c_int, ctypes.c_int, _dp]
    i32p = ctypes.POINTER(ctypes.c_int32)
    lib.orc_run.argtypes = [_dp, ctypes.c_int, i32p, i32p, i32p, _dp, _u64]
    lib.orc_run.restype = ctypes.c_int
    return lib


class Oracle:
    _lib = None

    def __init__(self):
        if Oracle._lib is None:
            Oracle._lib = _configure(ctypes.CDLL(build_oracle()))
        self.lib = Oracle._lib

    @classmethod
    def from_library(cls, path: str) -> "Oracle":
        """An oracle bound to another build of orc.c (tests/test_oracle_mutants.py compiles deliberately
        broken copies and checks that the pins catch every one)."""
        o = cls.__new__(cls)
        o.lib = _configure(ctypes.CDLL(path))
        return o

    # --- index math ---------------------------------------------------------------------------
    def pair_index(self, task: int, t: int):
        up, lo = _u64(), _u64()
        self.lib.orc_pair_index(task, t, ctypes.byref(up), ctypes.byref(lo))
        return up.value, lo.value

    # --- states --------------------------------------------------------------------------------
    def basis(self, n: int, x: int) -> np.ndarray:
        a = np.empty(1 << n, dtype=np.complex128)
        self.lib.orc_init_basis(_ptr(a), n, x)
        return a

    def random_state(self, n: int, seed: int) -> np.ndarray:
        a = np.empty(1 << n, dtype=np.complex128)
        self.lib.orc_init_random(_ptr(a), n, seed)
        return a

    def splitmix64(self, seed: int, j: int) -> int:
        return self.lib.orc_splitmix64(seed, j)

    def gauss2(self, seed: int, i: int):
        re, im = ctypes.c_double(), ctypes.c_double()
        self.lib.orc_gauss2(seed, i, ctypes.byref(re), ctypes.byref(im))
        return re.value, im.value

    def gauss2_range(self, seed: int, start: int, count: int, out: np.ndarray = None) -> np.ndarray:
        """Unnormalised gauss2(seed, i), i in [start, start + count) (orc_init_random before scaling)."""
        a = out if out is not None else np.empty(count, dtype=np.complex128)
        assert a.size == count
        self.lib.orc_gauss2_range(_ptr(a), seed, start, count)
        return a

    def norm2(self, a: np.ndarray) -> float:
        return self.lib.orc_norm2_count(_ptr(a), a.size)

    # --- gates (in place) -----------------------------------------------------------------------
    @staticmethod
    def _n(a):
        n = int(a.size).bit_length() - 1
        assert a.size == 1 << n
        return n

    def apply_1q(self, a, t, m):
        u = _mat(m)
        self.lib.orc_apply_1q(_ptr(a), self._n(a), t, u.ctypes.data_as(_dp))

    def apply_ctrl_1q(self, a, c, t, m):
        u = _mat(m)
        self.lib.orc_apply_ctrl_1q(_ptr(a), self._n(a), c, t, u.ctypes.data_as(_dp))

    def apply_2q(self, a, q0, q1, m):
        u = _mat(m)
        self.lib.orc_apply_2q(_ptr(a), self._n(a), q0, q1, u.ctypes.data_as(_dp))

    def run(self, a: np.ndarray, gates: Sequence) -> None:
        """Apply qsinputs.circuits.Gate objects in order (O7)."""
        G = len(gates)
        if G == 0:
            return
        kinds = {"1q": 0, "c1q": 1, "2q": 2}
        kind = np.array([kinds[g.kind] for g in gates], dtype=np.int32)
        q0 = np.array([g.q0 for g in gates], dtype=np.int32)
        q1 = np.array([g.q1 for g in gates], dtype=np.int32)
        mats = np.zeros((G, 32), dtype=np.float64)
        for k, g in enumerate(gates):
            f = _mat(g.m)
            mats[k, : f.size] = f
        i32p = ctypes.POINTER(ctypes.c_int32)
        rc = self.lib.orc_run(_ptr(a), self._n(a), kind.ctypes.data_as(i32p), q0.ctypes.data_as(i32p),
                              q1.ctypes.data_as(i32p), mats.ctypes.data_as(_dp), G)
        if rc != 0:
            raise ValueError("oracle rejected a gate")
