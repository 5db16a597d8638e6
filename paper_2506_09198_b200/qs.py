"""Thin ctypes binding of include/qs.h (argument marshalling only; every step runs in libqs_b200.so).

The functions keep the C names (qs_create, qs_apply_1q, ...).  ``QState`` is a small convenience
wrapper over the same calls.  There is no fallback: if the CUDA library is missing or the call
fails, an exception is raised.
"""
import ctypes
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libqs_b200.so")

QS_OK, QS_ERR_ARG, QS_ERR_RANGE, QS_ERR_OOM, QS_ERR_CUDA, QS_ERR_NCCL, QS_ERR_STATE, QS_ERR_UNSUPPORTED = range(8)
STATUS_NAMES = ["QS_OK", "QS_ERR_ARG", "QS_ERR_RANGE", "QS_ERR_OOM", "QS_ERR_CUDA", "QS_ERR_NCCL", "QS_ERR_STATE",
                "QS_ERR_UNSUPPORTED"]
QS_G_1Q, QS_G_C1Q, QS_G_2Q = 0, 1, 2
KIND_CODE = {"1q": QS_G_1Q, "c1q": QS_G_C1Q, "2q": QS_G_2Q}

GATE_DTYPE = np.dtype([("kind", "<i4"), ("q0", "<i4"), ("q1", "<i4"), ("flags", "<i4"), ("m", "<f8", (32,))])
assert GATE_DTYPE.itemsize == 272


class QSError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS_NAMES[code] if 0 <= code < len(STATUS_NAMES) else code}: {msg}")
        self.code = code


class _QSHandle(ctypes.Structure):
    pass


_H = ctypes.POINTER(_QSHandle)
_dp = ctypes.POINTER(ctypes.c_double)
_u64 = ctypes.c_uint64
_lib = None


def load_library():
    """Load libqs_b200.so (raises if it has not been built: there is no CPU path)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: run `python -m paper_2506_09198_b200.build` (no CPU fallback exists)")
    lib = ctypes.CDLL(LIB_PATH)
    S = ctypes.c_int
    sig = {
        "qs_create": (S, [ctypes.c_int, ctypes.c_int, ctypes.POINTER(_H)]),
        "qs_create_virtual": (S, [ctypes.c_int, ctypes.c_int, ctypes.POINTER(_H)]),
        "qs_get_unique_id": (S, [ctypes.c_void_p]),
        "qs_create_rank": (S, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(_H)]),
        "qs_destroy": (None, [_H]),
        "qs_init_basis": (S, [_H, _u64]),
        "qs_init_random": (S, [_H, _u64]),
        "qs_apply_1q": (S, [_H, ctypes.c_int, _dp]),
        "qs_apply_ctrl_1q": (S, [_H, ctypes.c_int, ctypes.c_int, _dp]),
        "qs_apply_2q": (S, [_H, ctypes.c_int, ctypes.c_int, _dp]),
        "qs_run_circuit": (S, [_H, ctypes.c_void_p, ctypes.c_size_t]),
        "qs_read_amps": (S, [_H, _u64, _u64, ctypes.c_void_p]),
        "qs_write_amps": (S, [_H, _u64, _u64, ctypes.c_void_p]),
        "qs_read_amps_async": (S, [_H, _u64, _u64, ctypes.c_void_p]),
        "qs_write_amps_async": (S, [_H, _u64, _u64, ctypes.c_void_p]),
        "qs_norm2": (S, [_H, _dp]),
        "qs_sync": (S, [_H]),
        "qs_last_error": (ctypes.c_char_p, [_H]),
        "qs_info": (S, [_H] + [ctypes.POINTER(ctypes.c_int)] * 5),
        "qs_launch_count": (_u64, [_H]),
        "qs_stream": (ctypes.c_void_p, [_H, ctypes.c_int]),
        "qs_set_option": (S, [_H, ctypes.c_char_p, ctypes.c_int64]),
        "qs_last_plan": (S, [_H, ctypes.POINTER(_u64), ctypes.POINTER(_u64)]),
        "qs_jit_stats": (S, [_H, ctypes.POINTER(_u64), ctypes.POINTER(_u64), ctypes.POINTER(_u64)]),
        "qs_plan_route": (S, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_int,
                              ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32), _dp]),
        "qs_plan_decompose": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]),
        "qs_plan_passes": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int,
                                          ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                          ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]),
        "qs_plan_remap": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p,
                                         ctypes.c_int, ctypes.c_void_p]),
        "qs_plan_hoist": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int,
                                         ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]),
        "qs_plan_tile_jit": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t,
                                            ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


EXPORTED = ["qs_create", "qs_create_virtual", "qs_get_unique_id", "qs_create_rank", "qs_destroy", "qs_init_basis",
            "qs_init_random", "qs_apply_1q", "qs_apply_ctrl_1q", "qs_apply_2q", "qs_run_circuit", "qs_read_amps",
            "qs_write_amps", "qs_read_amps_async", "qs_write_amps_async", "qs_norm2", "qs_sync", "qs_last_error", "qs_info", "qs_launch_count", "qs_stream",
            "qs_set_option", "qs_last_plan", "qs_jit_stats", "qs_plan_route", "qs_plan_decompose", "qs_plan_passes",
            "qs_plan_tile_jit", "qs_plan_remap", "qs_plan_hoist", "qs_jit_compile_file"]


def _check(code, h=None):
    if code != QS_OK:
        msg = load_library().qs_last_error(h)
        raise QSError(code, msg.decode() if msg else "")


def mat_flat(m) -> np.ndarray:
    m = np.ascontiguousarray(np.asarray(m, dtype=np.complex128))
    return m.reshape(-1).view(np.float64).copy()


def gates_array(gates) -> np.ndarray:
    """Marshal objects with .kind ('1q'/'c1q'/'2q' or 0/1/2), .q0, .q1, .m into a qs_gate array."""
    arr = np.zeros(len(gates), dtype=GATE_DTYPE)
    for i, g in enumerate(gates):
        arr[i]["kind"] = KIND_CODE.get(g.kind, g.kind) if isinstance(g.kind, str) else g.kind
        arr[i]["q0"] = g.q0
        arr[i]["q1"] = g.q1
        f = mat_flat(g.m)
        arr[i]["m"][: f.size] = f
    return arr


# ------------------------------------------------------------------------------------------------
# C-named functions
# ------------------------------------------------------------------------------------------------
def qs_create(n_qubits: int, n_gpus: int = 1):
    h = _H()
    _check(load_library().qs_create(n_qubits, n_gpus, ctypes.byref(h)))
    return h


def qs_create_virtual(n_qubits: int, n_shards: int):
    h = _H()
    _check(load_library().qs_create_virtual(n_qubits, n_shards, ctypes.byref(h)))
    return h


def qs_get_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(load_library().qs_get_unique_id(buf))
    return buf.raw


def qs_create_rank(n_qubits: int, world: int, rank: int, device: int, uid: bytes):
    h = _H()
    buf = ctypes.create_string_buffer(bytes(uid), 128)
    _check(load_library().qs_create_rank(n_qubits, world, rank, device, buf, ctypes.byref(h)))
    return h


def qs_destroy(h):
    load_library().qs_destroy(h)


def qs_init_basis(h, index: int):
    _check(load_library().qs_init_basis(h, index), h)


def qs_init_random(h, seed: int):
    _check(load_library().qs_init_random(h, seed), h)


def qs_apply_1q(h, target: int, u2):
    f = mat_flat(u2)
    _check(load_library().qs_apply_1q(h, target, f.ctypes.data_as(_dp)), h)


def qs_apply_ctrl_1q(h, ctrl: int, target: int, u2):
    f = mat_flat(u2)
    _check(load_library().qs_apply_ctrl_1q(h, ctrl, target, f.ctypes.data_as(_dp)), h)


def qs_apply_2q(h, q0: int, q1: int, u4):
    f = mat_flat(u4)
    _check(load_library().qs_apply_2q(h, q0, q1, f.ctypes.data_as(_dp)), h)


def qs_run_circuit(h, gates):
    arr = gates if isinstance(gates, np.ndarray) and gates.dtype == GATE_DTYPE else gates_array(gates)
    arr = np.ascontiguousarray(arr)
    _check(load_library().qs_run_circuit(h, arr.ctypes.data, arr.size), h)


def qs_read_amps(h, start: int, count: int, out: np.ndarray = None) -> np.ndarray:
    if out is None:
        out = np.empty(count, dtype=np.complex128)
    assert out.dtype == np.complex128 and out.flags.c_contiguous and out.size >= count
    _check(load_library().qs_read_amps(h, start, count, out.ctypes.data), h)
    return out


def qs_write_amps(h, start: int, data: np.ndarray):
    data = np.ascontiguousarray(data, dtype=np.complex128)
    _check(load_library().qs_write_amps(h, start, data.size, data.ctypes.data), h)


def qs_read_amps_async(h, start: int, count: int, out: np.ndarray):
    """Stream-ordered D2H into `out` (keep it alive, page-locked for overlap, until qs_sync)."""
    assert out.dtype == np.complex128 and out.flags.c_contiguous and out.size >= count
    _check(load_library().qs_read_amps_async(h, start, count, out.ctypes.data), h)


def qs_write_amps_async(h, start: int, data: np.ndarray):
    """Stream-ordered H2D from `data` (contiguous complex128; keep it alive until qs_sync)."""
    assert data.dtype == np.complex128 and data.flags.c_contiguous
    _check(load_library().qs_write_amps_async(h, start, data.size, data.ctypes.data), h)


def qs_norm2(h) -> float:
    v = ctypes.c_double()
    _check(load_library().qs_norm2(h, ctypes.byref(v)), h)
    return v.value


def qs_sync(h):
    _check(load_library().qs_sync(h), h)


def qs_last_error(h=None) -> str:
    return load_library().qs_last_error(h).decode()


def qs_info(h):
    vals = [ctypes.c_int() for _ in range(5)]
    _check(load_library().qs_info(h, *[ctypes.byref(v) for v in vals]), h)
    return dict(zip(["n", "P", "m", "owned", "first_rank"], [v.value for v in vals]))


def qs_launch_count(h) -> int:
    return load_library().qs_launch_count(h)


def qs_stream(h, i: int = 0) -> int:
    return load_library().qs_stream(h, i) or 0


def qs_set_option(h, key: str, value: int):
    _check(load_library().qs_set_option(h, key.encode(), int(value)), h)


def qs_last_plan(h):
    p, x = _u64(), _u64()
    _check(load_library().qs_last_plan(h, ctypes.byref(p), ctypes.byref(x)), h)
    return p.value, x.value


def qs_jit_stats(h):
    c, l, f = _u64(), _u64(), _u64()
    _check(load_library().qs_jit_stats(h, ctypes.byref(c), ctypes.byref(l), ctypes.byref(f)), h)
    return {"compiled": c.value, "launched": l.value, "failed": f.value}


# host-only planner hooks (include/qs_plan_abi.h)
def qs_plan_route(n: int, m: int, rank: int, gate, check_unitary: bool = True):
    arr = gates_array([gate])
    step = (ctypes.c_int32 * 5)()
    op = (ctypes.c_int32 * 4)()
    mm = (ctypes.c_double * 32)()
    code = load_library().qs_plan_route(n, m, rank, arr.ctypes.data, int(check_unitary), step, op, mm)
    _check(code)
    return {"action": step[0], "partner": step[1], "bit": step[2], "ctrl_local": step[3], "l": step[4],
            "kind": op[0], "q0": op[1], "q1": op[2], "touch": op[3], "m": np.array(mm[:])}


def qs_plan_decompose(n: int, m: int, gate):
    arr = gates_array([gate])
    out = np.zeros(8, dtype=GATE_DTYPE)
    k = load_library().qs_plan_decompose(n, m, arr.ctypes.data, out.ctypes.data, out.size)
    if k < 0:
        raise QSError(QS_ERR_ARG, qs_last_error(None))
    return out[:k]


def qs_plan_passes(n: int, m: int, gates, b: int = 11, L0: int = 5, fuse: bool = True, reorder: bool = False,
                   with_order: bool = False):
    arr = gates_array(gates)
    cap = max(1, len(gates)) * 2 + 4
    t = np.zeros(cap, np.int32)
    nops = np.zeros(cap, np.int32)
    first = np.zeros(cap, np.int32)
    mask = np.zeros(cap, np.uint64)
    order = np.full(max(1, len(gates)), -1, np.int32)
    k = load_library().qs_plan_passes(n, m, arr.ctypes.data, arr.size, b, L0, int(fuse), int(reorder), t.ctypes.data,
                                      nops.ctypes.data, first.ctypes.data, mask.ctypes.data, order.ctypes.data, cap)
    if k < 0:
        raise QSError(QS_ERR_ARG, qs_last_error(None))
    plan = [{"type": int(t[i]), "nops": int(nops[i]), "first": int(first[i]), "tile_mask": int(mask[i])}
            for i in range(k)]
    if with_order:
        return plan, [int(x) for x in order[:sum(p["nops"] for p in plan)]]
    return plan


def qs_plan_remap(n: int, m: int, gates):
    """Global-qubit remapped gate list (physical positions) as a qs_gate array, and the exchange volume
    {before, after} in half-shard units."""
    arr = gates_array(gates)
    cap = 3 * len(gates) + 2 * n + 4
    out = np.zeros(cap, dtype=GATE_DTYPE)
    cost = np.zeros(2, np.int32)
    k = load_library().qs_plan_remap(n, m, arr.ctypes.data, arr.size, out.ctypes.data, cap, cost.ctypes.data)
    if k < 0:
        raise QSError(QS_ERR_ARG, qs_last_error(None))
    return out[:k].copy(), (int(cost[0]), int(cost[1]))


def qs_plan_hoist(n: int, m: int, gates, b: int = 12, L0: int = 4, reorder: bool = True):
    """The op list after permutation hoisting (execution order, qs_gate array; empty if nothing was
    hoisted) and {passes before, passes after, passes with a fused permutation}."""
    arr = gates_array(gates)
    cap = 2 * len(gates) + 2 * n + 4
    out = np.zeros(cap, dtype=GATE_DTYPE)
    st = np.zeros(3, np.int32)
    k = load_library().qs_plan_hoist(n, m, arr.ctypes.data, arr.size, b, L0, int(reorder), out.ctypes.data, cap,
                                     st.ctypes.data)
    if k < 0:
        raise QSError(QS_ERR_ARG, qs_last_error(None))
    return out[:k].copy(), {"before": int(st[0]), "after": int(st[1]), "fused": int(st[2])}


def qs_plan_tile_jit(n: int, m: int, gates, rank: int = 0, b: int = 12, L0: int = 4, ladder_min: int = 4,
                     compile: bool = True, family: bool = False):
    """Tile passes of a circuit as qs_run_circuit builds them for shard `rank`; with compile, every
    distinct JIT source is compiled by NVRTC (no GPU needed); family: the sources' family form."""
    arr = gates_array(gates)
    st = np.zeros(10, np.int32)
    _check(load_library().qs_plan_tile_jit(n, m, rank, arr.ctypes.data, arr.size, b, L0, ladder_min,
                                           int(compile) | (2 if family else 0), st.ctypes.data))
    keys = ["passes", "tile_passes", "tile_ops", "ladders", "sources", "compiled", "batches", "source_hash",
            "warp_local", "group_local"]
    return dict(zip(keys, (int(x) for x in st)))


# ------------------------------------------------------------------------------------------------
class QState:
    """Owning wrapper: QState(n) on 1 GPU, QState(n, P) on P GPUs, QState(n, P, virtual=True) for
    P shards on one GPU, QState.rank(n, world, rank, device, uid) for one process per GPU."""

    def __init__(self, n: int, P: int = 1, virtual: bool = False, _handle=None):
        self.h = _handle if _handle is not None else (qs_create_virtual(n, P) if virtual else qs_create(n, P))
        self.info = qs_info(self.h)

    @classmethod
    def rank(cls, n, world, rank, device, uid):
        return cls(n, world, _handle=qs_create_rank(n, world, rank, device, uid))

    @property
    def n(self):
        return self.info["n"]

    def close(self):
        if self.h:
            qs_destroy(self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def init_basis(self, x):
        qs_init_basis(self.h, x)

    def init_random(self, seed):
        qs_init_random(self.h, seed)

    def apply_1q(self, t, u):
        qs_apply_1q(self.h, t, u)

    def apply_ctrl_1q(self, c, t, u):
        qs_apply_ctrl_1q(self.h, c, t, u)

    def apply_2q(self, q0, q1, u):
        qs_apply_2q(self.h, q0, q1, u)

    def apply(self, g):
        if g.kind == "1q":
            self.apply_1q(g.q0, g.m)
        elif g.kind == "c1q":
            self.apply_ctrl_1q(g.q0, g.q1, g.m)
        else:
            self.apply_2q(g.q0, g.q1, g.m)

    def run(self, gates):
        qs_run_circuit(self.h, gates)

    def read(self, start=0, count=None):
        if count is None:
            count = (1 << self.n) - start
        return qs_read_amps(self.h, start, count)

    def write(self, start, data):
        qs_write_amps(self.h, start, data)

    def norm2(self):
        return qs_norm2(self.h)

    def sync(self):
        qs_sync(self.h)

    def set_option(self, k, v):
        qs_set_option(self.h, k, v)

    def launches(self):
        return qs_launch_count(self.h)

    def stream(self, i=0):
        return qs_stream(self.h, i)

    def last_plan(self):
        return qs_last_plan(self.h)

    def jit_stats(self):
        return qs_jit_stats(self.h)
