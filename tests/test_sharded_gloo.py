"""World-size-2/4 multi-process test of the sharded path's host logic over torch.distributed (gloo,
CPU).  Each rank owns shard `rank` of an n-qubit state as a numpy array.  For every gate it asks
the library's planner (qs_plan_route / qs_plan_decompose — the code the CUDA path runs) what to do,
and executes that with gloo send/recv for the pairwise exchange and the oracle
for local arithmetic.  The gathered state must equal the oracle's unsharded simulation.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

SA_SKIP, SA_LOCAL, SA_XPAIR, SA_XSWAP_LG, SA_XSWAP_GG, SA_VIA_SWAP = range(6)
OP_PAIR, OP_CTRL, OP_QUAD, OP_DIAG, OP_SWAP = range(5)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _exchange(buf: np.ndarray, partner: int) -> np.ndarray:
    send = torch.from_numpy(buf.view(np.float64).copy())
    recv = torch.empty_like(send)
    reqs = dist.batch_isend_irecv([dist.P2POp(dist.isend, send, partner), dist.P2POp(dist.irecv, recv, partner)])
    for r in reqs:
        r.wait()
    return recv.numpy().view(np.complex128)


def _local(orc, shard, r):
    from qsinputs import gates as G
    k, q0, q1, mm = r["kind"], r["q0"], r["q1"], r["m"]
    U2 = mm[:8].view(np.complex128).reshape(2, 2)
    if k == OP_PAIR:
        orc.apply_1q(shard, q0, U2)
    elif k == OP_CTRL:
        orc.apply_ctrl_1q(shard, q0, q1, U2)
    elif k == OP_QUAD:
        orc.apply_2q(shard, q0, q1, mm.view(np.complex128).reshape(4, 4))
    elif k == OP_SWAP:
        orc.apply_2q(shard, q0, q1, G.SWAP)
    elif k == OP_DIAG:
        d = mm[:8].view(np.complex128)
        if q0 < 0:
            shard *= d[0]
        elif q1 < 0:
            orc.apply_1q(shard, q0, np.diag(d[:2]))
        else:
            orc.apply_2q(shard, q0, q1, np.diag(d))


def _apply(orc, shard, n, m, rank, gate):
    import paper_2506_09198_b200 as qs
    r = qs.qs_plan_route(n, m, rank, gate)
    act = r["action"]
    idx = np.arange(shard.size, dtype=np.int64)
    if act == SA_SKIP:
        return
    if act == SA_LOCAL:
        _local(orc, shard, r)
    elif act == SA_XPAIR:
        remote = _exchange(shard, r["partner"])
        U = r["m"][:8].view(np.complex128).reshape(2, 2)
        b = r["bit"]
        a0, a1 = (remote, shard) if b else (shard, remote)
        new = U[b, 0] * a0 + U[b, 1] * a1
        if r["ctrl_local"] >= 0:
            mask = ((idx >> r["ctrl_local"]) & 1) == 1
            shard[mask] = new[mask]
        else:
            shard[:] = new
    elif act == SA_XSWAP_LG:
        sel = ((idx >> r["l"]) & 1) == 1 - r["bit"]
        shard[sel] = _exchange(np.ascontiguousarray(shard[sel]), r["partner"])
    elif act == SA_XSWAP_GG:
        shard[:] = _exchange(shard, r["partner"])
    elif act == SA_VIA_SWAP:
        from qsinputs.circuits import Gate
        for g in qs.qs_plan_decompose(n, m, gate):
            kind = {0: "1q", 1: "c1q", 2: "2q"}[int(g["kind"])]
            d = 4 if kind == "2q" else 2
            mat = g["m"][: 2 * d * d].copy().view(np.complex128).reshape(d, d)
            _apply(orc, shard, n, m, rank, Gate(kind, int(g["q0"]), int(g["q1"]), mat))
    else:
        raise AssertionError(act)


def _physical(circ, n, m):
    """The global-qubit remapped gate list qs_run_circuit executes on a sharded state (qs_plan_remap)."""
    from paper_2506_09198_b200 import qs as qsmod
    from qsinputs.circuits import Gate
    arr, _ = qsmod.qs_plan_remap(n, m, circ)
    out = []
    for g in arr:
        kind = {0: "1q", 1: "c1q", 2: "2q"}[int(g["kind"])]
        d = 4 if kind == "2q" else 2
        out.append(Gate(kind, int(g["q0"]), int(g["q1"]), g["m"][: 2 * d * d].copy().view(np.complex128).reshape(d, d)))
    return out


def _worker(rank, world, port, n, case, out_q, remap=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import Oracle
        orc = Oracle()
        circ = _circuit(case, n)
        k = world.bit_length() - 1
        m = n - k
        if remap:
            circ = _physical(circ, n, m)
        full = orc.random_state(n, 2506)
        shard = full[rank << m:(rank + 1) << m].copy()
        for g in circ:
            _apply(orc, shard, n, m, rank, g)
        t = torch.from_numpy(shard.view(np.float64).copy())
        parts = [torch.empty_like(t) for _ in range(world)] if rank == 0 else None
        dist.gather(t, parts, dst=0)
        if rank == 0:
            out_q.put(np.concatenate([p.numpy().view(np.complex128) for p in parts]))
    finally:
        dist.destroy_process_group()


def _circuit(case, n):
    from qsinputs import circuits as C
    from qsinputs import gates as G
    rng = np.random.Generator(np.random.PCG64(77))
    if case == "config1":
        return C.config1(n)
    if case == "mixed":  # every routing class, on global and local qubits
        out = []
        for q in range(n):
            out.append(C.g1(q, G.haar(2, rng)))
        for (c, t) in [(n - 1, 2), (2, n - 1), (n - 1, n - 2), (n - 2, n - 1), (0, n - 1), (n - 1, 0), (3, 4)]:
            out.append(C.gc(c, t, G.haar(2, rng)))
            out.append(C.gc(c, t, G.X))
            out.append(C.gc(c, t, G.phase(rng.random() * 6)))
            out.append(C.g2(c, t, G.haar(4, rng)))
            out.append(C.g2(c, t, G.SWAP))
        out.append(C.g2(n - 1, n - 2, np.diag(np.exp(1j * rng.random(4)))))
        out.append(C.g1(n - 1, G.T))
        return out
    if case == "qft":
        return C.qft(n)
    if case == "rqc":
        return C.rqc_grid(12, depth=8)
    raise ValueError(case)


@pytest.mark.parametrize("world,case,remap", [(2, "config1", False), (2, "mixed", False), (4, "mixed", False),
                                              (2, "qft", False), (4, "rqc", False), (4, "rqc", True),
                                              (2, "qft", True), (4, "mixed", True)])
def test_sharded_plan_matches_oracle(world, case, remap):
    n = 12
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, case, q, remap)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    from oracle import Oracle
    orc = Oracle()
    ref = orc.random_state(n, 2506)
    orc.run(ref, _circuit(case, n))
    assert np.max(np.abs(got - ref)) <= 1e-13
