"""CPU-only checks of the C-ABI library (no GPU calls): it loads, exports every symbol the headers
declare, and its host planner (classification, §8(e) shard routing, swap-to-local decomposition,
tile-pass planning) behaves as specified."""
import math
import json
import os
import re
import sys

import numpy as np
import pytest

import paper_2506_09198_b200 as qs
from paper_2506_09198_b200 import qs as qsmod
from qsinputs import circuits as C
from qsinputs import gates as G

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def built():
    import importlib.util
    spec = importlib.util.spec_from_file_location("_b", os.path.join(ROOT, "paper_2506_09198_b200", "build.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    mod.build()
    qs.load_library()


def test_library_exports_every_declared_symbol():
    declared = set()
    for h in ("qs.h", "qs_plan_abi.h"):
        txt = open(os.path.join(ROOT, "include", h)).read()
        txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
        declared |= set(re.findall(r"\b(qs_[a-z0-9_]+)\s*\(", txt))
    assert len(declared) >= 24
    lib = qs.load_library()
    for name in sorted(declared):
        assert hasattr(lib, name), name
    assert declared == set(qsmod.EXPORTED)


def test_gate_struct_layout():
    assert qsmod.GATE_DTYPE.itemsize == 272


def _route(n, m, rank, g, check=True):
    return qs.qs_plan_route(n, m, rank, g, check)


SA = dict(SKIP=0, LOCAL=1, XPAIR=2, XSWAP_LG=3, XSWAP_GG=4, VIA_SWAP=5)
OP = dict(PAIR=0, CTRL=1, QUAD=2, DIAG=3, SWAP=4)


def test_classification():
    n = m = 6
    assert _route(n, m, 0, C.g1(2, G.X))["kind"] == OP["PAIR"]
    r = _route(n, m, 0, C.g1(2, G.T))
    assert r["kind"] == OP["DIAG"] and r["touch"] == 0b10
    r = _route(n, m, 0, C.gc(1, 4, G.phase(0.3)))
    assert r["kind"] == OP["DIAG"] and r["touch"] == 0b1000 and (r["q0"], r["q1"]) == (1, 4)
    assert abs(complex(*r["m"][6:8]) - complex(math.cos(0.3), math.sin(0.3))) == 0
    r = _route(n, m, 0, C.gc(1, 4, G.Z))  # CZ
    assert r["kind"] == OP["DIAG"] and r["touch"] == 0b1000
    assert _route(n, m, 0, C.gc(1, 4, G.X))["kind"] == OP["CTRL"]
    assert _route(n, m, 0, C.g2(1, 4, G.SWAP))["kind"] == OP["SWAP"]
    assert _route(n, m, 0, C.g2(1, 4, np.diag(np.exp(1j * np.arange(4)))))["kind"] == OP["DIAG"]
    assert _route(n, m, 0, C.g2(1, 4, G.haar(4, np.random.default_rng(0))))["kind"] == OP["QUAD"]
    # an exact identity is a DIAG that touches nothing; the router skips it
    assert _route(n, m, 0, C.g1(3, np.eye(2)))["action"] == SA["SKIP"]


def test_argument_errors():
    with pytest.raises(qs.QSError):
        _route(6, 6, 0, C.g1(6, G.X))
    with pytest.raises(qs.QSError):
        _route(6, 6, 0, C.gc(2, 2, G.X))
    with pytest.raises(qs.QSError):
        _route(6, 6, 0, C.g2(1, 1, G.SWAP))
    bad = np.array([[1, 1], [0, 1]], dtype=complex)
    with pytest.raises(qs.QSError):
        _route(6, 6, 0, C.g1(0, bad))
    assert _route(6, 6, 0, C.g1(0, bad), check=False)["kind"] == OP["PAIR"]


def test_sharded_routing_table():
    """SURVEY.md §8(e) table at n=10, P=4 (m=8, global qubits 8, 9)."""
    n, m = 10, 8
    U = G.haar(2, np.random.default_rng(1))
    for rank in range(4):
        b8, b9 = rank & 1, (rank >> 1) & 1
        assert _route(n, m, rank, C.g1(3, U))["action"] == SA["LOCAL"]
        r = _route(n, m, rank, C.g1(9, U))
        assert (r["action"], r["partner"], r["bit"], r["ctrl_local"]) == (SA["XPAIR"], rank ^ 2, b9, -1)
        r = _route(n, m, rank, C.gc(9, 2, G.phase(0.5)))
        if b9:
            assert r["action"] == SA["LOCAL"] and r["kind"] == OP["DIAG"] and r["q0"] == 2 and r["touch"] == 0b10
        else:
            assert r["action"] == SA["SKIP"]
        r = _route(n, m, rank, C.gc(8, 2, G.X))
        assert r["action"] == (SA["LOCAL"] if b8 else SA["SKIP"])
        if b8:
            assert r["kind"] == OP["PAIR"] and r["q0"] == 2
        r = _route(n, m, rank, C.gc(2, 9, G.X))
        assert (r["action"], r["ctrl_local"], r["partner"], r["bit"]) == (SA["XPAIR"], 2, rank ^ 2, b9)
        r = _route(n, m, rank, C.gc(8, 9, G.X))
        assert r["action"] == (SA["XPAIR"] if b8 else SA["SKIP"])
        r = _route(n, m, rank, C.g2(3, 9, G.SWAP))
        assert (r["action"], r["l"], r["bit"], r["partner"]) == (SA["XSWAP_LG"], 3, b9, rank ^ 2)
        r = _route(n, m, rank, C.g2(8, 9, G.SWAP))
        if b8 != b9:
            assert (r["action"], r["partner"]) == (SA["XSWAP_GG"], rank ^ 3)
        else:
            assert r["action"] == SA["SKIP"]
        assert _route(n, m, rank, C.g2(2, 9, G.haar(4, np.random.default_rng(2))))["action"] == SA["VIA_SWAP"]
        # diagonal gates never communicate
        r = _route(n, m, rank, C.g2(8, 9, np.diag([1, 1j, -1, -1j])))
        k = b8 + 2 * b9
        assert r["action"] == (SA["SKIP"] if k == 0 else SA["LOCAL"])


def test_decompose_via_swap():
    n, m = 10, 8
    U4 = G.haar(4, np.random.default_rng(3))
    seq = qs.qs_plan_decompose(n, m, C.g2(2, 9, U4))
    assert [(int(g["q0"]), int(g["q1"])) for g in seq] == [(7, 9), (2, 7), (7, 9)]
    assert np.array_equal(seq[1]["m"], qs.gates_array([C.g2(2, 9, U4)])[0]["m"])
    swap = qs.gates_array([C.g2(0, 1, G.SWAP)])[0]["m"]
    assert np.array_equal(seq[0]["m"], swap) and np.array_equal(seq[2]["m"], swap)
    seq = qs.qs_plan_decompose(n, m, C.g2(9, 8, U4))  # both global, q0 > q1
    assert [(int(g["q0"]), int(g["q1"])) for g in seq] == [(7, 9), (6, 8), (7, 6), (6, 8), (7, 9)]
    seq = qs.qs_plan_decompose(n, m, C.g2(7, 8, U4))  # free qubit skips 7 (used by the gate)
    assert [(int(g["q0"]), int(g["q1"])) for g in seq] == [(6, 8), (7, 6), (6, 8)]


def _check_plan(circ, n, m, b, fuse=True):
    plan = qs.qs_plan_passes(n, m, circ, b=b, L0=5, fuse=fuse)
    covered = []
    for p in plan:
        covered.append((p["first"], p["nops"]))
        if p["type"] == 1:
            mask = p["tile_mask"]
            assert bin(mask).count("1") == min(b, m)
            assert mask & 0b11111 == 0b11111
    firsts = [f for f, _ in covered]
    assert firsts == sorted(firsts)
    assert sum(k for _, k in covered) <= len(circ)
    return plan


def test_plan_qft_fuses():
    n = 30
    q = C.qft(n)
    plan = _check_plan(q, n, n, 12)
    assert sum(p["nops"] for p in plan) == len(q)
    assert len(plan) < 12, len(plan)
    # the final qubit reversal (n/2 disjoint SWAPs over all n qubits) is ONE permutation pass
    assert plan[-1]["type"] == 3 and plan[-1]["nops"] == n // 2 and plan[-1]["first"] == len(q) - n // 2
    assert sum(p["type"] == 3 for p in plan) == 1
    unf = _check_plan(q, n, n, 12, fuse=False)
    assert all(p["type"] == 0 for p in unf) and len(unf) == len(q)


def test_plan_rqc_and_sweeps():
    circ = C.rqc_grid(32)
    plan = _check_plan(circ, 32, 32, 12)
    assert len(plan) <= 100
    # the 1q sweep on distinct targets: high targets cannot share a tile beyond capacity
    sw = C.sweep_1q(30)
    plan = _check_plan(sw, 30, 30, 12)
    assert sum(p["nops"] for p in plan) == 30
    # with global qubits the exchange ops are their own passes
    plan = _check_plan(C.config1(20), 20, 17, 11)
    assert any(p["type"] == 2 for p in plan)


def test_phase_ladders_formed_and_jit_sources_compile():
    """PHASE LADDER merge on the QFT: every target's controlled-R_k run
    becomes one op, and the NVRTC straight-line source of every distinct pass structure compiles for
    sm_100a (compile only: NVRTC needs no GPU), with ladders on and off, single shard and a sharded rank."""
    n = 20
    q = C.qft(n)
    off = qsmod.qs_plan_tile_jit(n, n, q, ladder_min=0, compile=False)
    on = qsmod.qs_plan_tile_jit(n, n, q, ladder_min=4, compile=True)
    # the final n/2 SWAPs form one permutation pass (not tile ops); the H gates' factored scalar is one
    # whole-state scale op
    assert off["ladders"] == 0 and off["tile_ops"] == len(q) - n // 2 + 1
    # targets t >= 4 carry >= 4 controlled phases each: one ladder per target (t = 0..3 stay single ops)
    assert on["ladders"] == n - 4
    assert on["tile_ops"] == len(q) - n // 2 + 1 - sum(t for t in range(4, n)) + (n - 4)
    assert on["compiled"] == on["sources"] >= 1
    shard = qsmod.qs_plan_tile_jit(n, n - 3, q, rank=5, ladder_min=1, compile=True)
    assert shard["ladders"] > 0 and shard["compiled"] == shard["sources"]
    ring = qsmod.qs_plan_tile_jit(14, 14, C.rqc_ring(14, layers=2) + C.config1(14), ladder_min=1, compile=True)
    assert ring["compiled"] == ring["sources"]


def test_family_kernel_sources_depend_on_shape_only():
    """with the family form (monomial gates of the grid RQC's {sqrtX, sqrtY, sqrtW} select
    their member at run time) two seeds of the same circuit shape generate the
    SAME pass kernels — a never-seen seed compiles nothing — while the specialised form (every entry code a
    compile-time constant, the fastest kernel) differs between seeds.  Sources are generated, not compiled."""
    for n, mk in ((20, lambda s: C.rqc_grid(20, seed=s)), (25, lambda s: C.rqc_grid(25, depth=8, seed=s))):
        fam = [qsmod.qs_plan_tile_jit(n, n, mk(s), L0=3, compile=False, family=True) for s in (20, 21)]
        spec = [qsmod.qs_plan_tile_jit(n, n, mk(s), L0=3, compile=False) for s in (20, 21)]
        assert fam[0]["source_hash"] == fam[1]["source_hash"], n
        assert spec[0]["source_hash"] != spec[1]["source_hash"], n
        assert fam[0]["sources"] == spec[0]["sources"]
    one = qsmod.qs_plan_tile_jit(12, 12, C.rqc_grid(12, depth=6), L0=3, compile=True, family=True)
    assert one["compiled"] == one["sources"] >= 1


def test_warp_local_batch_transitions(tmp_path):
    """Warp- and group-local batch transitions (k_tile.cu align_warp_bits, jit_tile_source): a pass kernel
    separates two register batches with __syncwarp instead of a CTA barrier only when both batches map the
    warp-selecting sub-cube bits 5..7 (256 threads, 2^8 sub-cubes) onto the same tile positions — every warp
    then reads back exactly the amplitudes it wrote — and with a named barrier of a group of 2^k warps only
    when the bits 5+k..7 (which group) agree.  Checked on the generated sources of grid RQCs (the deps are
    compile-time constants of sub_deposit_ct); the alignment must find such transitions, and the sources
    with them compile for sm_100a."""
    import re
    import subprocess
    counts = {}
    for wl in ("0", "1"):
        dump = tmp_path / ("dump" + wl)
        dump.mkdir()
        env = dict(os.environ, QS_JIT_DUMP_DIR=str(dump), QS_WARP_LOCAL=wl)
        code = ("import sys, json; sys.path.insert(0, %r); import paper_2506_09198_b200 as q; "
                "from qsinputs import circuits as C; "
                "print(json.dumps([q.qs_plan_tile_jit(25, 25, C.rqc_grid(25, depth=8), L0=3, compile=True), "
                "q.qs_plan_tile_jit(20, 20, C.rqc_grid(20), L0=3, compile=False)]))" % ROOT)
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=900)
        assert r.returncode == 0, r.stderr[-2000:]
        st = json.loads(r.stdout.strip().splitlines()[-1])
        assert st[0]["compiled"] == st[0]["sources"] >= 1
        counts[wl] = st[0]["group_local"] + st[1]["group_local"]
        assert st[0]["group_local"] >= st[0]["warp_local"]
        nsync = 0
        for f in dump.glob("*.cubin.cu"):
            lines = f.read_text().splitlines()
            deps = [(i, int(m.group(1))) for i, l in enumerate(lines)
                    for m in [re.search(r"sub_deposit_ct<(\d+)ull, 8>", l)] if m]
            for i, l in enumerate(lines):
                m = re.search(r'"r"\(1 \+ \(c\.tid >> (\d+)\)\), "r"\((\d+)\)', l)
                if l.strip() == "__syncwarp();":
                    lo = 5  # every warp bit must agree
                elif m and "bar.sync" in l:
                    lo = int(m.group(1))  # a group of 2^(lo-5) warps: the bits above it must agree
                    assert int(m.group(2)) == 1 << lo  # the barrier counts exactly the group's threads
                else:
                    continue
                nsync += 1
                before = [d for j, d in deps if j < i][-1]
                after = [d for j, d in deps if j > i][0]
                assert all((before >> (4 * k)) & 15 == (after >> (4 * k)) & 15 for k in range(lo, 8)), f.name
        if wl == "1":
            assert nsync > 0
    assert counts["1"] > counts["0"], counts


def test_background_compiler_process(tmp_path):
    """The JIT's background compiler runs as a separate process (qs_jitc, beside the library): a source file
    in, its cubin in the on-disk cache under the same key the library looks up (the key the source dump of
    qs_plan_tile_jit uses), the input file deleted.  No GPU needed (NVRTC only)."""
    import subprocess
    dump, cache = tmp_path / "dump", tmp_path / "cache"
    dump.mkdir()
    cache.mkdir()
    env = dict(os.environ, QS_JIT_DUMP_DIR=str(dump))
    code = ("import sys; sys.path.insert(0, %r); import paper_2506_09198_b200 as q; from qsinputs import circuits as C; "
            "q.qs_plan_tile_jit(12, 12, C.rqc_grid(12, depth=3), L0=3, compile=True)" % ROOT)
    subprocess.run([sys.executable, "-c", code], env=env, check=True, timeout=600)
    srcs = sorted(dump.glob("*.cubin.cu"))
    assert srcs
    inp = tmp_path / "in.src"
    inp.write_bytes(srcs[0].read_bytes())
    exe = os.path.join(ROOT, "paper_2506_09198_b200", "qs_jitc")
    r = subprocess.run([exe, str(inp)], env=dict(os.environ, QS_JIT_CACHE=str(cache)), timeout=600)
    assert r.returncode == 0 and not inp.exists()
    key = srcs[0].name[: -len(".cu")]
    assert (cache / key).exists() and (cache / key).read_bytes() == (dump / key).read_bytes()


def _is_diag(g):
    return np.count_nonzero(g.m - np.diag(np.diag(g.m))) == 0


def test_reorder_schedule_is_a_valid_commutation_order():
    """Commutation-aware pass scheduling (qs_run_circuit's default): every gate runs exactly once and
    every pair of gates that share a qubit and do not commute keeps its order (diagonal gates commute
    with each other; anything else sharing a qubit does not) — on the grid RQC, the QFT, the paper's
    ring RQC, random circuits and sharded layouts.  The grid RQC needs far fewer HBM passes."""
    rng = np.random.Generator(np.random.PCG64(3))
    cases = [(C.rqc_grid(32), 32, 32), (C.rqc_grid(20), 20, 20), (C.qft(24), 24, 24), (C.rqc_ring(16, 5), 16, 16),
             (C.rqc_grid(20), 20, 17), (C.qft(20), 20, 18)]
    for _ in range(6):
        n = int(rng.integers(8, 16))
        circ = []
        for _ in range(120):
            a, b = (int(x) for x in rng.choice(n, 2, replace=False))
            r = rng.random()
            if r < 0.35:
                circ.append(C.g1(a, G.haar(2, rng) if rng.random() < 0.6 else G.T))
            elif r < 0.7:
                circ.append(C.gc(a, b, [G.X, G.phase(0.7), G.haar(2, rng)][int(rng.integers(3))]))
            else:
                circ.append(C.g2(a, b, [G.haar(4, rng), G.SWAP, np.diag(np.exp(1j * rng.random(4)))][int(rng.integers(3))]))
        cases.append((circ, n, n - int(rng.integers(0, 3))))
    for circ, n, m in cases:
        plan, order = qs.qs_plan_passes(n, m, circ, b=12, L0=4, reorder=True, with_order=True)
        assert sorted(order) == list(range(len(circ))), "every gate exactly once"
        pos = {g: k for k, g in enumerate(order)}
        qsets = [set(g.qubits()) for g in circ]
        dg = [_is_diag(g) for g in circ]
        for i in range(len(circ)):
            for j in range(i + 1, len(circ)):
                if qsets[i] & qsets[j] and not (dg[i] and dg[j]):
                    assert pos[i] < pos[j], (i, j, circ[i].kind, circ[j].kind)
        for p in plan:  # tile passes hold their non-diagonal qubits
            if p["type"] == 1:
                assert bin(p["tile_mask"]).count("1") == min(12, m)
    plan0 = qs.qs_plan_passes(32, 32, C.rqc_grid(32), b=12, L0=4, reorder=False)
    plan1 = qs.qs_plan_passes(32, 32, C.rqc_grid(32), b=12, L0=4, reorder=True)
    assert len(plan1) * 2 < len(plan0), (len(plan0), len(plan1))


def _gates_from_array(arr):
    out = []
    for g in arr:
        k, q0, q1 = int(g["kind"]), int(g["q0"]), int(g["q1"])
        m = g["m"].view(np.complex128)
        if k == 0:
            out.append(C.g1(q0, m[:4].reshape(2, 2)))
        elif k == 1:
            out.append(C.gc(q0, q1, m[:4].reshape(2, 2)))
        else:
            out.append(C.g2(q0, q1, m[:16].reshape(4, 4)))
    return out


def test_global_remap_equals_original_on_the_oracle(orc):
    """Global-qubit remapping (qs_run_circuit on sharded states): the physical gate list — swap-to-local
    SWAPs, relabelled SWAP gates, restoring SWAPs — run by the ORACLE gives the logical circuit's state
    bit for bit (same matrices on the same amplitude pairs), every gate that needs a qubit locally finds
    it local, and the grid RQC's exchange volume halves (3 half-shard swaps per cycle instead of 3 full
    exchanges)."""
    rng = np.random.Generator(np.random.PCG64(8))
    cases = [(C.rqc_grid(12), 12, 10), (C.qft(11), 11, 8), (C.config1(10), 10, 8), (C.rqc_ring(10, 3), 10, 9)]
    for _ in range(8):
        n = int(rng.integers(6, 12))
        circ = []
        for _ in range(80):
            a, b = (int(x) for x in rng.choice(n, 2, replace=False))
            r = rng.random()
            if r < 0.3:
                circ.append(C.g1(a, G.haar(2, rng) if rng.random() < 0.7 else G.T))
            elif r < 0.6:
                circ.append(C.gc(a, b, [G.X, G.phase(0.7), G.haar(2, rng)][int(rng.integers(3))]))
            else:
                circ.append(C.g2(a, b, [G.haar(4, rng), G.SWAP, np.diag(np.exp(1j * rng.random(4)))][int(rng.integers(3))]))
        cases.append((circ, n, n - int(rng.integers(1, 4))))
    for circ, n, m in cases:
        phys, (before, after) = qsmod.qs_plan_remap(n, m, circ)
        pg = _gates_from_array(phys)
        for g in pg:  # non-diagonal roles are local except swap-to-local / restoring SWAPs
            is_swap = g.kind == "2q" and np.array_equal(g.m, G.SWAP)
            diag = np.count_nonzero(g.m - np.diag(np.diag(g.m))) == 0
            if not is_swap and not diag:
                need = [g.q0] if g.kind == "1q" else [g.q1] if g.kind == "c1q" else [g.q0, g.q1]
                assert all(q < m for q in need), (g.kind, g.q0, g.q1, m)
        a = orc.random_state(n, 5)
        b = a.copy()
        orc.run(a, circ)
        orc.run(b, pg)
        assert np.array_equal(a, b), (n, m)
    _, (before, after) = qsmod.qs_plan_remap(20, 17, C.rqc_grid(20))
    assert before == 20 * 3 * 2 and after <= 20 * 3 + 12, (before, after)  # + restoring swaps


def test_plan_hoists_qft_reversal(orc):
    """Permutation hoisting (qs_plan.h hoist_permutation): the QFT's final reversal, too wide to join
    the last ladder pass, is split over two earlier tile passes (their stores), the gates in between
    relabelled — one HBM pass fewer.  The rewritten op list (execution order) must give the same state
    as the paper's circuit: both applied by the ORACLE, gate by gate, on a random state; relabelling
    changes no arithmetic, so the states are bitwise equal.  Also checked: every transposition of the
    reversal appears once, and the gate count is unchanged."""
    for n, b, L0 in ((12, 6, 2), (14, 7, 2), (16, 6, 2), (20, 6, 2), (20, 8, 3), (22, 10, 2)):
        circ = C.qft(n)
        out, st = qs.qs_plan_hoist(n, n, circ, b=b, L0=L0)
        assert st["after"] == st["before"] - 1 and st["fused"] >= 1, (n, b, L0, st)
        hg = _gates_from_array(out)
        assert len(hg) == len(circ)
        swaps = [(g.q0, g.q1) for g in hg if g.kind == "2q" and np.array_equal(g.m, G.SWAP)]
        assert sorted(tuple(sorted(p)) for p in swaps) == [(q, n - 1 - q) for q in range(n // 2)]
        a = orc.random_state(n, 11)
        c = a.copy()
        orc.run(a, circ)
        orc.run(c, hg)
        assert np.array_equal(a, c), (n, b, L0, float(np.max(np.abs(a - c))))
    # QFT(32) as the library plans it (12-qubit tiles, 4 low qubits): 4 ladder passes + the reversal
    # -> 4 passes, the reversal riding on two of them
    _, st = qs.qs_plan_hoist(32, 32, C.qft(32), b=12, L0=4)
    assert st == {"before": 5, "after": 4, "fused": 2}
    # nothing to hoist: grid RQC has no permutation pass
    out, st = qs.qs_plan_hoist(20, 20, C.rqc_grid(20), b=12, L0=4)
    assert len(out) == 0 and st["before"] == st["after"]


def test_plan_hoists_random_swap_runs(orc):
    """Permutation hoisting on random circuits (U2, CNOT, CPhase, U4, H around a run of disjoint SWAPs
    over the qubits, qsinputs.circuits.random_with_swap_run): wherever the planner removes the
    permutation pass, the rewritten op list (gate order kept: reorder = 0) applied by the ORACLE gives
    bitwise the input circuit's state — every gate kind relabelled, controls and U4 qubit order kept."""
    hits = 0
    for seed in range(40):
        n, b = 12 + seed % 5, 6 + seed % 3
        circ = C.random_with_swap_run(n, seed)
        out, st = qs.qs_plan_hoist(n, n, circ, b=b, L0=2, reorder=False)
        if not len(out):
            assert st["after"] == st["before"]
            continue
        hits += 1
        assert st["after"] == st["before"] - 1
        hg = _gates_from_array(out)
        a = orc.random_state(n, seed)
        c = a.copy()
        orc.run(a, circ)
        orc.run(c, hg)
        assert np.array_equal(a, c), (seed, n, b, float(np.max(np.abs(a - c))))
    assert hits >= 10, hits


def test_plan_fuses_qft_reversal():
    """The QFT's final reversal (a run of disjoint SWAPs) joins the last tile pass when that pass's
    qubits close under the permutation within 11 qubits: QFT(32) at tile_low 3 = 4 passes, the last
    one (type 4) on qubits {0..4} U {27..31}; at tile_low 4 the last pass is too wide and the reversal
    stays a permutation pass (type 3).  Every gate appears once in the execution order."""
    circ = C.qft(32)
    plan, order = qs.qs_plan_passes(32, 32, circ, b=12, L0=3, reorder=True, with_order=True)
    assert [p["type"] for p in plan] == [1, 1, 1, 4]
    assert plan[-1]["tile_mask"] == sum(1 << q for q in list(range(5)) + list(range(27, 32)))
    assert sorted(order) == list(range(len(circ)))
    assert all(circ[i].kind == circ[-1].kind for i in order[-16:])  # the SWAPs run last
    plan4 = qs.qs_plan_passes(32, 32, circ, b=12, L0=4, reorder=True)
    assert [p["type"] for p in plan4] == [1, 1, 1, 1, 3]
