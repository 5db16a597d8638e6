"""GPU: the tile-pass executor's process-wide shapes give bit-identical states.

The JIT pipeline options are read once per process from the environment (QS_TILE_DYN: dynamic tile
scheduling; QS_TILE_DIRECT: HBM I/O of the first / last register batch and the pipelined next-tile
gather; QS_PERM_DYN: dynamic scheduling of the permutation pass; QS_WARP_LOCAL: warp-aligned batch layouts
and __syncwarp between warp-local batches).  Each mode runs in its own process on
the same seeded inputs — QFT + grid RQC + configs[0] gates, on one shard and on two virtual shards —
and every final state must equal the default executor's bit for bit (the modes only move data
differently; the per-op arithmetic is the same template code).
"""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import hashlib, sys
sys.path.insert(0, %r)
import paper_2506_09198_b200 as qs
from qsinputs import circuits as C
out = []
for n, P, circ in ((20, 1, C.qft(20) + C.rqc_grid(20) + C.config1(20)), (18, 2, C.rqc_grid(12, depth=8) + C.qft(18)),
                   (25, 1, C.rqc_grid(25))):
    with qs.QState(n, P, virtual=P > 1) as st:
        st.set_option("jit_async", 0)
        st.init_random(2506)
        st.run(circ)
        a = st.read()
        out.append(hashlib.sha256(a.tobytes()).hexdigest() + ":" + str(st.jit_stats()["failed"]))
print(" ".join(out))
""" % ROOT

MODES = [
    {},
    {"QS_TILE_DYN": "0"},
    {"QS_TILE_DIRECT": "0"},
    {"QS_TILE_DIRECT": "1"},
    {"QS_TILE_DIRECT": "2"},
    {"QS_TILE_DIRECT": "3"},
    {"QS_TILE_DIRECT": "6"},
    {"QS_PERM_DYN": "0"},
    {"QS_TILE_NBUF": "2", "QS_TILE_CTAS": "1"},
    {"QS_WARP_LOCAL": "0"},  # round-2 lane layout, CTA barriers between all batches
    {"QS_WARP_LOCAL": "2"},  # warp alignment of shared-memory batches only
    {"QS_WARP_LOCAL": "3"},  # aligned layouts, CTA barriers kept
    {"QS_WARP_LOCAL": "4"},  # aligned layouts, warp barriers only (no named group barriers)
]


def _run(env_extra):
    env = dict(os.environ)
    env.update(env_extra)
    r = subprocess.run([sys.executable, "-c", SCRIPT], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return r.stdout.strip().splitlines()[-1]


def test_executor_modes_bitwise():
    base = _run(MODES[0])
    assert all(h.endswith(":0") for h in base.split()), base  # no failed JIT compilation
    for m in MODES[1:]:
        assert _run(m) == base, m


SCRIPT_STATE = r"""
import sys
import numpy as np
sys.path.insert(0, %r)
import paper_2506_09198_b200 as qs
from qsinputs import circuits as C
n = 20
with qs.QState(n) as st:
    st.set_option("jit_async", 0)
    st.init_random(2506)
    st.run(C.qft(n) + C.rqc_grid(20) + C.config1(n))
    np.save(sys.argv[1], st.read())
""" % ROOT


@pytest.mark.parametrize("env", [{"QS_PLAN_TRIALS": "1", "QS_BATCH_TRIALS": "1"},
                                 {"QS_PLAN_RESTARTS": "8"}, {"QS_PLAN_TRIALS": "200", "QS_BATCH_TRIALS": "64"}])
def test_schedule_search_options_keep_parity(orc, tmp_path, env):
    """The planner's search knobs change which commuting gates share a pass or a register batch (the
    rounding order, reading R21), never the result beyond the contract tolerance."""
    from gpu_util import assert_parity
    from qsinputs import circuits as C

    out = tmp_path / "state.npy"
    e = dict(os.environ)
    e.update(env)
    r = subprocess.run([sys.executable, "-c", SCRIPT_STATE, str(out)], env=e, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    got = np.load(out)
    n = 20
    circ = C.qft(n) + C.rqc_grid(20) + C.config1(n)
    ref = orc.random_state(n, 2506)
    orc.run(ref, circ)
    assert_parity(got, ref, len(circ), f"search options {env}")


SCRIPT_FAMILY = r"""
import json, sys
sys.path.insert(0, %r)
import paper_2506_09198_b200 as qs
from qsinputs import circuits as C
n = 20
with qs.QState(n) as st:
    if sys.argv[1] == "spec":
        st.set_option("jit_family", 0)
        st.set_option("jit_async", 0)
        st.init_basis(0); st.run(C.rqc_grid(n, seed=20)); st.sync()
        print(json.dumps(st.jit_stats()))
    else:
        st.init_basis(0); st.run(C.rqc_grid(n, seed=20)); st.sync()
        s0 = st.jit_stats()
        st.set_option("jit_wait", 1)
        s1 = st.jit_stats()
        st.init_basis(0); st.run(C.rqc_grid(n, seed=21)); st.sync()
        s2 = st.jit_stats()
        print(json.dumps([s0, s1, s2]))
""" % ROOT


def test_family_kernels_compiled_when_specialised_come_from_disk(tmp_path):
    """The hybrid JIT (jit_family = 1) keeps each pass's FAMILY kernel compiled even when the specialised
    kernel of the first seed comes straight from the disk cache: a first process fills the cache with
    specialised kernels only; a second runs seed 20 (specialised kernels loaded, nothing compiled in the
    foreground, the family forms compiled by the background helper), joins the helper, and then a
    never-seen seed 21 compiles nothing."""
    import json
    env = dict(os.environ, QS_JIT_CACHE=str(tmp_path / "cache"))
    r = subprocess.run([sys.executable, "-c", SCRIPT_FAMILY, "spec"], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert json.loads(r.stdout.strip().splitlines()[-1])["compiled"] > 0
    r = subprocess.run([sys.executable, "-c", SCRIPT_FAMILY, "default"], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    s0, s1, s2 = json.loads(r.stdout.strip().splitlines()[-1])
    assert s0["compiled"] == 0  # seed 20: every specialised kernel from the disk cache
    assert s1["compiled"] > 0  # the family kernels, compiled in the background
    assert s2["compiled"] == s1["compiled"] and s2["failed"] == 0  # seed 21: nothing compiled
