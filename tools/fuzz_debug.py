"""Reproduce one fuzz seed under option variants and report which differ from the unfused P=1 result."""
import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2506_09198_b200 as qs
from oracle import Oracle
from test_gpu_fuzz import random_circuit

seed = int(sys.argv[1])
rng = np.random.Generator(np.random.PCG64(1000 + seed))
P = [1, 1, 2, 4, 8][seed % 5]
k = P.bit_length() - 1
n = int(rng.integers(max(1, 8 + k if P > 1 else 1), 15))
circ = random_circuit(rng, n, int(rng.integers(20, 160)))
opts = {"fuse": 1, "tile_qubits": int(rng.integers(6, 13)), "jit": int(rng.integers(0, 2)), "tile_low": int(rng.integers(1, 7))}
chunk = P > 1 and rng.random() < 0.5
print("seed", seed, "n", n, "P", P, "gates", len(circ), "opts", opts, "chunk4096", chunk)
orc = Oracle()
ref = orc.random_state(n, 77 + seed); orc.run(ref, circ)
def run(P, virtual, o, chunk):
    with qs.QState(n, P, virtual=virtual) as st:
        for kk, v in o.items(): st.set_option(kk, v)
        if chunk: st.set_option("chunk_bytes", 4096)
        st.init_random(77 + seed); st.run(circ); return st.read()
base = run(1, False, {"fuse": 0}, False)
print("unfused vs oracle", np.max(np.abs(base - ref)))
for name, (PP, o, ch) in {
    "given": (P, opts, chunk), "P1_given": (1, opts, False), "P_unfused": (P, {"fuse": 0}, chunk),
    "P_unfused_nochunk": (P, {"fuse": 0}, False), "given_jit0": (P, dict(opts, jit=0), chunk),
    "given_jit1": (P, dict(opts, jit=1), chunk), "given_low5": (P, dict(opts, tile_low=5), chunk),
    "given_b12": (P, dict(opts, tile_qubits=12), chunk)}.items():
    g = run(PP, PP > 1, o, ch)
    print(f"{name:20s} equal={np.array_equal(g, base)} maxdiff={np.max(np.abs(g - base)):.3e} vs_oracle={np.max(np.abs(g - ref)):.3e}")
if not np.array_equal(run(1, False, {"fuse": 0}, False), base): print("nondeterministic!")
# bisect the circuit prefix for the 'given' config
lo, hi = 0, len(circ)
full = circ
while hi - lo > 1:
    mid = (lo + hi) // 2
    circ = full[:mid]
    b = run(1, False, {"fuse": 0}, False); g = run(P, P > 1, opts, chunk)
    if np.array_equal(b, g): lo = mid
    else: hi = mid
circ = full
print("first failing prefix length", hi, "gate", full[hi - 1].kind, full[hi - 1].q0, full[hi - 1].q1, full[hi-1].name)
print(np.round(full[hi-1].m, 3))
