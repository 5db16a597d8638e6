// qs_plan.h — host-side gate classification, sharding localisation and tile-pass planning.
//
// Pure host C++ (no CUDA types), so it is exercised on CPU through the C-ABI test hooks
// (qs_plan_* in qs_api.cu) and by the world-size-2 gloo tests.
//
// Terminology:
//   n qubits, P = 2^k shards, m = n - k local qubits; qubit q >= m is "global" = bit (q-m) of the
//   shard rank.  An Op is one gate after exact classification:
//     OP_PAIR      general 1q on target q0                       (§8(a) a5/a6)
//     OP_CTRL_PAIR general 1q on target q1 where bit q0 == 1     (a7 general / CNOT)
//     OP_QUAD      general 4x4 on (q0, q1), k = bit_q0 + 2 bit_q1 (a8 general)
//     OP_DIAG      diagonal over nq in {0,1,2} qubits: amp *= d[k]; only k with d[k] != 1 touched
//                  (a7 diagonal / CPhase / CZ; nq = 0 means "scale the whole shard")
//     OP_SWAP      exchange k=1 <-> k=2 on (q0, q1)              (a8 SWAP)
#pragma once
#include <cstdint>
#include <cstdlib>
#include <string>
#include <vector>

namespace qsb {

enum OpKind : int32_t { OP_PAIR = 0, OP_CTRL_PAIR = 1, OP_QUAD = 2, OP_DIAG = 3, OP_SWAP = 4 };

struct Op {
    int32_t kind = OP_PAIR;
    int32_t q0 = -1, q1 = -1;  // see OpKind
    uint32_t touch = 0;        // OP_DIAG: bit k set <=> d[k] != 1
    double m[32] = {0};        // PAIR/CTRL: U2 (8); QUAD: U4 (32); DIAG: d[k] at m[2k], m[2k+1]
    int32_t form = 0;          // PAIR after factor_scalars: 1 = entries are monomials or w(+-1+-i) with
                               // one shared real w (the tile executor may apply them with adds + 1 FMA)
};

// Exact classification of one qs_gate (kind/q0/q1/m as in qs.h).  Returns false (with msg) on a
// bad argument.  `check_unitary`: reject max|U^H U - I| > 1e-10.  An exact identity gate yields
// an OP_DIAG with touch == 0 (the executor skips it).
bool classify(int n, int32_t kind, int32_t q0, int32_t q1, const double *m, bool check_unitary, Op &out,
              std::string &msg);

// What a shard with rank `rank` must do for a (globally indexed) Op.  Local ops are rewritten
// in the shard's local qubit space (< m); the rank's global bits are folded in.
enum ShardAction : int32_t {
    SA_SKIP = 0,        // nothing to do on this shard
    SA_LOCAL = 1,       // run `local` on the shard (no communication)
    SA_XPAIR = 2,       // global-target 1q: exchange with `partner`, fused update (row `bit` of U);
                        //   `ctrl_local` >= 0: only amps whose local bit ctrl_local == 1 change
    SA_XSWAP_LG = 3,    // SWAP(local l, global g): pack local amps with bit l == 1-bit, exchange,
                        //   unpack into the same positions (`l` = local qubit, `bit` = rank bit)
    SA_XSWAP_GG = 4,    // SWAP(global, global) and this rank's two bits differ: swap whole shards
    SA_VIA_SWAP = 5     // non-diagonal 2q op touching global qubits: decomposed by the executor
                        //   into SWAP(g, free local) + local op + SWAP back (see decompose_via_swap)
};

struct ShardStep {
    int32_t action = SA_SKIP;
    int32_t partner = -1;
    int32_t bit = 0;
    int32_t ctrl_local = -1;
    int32_t l = -1;
    Op local;  // SA_LOCAL: the op in local qubit space; SA_XPAIR: U2 in local.m[0..7]
};

ShardStep localize(const Op &op, int n, int m, int rank);

// SWAP-to-local decomposition of a QUAD/SWAP/CTRL op whose non-diagonal qubits include global
// ones: returns the list of global-space ops [SWAP(g, f)..., op', SWAP(g, f)...] where f are the
// highest local qubits not used by op.  Every op of the result is either local or a
// SWAP(local, global), which localize() maps to SA_LOCAL / SA_XSWAP_LG / SA_SKIP.
std::vector<Op> decompose_via_swap(const Op &op, int m);

// Global-qubit remapping for sharded states (m < n).  Returns an equivalent
// op list in PHYSICAL qubit positions: a gate that needs a global qubit locally (1q target, controlled
// target, either qubit of a general 2q gate) first swaps it with the local position whose logical
// qubit is needed furthest in the future (Belady) — a half-shard exchange instead of a full one, and
// later gates on that qubit are local; a SWAP gate only relabels (no data moves); diagonal gates and
// global controls never move data.  Trailing SWAPs restore the canonical layout (logical q at bit q),
// so the state after the list is exactly the state after `ops`.  Amplitude arithmetic is unchanged
// (same matrices on the same amplitude pairs): results are bitwise those of the original list.
std::vector<Op> remap_global(const std::vector<Op> &ops, int n, int m);

// Scalar factoring (the RQC's sqrt(X), sqrt(Y), sqrt(W), H, ...): a 1q gate U = c M whose M has every
// entry in {0, +-1, +-i} EXACTLY is applied as M — additions and sign/component swaps only, no
// multiplies; entries w(+-1+-i) with one shared real w (sqrt(W) = ((1+i)/2) [[1, -h(1+i)], [h(1-i), 1]])
// cost one extra FMA per component (form = 1) —
// and the scalars c are multiplied into one global factor, applied at the end of the list by a
// whole-state scale op (DIAG over no qubit), or earlier when |log2 of the deferred factor| > 400.
// Scalars commute with every gate, so the product is the same unitary; rounding differs from
// applying U directly (reading R21).
std::vector<Op> factor_scalars(const std::vector<Op> &ops);
// 0, 1, -1, i, -i -> 0..4 for an exact entry (re, im); -1 otherwise
int mono_code(const double *e);
// as mono_code, plus w(1+i), w(1-i), w(-1+i), w(-1-i) -> 5..8 (w = |re| = |im| > 0, returned in *w;
// every such entry of one matrix must share w)
int mono_code_w(const double *e, double *w);

// Exchange volume of an op list on m local qubits, in half-shard units per rank (a full pairwise
// exchange = 2, a packed/SWAP half exchange = 1, a 2q gate via swap-to-local = 2 per global qubit).
int exchange_cost(const std::vector<Op> &ops, int m);

// ---------------------------------------------------------------------------------------------
// Tile-pass planning (§8(a) a9): ops whose non-diagonal LOCAL qubits fit one tile of `b` qubits (the
// tile always contains local qubits 0..L0-1 so that global-memory runs are >= 2^L0 amplitudes
// contiguous) are applied in one HBM pass.  Diagonal ops and global-control CTRL ops that reduce to
// local ones join any tile.  Exchange ops and permutation runs split the list into segments; inside a
// segment ops keep gate order (reorder = false) or are scheduled through their dependency DAG
// (reorder = true; commuting gates may swap).  Pass.ops lists the ops in execution order.
// ---------------------------------------------------------------------------------------------
struct Pass {
    int32_t type = 0;             // 0 = single op (direct kernel), 1 = tile pass, 2 = exchange op,
                                  // 3 = qubit-permutation pass (run of disjoint local SWAPs, k_perm.cu)
    std::vector<int32_t> ops;     // indices into the op list
    std::vector<int32_t> tile_q;  // tile qubits (local), ascending, |tile_q| = b, tile_q[i]=i for i<L
    int32_t L = 0;                // number of contiguous low qubits in the tile
    std::vector<int32_t> perm;    // type 3: local qubit permutation (an involution), size m; type 1: the
                                  // permutation run that follows the pass, fused into its store (empty: none)
    std::vector<int32_t> perm_ops;  // type 1 with perm: the SWAP ops of the fused run (execution order)
};

inline int default_trials() {  // QS_PLAN_TRIALS overrides (measurement)
    static const int t = getenv("QS_PLAN_TRIALS") ? atoi(getenv("QS_PLAN_TRIALS")) : 48;
    return t < 1 ? 1 : t;
}

inline int default_restarts() {  // QS_PLAN_RESTARTS overrides (measurement)
    static const int r = getenv("QS_PLAN_RESTARTS") ? atoi(getenv("QS_PLAN_RESTARTS")) : 0;
    return r < 0 ? 0 : r;
}

struct PlanConfig {
    int b = 11;        // tile qubits
    int L0 = 5;        // low qubits always in a tile
    bool fuse = true;
    int perm_low = 5;  // permutation passes gather runs of 2^perm_low amplitudes (0 = no permutation passes)
    int trials = default_trials();  // reorder: greedy schedules tried per segment (first deterministic)
    int restarts = default_restarts();  // reorder: randomized reschedules of the tail after each prefix
    bool perm_fuse = true;  // a permutation run right after a tile pass whose needed qubits Q satisfy
                            // |Q ∪ pi(Q)| <= perm_fuse_b joins that pass (tile pairs, tile_kernel PAIR)
    int perm_fuse_b = 12;  // tile pairs of 2^12 amplitudes: two 64-KiB buffers, 512 threads, one CTA per SM
    bool reorder = false;  // commutation-aware scheduling of each segment between exchanges (changes
                           // the order of commuting gates: results agree to rounding, not bitwise)
};

// Qubits an op needs inside the tile (non-diagonal roles, in GLOBAL numbering); returns false if
// the op cannot be in a tile at all (non-diagonal role on a global qubit).
bool tile_requirements(const Op &op, int m, std::vector<int> &need);

std::vector<Pass> plan_passes(const std::vector<Op> &ops, int n, int m, const PlanConfig &cfg);

// Permutation hoisting (the QFT's final reversal).  A
// permutation pass (type 3: a run of disjoint SWAPs, pi = a product of transpositions) that follows a
// run of tile passes is split over those passes: transposition (a, b) moves to the end of tile pass k
// — fused into its store (tile pairs, tile_kernel PAIR) — and every op between pass k and the old
// permutation pass is relabelled a <-> b (SWAP_ab G(a) = G(b) SWAP_ab, exact).  Each fused pass k needs
// C_k = Q_k ∪ sigma_k(Q_k) <= perm_fuse_b qubits, where Q_k are its (relabelled) needed qubits and the
// low qubits; a transposition with both qubits inside Q_k or both outside costs no tile slot.  A small
// search (<= 8 passes, 3 choices each) takes the assignment with the fewest fused passes that places
// every transposition; the permutation pass disappears (one HBM pass fewer).  Returns false (outputs
// untouched) when no permutation pass can be removed; else the new op list (relabelled ops, the SWAPs
// of each fused pass as its perm_ops) and plan.
bool hoist_permutation(const std::vector<Op> &ops, const std::vector<Pass> &plan, int m, const PlanConfig &cfg,
                       std::vector<Op> &ops_out, std::vector<Pass> &plan_out);

}  // namespace qsb
