/*
 * qs_plan_abi.h — host-only planner entry points of libqs_b200 (no GPU needed).
 *
 * They expose the exact host logic the library runs before launching kernels, so that it can be
 * tested on CPU: gate classification (SURVEY.md §8(a) a7/a8 specialisations), the per-shard
 * routing of a gate on a sharded state (§8(e) table), the swap-to-local decomposition of
 * 2-qubit gates on global qubits, and the tile-pass planner (§8(a) a9).
 * Same conventions as qs.h.  None of these allocate device memory or touch CUDA.
 */
#ifndef QS_PLAN_ABI_H
#define QS_PLAN_ABI_H

#include <stddef.h>
#include <stdint.h>

#include "qs.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Routing actions (ShardStep.action) */
enum {
    QS_SA_SKIP = 0,      /* shard does nothing                                               */
    QS_SA_LOCAL = 1,     /* shard runs a local op (out_op)                                   */
    QS_SA_XPAIR = 2,     /* global-target 1q: exchange with partner, row `bit` of U; ctrl_local
                            >= 0 restricts the update to local amps whose bit ctrl_local == 1 */
    QS_SA_XSWAP_LG = 3,  /* SWAP(local l, global): send local amps with bit l == 1-bit, receive
                            the partner's into the same positions                              */
    QS_SA_XSWAP_GG = 4,  /* SWAP(global, global), this rank's two bits differ: swap shards    */
    QS_SA_VIA_SWAP = 5   /* 2q op on a global qubit: see qs_plan_decompose                    */
};

/* Op kinds after classification (out_op[0]) */
enum { QS_OP_PAIR = 0, QS_OP_CTRL_PAIR = 1, QS_OP_QUAD = 2, QS_OP_DIAG = 3, QS_OP_SWAP = 4 };

/* Classify gate g on an n-qubit state and route it for shard `rank` of P = 2^(n-m) shards.
 * out_step[0..4] = {action, partner, bit, ctrl_local, l};
 * out_op[0..3]   = {kind, q0, q1, touch} of the local op (valid for QS_SA_LOCAL / QS_SA_XPAIR);
 * out_m[0..31]   = its matrix (PAIR/CTRL: U2 in [0..8); QUAD: U4; DIAG: d[k] at [2k, 2k+1]).
 * Returns QS_ERR_ARG on an invalid gate (message via qs_last_error(NULL)). */
qs_status qs_plan_route(int n, int m, int rank, const qs_gate *g, int check_unitary, int32_t out_step[5],
                        int32_t out_op[4], double out_m[32]);

/* SWAP-to-local decomposition of a non-diagonal 2q gate touching global qubits (m local qubits):
 * writes the gate sequence [SWAP(f, g)..., gate', SWAP(f, g)...] (SWAP as QS_G_2Q with the SWAP
 * matrix) to out (capacity max_out) and returns the count, or -1. */
int qs_plan_decompose(int n, int m, const qs_gate *g, qs_gate *out, int max_out);

/* Tile-pass plan of a circuit (m local qubits, tile of b qubits, L0 low qubits always in a tile;
 * reorder != 0: commutation-aware scheduling inside each segment between exchanges, as qs_run_circuit
 * does by default).  For pass i: out_type[i] (0 = single-op kernel, 1 = tile pass, 2 = exchange op,
 * 3 = qubit-permutation pass), out_nops[i], out_first[i] = index of its first gate in execution order,
 * out_tile_mask[i] = bitmask of its tile qubits (type 1).  out_order (may be NULL; capacity n_gates)
 * receives the gate indices of all passes concatenated in execution order (exact identities are
 * dropped).  Returns the number of passes (<= max_passes) or -1. */
int qs_plan_passes(int n, int m, const qs_gate *gates, size_t n_gates, int b, int L0, int fuse, int reorder,
                   int32_t *out_type, int32_t *out_nops, int32_t *out_first, uint64_t *out_tile_mask,
                   int32_t *out_order, int max_passes);

/* Global-qubit remapping of a circuit on m local qubits (what qs_run_circuit does on a sharded state
 * when it lowers the exchange volume): writes the equivalent gate list in PHYSICAL qubit positions —
 * swap-to-local SWAP(local, global) gates inserted before gates that need a global qubit locally, SWAP
 * gates of the input turned into relabellings, trailing SWAPs that restore the canonical layout —
 * to out (capacity max_out).  Diagonal gates come out as diagonal matrices.  out_cost = {exchange
 * volume of the input, of the output} in half-shard units per rank.  Returns the count, or -1. */
int qs_plan_remap(int n, int m, const qs_gate *gates, size_t n_gates, qs_gate *out, int max_out, int32_t out_cost[2]);

/* Permutation hoisting (qs_plan.h hoist_permutation, the QFT's final reversal): plan the
 * circuit (tile of b qubits, L0 low qubits, reorder = commutation-aware scheduling) and split its first
 * removable permutation pass over the tile passes before it.  Writes the resulting op list in
 * EXECUTION order — relabelled gates, each fused pass's SWAPs after its gates — to out (capacity
 * max_out; diagonal ops as diagonal matrices, SWAPs as 4x4 permutation matrices) and returns its length;
 * 0 if nothing was hoisted; -1 on bad input or capacity.  out_stats = {passes before, passes after,
 * passes with a fused permutation}.  Applying the output gates in order gives the same state as the
 * input circuit (tests/test_abi_cpu.py checks it with the oracle). */
int qs_plan_hoist(int n, int m, const qs_gate *gates, size_t n_gates, int b, int L0, int reorder, qs_gate *out,
                  int max_out, int32_t out_stats[3]);

/* Build the fused tile passes of a circuit exactly as qs_run_circuit would for shard `rank` (m local
 * qubits, tile of b qubits, L0 low qubits, PHASE LADDER merge of runs >= ladder_min; 0 = off), generate
 * the NVRTC source of each distinct pass structure and, if `compile`, compile it for sm_100a (NVRTC
 * only: no device, nothing loaded or cached).  `compile` bit 0: compile; bit 1: generate the FAMILY
 * form of each source (monomial gates of a known family select their member at run time, jit_tile.cu).
 * out_stats = {passes, tile passes, tile ops, ladders, distinct sources, sources compiled, register
 * batches, FNV-1a hash of all sources (low 31 bits), batch transitions separated by __syncwarp instead of
 * a CTA barrier (warp-local: both batches give each warp the same amplitudes, k_tile.cu align_warp_bits),
 * batch transitions separated by any barrier narrower than the CTA (a warp or a group of warps)}.  QS_ERR_ARG on bad input, QS_ERR_UNSUPPORTED if a source does not
 * compile (NVRTC log via qs_last_error(NULL)). */
qs_status qs_plan_tile_jit(int n, int m, int rank, const qs_gate *gates, size_t n_gates, int b, int L0, int ladder_min,
                           int compile, int32_t out_stats[10]);

/* Background-compiler entry (the qs_jitc helper process the JIT executor spawns): compile the NVRTC tile
 * source stored in the file `path` into the on-disk cubin cache ($QS_JIT_CACHE, else the user cache dir)
 * and delete the file.  0 on success.  No CUDA call. */
int qs_jit_compile_file(const char *path);

#ifdef __cplusplus
}
#endif
#endif /* QS_PLAN_ABI_H */
