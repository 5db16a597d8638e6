// qs_kernels.h — host-callable launchers for the sm_100a kernels (definitions in k_*.cu).
//
// All launchers are asynchronous on `st` and return the number of kernels they launched (for
// qs_launch_count).  `a` is a shard: 2^m amplitudes (double2 = {re, im}, AoS).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "qs_plan.h"
#include "qs_tile_types.h"

namespace qsb {

// ---- single-op kernels (k_gates.cu) ---------------------------------------------------------
// `op` must be local (all qubits < m).  Dispatches PAIR / CTRL_PAIR / QUAD / DIAG / SWAP.
int launch_op(double2 *a, int m, const Op &op, cudaStream_t st, int num_sms);

// ---- fused tile pass (k_tile.cu, jit_tile.cpp); descriptors in qs_tile_types.h ------------------
// Build one pass for one shard from LOCAL ops (appends to batches / ops; desc.batch0 and each
// batch's op0 index into those arrays).
// Runs of >= ladder_min consecutive pure-phase ops sharing one qubit become PHASE LADDER ops (records
// appended to lads; desc.lad_count of them; desc.lads must then be set to their device copy);
// ladder_min = 0 keeps every op (bitwise equal to the unfused path).  reorder_batches: batches are
// formed through the pass's dependency DAG (commuting ops may swap) instead of in the given order.
void make_tile_pass(const int *tile_q, int b, int L, int m, const Op *local_ops, int nops, TileDesc &desc,
                    std::vector<TileBatch> &batches, std::vector<TileOp> &ops, std::vector<TileLadder> &lads,
                    int ladder_min, bool reorder_batches = false);
// Fused permutation of a tile pass (TileDesc::perm): pi (size m, an involution) must map the pass's tile
// qubits onto themselves; fills out_pq and the tile-position permutation rho.  False if it does not.
bool set_tile_perm(TileDesc &desc, const int *tile_q, int b, const int *perm, int m);

// register slots per batch (QS_TILE_R = 3 or 4, default 4)
int tile_regs();
int tile_direct_io();  // bit 0: first batch reads HBM, bit 1: last batch writes HBM
int tile_warp_local();  // align warp positions of consecutive batches (make_tile_pass), default 1
// threads per CTA of a JIT tile kernel with 2^b-amplitude tiles and R register slots
int jit_tile_threads(int b, int R);
// consecutive batches with deps dep_a, dep_b hand every amplitude from a warp to the same warp (equal
// warp-selecting sub-cube bits 5 .. log2(tpb)-1): __syncwarp separates them (jit_tile_source)
bool warp_local_transition(uint64_t dep_a, uint64_t dep_b, int nsub_bits, int tpb);
// the smallest k such that the warp-selecting sub-cube bits 5 + k .. log2(tpb)-1 agree between the two deps:
// every group of 2^k consecutive warps then hands its amplitudes only to itself (0: warp-local; the number
// of warp bits: the whole CTA)
int transition_scope(uint64_t dep_a, uint64_t dep_b, int nsub_bits, int tpb);

// Launch one tile pass; ddesc / dbatches / dops point to DEVICE copies; hdesc is the host copy.
int launch_tile(double2 *a, int m, const TileDesc &hdesc, const TileDesc *ddesc, const TileBatch *dbatches,
                const TileOp *dops, cudaStream_t st, int num_sms);

// ---- fused peer-memory exchange (k_p2p.cu): one rank's half of a global-qubit gate, loading and
// storing both its own shard `loc` and the partner's `rem` (same device or peer-mapped).  action =
// SA_XPAIR (u2, ctrl = local control or -1), SA_XSWAP_LG (l), SA_XSWAP_GG (lower = rank < partner).
int launch_p2p_exchange(int action, double2 *loc, double2 *rem, int m, int bit, int ctrl, int l, bool lower,
                        const double *u2, cudaStream_t st, int num_sms);

// pairwise flag barrier between two ranks whose shards are peer-mapped (CUDA IPC), one-process-per-GPU
int launch_flag_barrier(unsigned long long *my_flags, unsigned long long *peer_flags, int me, int peer,
                        unsigned long long val, cudaStream_t st);

// ---- qubit-permutation pass (k_perm.cu): perm = involutive permutation of the m local qubits; tiles
// gather runs of 2^L amplitudes, L <= L0.  Returns -1 if perm is not usable (not an involution, ...).
// a zeroed-before-use global counter per (device, stream) for dynamic tile scheduling (jit_tile.cu)
unsigned long long *tile_counter(cudaStream_t st);
int launch_perm(double2 *a, int m, const int *perm, int L0, cudaStream_t st, int num_sms);

// ---- JIT executor of tile passes (jit_tile.cu) --------------------------------------------------
// Straight-line source of one pass (depends on its structure only), compile+cache (parallel NVRTC),
// launch (returns -1 if the source is not compiled or the pass does not fit).
// family = true: PAIR_MONO ops whose gate belongs to a monomial family (jit_tile.cu kMonoFamilies) select
// the member at run time (the source depends on the circuit's shape only); false: every entry code is a
// compile-time constant (the fastest kernel)
std::string jit_tile_source(const TileDesc &desc, const TileBatch *batches, const TileOp *ops, int R, bool family = false);
// async: disk-cached cubins load now, the others compile on background threads (launch_tile_jit
// returns -1 for a pass whose kernel is not ready: the interpreter runs it); jit_tile_wait joins them.
bool jit_tile_prepare(const std::vector<std::string> &sources, std::string &err, bool async = false);
void jit_tile_wait();
// compile src into the on-disk cubin cache (no CUDA call; the qs_jitc helper process runs this)
bool jit_compile_to_disk(const std::string &src, std::string &err);
// per pass: specialised source spec[i], family source fam[i] (== spec[i] without family ops); picks which
// to launch (use_family[i]) by `mode` and the caches, compiling what is needed now and the rest in the
// background (jit_tile.cu)
bool jit_tile_prepare_pair(const std::vector<std::string> &spec, const std::vector<std::string> &fam, int mode,
                           std::vector<int> &use_family, std::string &err, bool async,
                           std::vector<std::string> *deferred = nullptr);
// start background compilations (helper processes) of sources a prepare_pair call deferred
void jit_tile_background(const std::vector<std::string> &sources);
int launch_tile_jit(const std::string &src, double2 *a, int m, const TileDesc &hdesc, const TileDesc *ddesc,
                    const TileBatch *dbatches, const TileOp *dops, cudaStream_t st, int num_sms);
// NVRTC compile only (no device, no cache): CPU check that a pass's generated source builds
bool jit_tile_compile_check(const std::string &src, size_t *cubin_bytes, std::string &err);
void jit_tile_stats(uint64_t *compiled, uint64_t *launched, uint64_t *failed);

// ---- state kernels (k_state.cu) ----------------------------------------------------------------
int launch_set_amp(double2 *a, uint64_t index, double re, double im, cudaStream_t st);
int launch_scale(double2 *a, uint64_t count, double s, cudaStream_t st, int num_sms);
// Deterministic sum |a|^2 of count = 2^j amplitudes: leaves of 2^leaf_log2 amplitudes (>= 2), then a
// perfect binary tree.  `scratch` holds >= count/2^leaf_log2 + 1024 doubles.  Result at *d_out.
constexpr int NORM_LEAF_LOG2 = 13;
// leaf size for an n-qubit state: 2^min(13, n-3) (>= 2) never spans a shard for P <= 8, so every shard
// count sums the same leaves in the same tree and the norm is bitwise P-invariant
inline int norm_leaf_log2(int n) { return n - 3 < 1 ? 1 : (n - 3 > NORM_LEAF_LOG2 ? NORM_LEAF_LOG2 : n - 3); }
int launch_norm2(const double2 *a, uint64_t count, int leaf_log2, double *scratch, double *d_out, cudaStream_t st,
                 int num_sms);
// launch_init_random + launch_norm2 in one HBM pass: the generated amplitudes are stored and their leaf
// sums formed as they are generated (bitwise the sums launch_norm2 would form from the stored state)
int launch_init_random_norm(double2 *a, uint64_t count, uint64_t global_base, uint64_t seed, int leaf_log2,
                            double *scratch, double *d_out, cudaStream_t st, int num_sms);

// ---- exchange kernels (k_state.cu) -------------------------------------------------------------
// Fused global-qubit update of one chunk (§8(e)): for i in [0, count):
//   if ctrl < 0 or bit ctrl of (local_offset + i) is 1:
//     bit == 0: a[i] = u00 a[i] + u01 r[i];  bit == 1: a[i] = u10 r[i] + u11 a[i]
// (operand order equal to the local PAIR kernel, so the result is bitwise P-invariant).
int launch_xpair_update(double2 *a, const double2 *r, uint64_t count, uint64_t local_offset, int ctrl,
                        int bit, const double *u2, cudaStream_t st, int num_sms);
// controlled 1q, local control c, global target: fused update of the packed control-1 half
// (elements [j0, j0+count) of {i : bit c == 1}) with the partner's packed half r
int launch_xpair_packed(double2 *a, const double2 *r, int c, uint64_t j0, uint64_t count, int bit, const double *u2,
                        cudaStream_t st, int num_sms);
// pack/unpack the sub-lattice {local index i : bit l of i == v}, elements [j0, j0 + count) of it.
int launch_pack(const double2 *a, double2 *buf, int l, int v, uint64_t j0, uint64_t count, cudaStream_t st,
                int num_sms);
int launch_unpack(double2 *a, const double2 *buf, int l, int v, uint64_t j0, uint64_t count, cudaStream_t st,
                  int num_sms);

}  // namespace qsb
