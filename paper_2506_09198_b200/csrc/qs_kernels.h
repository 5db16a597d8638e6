// qs_kernels.h — host-callable launchers for the sm_100a kernels (definitions in k_*.cu).
//
// All launchers are asynchronous on `st` and return the number of kernels they launched (for
// qs_launch_count).  `a` is a shard: 2^m amplitudes (double2 = {re, im}, AoS).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "qs_plan.h"

namespace qsb {

// ---- single-op kernels (k_gates.cu) ---------------------------------------------------------
// `op` must be local (all qubits < m).  Dispatches PAIR / CTRL_PAIR / QUAD / DIAG / SWAP.
int launch_op(double2 *a, int m, const Op &op, cudaStream_t st, int num_sms);

// ---- fused tile pass (k_tile.cu) ---------------------------------------------------------------
constexpr int TILE_MAX_Q = 13;  // 2^13 amplitudes = 128 KiB of shared memory

struct TileOp {  // one op in tile coordinates
    int32_t kind;          // OpKind
    int32_t p0, p1;        // tile-local bit positions of q0 / q1, or -1 when outside the tile
    int32_t q0, q1;        // local qubit numbers (-1 if absent); used for outside-tile fixed bits
    uint32_t touch;        // DIAG
    int32_t pad[2];
    double2 m[16];         // PAIR/CTRL: m[0..3]; QUAD: m[0..15]; DIAG: d[k] = m[k]
};

struct TileDesc {
    int32_t b;             // tile qubits
    int32_t L;             // contiguous low qubits 0..L-1 in the tile
    int32_t n_hi;          // b - L
    int32_t n_out;         // number of local qubits outside the tile (m - b)
    int32_t hi_q[TILE_MAX_Q];   // local qubit of tile bit L+i
    int32_t out_q[40];     // local qubits outside the tile, ascending (tile-id bit i -> out_q[i])
    int32_t nops;
    int32_t op0;           // index of the first TileOp in the op array
};

// Build the tile-coordinate op list of one pass for one shard from LOCAL ops.
void make_tile_pass(const int *tile_q, int b, int L, int m, const Op *local_ops, int nops, TileDesc &desc,
                    TileOp *out_ops);

// Launch one tile pass; desc/ops point to DEVICE memory; the host copy `hdesc` gives sizes.
int launch_tile(double2 *a, int m, const TileDesc &hdesc, const TileDesc *ddesc, const TileOp *dops,
                cudaStream_t st, int num_sms);

// ---- state kernels (k_state.cu) ----------------------------------------------------------------
int launch_init_random(double2 *a, uint64_t count, uint64_t global_base, uint64_t seed, cudaStream_t st,
                       int num_sms);
int launch_set_amp(double2 *a, uint64_t index, double re, double im, cudaStream_t st);
int launch_scale(double2 *a, uint64_t count, double s, cudaStream_t st, int num_sms);
// Deterministic sum |a|^2 of count = 2^j amplitudes: leaves of min(count, 2^13) amplitudes, then a
// perfect binary tree.  `scratch` holds >= count/2^13 + 1024 doubles.  Result at *d_out.
constexpr int NORM_LEAF_LOG2 = 13;
int launch_norm2(const double2 *a, uint64_t count, double *scratch, double *d_out, cudaStream_t st,
                 int num_sms);

// ---- exchange kernels (k_state.cu) -------------------------------------------------------------
// Fused global-qubit update of one chunk (§8(e)): for i in [0, count):
//   if ctrl < 0 or bit ctrl of (local_offset + i) is 1:
//     bit == 0: a[i] = u00 a[i] + u01 r[i];  bit == 1: a[i] = u10 r[i] + u11 a[i]
// (operand order equal to the local PAIR kernel, so the result is bitwise P-invariant).
int launch_xpair_update(double2 *a, const double2 *r, uint64_t count, uint64_t local_offset, int ctrl,
                        int bit, const double *u2, cudaStream_t st, int num_sms);
// pack/unpack the sub-lattice {local index i : bit l of i == v}, elements [j0, j0 + count) of it.
int launch_pack(const double2 *a, double2 *buf, int l, int v, uint64_t j0, uint64_t count, cudaStream_t st,
                int num_sms);
int launch_unpack(double2 *a, const double2 *buf, int l, int v, uint64_t j0, uint64_t count, cudaStream_t st,
                  int num_sms);

}  // namespace qsb
