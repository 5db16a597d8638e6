// qs_kernels.h — host-callable launchers for the sm_100a kernels (definitions in k_*.cu).
//
// All launchers are asynchronous on `st` and return the number of kernels they launched (for
// qs_launch_count).  `a` is a shard: 2^m amplitudes (double2 = {re, im}, AoS).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "qs_plan.h"

namespace qsb {

// ---- single-op kernels (k_gates.cu) ---------------------------------------------------------
// `op` must be local (all qubits < m).  Dispatches PAIR / CTRL_PAIR / QUAD / DIAG / SWAP.
int launch_op(double2 *a, int m, const Op &op, cudaStream_t st, int num_sms);
// TMA bulk-copy streaming variant of the 1q gate (k_bulk.cu); needs m >= 11
int launch_pair_bulk(double2 *a, int m, int t, const double *m8, cudaStream_t st, int num_sms);

// ---- fused tile pass (k_tile.cu) ---------------------------------------------------------------
// A tile = 2^b amplitudes whose local indices differ only in the tile qubits (local qubits 0..L-1
// plus b-L higher ones).  Inside a tile the ops are grouped into BATCHES: a batch names R = 4 tile
// positions ("register slots"); every thread holds the 2^R = 16 amplitudes of one sub-cube spanned
// by those positions in registers and applies all ops of the batch there.  Non-diagonal ops of a
// batch act only on its register slots; diagonal ops and controls may use any bit (bits outside the
// slots are constants of the sub-cube or of the tile).
constexpr int TILE_MAX_Q = 12;  // 2 x 2^12 amplitudes = 128 KiB of shared memory (double buffer)
constexpr int TILE_MIN_Q = 6;
constexpr int TILE_R = 4;       // register slots per batch

struct TileOp {        // one op in batch coordinates (272 B); the first 16 B are the header
    int32_t code;      // host-decoded opcode (k_tile.cu apply_op): kind x register slots
    int32_t src0, src1;  // bit source of a non-register qubit: >= 0 tile position (bit of the
                         // sub-cube index), -1 constant 0, <= -2 local qubit -2-src (tile base)
    uint32_t touch;    // DIAG: bit k set <=> d[k] != 1; QUAD: index of its matrix among the pass's QUADs
    double2 m[16];     // PAIR/CTRL: m[0..3]; QUAD: m[0..15]; DIAG: d[k] = m[k]
};
// shared-memory budget for the op stream of one pass: 80 B per op + 256 B per QUAD matrix
constexpr int TILE_OP_SMEM = 80 * 1024;

struct TileBatch {
    int32_t rp[TILE_R];    // tile position of register slot i (ascending)
    uint32_t swo[16];      // swizzled shared-memory offset of register combination r
    int32_t op0, nops;     // ops[op0 .. op0+nops)
    int32_t pad[2];
};

struct TileDesc {
    int32_t b;             // tile qubits
    int32_t L;             // contiguous low qubits 0..L-1 in the tile
    int32_t n_hi;          // b - L
    int32_t n_out;         // number of local qubits outside the tile (m - b)
    int32_t hi_q[TILE_MAX_Q];   // local qubit of tile bit L+i
    int32_t out_q[40];     // local qubits outside the tile, ascending (tile-id bit i -> out_q[i])
    int32_t batch0, nbatch;     // batches[batch0 .. batch0+nbatch)
    int32_t op_begin, op_count; // ops of the whole pass (batch op0 values are absolute)
    int32_t quad_count;         // QUAD ops of the pass
    int32_t pad;
};

// Build one pass for one shard from LOCAL ops (appends to batches / ops; desc.batch0 and each
// batch's op0 index into those arrays).
void make_tile_pass(const int *tile_q, int b, int L, int m, const Op *local_ops, int nops, TileDesc &desc,
                    std::vector<TileBatch> &batches, std::vector<TileOp> &ops);

// Launch one tile pass; ddesc / dbatches / dops point to DEVICE copies; hdesc is the host copy.
int launch_tile(double2 *a, int m, const TileDesc &hdesc, const TileDesc *ddesc, const TileBatch *dbatches,
                const TileOp *dops, cudaStream_t st, int num_sms);

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
