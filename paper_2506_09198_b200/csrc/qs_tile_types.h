// qs_tile_types.h — device-visible descriptors of a fused tile pass (k_tile.cu, JIT kernels).
// Plain structs, includable by nvcc and by NVRTC (the JIT tile kernels, jit_tile.cpp).
#pragma once
#ifdef __CUDACC_RTC__
typedef int int32_t;
typedef unsigned int uint32_t;
typedef unsigned short uint16_t;
typedef unsigned long long uint64_t;
#else
#include <cuda_runtime.h>

#include <cstdint>
#endif

namespace qsb {

// A tile = 2^b amplitudes whose local indices differ only in the tile qubits (local qubits 0..L-1
// plus b-L higher ones).  Inside a tile the ops are grouped into BATCHES: a batch names R tile
// positions ("register slots"); every thread holds the 2^R amplitudes of one sub-cube spanned by
// those positions in registers and applies all ops of the batch there.  Non-diagonal ops of a batch
// act only on its register slots; diagonal ops and controls may use any bit (bits outside the slots
// are constants of the sub-cube or of the tile).
constexpr int TILE_MAX_Q = 12;  // 2 x 2^12 amplitudes = 128 KiB of shared memory (double buffer)
constexpr int TILE_MIN_Q = 6;
constexpr int TILE_R = 4;       // register slots per batch (max)

struct TileOp {        // one op in batch coordinates (272 B); the first 16 B are the header
    int32_t code;      // host-decoded opcode (qs_tile_ops.cuh): kind x register slots
    int32_t src0, src1;  // bit source of a non-register qubit: >= 0 tile position (bit of the
                         // sub-cube index), -1 constant 0, <= -2 local qubit -2-src (tile base),
                         // <= -1000 no constraint (phase ops)
    uint32_t touch;    // DIAG: bit k set <=> d[k] != 1; QUAD: index of its matrix among the pass's QUADs
    double2 m[16];     // PAIR/CTRL: m[0..3]; QUAD: m[0..15]; DIAG: d[k] = m[k]; PHASE: m[0]
};
// shared-memory budget for the op stream of one pass: 80 B per op + 256 B per QUAD matrix
constexpr int TILE_OP_SMEM = 80 * 1024;

struct TileBatch {
    int32_t rp[TILE_R];    // tile position of register slot i (ascending)
    uint32_t swo[16];      // swizzled shared-memory offset of register combination r
    int32_t op0, nops;     // ops[op0 .. op0+nops)
    uint64_t dep;          // sub-cube index bit i -> tile position (dep >> 4i) & 15 (the non-slot
                           // positions; the first five are the lane bits, chosen so the 32 lanes of a
                           // warp cover all 8 shared-memory columns of the swizzle: no bank conflicts)
};

// A PHASE LADDER: a run of consecutive pure-phase diagonal ops of one batch that all carry the
// constraint bit t (or, when t < 0, single-bit phases on different qubits), merged into one op:
//   amp *= [bit t of i] * k0 * prod_{c in C} (bit c of i ? x_c : 1)
// (the QFT's controlled-R_k ladder).  The control set C is split by
// where the bit lives: register slots (xs, compile-time in the opcode mask), sub-cube tile positions
// (tj: three 16-entry product tables by tile-position nibble, looked up with the sub-cube index jb)
// and qubits outside the tile (bq/bx: their product is a constant of the tile, formed once per tile
// by one warp, TileCtx::lad_k).  One factor per amplitude instead of one multiply per gate; the
// rounding of the factor product differs from gate-by-gate by a few ulp (reading R21).
constexpr int TILE_MAX_LADDERS = 24;  // per pass (lad_k in static shared memory)
constexpr int TILE_LADDER_BASE = 28;  // controls outside the tile (n_out <= 27)
struct TileLadder {
    double2 k0;                       // constant factor (ops on t alone; global control bits folded)
    double2 xs[4];                    // factor of register slot s (1 if slot s is not a control)
    double2 tj[3][16];                // tj[k][x] = product of x_p over set bits i of x, p = 4k+i a control
    double2 bx[TILE_LADDER_BASE];     // factors of the controls outside the tile
    int32_t bq[TILE_LADDER_BASE];     // their local qubit (bit of the tile base index)
    int32_t nb, pad[3];
};

struct TileDesc {
    int32_t b;             // tile qubits
    int32_t L;             // contiguous low qubits 0..L-1 in the tile
    int32_t n_hi;          // b - L
    int32_t n_out;         // number of local qubits outside the tile (m - b)
    int32_t hi_q[TILE_MAX_Q];   // local qubit of tile bit L+i
    int32_t out_q[40];     // local qubits outside the tile, ascending (tile-id bit i -> out_q[i]; a fused
                           // permutation reorders them, set_tile_perm)
    int32_t batch0, nbatch;     // batches[batch0 .. batch0+nbatch)
    int32_t op_begin, op_count; // ops of the whole pass (batch op0 values are absolute)
    int32_t quad_count;         // QUAD ops of the pass
    int32_t lad_count;          // PHASE LADDER ops of the pass (records at lads[0 .. lad_count))
    const TileLadder *lads;     // device address of the pass's ladder records
    // Fused qubit permutation (perm = 1; tile_kernel PAIR): the run of disjoint SWAPs that follows the
    // pass, an involution pi with pi(tile qubits) = tile qubits.  Tile T (base B) is stored onto tile
    // pi(B) with its positions permuted: destination position j <- source position rho(j).
    int32_t perm, pad_perm;
    int32_t out_pq[40];         // pi(out_q[i])
    uint16_t rho[3][16];        // rho(j) = OR_k rho[k][(j >> 4k) & 15]
};

#ifndef __CUDACC_RTC__
// shared-memory bytes of a pass's op stream (ops + QUAD matrices + ladder records)
inline unsigned long long tile_op_bytes(const TileDesc &d) {
    return 80ull * (unsigned long long)d.op_count + 256ull * (unsigned long long)d.quad_count +
           (unsigned long long)sizeof(TileLadder) * (unsigned long long)d.lad_count;
}
#endif

}  // namespace qsb
