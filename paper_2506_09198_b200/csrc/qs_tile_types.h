// qs_tile_types.h — device-visible descriptors of a fused tile pass (k_tile.cu, JIT kernels).
// Plain structs, includable by nvcc and by NVRTC (the JIT tile kernels, jit_tile.cpp).
#pragma once
#ifdef __CUDACC_RTC__
typedef int int32_t;
typedef unsigned int uint32_t;
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
constexpr int TILE_NBUF_MAX = 3; // tile buffers per CTA (tiles k+1..k+NBUF-1 in flight)

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

}  // namespace qsb
