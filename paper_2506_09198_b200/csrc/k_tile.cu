// k_tile.cu — fused tile pass (paper: cache blocking / gate fusion "traverse the
// state fewer times", blocked QFT L295).
//
// Two-level blocking of a run of consecutive ops:
//  1. TILE (HBM <-> shared memory): a persistent CTA gathers 2^b amplitudes — local qubits 0..L-1
//     (contiguous runs of >= 512 B, coalesced) plus b-L higher qubits (qsim-style gathered tile,
//     SURVEY.md §8(f) rank 1) — into shared memory, applies the run, writes it back: one HBM
//     read + write for the whole run instead of one per gate.  The next tile is prefetched with
//     cp.async into the second of two buffers while the current one is processed.
//  2. BATCH (shared memory <-> registers): ops are grouped so that the non-diagonal ones of a batch
//     act on at most R tile positions ("register slots"); each thread loads the 2^R amplitudes of
//     one sub-cube spanned by those positions into registers, applies every op of the batch with
//     compile-time register indices, and stores them back: one shared-memory round trip per batch.
//     Diagonal ops and controls may use any bit: outside the register slots the bit is a constant
//     of the sub-cube (tile position) or of the tile (qubit outside the tile).
// The host pre-decodes every op into one opcode (kind x register slots -> one jump-table switch),
// and every batch into its 16 swizzled register offsets; each CTA stages the pass's op stream
// (80 B per op + 256 B per 4x4 matrix) in shared memory once.
// Shared memory is XOR-swizzled on 16-B slots (index bits 0..2 ^= bits 3..5 ^ 6..8 ^ 9..11), so the
// 8 lanes of a quarter-warp hit distinct bank groups for the common register-slot choices.
// Per-op arithmetic is the qs_device.cuh chain in gate order: bitwise identical to the unfused path.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "qs_device.cuh"
#include "qs_kernels.h"

namespace qsb {

constexpr int MAX_SEG = 1 << 7;  // 2^(b-L) <= 2^(TILE_MAX_Q - 5) contiguous runs per tile
constexpr int DEP_BITS = 9;      // tile-index deposit tables: 3 x 512 entries (n_out <= 27)

inline uint32_t swz_host(uint32_t j) { return j ^ (((j >> 3) ^ (j >> 6) ^ (j >> 9)) & 7u); }
__device__ __forceinline__ uint32_t swz(uint32_t j) { return j ^ (((j >> 3) ^ (j >> 6) ^ (j >> 9)) & 7u); }
__device__ __forceinline__ uint32_t smem_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ int fixed_bit(int src, uint32_t jb, uint64_t base) {
    if (src >= 0) return (int)((jb >> src) & 1u);
    if (src == -1) return 0;
    return (int)((base >> (-2 - src)) & 1ull);
}

// ------------------------------------------------------------------------------------------------
// ops on 2^R register amplitudes; slot indices are compile-time (slots >= R compile to nothing)
// ------------------------------------------------------------------------------------------------
template <int R, int S>
__device__ __forceinline__ void c_pair(double2 (&v)[1 << R], const double2 (&mm)[4]) {
    if constexpr (S < R) {
        const double2 u0 = mm[0], u1 = mm[1], u2 = mm[2], u3 = mm[3];
#pragma unroll
        for (int r = 0; r < (1 << R); ++r)
            if (!((r >> S) & 1)) {
                const double2 x = v[r], y = v[r | (1 << S)];
                v[r] = cmac2(u0, x, u1, y);
                v[r | (1 << S)] = cmac2(u2, x, u3, y);
            }
    }
}

template <int R, int SC, int ST>
__device__ __forceinline__ void c_ctrl(double2 (&v)[1 << R], const double2 (&mm)[4]) {
    if constexpr (SC < R && ST < R) {
        const double2 u0 = mm[0], u1 = mm[1], u2 = mm[2], u3 = mm[3];
#pragma unroll
        for (int r = 0; r < (1 << R); ++r)
            if (!((r >> ST) & 1) && ((r >> SC) & 1)) {
                const double2 x = v[r], y = v[r | (1 << ST)];
                v[r] = cmac2(u0, x, u1, y);
                v[r | (1 << ST)] = cmac2(u2, x, u3, y);
            }
    }
}

template <int R, int S0, int S1>
__device__ __forceinline__ void c_quad(double2 (&v)[1 << R], const double2 *gu) {
    if constexpr (S0 < R && S1 < R) {
        double2 u[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) u[i] = gu[i];
#pragma unroll
        for (int r = 0; r < (1 << R); ++r)
            if (!((r >> S0) & 1) && !((r >> S1) & 1)) {
                constexpr int o1 = 1 << S0, o2 = 1 << S1;
                const double2 v0 = v[r], v1 = v[r | o1], v2 = v[r | o2], v3 = v[r | o1 | o2];
                v[r] = cmac4(&u[0], v0, v1, v2, v3);
                v[r | o1] = cmac4(&u[4], v0, v1, v2, v3);
                v[r | o2] = cmac4(&u[8], v0, v1, v2, v3);
                v[r | o1 | o2] = cmac4(&u[12], v0, v1, v2, v3);
            }
    }
}

template <int R, int S0, int S1>
__device__ __forceinline__ void c_swap(double2 (&v)[1 << R]) {
    if constexpr (S0 < R && S1 < R) {
#pragma unroll
        for (int r = 0; r < (1 << R); ++r)
            if (!((r >> S0) & 1) && !((r >> S1) & 1)) {
                const double2 x = v[r | (1 << S0)];
                v[r | (1 << S0)] = v[r | (1 << S1)];
                v[r | (1 << S1)] = x;
            }
    }
}

// DIAG ops are branch-free (runtime ifs inside an op body make ptxas re-copy the whole register
// array at the merge).  Two forms:
//  * c_phase<R, S0, S1>: a single factor x on the amplitudes whose constrained bits are all 1
//    (CZ, CPhase, S, T, Z, phase: one touched k).  Constraints on register slots select a
//    compile-time register subset; constraints on other bits give a runtime predicate p, applied as
//    the factor (p ? x : 1) — multiplying by exactly 1 leaves the value unchanged.  Slot 4 = none.
//  * c_diag<R, S0, S1>: general diagonal: factor d[k(r)] selected per register (slot 4 = fixed bit).
__device__ __forceinline__ double2 sel4(const double2 (&dd)[4], int k) {
    double2 d = dd[0];
    d = k == 1 ? dd[1] : d;
    d = k == 2 ? dd[2] : d;
    d = k == 3 ? dd[3] : d;
    return d;
}

// predicate of a fixed constraint: src <= -1000 means "no constraint" (true)
__device__ __forceinline__ bool fixed_true(int src, uint32_t jb, uint64_t base) {
    return src <= -1000 ? true : fixed_bit(src, jb, base) != 0;
}

template <int R, int S0, int S1>
__device__ __forceinline__ void c_phase(double2 (&v)[1 << R], const double2 (&mm)[4], int4 h, uint32_t jb, uint64_t base) {
    if constexpr ((S0 < R || S0 == 4) && (S1 < R || S1 == 4)) {
        const bool p = fixed_true(h.y, jb, base) && fixed_true(h.z, jb, base);
        double2 x = mm[0];
        x.x = p ? x.x : 1.0;
        x.y = p ? x.y : 0.0;
#pragma unroll
        for (int r = 0; r < (1 << R); ++r) {
            const bool m0 = S0 == 4 || ((r >> (S0 & 3)) & 1);
            const bool m1 = S1 == 4 || ((r >> (S1 & 3)) & 1);
            if (m0 && m1) v[r] = cmul(x, v[r]);
        }
    }
}

template <int R, int S0, int S1>
__device__ __forceinline__ void c_diag(double2 (&v)[1 << R], const double2 (&dd)[4], int4 h, uint32_t jb, uint64_t base) {
    if constexpr ((S0 < R || S0 == 4) && (S1 < R || S1 == 4)) {
        const int f0 = S0 == 4 ? fixed_bit(h.y, jb, base) : 0;
        const int f1 = S1 == 4 ? fixed_bit(h.z, jb, base) : 0;
#pragma unroll
        for (int r = 0; r < (1 << R); ++r) {
            const int b0 = S0 < 4 ? ((r >> (S0 & 3)) & 1) : f0;
            const int b1 = S1 < 4 ? ((r >> (S1 & 3)) & 1) : f1;
            v[r] = cmul(sel4(dd, b0 | (b1 << 1)), v[r]);  // untouched k carry the exact factor 1
        }
    }
}

// controlled pair whose control is a constant of the sub-cube: branch-free, the matrix becomes the
// identity when the control bit is 0 (1*x + 0*y == x exactly)
template <int R, int S>
__device__ __forceinline__ void c_ctrl_fixed(double2 (&v)[1 << R], const double2 (&mm)[4], int4 h, uint32_t jb,
                                             uint64_t base) {
    const bool on = fixed_bit(h.y, jb, base) != 0;
    double2 u[4];
    u[0] = on ? mm[0] : make_double2(1.0, 0.0);
    u[1] = on ? mm[1] : make_double2(0.0, 0.0);
    u[2] = on ? mm[2] : make_double2(0.0, 0.0);
    u[3] = on ? mm[3] : make_double2(1.0, 0.0);
    c_pair<R, S>(v, u);
}

// dense opcodes 0..69 (one jump table; encoded on the host by tile_opcode / tile_phase_opcode):
//   PAIR(slot) | CTRL(ctrl slot, target slot) | CTRL(fixed control, target) | QUAD | SWAP | DIAG (slot 4 =
//   fixed bit) | PHASE (single factor; constrained slots, 4 = none)
template <int R>
__device__ __forceinline__ void apply_op(double2 (&v)[1 << R], int4 h, const double2 (&mm)[4], const double2 *m,
                                         uint32_t jb, uint64_t base) {
    switch (h.x) {
        case 0: c_pair<R, 0>(v, mm); break;
        case 1: c_pair<R, 1>(v, mm); break;
        case 2: c_pair<R, 2>(v, mm); break;
        case 3: c_pair<R, 3>(v, mm); break;
        case 4: c_ctrl<R, 0, 1>(v, mm); break;
        case 5: c_ctrl<R, 0, 2>(v, mm); break;
        case 6: c_ctrl<R, 0, 3>(v, mm); break;
        case 7: c_ctrl<R, 1, 0>(v, mm); break;
        case 8: c_ctrl<R, 1, 2>(v, mm); break;
        case 9: c_ctrl<R, 1, 3>(v, mm); break;
        case 10: c_ctrl<R, 2, 0>(v, mm); break;
        case 11: c_ctrl<R, 2, 1>(v, mm); break;
        case 12: c_ctrl<R, 2, 3>(v, mm); break;
        case 13: c_ctrl<R, 3, 0>(v, mm); break;
        case 14: c_ctrl<R, 3, 1>(v, mm); break;
        case 15: c_ctrl<R, 3, 2>(v, mm); break;
        case 16: c_ctrl_fixed<R, 0>(v, mm, h, jb, base); break;
        case 17: c_ctrl_fixed<R, 1>(v, mm, h, jb, base); break;
        case 18: c_ctrl_fixed<R, 2>(v, mm, h, jb, base); break;
        case 19: c_ctrl_fixed<R, 3>(v, mm, h, jb, base); break;
        case 20: c_quad<R, 0, 1>(v, m); break;
        case 21: c_quad<R, 0, 2>(v, m); break;
        case 22: c_quad<R, 0, 3>(v, m); break;
        case 23: c_quad<R, 1, 0>(v, m); break;
        case 24: c_quad<R, 1, 2>(v, m); break;
        case 25: c_quad<R, 1, 3>(v, m); break;
        case 26: c_quad<R, 2, 0>(v, m); break;
        case 27: c_quad<R, 2, 1>(v, m); break;
        case 28: c_quad<R, 2, 3>(v, m); break;
        case 29: c_quad<R, 3, 0>(v, m); break;
        case 30: c_quad<R, 3, 1>(v, m); break;
        case 31: c_quad<R, 3, 2>(v, m); break;
        case 32: c_swap<R, 0, 1>(v); break;
        case 33: c_swap<R, 0, 2>(v); break;
        case 34: c_swap<R, 0, 3>(v); break;
        case 35: c_swap<R, 1, 2>(v); break;
        case 36: c_swap<R, 1, 3>(v); break;
        case 37: c_swap<R, 2, 3>(v); break;
        case 38: c_diag<R, 0, 1>(v, mm, h, jb, base); break;
        case 39: c_diag<R, 0, 2>(v, mm, h, jb, base); break;
        case 40: c_diag<R, 0, 3>(v, mm, h, jb, base); break;
        case 41: c_diag<R, 0, 4>(v, mm, h, jb, base); break;
        case 42: c_diag<R, 1, 0>(v, mm, h, jb, base); break;
        case 43: c_diag<R, 1, 2>(v, mm, h, jb, base); break;
        case 44: c_diag<R, 1, 3>(v, mm, h, jb, base); break;
        case 45: c_diag<R, 1, 4>(v, mm, h, jb, base); break;
        case 46: c_diag<R, 2, 0>(v, mm, h, jb, base); break;
        case 47: c_diag<R, 2, 1>(v, mm, h, jb, base); break;
        case 48: c_diag<R, 2, 3>(v, mm, h, jb, base); break;
        case 49: c_diag<R, 2, 4>(v, mm, h, jb, base); break;
        case 50: c_diag<R, 3, 0>(v, mm, h, jb, base); break;
        case 51: c_diag<R, 3, 1>(v, mm, h, jb, base); break;
        case 52: c_diag<R, 3, 2>(v, mm, h, jb, base); break;
        case 53: c_diag<R, 3, 4>(v, mm, h, jb, base); break;
        case 54: c_diag<R, 4, 0>(v, mm, h, jb, base); break;
        case 55: c_diag<R, 4, 1>(v, mm, h, jb, base); break;
        case 56: c_diag<R, 4, 2>(v, mm, h, jb, base); break;
        case 57: c_diag<R, 4, 3>(v, mm, h, jb, base); break;
        case 58: c_diag<R, 4, 4>(v, mm, h, jb, base); break;
        case 59: c_phase<R, 0, 1>(v, mm, h, jb, base); break;
        case 60: c_phase<R, 0, 2>(v, mm, h, jb, base); break;
        case 61: c_phase<R, 0, 3>(v, mm, h, jb, base); break;
        case 62: c_phase<R, 0, 4>(v, mm, h, jb, base); break;
        case 63: c_phase<R, 1, 2>(v, mm, h, jb, base); break;
        case 64: c_phase<R, 1, 3>(v, mm, h, jb, base); break;
        case 65: c_phase<R, 1, 4>(v, mm, h, jb, base); break;
        case 66: c_phase<R, 2, 3>(v, mm, h, jb, base); break;
        case 67: c_phase<R, 2, 4>(v, mm, h, jb, base); break;
        case 68: c_phase<R, 3, 4>(v, mm, h, jb, base); break;
        case 69: c_phase<R, 4, 4>(v, mm, h, jb, base); break;
        default: break;
    }
}

__device__ __forceinline__ void cp_async16(uint32_t dst_smem, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst_smem), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Persistent CTA (one per SM): tiles blockIdx.x, +gridDim.x, ...; the gathered load of the NEXT tile
// is issued with cp.async (16 B per lane, swizzled shared destination, no registers) before the
// current tile's batches run, so HBM reads overlap compute.
constexpr int NBUF = 2;  // tile k+1 in flight while tile k is processed

template <int R, int TPB>
__global__ void __launch_bounds__(TPB, 1) k_tile(double2 *__restrict__ a, uint64_t ntiles, const TileDesc *__restrict__ dd,
                                                 const TileBatch *__restrict__ bats, const TileOp *__restrict__ ops) {
    constexpr int NV = 1 << R;
    extern __shared__ __align__(16) double2 sm[];  // NBUF buffers of 2^b amplitudes
    __shared__ uint64_t seg_off[MAX_SEG];
    __shared__ uint64_t dep[3][1 << DEP_BITS];
    __shared__ TileDesc desc;
    const int tid = threadIdx.x;
    if (tid == 0) desc = *dd;
    __syncthreads();
    const int b = desc.b, L = desc.L, n_hi = desc.n_hi, n_out = desc.n_out;
    for (int s = tid; s < (1 << n_hi); s += TPB) {
        uint64_t o = 0;
        for (int i = 0; i < n_hi; ++i) o |= (uint64_t)((s >> i) & 1) << desc.hi_q[i];
        seg_off[s] = o;
    }
    for (int s = tid; s < 3 * (1 << DEP_BITS); s += TPB) {  // tile index -> base deposit tables
        const int tbl = s >> DEP_BITS, x = s & ((1 << DEP_BITS) - 1);
        uint64_t o = 0;
        for (int i = 0; i < DEP_BITS; ++i) {
            const int bit = tbl * DEP_BITS + i;
            if (bit < n_out) o |= (uint64_t)((x >> i) & 1) << desc.out_q[bit];
        }
        dep[tbl][x] = o;
    }
    const uint32_t namp = 1u << b;
    const uint32_t nsub = 1u << (b - R);
    const uint32_t lmask = (1u << L) - 1;
    const uint32_t sm_base = smem_addr(sm);
    // stage the pass's op stream once per CTA: 5 x 16 B per op (header + 4 matrix entries), then the
    // QUAD matrices (16 x 16 B each)
    int4 *ops_sm = reinterpret_cast<int4 *>(sm + (size_t)NBUF * namp);
    double2 *quad_sm = reinterpret_cast<double2 *>(ops_sm + 5 * desc.op_count);
    {
        const TileOp *g = ops + desc.op_begin;
        for (int i = tid; i < 5 * desc.op_count; i += TPB) {
            const int o = i / 5, w = i % 5;
            ops_sm[i] = reinterpret_cast<const int4 *>(g + o)[w];
        }
        __syncthreads();
        for (int i = tid; i < 16 * desc.op_count; i += TPB) {  // QUAD matrices by their pass index
            const int o = i >> 4, e = i & 15;
            const int4 hd = ops_sm[5 * o];
            if (hd.x >= 20 && hd.x <= 31) quad_sm[16 * hd.w + e] = g[o].m[e];  // QUAD opcodes
        }
    }
    __syncthreads();
    auto tile_base = [&](uint64_t tile) {
        return dep[0][tile & 511] | dep[1][(tile >> 9) & 511] | dep[2][(tile >> 18) & 511];
    };
    auto prefetch = [&](uint64_t tile, int buf) {
        const uint64_t base = tile_base(tile);
        const uint32_t dst0 = sm_base + (uint32_t)buf * namp * 16u;
        for (uint32_t j = tid; j < namp; j += TPB)
            cp_async16(dst0 + swz(j) * 16u, a + (base | seg_off[j >> L] | (j & lmask)));
        cp_async_commit();
    };

    uint64_t tile = blockIdx.x;
    int buf = 0;
#pragma unroll
    for (int k = 0; k < NBUF - 1; ++k) {  // always commit NBUF-1 groups (possibly empty)
        const uint64_t t = tile + (uint64_t)k * gridDim.x;
        if (t < ntiles)
            prefetch(t, k);
        else
            cp_async_commit();
    }
    for (; tile < ntiles; tile += gridDim.x, buf = buf == NBUF - 1 ? 0 : buf + 1) {
        const uint64_t ahead = tile + (uint64_t)(NBUF - 1) * gridDim.x;
        const int abuf = buf == 0 ? NBUF - 1 : buf - 1;  // the buffer freed by the previous tile
        if (ahead < ntiles)
            prefetch(ahead, abuf);
        else
            cp_async_commit();
        cp_async_wait<NBUF - 1>();  // the group of `tile` has landed
        __syncthreads();
        double2 *smb = sm + (size_t)buf * namp;
        const uint64_t base = tile_base(tile);
        for (int bi = 0; bi < desc.nbatch; ++bi) {
            const TileBatch *bt = bats + desc.batch0 + bi;
            int p[R];
#pragma unroll
            for (int i = 0; i < R; ++i) p[i] = bt->rp[i];
            uint32_t swo[NV];
#pragma unroll
            for (int r = 0; r < NV; ++r) swo[r] = bt->swo[r];
            const int nops = bt->nops;
            for (uint32_t s = tid; s < nsub; s += TPB) {
                uint32_t jb = s;
#pragma unroll
                for (int i = 0; i < R; ++i) jb = (uint32_t)ins0(jb, p[i]);
                const uint32_t sjb = swz(jb);
                double2 v[NV];
#pragma unroll
                for (int r = 0; r < NV; ++r) v[r] = smb[sjb ^ swo[r]];
                const int4 *op_rec = ops_sm + 5 * (bt->op0 - desc.op_begin);
                for (int o = 0; o < nops; ++o) {
                    const int4 *rec = op_rec + 5 * o;
                    const int4 cur = rec[0];
                    double2 mm[4];
#pragma unroll
                    for (int k = 0; k < 4; ++k) mm[k] = reinterpret_cast<const double2 *>(rec + 1)[k];
                    apply_op<R>(v, cur, mm, quad_sm + 16 * cur.w, jb, base);
                }
#pragma unroll
                for (int r = 0; r < NV; ++r) smb[sjb ^ swo[r]] = v[r];
            }
            __syncthreads();
        }
        for (uint32_t j = tid; j < namp; j += TPB) stg1(a + (base | seg_off[j >> L] | (j & lmask)), smb[swz(j)]);
        __syncthreads();  // this buffer is refilled by the prefetch of the next iteration
    }
}

// ------------------------------------------------------------------------------------------------
// host: batch formation and op decoding
// ------------------------------------------------------------------------------------------------
int tile_regs() {  // register slots per batch: 4 (16 amplitudes / thread, 256 threads) or 3
    static int r = getenv("QS_TILE_R") ? atoi(getenv("QS_TILE_R")) : 4;
    return r == 3 ? 3 : 4;
}

int tile_opcode(int kind, int s0, int s1) {  // dense opcode of k_tile's apply_op switch
    static const int ctrl[4][4] = {{-1,4,5,6},{7,-1,8,9},{10,11,-1,12},{13,14,15,-1}};
    static const int quad[4][4] = {{-1,20,21,22},{23,-1,24,25},{26,27,-1,28},{29,30,31,-1}};
    static const int swp[4][4] = {{-1,32,33,34},{-1,-1,35,36},{-1,-1,-1,37},{-1,-1,-1,-1}};
    static const int diag[5][5] = {{-1,38,39,40,41},{42,-1,43,44,45},{46,47,-1,48,49},{50,51,52,-1,53},{54,55,56,57,58}};
    switch (kind) {
    case OP_PAIR: return s0;
    case OP_CTRL_PAIR: return s0 == 4 ? 16 + s1 : ctrl[s0][s1];
    case OP_QUAD: return quad[s0][s1];
    case OP_SWAP: return swp[std::min(s0, s1)][std::max(s0, s1)];
    default: return diag[s0][s1];
    }
}

int tile_phase_opcode(int a, int b) {  // single-factor phase op, constrained slots a, b (4 = none)
    static const int ph[5][5] = {{-1,59,60,61,62},{59,-1,63,64,65},{60,63,-1,66,67},{61,64,66,-1,68},{62,65,67,68,69}};
    return ph[a][b];
}

namespace {

void needs(const Op &op, const int *pos, std::vector<int> &need) {
    need.clear();
    switch (op.kind) {
    case OP_PAIR: need.push_back(pos[op.q0]); break;
    case OP_CTRL_PAIR: need.push_back(pos[op.q1]); break;
    case OP_QUAD:
    case OP_SWAP:
        need.push_back(pos[op.q0]);
        need.push_back(pos[op.q1]);
        break;
    default: break;
    }
}

}  // namespace

void make_tile_pass(const int *tile_q, int b, int L, int m, const Op *local_ops, int nops, TileDesc &desc,
                    std::vector<TileBatch> &batches, std::vector<TileOp> &ops) {
    const int R = tile_regs();
    desc = TileDesc();
    desc.b = b;
    desc.L = L;
    desc.n_hi = b - L;
    for (int i = 0; i < b - L; ++i) desc.hi_q[i] = tile_q[L + i];
    int pos[64];
    for (int q = 0; q < 64; ++q) pos[q] = -1;
    for (int i = 0; i < b; ++i) pos[tile_q[i]] = i;
    int no = 0;
    for (int q = 0; q < m; ++q)
        if (pos[q] < 0) desc.out_q[no++] = q;
    desc.n_out = no;
    desc.batch0 = (int32_t)batches.size();
    desc.op_begin = (int32_t)ops.size();
    int nquad = 0;

    // greedy batches: non-diagonal ops of a batch use <= R tile positions; order kept
    std::vector<int> cur, need;
    std::vector<int> members;
    auto close = [&]() {
        if (members.empty()) return;
        std::vector<int> rp = cur;
        for (int p = b - 1; (int)rp.size() < R && p >= 0; --p)  // fill with the highest free positions
            if (std::find(rp.begin(), rp.end(), p) == rp.end()) rp.push_back(p);
        std::sort(rp.begin(), rp.end());
        TileBatch bt = TileBatch();
        for (int i = 0; i < TILE_R; ++i) bt.rp[i] = i < R ? rp[i] : 31;
        for (int r = 0; r < 16; ++r) {
            uint32_t off = 0;
            for (int i = 0; i < R; ++i) off |= (uint32_t)((r >> i) & 1) << rp[i];
            bt.swo[r] = r < (1 << R) ? swz_host(off) : 0;
        }
        bt.op0 = (int32_t)ops.size();
        bt.nops = (int32_t)members.size();
        // slot of qubit q in this batch (0..R-1) or 4 (not a register slot) with its bit source
        auto slot_src = [&](int q, int &slot, int32_t &src) {
            slot = 4;
            src = -1;
            if (q < 0) return;
            const int p = pos[q];
            for (int i = 0; i < R; ++i)
                if (rp[i] == p) slot = i;
            if (slot == 4) src = p >= 0 ? p : -2 - q;
        };
        for (int oi : members) {
            const Op &op = local_ops[oi];
            TileOp t = TileOp();
            int s0, s1;
            slot_src(op.q0, s0, t.src0);
            slot_src(op.q1, s1, t.src1);
            t.code = tile_opcode(op.kind, s0, s1);
            t.touch = op.kind == OP_QUAD ? (uint32_t)nquad++ : op.touch;
            const int nm = op.kind == OP_QUAD ? 16 : 4;
            for (int k = 0; k < nm; ++k) t.m[k] = make_double2(op.m[2 * k], op.m[2 * k + 1]);
            if (op.kind == OP_DIAG) {  // single touched k with all constrained bits 1 -> phase form
                const int nq = op.q0 < 0 ? 0 : (op.q1 < 0 ? 1 : 2);
                const uint32_t kall = (1u << nq) - 1;
                if (op.touch == (1u << kall)) {
                    int a = 4, bb = 4;
                    int32_t fa = -1000, fb = -1000;
                    const int qs[2] = {op.q0, op.q1};
                    const int ss[2] = {s0, s1};
                    const int32_t srcs[2] = {t.src0, t.src1};
                    for (int j2 = 0; j2 < nq; ++j2) {
                        if (ss[j2] < 4) {
                            if (a == 4) a = ss[j2]; else bb = ss[j2];
                        } else {
                            if (fa == -1000) fa = srcs[j2]; else fb = srcs[j2];
                        }
                        (void)qs;
                    }
                    t.code = tile_phase_opcode(a, bb);
                    t.src0 = fa;
                    t.src1 = fb;
                    t.m[0] = make_double2(op.m[2 * kall], op.m[2 * kall + 1]);
                }
            }
            ops.push_back(t);
        }
        batches.push_back(bt);
        members.clear();
        cur.clear();
    };
    for (int i = 0; i < nops; ++i) {
        needs(local_ops[i], pos, need);
        std::vector<int> u = cur;
        for (int p : need)
            if (std::find(u.begin(), u.end(), p) == u.end()) u.push_back(p);
        if ((int)u.size() > R) {
            close();
            u = need;
        }
        cur = u;
        members.push_back(i);
    }
    close();
    desc.nbatch = (int32_t)batches.size() - desc.batch0;
    desc.op_count = (int32_t)ops.size() - desc.op_begin;
    desc.quad_count = nquad;
}

int launch_tile(double2 *a, int m, const TileDesc &hdesc, const TileDesc *ddesc, const TileBatch *dbatches,
                const TileOp *dops, cudaStream_t st, int num_sms) {
    static uint64_t attr_mask = 0;  // per device
    const size_t smem = (size_t)NBUF * (16 << hdesc.b) + 80 * (size_t)hdesc.op_count + 256 * (size_t)hdesc.quad_count;
    const int maxsmem = (int)((size_t)NBUF * (16 << TILE_MAX_Q) + TILE_OP_SMEM);
    if (80 * hdesc.op_count + 256 * hdesc.quad_count > TILE_OP_SMEM) return -1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (!((attr_mask >> dev) & 1)) {
        cudaFuncSetAttribute(k_tile<4, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsmem);
        cudaFuncSetAttribute(k_tile<4, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsmem);
        cudaFuncSetAttribute(k_tile<3, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsmem);
        cudaFuncSetAttribute(k_tile<3, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsmem);
        attr_mask |= 1ull << dev;
    }
    if (hdesc.n_out > 3 * DEP_BITS) return -1;
    const uint64_t ntiles = 1ull << (m - hdesc.b);
    uint64_t g = (uint64_t)num_sms;
    if (g > ntiles) g = ntiles;
    const int R = tile_regs();
    const int sub = 1 << (hdesc.b - R);
    if (R == 4) {
        if (sub >= 256)
            k_tile<4, 256><<<(unsigned)g, 256, smem, st>>>(a, ntiles, ddesc, dbatches, dops);
        else
            k_tile<4, 64><<<(unsigned)g, 64, smem, st>>>(a, ntiles, ddesc, dbatches, dops);
    } else {
        if (sub >= 512)
            k_tile<3, 512><<<(unsigned)g, 512, smem, st>>>(a, ntiles, ddesc, dbatches, dops);
        else
            k_tile<3, 64><<<(unsigned)g, 64, smem, st>>>(a, ntiles, ddesc, dbatches, dops);
    }
    return 1;
}

}  // namespace qsb
