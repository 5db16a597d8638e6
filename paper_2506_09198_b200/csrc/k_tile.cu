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
// Shared memory is XOR-swizzled on 16-B slots (index bits 0..2 ^= bits 3..5 ^ 6..8 ^ 9..11), so the
// 8 lanes of a quarter-warp hit distinct bank groups for the common register-slot choices.
// Op headers are read one op ahead (software pipelined) to hide the L1 latency of the op stream.
// Per-op arithmetic is the qs_device.cuh chain in gate order: bitwise identical to the unfused path.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "qs_device.cuh"
#include "qs_kernels.h"

namespace qsb {

constexpr int MAX_SEG = 1 << 7;  // 2^(b-L) <= 2^(TILE_MAX_Q - 5) contiguous runs per tile

__device__ __forceinline__ uint32_t smem_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint32_t swz(uint32_t j) { return j ^ (((j >> 3) ^ (j >> 6) ^ (j >> 9)) & 7u); }

__device__ __forceinline__ double2 ldu(const double2 *p) {  // L1-resident op data
    double2 v;
    asm volatile("ld.global.nc.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
}

__device__ __forceinline__ int4 ldh(const TileOp *p) {  // first 16 B of an op: kind, s0, s1, src0
    int4 v;
    asm volatile("ld.global.nc.v4.s32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}

// ------------------------------------------------------------------------------------------------
// ops on NV = 2^R register amplitudes; slot indices are compile-time
// ------------------------------------------------------------------------------------------------
template <int NV, int S>
__device__ __forceinline__ void ap_pair(double2 (&v)[NV], double2 u0, double2 u1, double2 u2, double2 u3) {
#pragma unroll
    for (int r = 0; r < NV; ++r)
        if (!((r >> S) & 1)) {
            const double2 x = v[r], y = v[r | (1 << S)];
            v[r] = cmac2(u0, x, u1, y);
            v[r | (1 << S)] = cmac2(u2, x, u3, y);
        }
}

template <int NV, int SC, int ST>
__device__ __forceinline__ void ap_ctrl(double2 (&v)[NV], double2 u0, double2 u1, double2 u2, double2 u3) {
#pragma unroll
    for (int r = 0; r < NV; ++r)
        if (!((r >> ST) & 1) && ((r >> SC) & 1)) {
            const double2 x = v[r], y = v[r | (1 << ST)];
            v[r] = cmac2(u0, x, u1, y);
            v[r | (1 << ST)] = cmac2(u2, x, u3, y);
        }
}

template <int NV, int S0, int S1>
__device__ __forceinline__ void ap_quad(double2 (&v)[NV], const double2 *gu) {
#pragma unroll
    for (int r = 0; r < NV; ++r)
        if (!((r >> S0) & 1) && !((r >> S1) & 1)) {
            constexpr int o1 = 1 << S0, o2 = 1 << S1;
            const double2 v0 = v[r], v1 = v[r | o1], v2 = v[r | o2], v3 = v[r | o1 | o2];
            double2 out[4];
#pragma unroll
            for (int row = 0; row < 4; ++row) {
                double2 u[4];
#pragma unroll
                for (int c = 0; c < 4; ++c) u[c] = ldu(gu + 4 * row + c);
                out[row] = cmac4(u, v0, v1, v2, v3);
            }
            v[r] = out[0];
            v[r | o1] = out[1];
            v[r | o2] = out[2];
            v[r | o1 | o2] = out[3];
        }
}

template <int NV, int S0, int S1>
__device__ __forceinline__ void ap_swap(double2 (&v)[NV]) {
#pragma unroll
    for (int r = 0; r < NV; ++r)
        if (!((r >> S0) & 1) && !((r >> S1) & 1)) {
            const double2 x = v[r | (1 << S0)];
            v[r | (1 << S0)] = v[r | (1 << S1)];
            v[r | (1 << S1)] = x;
        }
}

// DIAG with slot S = R meaning "bit constant for the sub-cube" (value f0 / f1)
template <int NV, int R, int S0, int S1>
__device__ __forceinline__ void ap_diag(double2 (&v)[NV], const double2 *d, uint32_t touch, int f0, int f1) {
    double2 dd[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) dd[k] = ldu(d + k);
#pragma unroll
    for (int r = 0; r < NV; ++r) {
        const int b0 = S0 < R ? ((r >> (S0 < R ? S0 : 0)) & 1) : f0;
        const int b1 = S1 < R ? ((r >> (S1 < R ? S1 : 0)) & 1) : f1;
        const int k = b0 | (b1 << 1);
        if ((touch >> k) & 1) {
            double2 f = dd[0];
            f = k == 1 ? dd[1] : f;
            f = k == 2 ? dd[2] : f;
            f = k == 3 ? dd[3] : f;
            v[r] = cmul(f, v[r]);
        }
    }
}

__device__ __forceinline__ int fixed_bit(int src, uint32_t jb, uint64_t base) {
    if (src >= 0) return (int)((jb >> src) & 1u);
    if (src == -1) return 0;
    return (int)((base >> (-2 - src)) & 1ull);
}

// header h = {kind, s0, s1, src0}; src1 / touch / matrix are read on demand
template <int R>
__device__ __forceinline__ void apply_op(double2 (&v)[1 << R], int4 h, const TileOp *op, uint32_t jb, uint64_t base) {
    constexpr int NV = 1 << R;
    const int kind = h.x, s0 = h.y, s1 = h.z;
    const double2 *m = op->m;
    if (kind == OP_PAIR || (kind == OP_CTRL_PAIR && s0 == R)) {
        if (kind == OP_CTRL_PAIR && !fixed_bit(h.w, jb, base)) return;  // control constant 0
        const int st = kind == OP_PAIR ? s0 : s1;
        const double2 u0 = ldu(m), u1 = ldu(m + 1), u2 = ldu(m + 2), u3 = ldu(m + 3);
        switch (st) {
        case 0: ap_pair<NV, 0>(v, u0, u1, u2, u3); break;
        case 1: ap_pair<NV, 1>(v, u0, u1, u2, u3); break;
        case 2: ap_pair<NV, 2>(v, u0, u1, u2, u3); break;
        default:
            if constexpr (R > 3) ap_pair<NV, R - 1>(v, u0, u1, u2, u3);
            break;
        }
        return;
    }
    if (kind == OP_CTRL_PAIR) {
        const double2 u0 = ldu(m), u1 = ldu(m + 1), u2 = ldu(m + 2), u3 = ldu(m + 3);
        switch (s0 * 8 + s1) {
        case 0 * 8 + 1: ap_ctrl<NV, 0, 1>(v, u0, u1, u2, u3); break;
        case 0 * 8 + 2: ap_ctrl<NV, 0, 2>(v, u0, u1, u2, u3); break;
        case 1 * 8 + 0: ap_ctrl<NV, 1, 0>(v, u0, u1, u2, u3); break;
        case 1 * 8 + 2: ap_ctrl<NV, 1, 2>(v, u0, u1, u2, u3); break;
        case 2 * 8 + 0: ap_ctrl<NV, 2, 0>(v, u0, u1, u2, u3); break;
        case 2 * 8 + 1: ap_ctrl<NV, 2, 1>(v, u0, u1, u2, u3); break;
        default:
            if constexpr (R > 3) {
                switch (s0 * 8 + s1) {
                case 0 * 8 + 3: ap_ctrl<NV, 0, R - 1>(v, u0, u1, u2, u3); break;
                case 1 * 8 + 3: ap_ctrl<NV, 1, R - 1>(v, u0, u1, u2, u3); break;
                case 2 * 8 + 3: ap_ctrl<NV, 2, R - 1>(v, u0, u1, u2, u3); break;
                case 3 * 8 + 0: ap_ctrl<NV, R - 1, 0>(v, u0, u1, u2, u3); break;
                case 3 * 8 + 1: ap_ctrl<NV, R - 1, 1>(v, u0, u1, u2, u3); break;
                default: ap_ctrl<NV, R - 1, 2>(v, u0, u1, u2, u3); break;
                }
            }
        }
        return;
    }
    if (kind == OP_QUAD) {
        switch (s0 * 8 + s1) {
        case 0 * 8 + 1: ap_quad<NV, 0, 1>(v, m); break;
        case 0 * 8 + 2: ap_quad<NV, 0, 2>(v, m); break;
        case 1 * 8 + 0: ap_quad<NV, 1, 0>(v, m); break;
        case 1 * 8 + 2: ap_quad<NV, 1, 2>(v, m); break;
        case 2 * 8 + 0: ap_quad<NV, 2, 0>(v, m); break;
        case 2 * 8 + 1: ap_quad<NV, 2, 1>(v, m); break;
        default:
            if constexpr (R > 3) {
                switch (s0 * 8 + s1) {
                case 0 * 8 + 3: ap_quad<NV, 0, R - 1>(v, m); break;
                case 1 * 8 + 3: ap_quad<NV, 1, R - 1>(v, m); break;
                case 2 * 8 + 3: ap_quad<NV, 2, R - 1>(v, m); break;
                case 3 * 8 + 0: ap_quad<NV, R - 1, 0>(v, m); break;
                case 3 * 8 + 1: ap_quad<NV, R - 1, 1>(v, m); break;
                default: ap_quad<NV, R - 1, 2>(v, m); break;
                }
            }
        }
        return;
    }
    if (kind == OP_SWAP) {
        const int a = min(s0, s1), b = max(s0, s1);
        switch (a * 8 + b) {
        case 0 * 8 + 1: ap_swap<NV, 0, 1>(v); break;
        case 0 * 8 + 2: ap_swap<NV, 0, 2>(v); break;
        case 1 * 8 + 2: ap_swap<NV, 1, 2>(v); break;
        default:
            if constexpr (R > 3) {
                switch (a * 8 + b) {
                case 0 * 8 + 3: ap_swap<NV, 0, R - 1>(v); break;
                case 1 * 8 + 3: ap_swap<NV, 1, R - 1>(v); break;
                default: ap_swap<NV, 2, R - 1>(v); break;
                }
            }
        }
        return;
    }
    // OP_DIAG
    const int src1 = op->src1;
    const uint32_t touch = op->touch;
    const int f0 = s0 == R ? fixed_bit(h.w, jb, base) : 0;
    const int f1 = s1 == R ? fixed_bit(src1, jb, base) : 0;
    if (s0 == R && s1 == R) {  // one factor (or none) for the whole sub-cube
        const int k = f0 | (f1 << 1);
        if ((touch >> k) & 1) {
            const double2 d = ldu(m + k);
#pragma unroll
            for (int r = 0; r < NV; ++r) v[r] = cmul(d, v[r]);
        }
        return;
    }
    switch (s0 * 8 + s1) {
#define QS_D(A, B) \
    case (A)*8 + (B): ap_diag<NV, R, A, B>(v, m, touch, f0, f1); break;
        QS_D(0, 1) QS_D(0, 2) QS_D(1, 0) QS_D(1, 2) QS_D(2, 0) QS_D(2, 1)
        QS_D(0, R) QS_D(1, R) QS_D(2, R) QS_D(R, 0) QS_D(R, 1) QS_D(R, 2)
    default:
        if constexpr (R > 3) {
            switch (s0 * 8 + s1) {
                QS_D(0, 3) QS_D(1, 3) QS_D(2, 3) QS_D(3, 0) QS_D(3, 1) QS_D(3, 2) QS_D(3, R) QS_D(R, 3)
            default: break;
            }
        }
#undef QS_D
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
template <int R, int TPB>
__global__ void __launch_bounds__(TPB, 1) k_tile(double2 *__restrict__ a, uint64_t ntiles, const TileDesc *__restrict__ dd,
                                                 const TileBatch *__restrict__ bats, const TileOp *__restrict__ ops) {
    constexpr int NV = 1 << R;
    extern __shared__ __align__(16) double2 sm[];  // 2 buffers of 2^b amplitudes
    __shared__ uint64_t seg_off[MAX_SEG];
    __shared__ TileDesc desc;
    const int tid = threadIdx.x;
    if (tid == 0) desc = *dd;
    __syncthreads();
    const int b = desc.b, L = desc.L, n_hi = desc.n_hi;
    for (int s = tid; s < (1 << n_hi); s += TPB) {
        uint64_t o = 0;
        for (int i = 0; i < n_hi; ++i) o |= (uint64_t)((s >> i) & 1) << desc.hi_q[i];
        seg_off[s] = o;
    }
    const uint32_t namp = 1u << b;
    const uint32_t nsub = 1u << (b - R);
    const uint32_t lmask = (1u << L) - 1;
    const uint32_t sm_base = smem_addr(sm);
    __syncthreads();

    auto tile_base = [&](uint64_t tile) {
        uint64_t base = 0;
        for (int i = 0; i < desc.n_out; ++i) base |= ((tile >> i) & 1ull) << desc.out_q[i];
        return base;
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
    if (tile < ntiles) prefetch(tile, 0);
    for (; tile < ntiles; tile += gridDim.x, buf ^= 1) {
        const uint64_t next = tile + gridDim.x;
        if (next < ntiles) {
            prefetch(next, buf ^ 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        double2 *smb = sm + (size_t)buf * namp;
        const uint64_t base = tile_base(tile);
        for (int bi = 0; bi < desc.nbatch; ++bi) {
            const TileBatch &bt = bats[desc.batch0 + bi];
            int p[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) p[i] = bt.rp[i];
            uint32_t swo[NV];
#pragma unroll
            for (int r = 0; r < NV; ++r) {
                uint32_t off = 0;
#pragma unroll
                for (int i = 0; i < R; ++i) off |= (uint32_t)((r >> i) & 1) << p[i];
                swo[r] = swz(off);
            }
            const TileOp *bops = ops + bt.op0;
            const int nops = bt.nops;
            for (uint32_t s = tid; s < nsub; s += TPB) {
                uint32_t jb = s;
#pragma unroll
                for (int i = 0; i < R; ++i) jb = (uint32_t)ins0(jb, p[i]);
                const uint32_t sjb = swz(jb);
                double2 v[NV];
#pragma unroll
                for (int r = 0; r < NV; ++r) v[r] = smb[sjb ^ swo[r]];
                int4 h = nops > 0 ? ldh(bops) : make_int4(0, 0, 0, 0);
                for (int o = 0; o < nops; ++o) {
                    const int4 cur = h;
                    if (o + 1 < nops) h = ldh(bops + o + 1);  // next header in flight
                    apply_op<R>(v, cur, bops + o, jb, base);
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
// host: batch formation
// ------------------------------------------------------------------------------------------------
int tile_regs() {  // register slots per batch: 3 (8 amplitudes / thread, 512 threads) or 4
    static int r = getenv("QS_TILE_R") ? atoi(getenv("QS_TILE_R")) : 3;
    return r == 4 ? 4 : 3;
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
        for (int i = 0; i < 4; ++i) bt.rp[i] = i < R ? rp[i] : 31;
        int nn = 0;
        for (int p = 0; p < b; ++p)
            if (std::find(rp.begin(), rp.end(), p) == rp.end()) bt.nr_pos[nn++] = p;
        bt.n_nr = nn;
        bt.op0 = (int32_t)ops.size();
        bt.nops = (int32_t)members.size();
        auto slot_src = [&](int q, int32_t &slot, int32_t &src) {
            if (q < 0) {
                slot = R;
                src = -1;
                return;
            }
            const int p = pos[q];
            int sl = R;
            for (int i = 0; i < R; ++i)
                if (rp[i] == p) sl = i;
            slot = sl;
            src = sl < R ? 0 : (p >= 0 ? p : -2 - q);
        };
        for (int oi : members) {
            const Op &op = local_ops[oi];
            TileOp t = TileOp();
            t.kind = op.kind;
            slot_src(op.q0, t.s0, t.src0);
            slot_src(op.q1, t.s1, t.src1);
            if (op.kind == OP_PAIR) t.s1 = R;
            t.touch = op.touch;
            const int nm = op.kind == OP_QUAD ? 16 : 4;
            for (int k = 0; k < nm; ++k) t.m[k] = make_double2(op.m[2 * k], op.m[2 * k + 1]);
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
}

int launch_tile(double2 *a, int m, const TileDesc &hdesc, const TileDesc *ddesc, const TileBatch *dbatches,
                const TileOp *dops, cudaStream_t st, int num_sms) {
    static uint64_t attr_mask = 0;  // per device
    const size_t smem = (size_t)2 * (16 << hdesc.b);
    const int maxsmem = (int)((size_t)2 * (16 << TILE_MAX_Q));
    int dev = 0;
    cudaGetDevice(&dev);
    if (!((attr_mask >> dev) & 1)) {
        cudaFuncSetAttribute(k_tile<3, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsmem);
        cudaFuncSetAttribute(k_tile<3, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsmem);
        cudaFuncSetAttribute(k_tile<3, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsmem);
        cudaFuncSetAttribute(k_tile<4, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsmem);
        cudaFuncSetAttribute(k_tile<4, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsmem);
        attr_mask |= 1ull << dev;
    }
    const uint64_t ntiles = 1ull << (m - hdesc.b);
    uint64_t g = (uint64_t)num_sms;
    if (g > ntiles) g = ntiles;
    const int R = tile_regs();
    const int sub = 1 << (hdesc.b - R);
    if (R == 3) {
        if (sub >= 512)
            k_tile<3, 512><<<(unsigned)g, 512, smem, st>>>(a, ntiles, ddesc, dbatches, dops);
        else if (sub >= 256)
            k_tile<3, 256><<<(unsigned)g, 256, smem, st>>>(a, ntiles, ddesc, dbatches, dops);
        else
            k_tile<3, 64><<<(unsigned)g, 64, smem, st>>>(a, ntiles, ddesc, dbatches, dops);
    } else {
        if (sub >= 256)
            k_tile<4, 256><<<(unsigned)g, 256, smem, st>>>(a, ntiles, ddesc, dbatches, dops);
        else
            k_tile<4, 64><<<(unsigned)g, 64, smem, st>>>(a, ntiles, ddesc, dbatches, dops);
    }
    return 1;
}

}  // namespace qsb
