// k_tile.cu — fused tile pass (paper: cache blocking / gate fusion "traverse the
// state fewer times", blocked QFT L295).
//
// A CTA stages one tile of 2^b amplitudes in shared memory, applies a run of consecutive ops whose
// non-diagonal qubits all lie in the tile, and writes the tile back: one HBM read + one write for
// the whole run instead of one per gate.  The tile is a *gathered* set of qubits: local qubits
// 0..L-1 (contiguous 2^L-amplitude runs, >= 512 B, coalesced 256-bit accesses) plus b-L arbitrary
// higher qubits, so runs of gates on high qubits fuse too (qsim-style).
// Diagonal ops may act on any qubit: outside the tile their bits are constants of the tile.
// Per-op arithmetic is the same qs_device.cuh chain as the single-op kernels, in the same order,
// so the result is bitwise identical to the unfused path.
#include <cstdio>

#include "qs_device.cuh"
#include "qs_kernels.h"

namespace qsb {

constexpr int TILE_TPB = 256;
constexpr int MAX_SEG = 1 << 9;  // 2^(b-L) <= 2^(TILE_MAX_Q - 5) segments of contiguous amplitudes

__global__ void __launch_bounds__(TILE_TPB)
    k_tile(double2 *__restrict__ a, uint64_t ntiles, const TileDesc *__restrict__ dd, const TileOp *__restrict__ dops) {
    extern __shared__ double2 sm[];
    __shared__ uint64_t seg_off[MAX_SEG];
    __shared__ TileDesc desc;
    const int tid = threadIdx.x;
    if (tid == 0) desc = *dd;
    __syncthreads();
    const int b = desc.b, L = desc.L, n_hi = desc.n_hi;
    const int nseg = 1 << n_hi;
    for (int s = tid; s < nseg; s += TILE_TPB) {
        uint64_t o = 0;
        for (int i = 0; i < n_hi; ++i) o |= (uint64_t)((s >> i) & 1) << desc.hi_q[i];
        seg_off[s] = o;
    }
    const TileOp *ops = dops + desc.op0;
    const int nops = desc.nops;
    const uint32_t nchunk = 1u << (b - 1);   // 256-bit chunks per tile
    const uint32_t lmask = (1u << L) - 1;
    __syncthreads();

    for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        uint64_t base = 0;
        for (int i = 0; i < desc.n_out; ++i) base |= ((tile >> i) & 1ull) << desc.out_q[i];
        // ---- gather load -----------------------------------------------------------------------
        for (uint32_t c = tid; c < nchunk; c += TILE_TPB) {
            const uint32_t j = 2 * c;
            const Amp2 v = ldg2(a + (base | seg_off[j >> L] | (j & lmask)));
            sm[j] = v.a;
            sm[j + 1] = v.b;
        }
        __syncthreads();
        // ---- ops in order ------------------------------------------------------------------------
        for (int o = 0; o < nops; ++o) {
            const TileOp &op = ops[o];
            const int kind = op.kind;
            if (kind == OP_PAIR || (kind == OP_CTRL_PAIR && op.p0 < 0)) {
                if (kind == OP_CTRL_PAIR && !((base >> op.q0) & 1)) continue;  // uniform per tile
                const int p = kind == OP_PAIR ? op.p0 : op.p1;
                const double2 u0 = op.m[0], u1 = op.m[1], u2 = op.m[2], u3 = op.m[3];
                for (uint32_t q = tid; q < (nchunk); q += TILE_TPB) {
                    const uint32_t j0 = (uint32_t)ins0(q, p), j1 = j0 | (1u << p);
                    const double2 x = sm[j0], y = sm[j1];
                    sm[j0] = cmac2(u0, x, u1, y);
                    sm[j1] = cmac2(u2, x, u3, y);
                }
            } else if (kind == OP_CTRL_PAIR) {
                const int pc = op.p0, pt = op.p1;
                const int lo = min(pc, pt), hi = max(pc, pt);
                const double2 u0 = op.m[0], u1 = op.m[1], u2 = op.m[2], u3 = op.m[3];
                for (uint32_t q = tid; q < (nchunk >> 1); q += TILE_TPB) {
                    const uint32_t j0 = (uint32_t)ins00(q, lo, hi) | (1u << pc), j1 = j0 | (1u << pt);
                    const double2 x = sm[j0], y = sm[j1];
                    sm[j0] = cmac2(u0, x, u1, y);
                    sm[j1] = cmac2(u2, x, u3, y);
                }
            } else if (kind == OP_QUAD) {
                const int p0 = op.p0, p1 = op.p1;
                const int lo = min(p0, p1), hi = max(p0, p1);
                const uint32_t o1 = 1u << p0, o2 = 1u << p1, o3 = o1 | o2;
                double2 u[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) u[i] = op.m[i];
                for (uint32_t q = tid; q < (nchunk >> 1); q += TILE_TPB) {
                    const uint32_t j = (uint32_t)ins00(q, lo, hi);
                    const double2 v0 = sm[j], v1 = sm[j | o1], v2 = sm[j | o2], v3 = sm[j | o3];
                    sm[j] = cmac4(&u[0], v0, v1, v2, v3);
                    sm[j | o1] = cmac4(&u[4], v0, v1, v2, v3);
                    sm[j | o2] = cmac4(&u[8], v0, v1, v2, v3);
                    sm[j | o3] = cmac4(&u[12], v0, v1, v2, v3);
                }
            } else if (kind == OP_SWAP) {
                const int p0 = op.p0, p1 = op.p1;
                const int lo = min(p0, p1), hi = max(p0, p1);
                const uint32_t o1 = 1u << p0, o2 = 1u << p1;
                for (uint32_t q = tid; q < (nchunk >> 1); q += TILE_TPB) {
                    const uint32_t j = (uint32_t)ins00(q, lo, hi);
                    const double2 x = sm[j | o1];
                    sm[j | o1] = sm[j | o2];
                    sm[j | o2] = x;
                }
            } else {  // OP_DIAG
                const int nq = op.q0 < 0 ? 0 : (op.q1 < 0 ? 1 : 2);
                const int qs[2] = {op.q0, op.q1};
                const int ps[2] = {op.p0, op.p1};
                int kfix = 0, kfix_mask = 0, nin = 0, pin[2] = {0, 0}, sin_[2] = {0, 0};
                for (int s = 0; s < nq; ++s) {
                    if (ps[s] < 0) {
                        kfix |= (int)((base >> qs[s]) & 1) << s;
                        kfix_mask |= 1 << s;
                    } else {
                        pin[nin] = ps[s];
                        sin_[nin] = s;
                        ++nin;
                    }
                }
                const int plo = nin == 2 ? min(pin[0], pin[1]) : pin[0];
                const int phi = nin == 2 ? max(pin[0], pin[1]) : pin[0];
                const uint32_t cnt = 1u << (b - nin);
                for (int k = 0; k < (1 << nq); ++k) {
                    if (!((op.touch >> k) & 1) || (k & kfix_mask) != kfix) continue;
                    uint32_t set = 0;
                    for (int i = 0; i < nin; ++i) set |= (uint32_t)((k >> sin_[i]) & 1) << pin[i];
                    const double2 d = op.m[k];
                    for (uint32_t q = tid; q < cnt; q += TILE_TPB) {
                        const uint32_t j = (nin == 0 ? q : nin == 1 ? (uint32_t)ins0(q, plo) : (uint32_t)ins00(q, plo, phi)) | set;
                        sm[j] = cmul(d, sm[j]);
                    }
                }
            }
            __syncthreads();
        }
        // ---- scatter store -----------------------------------------------------------------------
        for (uint32_t c = tid; c < nchunk; c += TILE_TPB) {
            const uint32_t j = 2 * c;
            Amp2 v;
            v.a = sm[j];
            v.b = sm[j + 1];
            stg2(a + (base | seg_off[j >> L] | (j & lmask)), v);
        }
        __syncthreads();
    }
}

void make_tile_pass(const int *tile_q, int b, int L, int m, const Op *local_ops, int nops, TileDesc &desc,
                    TileOp *out_ops) {
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
    desc.nops = nops;
    for (int i = 0; i < nops; ++i) {
        const Op &op = local_ops[i];
        TileOp &t = out_ops[i];
        t = TileOp();
        t.kind = op.kind;
        t.q0 = op.q0;
        t.q1 = op.q1;
        t.p0 = op.q0 >= 0 ? pos[op.q0] : -1;
        t.p1 = op.q1 >= 0 ? pos[op.q1] : -1;
        t.touch = op.touch;
        int nm = op.kind == OP_QUAD ? 16 : 4;
        for (int k = 0; k < nm; ++k) t.m[k] = make_double2(op.m[2 * k], op.m[2 * k + 1]);
    }
}

int launch_tile(double2 *a, int m, const TileDesc &hdesc, const TileDesc *ddesc, const TileOp *dops, cudaStream_t st,
                int num_sms) {
    static uint64_t attr_set_mask = 0;  // per device
    const size_t smem = (size_t)16 << hdesc.b;
    int dev = 0;
    cudaGetDevice(&dev);
    if (!((attr_set_mask >> dev) & 1)) {
        cudaFuncSetAttribute(k_tile, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)((size_t)16 << TILE_MAX_Q));
        attr_set_mask |= 1ull << dev;
    }
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tile, TILE_TPB, smem);
    if (per_sm < 1) per_sm = 1;
    const uint64_t ntiles = 1ull << (m - hdesc.b);
    uint64_t g = (uint64_t)per_sm * num_sms;
    if (g > ntiles) g = ntiles;
    k_tile<<<(unsigned)g, TILE_TPB, smem, st>>>(a, ntiles, ddesc, dops);
    return 1;
}

}  // namespace qsb
