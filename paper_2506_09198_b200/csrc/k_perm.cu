// k_perm.cu — qubit-permutation pass: a run of consecutive disjoint local SWAP gates (the QFT's final
// qubit reversal, "swaps"; SURVEY.md §8(a) a8 SWAP, §8(f) rank 2) applied in ONE HBM
// read + write, in place.
//
// A run of disjoint SWAPs is a bit permutation pi of the local index that is an involution.  Pick a
// tile qubit set Q = {0..L-1} ∪ pi({0..L-1}): pi maps Q onto Q and the other ("base") qubits onto
// themselves, so tile T (base bits B) lands exactly on tile T' (base bits pi(B)) with its in-tile
// positions permuted by rho = pi restricted to Q.  One CTA owns the pair {T, T'} (T' = T when pi(B) =
// B): it gathers both into shared memory (runs of 2^L contiguous amplitudes), then scatters each to
// the other's place in destination order (runs of 2^L again) — no other CTA touches either tile, so
// the pass is race-free in place.  Pure data movement: results are bitwise identical to the SWAPs.
// (A variant with two buffer sets per CTA, the next pair's gather in flight during the current pair's
// scatter, measured slower on the QFT(32) reversal: 33.2 vs 31.2 ms; occupancy hides the latency.)
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "qs_kernels.h"
#include "qs_tile_ops.cuh"

namespace qsb {

constexpr int PERM_TPB = 256;

struct PermDesc {            // kernel parameter (by value)
    int32_t b, L, n_out, pad;
    int32_t hi_q[TILE_MAX_Q];    // local qubit of tile position L+i
    int32_t out_q[40];           // base qubits (tile-index bit i -> local qubit out_q[i])
    int32_t out_pq[40];          // pi(out_q[i])
    uint16_t rho[3][16];         // rho(j) = OR_k rho[k][(j >> 4k) & 15] (tile position permutation)
};

// ctr (optional): dynamic tile scheduling from a zeroed global counter (pairs in flight stay a contiguous
// window of tile indices; CTAs that draw non-representative indices move on at once)
__global__ void __launch_bounds__(PERM_TPB) k_perm(double2 *__restrict__ a, uint64_t ntiles, const PermDesc d,
                                                   unsigned long long *ctr) {
    extern __shared__ __align__(16) double2 sm[];  // two tiles of 2^b amplitudes (swizzled)
    __shared__ uint64_t seg[2][16];                 // tile positions L.. L+7 -> address offset
    __shared__ uint16_t rho[3][16];                 // lane-divergent lookups: shared, not param space
    const int tid = threadIdx.x;
    if (tid < 48) rho[tid >> 4][tid & 15] = d.rho[tid >> 4][tid & 15];
    const int n_hi = d.b - d.L;
    if (tid < 32) {
        const int tbl = tid >> 4, x = tid & 15;
        uint64_t o = 0;
        for (int i = 0; i < 4; ++i) {
            const int bit = 4 * tbl + i;
            if (bit < n_hi && ((x >> i) & 1)) o |= 1ull << d.hi_q[bit];
        }
        seg[tbl][x] = o;
    }
    __syncthreads();
    const uint32_t namp = 1u << d.b, lmask = (1u << d.L) - 1;
    double2 *buf0 = sm, *buf1 = sm + namp;
    auto addr = [&](uint64_t base, uint32_t j) {
        const uint32_t h = j >> d.L;
        return base | seg[0][h & 15] | seg[1][(h >> 4) & 15] | (uint64_t)(j & lmask);
    };
    // tile index -> base B and partner base pi(B): nibble deposit tables (an unrolled 22-bit loop
    // per tile made the pass instruction-bound: ncu 16.5e9 warp instructions, 36% uniform shifts/ops)
    __shared__ uint64_t tB[10][16], tBp[10][16];
    for (int e = tid; e < 10 * 16; e += PERM_TPB) {
        const int k = e >> 4, x = e & 15;
        uint64_t b0 = 0, b1 = 0;
        for (int i = 0; i < 4; ++i) {
            const int bit = 4 * k + i;
            if (bit < d.n_out && ((x >> i) & 1)) {
                b0 |= 1ull << d.out_q[bit];
                b1 |= 1ull << d.out_pq[bit];
            }
        }
        tB[k][x] = b0;
        tBp[k][x] = b1;
    }
    __shared__ uint64_t next_t;
    __syncthreads();
    // the pair of tile t (t = the representative: base B <= pi(B)) gathered, permuted, scattered
    auto do_pair = [&](uint64_t t) {
        uint64_t B = 0, Bp = 0;
#pragma unroll
        for (int k = 0; k < 10; ++k) {
            const uint32_t x = (uint32_t)(t >> (4 * k)) & 15u;
            B |= tB[k][x];
            Bp |= tBp[k][x];
        }
        if (Bp < B) return;  // the pair is owned by the CTA of the smaller base
        const bool two = Bp != B;
        const uint32_t s0 = smem_addr(buf0), s1 = smem_addr(buf1);
        for (uint32_t j = tid; j < namp; j += PERM_TPB) {
            cp_async16(s0 + swz(j) * 16u, a + addr(B, j));
            if (two) cp_async16(s1 + swz(j) * 16u, a + addr(Bp, j));
        }
        cp_async_commit();
        cp_async_wait<0>();
        __syncthreads();
        for (uint32_t j = tid; j < namp; j += PERM_TPB) {  // destination order: coalesced runs
            const uint32_t src = rho[0][j & 15] | rho[1][(j >> 4) & 15] | rho[2][(j >> 8) & 15];
            stg1(a + addr(Bp, j), buf0[swz(src)]);
            if (two) stg1(a + addr(B, j), buf1[swz(src)]);
        }
        __syncthreads();
    };
    if (!ctr) {
        for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) do_pair(t);
        return;
    }
    // dynamic scheduling in chunks of PERM_CHUNK tile indices: about half of all indices are not
    // representatives and cost only the check, so one atomic per chunk (taken a chunk ahead, its latency
    // under the current chunk's work) instead of one per index
    constexpr uint64_t PERM_CHUNK = 8;
    if (tid == 0) next_t = atomicAdd(ctr, PERM_CHUNK);
    __syncthreads();
    uint64_t t0 = next_t;
    while (t0 < ntiles) {
        unsigned long long nt = 0;
        if (tid == 0) nt = atomicAdd(ctr, PERM_CHUNK);
        for (uint64_t t = t0; t < t0 + PERM_CHUNK && t < ntiles; ++t) do_pair(t);
        __syncthreads();  // every thread has read next_t (a chunk without a pair has no barrier)
        if (tid == 0) next_t = nt;
        __syncthreads();
        t0 = next_t;
    }
}

namespace {

bool build_perm_desc(const int *perm, int m, int L0, PermDesc &d, std::vector<int> &tile_q) {
    std::memset(&d, 0, sizeof d);
    // Q = {0..L-1} ∪ pi({0..L-1}); the largest L <= L0 whose Q has <= TILE_MAX_Q qubits
    int L = std::min(L0, m);
    std::vector<int> q;
    for (;; --L) {
        if (L < 1) return false;
        q.clear();
        for (int i = 0; i < L; ++i) {
            q.push_back(i);
            q.push_back(perm[i]);
        }
        std::sort(q.begin(), q.end());
        q.erase(std::unique(q.begin(), q.end()), q.end());
        if ((int)q.size() <= TILE_MAX_Q) break;
    }
    for (int x : q)
        if (perm[x] < 0 || perm[x] >= m || perm[perm[x]] != x) return false;  // not an involution on Q
    int Lc = 0;
    while (Lc < (int)q.size() && q[Lc] == Lc) ++Lc;
    const int b = (int)q.size();
    if (m - b > 40 || b - Lc > 8) return false;  // (tile index: <= 40 bits = 5 deposit-table bytes)
    d.b = b;
    d.L = Lc;
    for (int i = Lc; i < b; ++i) d.hi_q[i - Lc] = q[i];
    int pos[64];
    for (int i = 0; i < 64; ++i) pos[i] = -1;
    for (int i = 0; i < b; ++i) pos[q[i]] = i;
    int no = 0;
    for (int x = 0; x < m; ++x)
        if (pos[x] < 0) {
            if (pos[perm[x]] >= 0) return false;  // Q not closed under pi
            d.out_q[no] = x;
            d.out_pq[no] = perm[x];
            ++no;
        }
    d.n_out = no;
    for (int k = 0; k < 3; ++k)
        for (int x = 0; x < 16; ++x) {
            uint32_t r = 0;
            for (int i = 0; i < 4; ++i) {
                const int p = 4 * k + i;
                if (p < b && ((x >> i) & 1)) r |= 1u << pos[perm[q[p]]];
            }
            d.rho[k][x] = (uint16_t)r;
        }
    tile_q = q;
    return true;
}

}  // namespace

int launch_perm(double2 *a, int m, const int *perm, int L0, cudaStream_t st, int num_sms) {
    PermDesc d;
    std::vector<int> q;
    if (!build_perm_desc(perm, m, L0, d, q)) return -1;
    static uint64_t attr_mask = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    if (!((attr_mask >> dev) & 1)) {
        cudaFuncSetAttribute(k_perm, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * (16 << TILE_MAX_Q));
        attr_mask |= 1ull << dev;
    }
    const size_t smem = (size_t)2 * (16u << d.b);
    const int per_sm = std::max(1, std::min(8, (int)((200u * 1024u) / (smem + 4096))));
    const uint64_t ntiles = 1ull << (m - d.b);
    uint64_t g = (uint64_t)num_sms * per_sm;
    if (g > ntiles) g = ntiles;
    static const bool dyn = getenv("QS_PERM_DYN") ? atoi(getenv("QS_PERM_DYN")) != 0 : true;
    unsigned long long *ctr = dyn ? tile_counter(st) : nullptr;
    if (ctr && cudaMemsetAsync(ctr, 0, sizeof(unsigned long long), st) != cudaSuccess) ctr = nullptr;
    k_perm<<<(unsigned)g, PERM_TPB, smem, st>>>(a, ntiles, d, ctr);
    return 1;
}

}  // namespace qsb
