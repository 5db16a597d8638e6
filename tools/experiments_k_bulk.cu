// MEASUREMENT RECORD, not built into the library (moved out of csrc/ in round 2): the TMA bulk-copy
// ring variant of the 1q gate measured at 6.41 TB/s vs 6.96 TB/s for the one-shot k_pair_hi.
// k_bulk.cu — TMA (cp.async.bulk) streaming variant of the 1q gate.
//
// A persistent CTA per SM streams units of 2 x 2^SEG amplitudes through a ring of STAGES shared-
// memory buffers: one elected thread issues bulk global->shared copies (completion on an mbarrier)
// and bulk shared->global stores; all threads apply the 2x2 update in shared memory.  For t >= SEG
// a unit is the lower segment [blk*2^(t+1) + off, +2^SEG) and the upper one at +2^t; for t < SEG a
// unit is 2^(SEG+1) contiguous amplitudes that contain whole pairs.  No register staging of the
// stream, deep memory-level parallelism (STAGES-2 units in flight per CTA).
#include "qs_device.cuh"
#include "qs_kernels.h"
#include "qs_tma.cuh"

namespace qsb {

constexpr int BK_TPB = 256;

template <int SEG, int STAGES>
__global__ void __launch_bounds__(BK_TPB, 1) k_pair_bulk(double2 *__restrict__ a, uint64_t nunits, int t, U2 u) {
    extern __shared__ __align__(128) double2 sm[];  // STAGES x 2^(SEG+1)
    __shared__ __align__(8) uint64_t full[STAGES];
    constexpr uint32_t S = 1u << SEG;
    constexpr uint32_t UNIT = 2 * S;
    const int tid = threadIdx.x;
    const bool split = t >= SEG;
    const int tt = split ? SEG : t;
    const uint64_t first = blockIdx.x, step = gridDim.x;
    const uint64_t mine = first < nunits ? (nunits - first + step - 1) / step : 0;

    auto unit_addr = [&](uint64_t k, uint64_t &lo) {
        const uint64_t uidx = first + k * step;
        if (split) {
            const int sh = t - SEG;
            const uint64_t blk = uidx >> sh, off = (uidx & ((1ull << sh) - 1)) << SEG;
            lo = (blk << (t + 1)) | off;
        } else {
            lo = uidx * UNIT;
        }
    };
    auto issue_load = [&](uint64_t k) {
        const int s = (int)(k % STAGES);
        uint64_t lo;
        unit_addr(k, lo);
        double2 *dst = sm + (size_t)s * UNIT;
        mbar_expect_tx(&full[s], UNIT * 16);
        if (split) {
            bulk_g2s(dst, a + lo, S * 16, &full[s]);
            bulk_g2s(dst + S, a + lo + (1ull << t), S * 16, &full[s]);
        } else {
            bulk_g2s(dst, a + lo, UNIT * 16, &full[s]);
        }
    };
    auto issue_store = [&](uint64_t k) {
        const int s = (int)(k % STAGES);
        uint64_t lo;
        unit_addr(k, lo);
        const double2 *src = sm + (size_t)s * UNIT;
        if (split) {
            bulk_s2g(a + lo, src, S * 16);
            bulk_s2g(a + lo + (1ull << t), src + S, S * 16);
        } else {
            bulk_s2g(a + lo, src, UNIT * 16);
        }
        bulk_commit();
    };

    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0)
        for (uint64_t k = 0; k < (uint64_t)STAGES && k < mine; ++k) issue_load(k);

    const double2 u0 = u.u[0], u1 = u.u[1], u2 = u.u[2], u3 = u.u[3];
    for (uint64_t k = 0; k < mine; ++k) {
        const int s = (int)(k % STAGES);
        mbar_wait(&full[s], (uint32_t)((k / STAGES) & 1));
        double2 *b = sm + (size_t)s * UNIT;
#pragma unroll 4
        for (uint32_t q = tid; q < S; q += BK_TPB) {
            const uint32_t j0 = (uint32_t)ins0(q, tt), j1 = j0 + (1u << tt);
            const double2 x = b[j0], y = b[j1];
            b[j0] = cmac2(u0, x, u1, y);
            b[j1] = cmac2(u2, x, u3, y);
        }
        fence_proxy_async_smem();
        __syncthreads();
        if (tid == 0) {
            issue_store(k);
            if (k >= 1 && k - 1 + STAGES < mine) {
                bulk_wait_read<1>();  // the store of unit k-1 has left its stage
                issue_load(k - 1 + STAGES);
            }
        }
    }
    if (tid == 0) bulk_wait<0>();
}

int launch_pair_bulk(double2 *a, int m, int t, const double *m8, cudaStream_t st, int num_sms) {
    constexpr int SEG = 10, STAGES = 4;
    U2 u;
    for (int i = 0; i < 4; ++i) u.u[i] = make_double2(m8[2 * i], m8[2 * i + 1]);
    const size_t smem = (size_t)STAGES * (2u << SEG) * 16;
    static uint64_t attr_mask = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    if (!((attr_mask >> dev) & 1)) {
        cudaFuncSetAttribute(k_pair_bulk<SEG, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr_mask |= 1ull << dev;
    }
    const uint64_t nunits = (1ull << m) >> (SEG + 1);
    uint64_t g = (uint64_t)num_sms;
    if (g > nunits) g = nunits;
    k_pair_bulk<SEG, STAGES><<<(unsigned)g, BK_TPB, smem, st>>>(a, nunits, t, u);
    return 1;
}

}  // namespace qsb
