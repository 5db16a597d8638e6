// tile_copy_bench.cu — memory-only microbenchmark of the fused tile pass data path (measurement tool, not
// part of the library): a 2^n complex128 state is gathered tile by tile into shared memory and scattered
// back in place, with no arithmetic, under several load/store schemes.  Tile = 2^12 amplitudes: local
// qubits 0..L-1 (contiguous runs) + 12-L high qubits starting at h0.  Dynamic tile scheduling (global
// counter), 256 threads, CTAs per SM as given.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tcb tools/tile_copy_bench.cu
//   /tmp/tcb [n=32] [h0=24]
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                                  \
    do {                                                                                       \
        cudaError_t e_ = (x);                                                                  \
        if (e_ != cudaSuccess) {                                                               \
            printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__);           \
            exit(1);                                                                           \
        }                                                                                      \
    } while (0)

constexpr int TPB = 256, B = 12, NAMP = 1 << B;

__device__ __forceinline__ uint32_t swz(uint32_t j) { return j ^ (((j >> 3) ^ (j >> 6) ^ (j >> 9)) & 7u); }
__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

struct Geo {
    int L, h0, n;
    uint64_t outmask;  // bits of the tile base
};

__device__ __forceinline__ uint64_t pdep(uint64_t x, uint64_t mask) {
    uint64_t r = 0;
    for (int b = 0; mask; mask &= mask - 1, ++b)
        if ((x >> b) & 1) r |= mask & (~mask + 1);
    return r;
}
__device__ __forceinline__ uint64_t eaddr(const Geo &g, uint64_t base, uint32_t j) {
    const uint32_t lm = (1u << g.L) - 1;
    return base | (j & lm) | ((uint64_t)(j >> g.L) << g.h0);
}
__device__ __forceinline__ bool next_tile(unsigned long long *ctr, uint64_t ntiles, const Geo &g, uint64_t &base) {
    __shared__ uint64_t sh_t, sh_base;
    if (threadIdx.x == 0) {
        sh_t = atomicAdd(ctr, 1ull);
        sh_base = pdep(sh_t, g.outmask);
    }
    __syncthreads();
    base = sh_base;
    return sh_t < ntiles;
}

// A: cp.async 16 B gather, 16-B stores (the library's skeleton)
// C: cp.async 16 B gather, 32-B stores (two adjacent amplitudes per thread)
template <int STORE32>
__global__ void __launch_bounds__(TPB, 2) k_async(double2 *a, uint64_t ntiles, Geo g, unsigned long long *ctr) {
    extern __shared__ __align__(16) double2 sm[];
    uint64_t base;
    while (next_tile(ctr, ntiles, g, base)) {
        for (uint32_t j = threadIdx.x; j < NAMP; j += TPB)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa(sm + swz(j))), "l"(a + eaddr(g, base, j)) : "memory");
        asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
        __syncthreads();
        if (STORE32) {
            for (uint32_t p = threadIdx.x; p < NAMP / 2; p += TPB) {
                const uint32_t j = 2 * p;
                const double2 x = sm[swz(j)], y = sm[swz(j + 1)];
                asm volatile("st.global.L1::no_allocate.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(a + eaddr(g, base, j)), "d"(x.x),
                             "d"(x.y), "d"(y.x), "d"(y.y)
                             : "memory");
            }
        } else {
            for (uint32_t j = threadIdx.x; j < NAMP; j += TPB) {
                const double2 x = sm[swz(j)];
                asm volatile("st.global.L1::no_allocate.v2.f64 [%0], {%1, %2};" ::"l"(a + eaddr(g, base, j)), "d"(x.x), "d"(x.y)
                             : "memory");
            }
        }
        __syncthreads();
    }
}

// B: register gather with 32-B loads, smem round trip, 32-B stores
__global__ void __launch_bounds__(TPB, 2) k_reg(double2 *a, uint64_t ntiles, Geo g, unsigned long long *ctr) {
    extern __shared__ __align__(16) double2 sm[];
    uint64_t base;
    while (next_tile(ctr, ntiles, g, base)) {
        double2 v[16];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint32_t j = 2 * (threadIdx.x + k * TPB);
            asm volatile("ld.global.L1::no_allocate.v4.f64 {%0, %1, %2, %3}, [%4];"
                         : "=d"(v[2 * k].x), "=d"(v[2 * k].y), "=d"(v[2 * k + 1].x), "=d"(v[2 * k + 1].y)
                         : "l"(a + eaddr(g, base, j)));
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint32_t j = 2 * (threadIdx.x + k * TPB);
            sm[swz(j)] = v[2 * k];
            sm[swz(j + 1)] = v[2 * k + 1];
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint32_t j = 2 * (threadIdx.x + k * TPB);
            const double2 x = sm[swz(j)], y = sm[swz(j + 1)];
            asm volatile("st.global.L1::no_allocate.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(a + eaddr(g, base, j)), "d"(x.x),
                         "d"(x.y), "d"(y.x), "d"(y.y)
                         : "memory");
        }
        __syncthreads();
    }
}

// D: TMA bulk copies, one per contiguous run (unswizzled smem), mbarrier completion, bulk stores
__global__ void __launch_bounds__(TPB, 2) k_bulk(double2 *a, uint64_t ntiles, Geo g, unsigned long long *ctr) {
    extern __shared__ __align__(128) double2 sm[];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    const uint32_t run = 1u << g.L, nruns = NAMP >> g.L, rbytes = run * 16;
    uint32_t phase = 0;
    uint64_t base;
    while (next_tile(ctr, ntiles, g, base)) {
        if (threadIdx.x == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(NAMP * 16) : "memory");
        __syncthreads();
        for (uint32_t r = threadIdx.x; r < nruns; r += TPB)
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                             sa(sm + r * run)),
                         "l"(a + eaddr(g, base, r * run)), "r"(rbytes), "r"(sa(&bar))
                         : "memory");
        asm volatile(
            "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(sa(&bar)),
            "r"(phase)
            : "memory");
        phase ^= 1;
        for (uint32_t r = threadIdx.x; r < nruns; r += TPB)
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(a + eaddr(g, base, r * run)),
                         "r"(sa(sm + r * run)), "r"(rbytes)
                         : "memory");
        asm volatile("cp.async.bulk.commit_group;\ncp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncthreads();
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// in-place streaming reference: one-shot grid, 32-B loads and stores
__global__ void __launch_bounds__(256) k_stream(double2 *a, uint64_t n2) {
    const uint64_t i = ((uint64_t)blockIdx.x * 256 + threadIdx.x) * 2;
    if (i >= n2) return;
    double2 x, y;
    asm volatile("ld.global.L1::no_allocate.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(x.x), "=d"(x.y), "=d"(y.x), "=d"(y.y) : "l"(a + i));
    asm volatile("st.global.L1::no_allocate.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(a + i), "d"(x.x), "d"(x.y), "d"(y.x), "d"(y.y)
                 : "memory");
}

int main(int argc, char **argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 32;
    const int h0 = argc > 2 ? atoi(argv[2]) : 24;
    const uint64_t N = 1ull << n;
    double2 *a;
    CK(cudaMalloc(&a, N * 16));
    CK(cudaMemset(a, 0, N * 16));
    unsigned long long *ctr;
    CK(cudaMalloc(&ctr, 8));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    const double bytes = 2.0 * 16.0 * (double)N;
    auto timeit = [&](const char *name, auto launch) {
        float best = 1e30f;
        for (int r = 0; r < 4; ++r) {
            CK(cudaMemset(ctr, 0, 8));
            CK(cudaEventRecord(e0));
            launch();
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            CK(cudaGetLastError());
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            if (r > 0 && ms < best) best = ms;
        }
        printf("{\"n\": %d, \"h0\": %d, \"variant\": \"%s\", \"ms\": %.3f, \"GBps\": %.1f}\n", n, h0, name, best, bytes / best / 1e6);
        fflush(stdout);
    };
    timeit("stream_v4_oneshot", [&]() { k_stream<<<(unsigned)(N / 2 / 256), 256>>>(a, N); });
    for (int L : {3, 4}) {
        Geo g;
        g.L = L;
        g.h0 = h0;
        g.n = n;
        const uint64_t tmask = ((1ull << L) - 1) | (((1ull << (B - L)) - 1) << h0);
        g.outmask = (N - 1) & ~tmask;
        const uint64_t ntiles = N >> B;
        const size_t smem = NAMP * 16;
        CK(cudaFuncSetAttribute(k_async<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        CK(cudaFuncSetAttribute(k_async<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        CK(cudaFuncSetAttribute(k_reg, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        CK(cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        char nm[64];
        for (int ctas : {2, 3}) {
            const unsigned grid = (unsigned)(sms * ctas);
            snprintf(nm, sizeof nm, "L%d_c%d_async16_st16", L, ctas);
            timeit(nm, [&]() { k_async<0><<<grid, TPB, smem>>>(a, ntiles, g, ctr); });
            snprintf(nm, sizeof nm, "L%d_c%d_async16_st32", L, ctas);
            timeit(nm, [&]() { k_async<1><<<grid, TPB, smem>>>(a, ntiles, g, ctr); });
            snprintf(nm, sizeof nm, "L%d_c%d_reg32_st32", L, ctas);
            timeit(nm, [&]() { k_reg<<<grid, TPB, smem>>>(a, ntiles, g, ctr); });
            if (L >= 4) {  // (bulk copies of 128-B runs fail on this pattern: skipped)
                snprintf(nm, sizeof nm, "L%d_c%d_bulk", L, ctas);
                timeit(nm, [&]() { k_bulk<<<grid, TPB, smem>>>(a, ntiles, g, ctr); });
            }
        }
    }
    return 0;
}
