// qs_device.cuh — device helpers shared by every sm_100a kernel of the library.
//
// Arithmetic contract: every complex multiply-accumulate is an explicit
// __dmul_rn/__fma_rn chain in ONE fixed order, so a gate produces bitwise-identical amplitudes in
// the single-gate kernels, the fused tile kernel and the sharded exchange update (the FMA of
// PAPER.md:L187 / Alg. 2; reading R7).
#pragma once
#ifdef __CUDACC_RTC__
typedef unsigned long long uint64_t;
#else
#include <cuda_runtime.h>

#include <cstdint>
#endif

namespace qsb {

// u_a * x + u_b * y  (one row of a 2x2 matrix-vector product)
__device__ __forceinline__ double2 cmac2(double2 ua, double2 x, double2 ub, double2 y) {
    double re = __dmul_rn(ua.x, x.x);
    re = __fma_rn(-ua.y, x.y, re);
    re = __fma_rn(ub.x, y.x, re);
    re = __fma_rn(-ub.y, y.y, re);
    double im = __dmul_rn(ua.x, x.y);
    im = __fma_rn(ua.y, x.x, im);
    im = __fma_rn(ub.x, y.y, im);
    im = __fma_rn(ub.y, y.x, im);
    return make_double2(re, im);
}

// sum_{s=0..3} u[s] * v[s]  (one row of a 4x4 matrix-vector product), s ascending
__device__ __forceinline__ double2 cmac4(const double2 *u, double2 v0, double2 v1, double2 v2, double2 v3) {
    double re = __dmul_rn(u[0].x, v0.x);
    re = __fma_rn(-u[0].y, v0.y, re);
    re = __fma_rn(u[1].x, v1.x, re);
    re = __fma_rn(-u[1].y, v1.y, re);
    re = __fma_rn(u[2].x, v2.x, re);
    re = __fma_rn(-u[2].y, v2.y, re);
    re = __fma_rn(u[3].x, v3.x, re);
    re = __fma_rn(-u[3].y, v3.y, re);
    double im = __dmul_rn(u[0].x, v0.y);
    im = __fma_rn(u[0].y, v0.x, im);
    im = __fma_rn(u[1].x, v1.y, im);
    im = __fma_rn(u[1].y, v1.x, im);
    im = __fma_rn(u[2].x, v2.y, im);
    im = __fma_rn(u[2].y, v2.x, im);
    im = __fma_rn(u[3].x, v3.y, im);
    im = __fma_rn(u[3].y, v3.x, im);
    return make_double2(re, im);
}

// d * a
__device__ __forceinline__ double2 cmul(double2 d, double2 a) {
    double re = __dmul_rn(d.x, a.x);
    re = __fma_rn(-d.y, a.y, re);
    double im = __dmul_rn(d.x, a.y);
    im = __fma_rn(d.y, a.x, im);
    return make_double2(re, im);
}

// insert a 0 bit at position p
__device__ __forceinline__ uint64_t ins0(uint64_t x, int p) {
    const uint64_t lo = x & ((1ull << p) - 1);
    return ((x ^ lo) << 1) | lo;
}
// insert 0 bits at positions lo < hi (final positions)
__device__ __forceinline__ uint64_t ins00(uint64_t x, int lo, int hi) { return ins0(ins0(x, lo), hi); }

// 256-bit global accesses: two amplitudes per instruction (LDG.E.ENL2.256 / STG.E.ENL2.256).
struct __align__(32) Amp2 {
    double2 a, b;
};

__device__ __forceinline__ Amp2 ldg2(const double2 *p) {
    Amp2 v;
    asm volatile("ld.global.L1::no_allocate.v4.f64 {%0, %1, %2, %3}, [%4];"
                 : "=d"(v.a.x), "=d"(v.a.y), "=d"(v.b.x), "=d"(v.b.y)
                 : "l"(p));
    return v;
}
__device__ __forceinline__ void stg2(double2 *p, const Amp2 &v) {
    asm volatile("st.global.L1::no_allocate.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(v.a.x), "d"(v.a.y),
                 "d"(v.b.x), "d"(v.b.y)
                 : "memory");
}
__device__ __forceinline__ double2 ldg1(const double2 *p) {
    double2 v;
    asm volatile("ld.global.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
}
__device__ __forceinline__ void stg1(double2 *p, double2 v) {
    asm volatile("st.global.L1::no_allocate.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
}

// kernel-parameter matrices
struct U2 {
    double2 u[4];  // u00, u01, u10, u11
};
struct U4 {
    double2 u[16];  // row-major, k = bit_q0 + 2 bit_q1
};
struct D4 {
    double2 d[4];
};

#ifndef __CUDACC_RTC__
// one-shot grid (see k_gates.cu): one work item per thread, the block scheduler streams the blocks
inline int grid_for(uint64_t work_items, int threads, int /*num_sms*/) {
    uint64_t blocks = (work_items + threads - 1) / threads;
    if (blocks > 0x7fffffffull) blocks = 0x7fffffffull;
    if (blocks < 1) blocks = 1;
    return (int)blocks;
}
#endif

}  // namespace qsb
