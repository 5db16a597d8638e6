// qs_tile_ops.cuh — device side of the fused tile pass, shared by the interpreter kernel
// (k_tile.cu) and the NVRTC-compiled straight-line kernels (jit_tile.cpp), so both run the very
// same per-op arithmetic (qs_device.cuh chains) and stay bitwise identical to the unfused path.
//
//  * op templates c_*: apply one op to the 2^R register amplitudes v of a sub-cube; register slots
//    are compile-time; every body is branch-free (a runtime `if` around register updates makes ptxas
//    re-copy the whole register array at the merge);
//  * tile_kernel<R, TPB, Prog>: the persistent-CTA skeleton (gathered cp.async double-buffered tile
//    loads into XOR-swizzled shared memory, the pass's op stream staged in shared memory once, the
//    scatter store); Prog::run applies the batches of one tile.
#pragma once
#include "qs_device.cuh"
#include "qs_tile_types.h"

namespace qsb {

constexpr int TILE_SEG_BITS = 6;     // segment-offset tables: 2 x 64 entries (n_hi = b - L <= 12)
constexpr int TILE_OPC_QUAD_LO = 20, TILE_OPC_QUAD_HI = 31;  // QUAD opcodes in qs_tile_opcodes.inc
__host__ __device__ constexpr bool tile_quad_code(int c) { return c >= TILE_OPC_QUAD_LO && c <= TILE_OPC_QUAD_HI; }

// XOR swizzle of 16-B slots: index bits 0..2 ^= bits 3..5 ^ 6..8 ^ 9..11 (a bijection, linear over XOR)
__host__ __device__ __forceinline__ uint32_t swz(uint32_t j) { return j ^ (((j >> 3) ^ (j >> 6) ^ (j >> 9)) & 7u); }
// sub-cube index s -> tile-position index jb (TileBatch::dep; nbits = b - R)
__device__ __forceinline__ uint32_t sub_deposit(uint32_t s, uint64_t dep, int nbits) {
    uint32_t jb = 0;
#pragma unroll
    for (int i = 0; i < 12; ++i)
        if (i < nbits) jb |= ((s >> i) & 1u) << (uint32_t)((dep >> (4 * i)) & 15u);
    return jb;
}
// compile-time form (JIT kernels): DEP and NBITS are constants of the batch
template <unsigned long long DEP, int NBITS>
__device__ __forceinline__ uint32_t sub_deposit_ct(uint32_t s) {
    uint32_t jb = 0;
#pragma unroll
    for (int i = 0; i < NBITS; ++i) {
        const int p = (int)((DEP >> (4 * i)) & 15ull);
        jb |= p >= i ? (s & (1u << i)) << (p - i) : (s & (1u << i)) >> (i - p);
    }
    return jb;
}
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

// real 2x2 matrix (all imaginary parts exactly 0, e.g. H): the cmac2 chain with its zero terms
// dropped — identical values (adding an exact 0 product never changes a nonzero sum; only the sign
// of an exact zero result may differ), half the FP64 instructions
template <int R, int S>
__device__ __forceinline__ void c_pair_real(double2 (&v)[1 << R], const double2 (&mm)[4]) {
    if constexpr (S < R) {
        const double u0 = mm[0].x, u1 = mm[1].x, u2 = mm[2].x, u3 = mm[3].x;
#pragma unroll
        for (int r = 0; r < (1 << R); ++r)
            if (!((r >> S) & 1)) {
                const double2 x = v[r], y = v[r | (1 << S)];
                v[r] = make_double2(__fma_rn(u1, y.x, __dmul_rn(u0, x.x)), __fma_rn(u1, y.y, __dmul_rn(u0, x.y)));
                v[r | (1 << S)] = make_double2(__fma_rn(u3, y.x, __dmul_rn(u2, x.x)), __fma_rn(u3, y.y, __dmul_rn(u2, x.y)));
            }
    }
}

// MONOMIAL-entry 2x2 matrix (every entry exactly 0, +-1 or +-i; code 0..4): each output is a signed
// component pick of x plus one of y — one DADD per component, no multiply.  The same values as the
// cmac2 chain on that matrix (its extra terms are exact zeros / exact +-x products).  Compile-time codes
// (JIT) and runtime codes (interpreter) give identical results.
template <int E>
__device__ __forceinline__ double2 mono_term(double2 z) {  // e z for codes 1..4; (a+bi) z for 5..8
    if constexpr (E == 1) return z;
    else if constexpr (E == 2) return make_double2(-z.x, -z.y);
    else if constexpr (E == 3) return make_double2(-z.y, z.x);
    else if constexpr (E == 4) return make_double2(z.y, -z.x);
    else if constexpr (E == 5) return make_double2(__dsub_rn(z.x, z.y), __dadd_rn(z.y, z.x));  // (1+i) z
    else if constexpr (E == 6) return make_double2(__dadd_rn(z.x, z.y), __dsub_rn(z.y, z.x));  // (1-i) z
    else if constexpr (E == 7) return make_double2(__dsub_rn(-z.x, z.y), __dsub_rn(z.x, z.y));  // (-1+i) z
    else return make_double2(__dsub_rn(z.y, z.x), __dsub_rn(-z.y, z.x));                        // (-1-i) z
}
__device__ __forceinline__ double2 c_add(double2 a, double2 b) { return make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y)); }
__device__ __forceinline__ double2 c_scale(double w, double2 a) { return make_double2(__dmul_rn(w, a.x), __dmul_rn(w, a.y)); }
__device__ __forceinline__ double2 c_fma(double w, double2 a, double2 b) {
    return make_double2(__fma_rn(w, a.x, b.x), __fma_rn(w, a.y, b.y));
}
// one output row e_a x + e_b y; codes 5..8 carry the real factor w
template <int EA, int EB>
__device__ __forceinline__ double2 mono_row(double2 x, double2 y, double w = 1.0) {
    constexpr bool WA = EA >= 5, WB = EB >= 5;
    if constexpr (EA == 0 && EB == 0) return make_double2(0.0, 0.0);
    else if constexpr (EA == 0) return WB ? c_scale(w, mono_term<EB>(y)) : mono_term<EB>(y);
    else if constexpr (EB == 0) return WA ? c_scale(w, mono_term<EA>(x)) : mono_term<EA>(x);
    else if constexpr (!WA && !WB) return c_add(mono_term<EA>(x), mono_term<EB>(y));
    else if constexpr (WA && !WB) return c_fma(w, mono_term<EA>(x), mono_term<EB>(y));
    else if constexpr (!WA && WB) return c_fma(w, mono_term<EB>(y), mono_term<EA>(x));
    else return c_scale(w, c_add(mono_term<EA>(x), mono_term<EB>(y)));
}
template <int R, int S, int E0, int E1, int E2, int E3>
__device__ __forceinline__ void c_pair_mono(double2 (&v)[1 << R], const double2 (&mm)[4]) {
    if constexpr (S < R) {
        const double w = mm[0].x;  // shared real factor of the w(+-1+-i) entries (codes 5..8)
#pragma unroll
        for (int r = 0; r < (1 << R); ++r)
            if (!((r >> S) & 1)) {
                const double2 x = v[r], y = v[r | (1 << S)];
                v[r] = mono_row<E0, E1>(x, y, w);
                v[r | (1 << S)] = mono_row<E2, E3>(x, y, w);
            }
    }
}
__device__ __forceinline__ double2 mono_term_rt(int e, double2 z) {
    const bool sw = e == 3 || e == 4;
    double re = sw ? z.y : z.x, im = sw ? z.x : z.y;
    re = (e == 2 || e == 3) ? -re : re;
    im = (e == 2 || e == 4) ? -im : im;
    // codes 5..8: (a + b i) z = (a zr - b zi, a zi + b zr), the same operations as mono_term<5..8>
    const double2 w5 = make_double2(__dsub_rn(z.x, z.y), __dadd_rn(z.y, z.x));
    const double2 w6 = make_double2(__dadd_rn(z.x, z.y), __dsub_rn(z.y, z.x));
    const double2 w7 = make_double2(__dsub_rn(-z.x, z.y), __dsub_rn(z.x, z.y));
    const double2 w8 = make_double2(__dsub_rn(z.y, z.x), __dsub_rn(-z.y, z.x));
    double2 r = make_double2(re, im);
    r = e == 5 ? w5 : r;
    r = e == 6 ? w6 : r;
    r = e == 7 ? w7 : r;
    r = e == 8 ? w8 : r;
    return r;
}
__device__ __forceinline__ double2 mono_row_rt(int ea, int eb, double2 x, double2 y, double w = 1.0) {
    const double2 a = mono_term_rt(ea, x), b = mono_term_rt(eb, y);
    const bool wa = ea >= 5, wb = eb >= 5;
    const double2 sa = wa ? c_scale(w, a) : a, sb = wb ? c_scale(w, b) : b;
    double2 r;
    if (ea == 0 && eb == 0) r = make_double2(0.0, 0.0);
    else if (ea == 0) r = sb;
    else if (eb == 0) r = sa;
    else if (!wa && !wb) r = c_add(a, b);
    else if (wa && !wb) r = c_fma(w, a, b);
    else if (!wa && wb) r = c_fma(w, b, a);
    else r = c_scale(w, c_add(a, b));
    return r;
}
// runtime codes: h.w = e0 | e1 << 4 | e2 << 8 | e3 << 12; w in the op record's first entry
template <int R, int S>
__device__ __forceinline__ void c_pair_mono_rt(double2 (&v)[1 << R], const double2 (&mm)[4], int4 h) {
    if constexpr (S < R) {
        const int e0 = h.w & 15, e1 = (h.w >> 4) & 15, e2 = (h.w >> 8) & 15, e3 = (h.w >> 12) & 15;
        const double w = mm[0].x;
#pragma unroll
        for (int r = 0; r < (1 << R); ++r)
            if (!((r >> S) & 1)) {
                const double2 x = v[r], y = v[r | (1 << S)];
                v[r] = mono_row_rt(e0, e1, x, y, w);
                v[r | (1 << S)] = mono_row_rt(e2, e3, x, y, w);
            }
    }
}

// member index (0, 1, 2) of a 3-member monomial family given its packed entry codes (JIT family kernels)
__device__ __forceinline__ uint32_t fam_member(uint32_t w, uint32_t c0, uint32_t c1) {
    return w == c0 ? 0u : (w == c1 ? 1u : 2u);
}

// controlled MONOMIAL matrix (CNOT, CY, CZ-as-matrix ...): compile-time / runtime entry codes
template <int R, int SC, int ST, int E0, int E1, int E2, int E3>
__device__ __forceinline__ void c_ctrl_mono(double2 (&v)[1 << R]) {
    if constexpr (SC < R && ST < R) {
#pragma unroll
        for (int r = 0; r < (1 << R); ++r)
            if (!((r >> ST) & 1) && ((r >> SC) & 1)) {
                const double2 x = v[r], y = v[r | (1 << ST)];
                v[r] = mono_row<E0, E1>(x, y);
                v[r | (1 << ST)] = mono_row<E2, E3>(x, y);
            }
    }
}
template <int R, int SC, int ST>
__device__ __forceinline__ void c_ctrl_mono_rt(double2 (&v)[1 << R], int4 h) {
    if constexpr (SC < R && ST < R) {
        const int e0 = h.w & 15, e1 = (h.w >> 4) & 15, e2 = (h.w >> 8) & 15, e3 = (h.w >> 12) & 15;
#pragma unroll
        for (int r = 0; r < (1 << R); ++r)
            if (!((r >> ST) & 1) && ((r >> SC) & 1)) {
                const double2 x = v[r], y = v[r | (1 << ST)];
                v[r] = mono_row_rt(e0, e1, x, y);
                v[r | (1 << ST)] = mono_row_rt(e2, e3, x, y);
            }
    }
}
// control outside the register slots (a constant of the sub-cube / tile): select old or new
__device__ __forceinline__ double2 sel2(bool on, double2 a, double2 b) {
    return make_double2(on ? a.x : b.x, on ? a.y : b.y);
}
template <int R, int S, int E0, int E1, int E2, int E3>
__device__ __forceinline__ void c_ctrl_fixed_mono(double2 (&v)[1 << R], int4 h, uint32_t jb, uint64_t base) {
    if constexpr (S < R) {
        const bool on = fixed_bit(h.y, jb, base) != 0;
#pragma unroll
        for (int r = 0; r < (1 << R); ++r)
            if (!((r >> S) & 1)) {
                const double2 x = v[r], y = v[r | (1 << S)];
                v[r] = sel2(on, mono_row<E0, E1>(x, y), x);
                v[r | (1 << S)] = sel2(on, mono_row<E2, E3>(x, y), y);
            }
    }
}
template <int R, int S>
__device__ __forceinline__ void c_ctrl_fixed_mono_rt(double2 (&v)[1 << R], int4 h, uint32_t jb, uint64_t base) {
    if constexpr (S < R) {
        const bool on = fixed_bit(h.y, jb, base) != 0;
        const int e0 = h.w & 15, e1 = (h.w >> 4) & 15, e2 = (h.w >> 8) & 15, e3 = (h.w >> 12) & 15;
#pragma unroll
        for (int r = 0; r < (1 << R); ++r)
            if (!((r >> S) & 1)) {
                const double2 x = v[r], y = v[r | (1 << S)];
                v[r] = sel2(on, mono_row_rt(e0, e1, x, y), x);
                v[r | (1 << S)] = sel2(on, mono_row_rt(e2, e3, x, y), y);
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

// PHASE form with factor exactly -1 (CZ, Z): a sign flip of both components — integer XOR on the
// sign bits, no FP64 instruction (equal to the cmul by -1 up to the sign of an exact zero)
__device__ __forceinline__ double2 negate_if(double2 a, bool p) {
    const unsigned long long m = (unsigned long long)p << 63;
    return make_double2(__longlong_as_double(__double_as_longlong(a.x) ^ m),
                        __longlong_as_double(__double_as_longlong(a.y) ^ m));
}

template <int R, int S0, int S1>
__device__ __forceinline__ void c_neg(double2 (&v)[1 << R], int4 h, uint32_t jb, uint64_t base) {
    if constexpr ((S0 < R || S0 == 4) && (S1 < R || S1 == 4)) {
        const bool p = fixed_true(h.y, jb, base) && fixed_true(h.z, jb, base);
#pragma unroll
        for (int r = 0; r < (1 << R); ++r) {
            const bool m0 = S0 == 4 || ((r >> (S0 & 3)) & 1);
            const bool m1 = S1 == 4 || ((r >> (S1 & 3)) & 1);
            if (m0 && m1) v[r] = negate_if(v[r], p);
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

// PHASE LADDER (qs_tile_types.h): amp *= [bit t] k0 prod_c (bit c ? x_c : 1).  The tile factor kt
// (k0 times the controls outside the tile) comes from the per-tile prologue; the sub-cube factor from
// three table lookups; the register-slot factors are multiplied into the 2^|MASK| subset products.
// ST < 4: t is register slot ST (only registers with that bit are touched); ST == 4: t is a fixed
// bit of the sub-cube / tile (source h.y; h.y <= -1000: no target bit, every amplitude).
template <int R, int ST, int MASK>
__device__ __forceinline__ void c_ladder(double2 (&v)[1 << R], const TileLadder &L, double2 kt, int4 h, uint32_t jb,
                                         uint64_t base) {
    if constexpr ((ST < R || ST == 4) && (MASK >> R) == 0 && !(ST < 4 && ((MASK >> ST) & 1))) {
        double2 k = cmul(L.tj[0][jb & 15u], kt);
        k = cmul(L.tj[1][(jb >> 4) & 15u], k);
        k = cmul(L.tj[2][(jb >> 8) & 15u], k);
        double2 f[1 << R];
        f[0] = k;
#pragma unroll
        for (int r = 1; r < (1 << R); ++r)
            if ((r & ~MASK) == 0) {
                int s = 0;
                while (!((r >> s) & 1)) ++s;  // lowest set slot (compile time)
                f[r] = cmul(L.xs[s], f[r & (r - 1)]);
            }
        bool p = true;
        if constexpr (ST == 4) p = fixed_true(h.y, jb, base);
#pragma unroll
        for (int r = 0; r < (1 << R); ++r)
            if (ST == 4 || ((r >> (ST & 3)) & 1)) {
                const double2 y = cmul(f[r & MASK], v[r]);
                v[r].x = p ? y.x : v[r].x;
                v[r].y = p ? y.y : v[r].y;
            }
    }
}

// per-tile factor of every ladder of the pass: k0 times the product of the controls outside the
// tile whose bit is set in the tile base.  One warp per ladder, one control per lane, a fixed
// butterfly (the same tree for every tile), written to lad_k before the tile's first barrier.
template <int TPB>
__device__ __forceinline__ void ladder_prologue(const TileLadder *lad_sm, double2 *lad_k, int nlad, uint64_t base,
                                                int tid) {
    const int warp = tid >> 5, lane = tid & 31;
    for (int l = warp; l < nlad; l += TPB / 32) {
        const TileLadder &L = lad_sm[l];
        double2 f = make_double2(1.0, 0.0);
        if (lane < L.nb && ((base >> L.bq[lane]) & 1ull)) f = L.bx[lane];
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            double2 o;
            o.x = __shfl_xor_sync(0xffffffffu, f.x, off);
            o.y = __shfl_xor_sync(0xffffffffu, f.y, off);
            f = (lane & off) ? cmul(o, f) : cmul(f, o);  // (lower lanes) * (upper lanes)
        }
        if (lane == 0) lad_k[l] = cmul(L.k0, f);
    }
}

__device__ __forceinline__ void cp_async16(uint32_t dst_smem, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst_smem), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }

template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// per-tile state handed to Prog::run
struct TileCtx {
    // direct-I/O batches and the pipelined gather of the next tile (tile_kernel DIRECT)
    double2 *a;
    const uint64_t *seg_off;
    uint32_t lmask;
    int L;
    uint32_t pf_dst;         // shared address of the buffer the next tile is gathered into
    uint64_t nbase;          // base of the tile to prefetch, if pf_valid
    int pf_valid;
    double2 *smb;            // this tile's shared-memory buffer (swizzled)
    uint64_t base;           // tile base index (bits outside the tile)
    uint64_t bswap;          // fused permutation (tile pairs): base ^ destination base of the direct stores
    const TileBatch *bats;   // all batches (device)
    const int4 *ops_sm;      // the pass's op stream in shared memory: 5 x 16 B per op
    const double2 *quad_sm;  // the pass's QUAD matrices in shared memory: 16 x 16 B each
    const TileLadder *lad_sm;  // the pass's PHASE LADDER records in shared memory
    const double2 *lad_k;      // per-tile factor of each ladder (ladder_prologue)
    const int32_t *tq;         // tile position -> local qubit (direct-I/O batches)
    int batch0, op_begin, nbatch;
    uint32_t nsub;           // sub-cubes per tile
    int nsub_bits;           // log2(nsub) = b - R
    int tid;
};

// ---------------------------------------------------------------------------------------------
// Pass with a fused qubit permutation (TileDesc::perm, the QFT's final
// reversal): the pass's ops, then the run of disjoint SWAPs that follows it — an
// involution pi with pi(tile qubits) = tile qubits — in the same HBM pass.  Tile T (base B) lands on
// tile T' (base pi(B)) with its positions permuted by rho.  tile_kernel<..., PAIR = true> runs the pair
// {T, T'} on a CLUSTER OF TWO CTAs (__cluster_dims__(2, 1, 1)): rank 0 owns tile B, rank 1 its partner
// pi(B), each a plain one-buffer tile CTA (two per SM) with the direct HBM I/O of the plain passes.  The
// only coupling is the cluster barrier, split in two: a CTA ARRIVES once its own tile has left HBM
// (after the direct first batch, or the gather) and WAITS just before it stores onto the partner's
// place (the last batch's direct stores — when rho is the identity — or the scatter in destination
// order).  Tiles pi maps onto themselves run on rank 0 alone (rank 1 still takes part in the barrier).
// Dynamic schedule: the cluster takes chunks of indices from a counter and skips non-representatives
// (pi(B) < B) — the same decision on both ranks.  Bitwise the pass followed by k_perm.
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t cluster_idx() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t cluster_count() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
    return r;
}
// store v into the shared variable *p of cluster CTA `rank` (distributed shared memory)
__device__ __forceinline__ void st_cluster_u64(uint64_t *p, uint32_t rank, uint64_t v) {
    uint32_t ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_addr(p)), "r"(rank));
    asm volatile("st.shared::cluster.u64 [%0], %1;" ::"r"(ra), "l"(v) : "memory");
}
__device__ __forceinline__ void cluster_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }

// Persistent CTA (one per SM): tiles blockIdx.x, +gridDim.x, ...; the gathered load of the NEXT tile
// is issued with cp.async (16 B per lane, swizzled shared destination, no registers) before the
// current tile's batches run, so HBM reads overlap compute.
// ctr (NBUF = 1 only, optional): dynamic tile scheduling — each tile index is taken from a zeroed global
// counter, so the tiles in flight stay a contiguous window of the state (DRAM page locality) instead of
// drifting apart as the CTAs of a grid-stride loop do.
// DIRECT (with ctr): Prog's first batch loads the tile from HBM into registers and its last batch stores
// it from registers (no gather into / scatter out of shared memory, which then only carries the tile
// between batches)
template <int R, int TPB, int NBUF, class Prog, int DIRECT = 0, bool PAIR = false>
__device__ __forceinline__ void tile_kernel(double2 *__restrict__ a, uint64_t ntiles, const TileDesc *__restrict__ dd,
                                            const TileBatch *__restrict__ bats, const TileOp *__restrict__ ops,
                                            unsigned long long *ctr = nullptr) {
    extern __shared__ __align__(16) double2 sm[];  // NBUF tile buffers, then the op stream
    __shared__ uint64_t seg_off[2 << TILE_SEG_BITS];
    __shared__ uint64_t dep[7][16];  // tile index nibble k -> base bits (n_out <= 27)
    __shared__ TileDesc desc;
    const int tid = threadIdx.x;
    if (tid == 0) desc = *dd;
    __syncthreads();
    const int b = desc.b, L = desc.L, n_hi = desc.n_hi, n_out = desc.n_out;
    for (int s = tid; s < 2 << TILE_SEG_BITS; s += TPB) {  // segment index -> offset, two tables
        const int tbl = s >> TILE_SEG_BITS, x = s & ((1 << TILE_SEG_BITS) - 1);
        uint64_t o = 0;
        for (int i = 0; i < TILE_SEG_BITS; ++i) {
            const int bit = tbl * TILE_SEG_BITS + i;
            if (bit < n_hi) o |= (uint64_t)((x >> i) & 1) << desc.hi_q[bit];
        }
        seg_off[s] = o;
    }
    for (int s = tid; s < 7 * 16; s += TPB) {  // tile index -> base deposit tables (nibbles)
        const int tbl = s >> 4, x = s & 15;
        uint64_t o = 0;
        for (int i = 0; i < 4; ++i) {
            const int bit = 4 * tbl + i;
            if (bit < n_out) o |= (uint64_t)((x >> i) & 1) << desc.out_q[bit];
        }
        dep[tbl][x] = o;
    }
    const uint32_t namp = 1u << b;
    const uint32_t lmask = (1u << L) - 1;
    const uint32_t sm_base = smem_addr(sm);
    // the pass's op stream, staged once per CTA: 5 x 16 B per op (header + 4 matrix entries), then
    // the QUAD matrices (16 x 16 B each, at their pass index)
    int4 *ops_sm = reinterpret_cast<int4 *>(sm + (size_t)NBUF * namp);
    double2 *quad_sm = reinterpret_cast<double2 *>(ops_sm + 5 * desc.op_count);
    TileLadder *lad_sm = reinterpret_cast<TileLadder *>(quad_sm + 16 * desc.quad_count);
    __shared__ double2 lad_k[TILE_MAX_LADDERS];
    {
        const TileOp *g = ops + desc.op_begin;
        for (int i = tid; i < 5 * desc.op_count; i += TPB) {
            const int o = i / 5, w = i % 5;
            ops_sm[i] = reinterpret_cast<const int4 *>(g + o)[w];
        }
        for (int i = tid; i < 16 * desc.op_count; i += TPB) {
            const int o = i >> 4, e = i & 15;
            if (g[o].touch < (uint32_t)desc.quad_count && tile_quad_code(g[o].code)) quad_sm[16 * g[o].touch + e] = g[o].m[e];
        }
        const int4 *gl = reinterpret_cast<const int4 *>(desc.lads);
        int4 *sl = reinterpret_cast<int4 *>(lad_sm);
        for (int i = tid; i < desc.lad_count * (int)(sizeof(TileLadder) / 16); i += TPB) sl[i] = gl[i];
    }
    __syncthreads();

    auto tile_base = [&](uint64_t tile) {
        uint64_t o = 0;
#pragma unroll
        for (int k = 0; k < 7; ++k) o |= dep[k][(tile >> (4 * k)) & 15];
        return o;
    };
    auto prefetch = [&](uint64_t tile, int buf) {
        const uint64_t base = tile_base(tile);
        const uint32_t dst0 = sm_base + (uint32_t)buf * namp * 16u;
        for (uint32_t j = tid; j < namp; j += TPB)
            cp_async16(dst0 + swz(j) * 16u, a + (base | (seg_off[(j >> L) & 63] | seg_off[64 + ((j >> L) >> 6)]) | (j & lmask)));
        cp_async_commit();
    };

    TileCtx ctx;
    ctx.bats = bats;
    ctx.ops_sm = ops_sm;
    ctx.quad_sm = quad_sm;
    ctx.lad_sm = lad_sm;
    ctx.lad_k = lad_k;
    ctx.batch0 = desc.batch0;
    ctx.op_begin = desc.op_begin;
    ctx.nbatch = desc.nbatch;
    ctx.nsub = 1u << (b - R);
    ctx.nsub_bits = b - R;
    ctx.tid = tid;
    ctx.bswap = 0;
    if constexpr (NBUF == 1 && PAIR) {
        __shared__ uint64_t depp[7][16];  // tile index nibble -> partner base bits pi(B)
        __shared__ uint64_t koff[64];     // in-tile HBM offset of position k * TPB (namp / TPB <= 64)
        __shared__ uint16_t rho_sm[3][16];
        __shared__ uint16_t rk[64];       // rho(k * TPB)
        __shared__ int32_t tq[TILE_MAX_Q];
        for (int s = tid; s < 7 * 16; s += TPB) {
            const int tbl = s >> 4, x = s & 15;
            uint64_t o = 0;
            for (int i = 0; i < 4; ++i) {
                const int bit = 4 * tbl + i;
                if (bit < n_out && ((x >> i) & 1)) o |= 1ull << desc.out_pq[bit];
            }
            depp[tbl][x] = o;
        }
        if (tid < 48) rho_sm[tid >> 4][tid & 15] = desc.rho[tid >> 4][tid & 15];
        if (tid < b) tq[tid] = tid < L ? tid : desc.hi_q[tid - L];
        __syncthreads();
        // position j = tid + k * TPB (disjoint bits): its HBM offset and its rho image are ORs of a
        // per-thread and a per-k part (bit deposits), so the gather / scatter loops do one table load
        auto inner = [&](uint32_t j) {
            return (uint64_t)(j & lmask) | seg_off[(j >> L) & 63] | seg_off[64 + ((j >> L) >> 6)];
        };
        auto rho_of = [&](uint32_t j) {
            return (uint32_t)(rho_sm[0][j & 15] | rho_sm[1][(j >> 4) & 15] | rho_sm[2][(j >> 8) & 15]);
        };
        const uint32_t nk = namp / TPB;
        if (tid < (int)nk) {
            koff[tid] = inner(tid * TPB);
            rk[tid] = (uint16_t)rho_of(tid * TPB);
        }
        const uint64_t in_tid = inner(tid);
        const uint32_t rho_tid = rho_of(tid);
        ctx.a = a;
        ctx.seg_off = seg_off;
        ctx.lmask = lmask;
        ctx.L = L;
        ctx.tq = tq;
        ctx.smb = sm;
        __syncthreads();
        const uint32_t rank = cluster_rank();
        // dynamic schedule in chunks of 8 indices (about half are not pair representatives): rank 0 takes
        // a chunk from the counter and writes it into both CTAs' shared memory (two alternating slots: a
        // slot is rewritten only two cluster barriers later, after every thread has read it); a cluster
        // barrier publishes it.  The counter keeps the pairs in flight a window of consecutive indices.
        constexpr uint64_t CHUNK = 8;
        __shared__ uint64_t chunk_at[2];
        uint32_t slot = 0;
        auto grab = [&]() {
            if (rank == 0 && tid == 0) {
                const uint64_t v = atomicAdd(ctr, CHUNK);
                chunk_at[slot] = v;
                st_cluster_u64(&chunk_at[slot], 1, v);
            }
            cluster_arrive();
            cluster_wait();
            const uint64_t v = chunk_at[slot];
            slot ^= 1u;
            return v;
        };
        for (uint64_t t0 = grab(); t0 < ntiles; t0 = grab())
        for (uint64_t t = t0; t < t0 + CHUNK && t < ntiles; ++t) {
            uint64_t B = 0, Bp = 0;
#pragma unroll
            for (int k = 0; k < 7; ++k) {
                const uint32_t x = (uint32_t)(t >> (4 * k)) & 15u;
                B |= dep[k][x];
                Bp |= depp[k][x];
            }
            if (Bp < B) continue;  // owned by the cluster of the smaller base (both ranks skip)
            if (rank != 0 && Bp == B) {  // pi maps the tile onto itself: rank 0 alone
                cluster_arrive();
                cluster_wait();
                continue;
            }
            const uint64_t mine = rank == 0 ? B : Bp, dest = rank == 0 ? Bp : B;
            ctx.base = mine;
            ctx.bswap = mine ^ dest;
            if (DIRECT & 1) {
                if (desc.lad_count) {
                    ladder_prologue<TPB>(lad_sm, lad_k, desc.lad_count, mine, tid);
                    __syncthreads();
                }
                Prog::template run<R, TPB>(ctx);  // arrives after its first batch (QS_PAIR_READ)
            } else {
                for (uint32_t k = 0; k < nk; ++k)
                    cp_async16(sm_base + swz(tid + k * TPB) * 16u, a + (mine | in_tid | koff[k]));
                cp_async_commit();
                if (desc.lad_count) ladder_prologue<TPB>(lad_sm, lad_k, desc.lad_count, mine, tid);
                cp_async_wait<0>();
                __syncthreads();
                cluster_arrive();  // this tile has left HBM: the partner may store onto its place
                Prog::template run<R, TPB>(ctx);
            }
            if (!(DIRECT & 2)) {  // (with direct stores, Prog's last batch waited: QS_PAIR_WAIT)
                cluster_wait();   // the partner's tile has left HBM
                for (uint32_t k = 0; k < nk; ++k) stg1(a + (dest | in_tid | koff[k]), sm[swz(rho_tid | rk[k])]);
                __syncthreads();  // the buffer is refilled by the next tile
            }
        }
        return;
    }
    if constexpr (NBUF == 1) {
        if (ctr) {
            __shared__ uint64_t next_tile;
            __shared__ int32_t tq[TILE_MAX_Q];
            if (DIRECT) {  // bit 0: Prog's first batch loads from HBM; bit 1: its last batch stores to HBM
                if (tid < b) tq[tid] = tid < L ? tid : desc.hi_q[tid - L];
                ctx.a = a;
                ctx.seg_off = seg_off;
                ctx.lmask = lmask;
                ctx.L = L;
                ctx.tq = tq;
                ctx.smb = sm;
            }
            if (DIRECT & 4) {
                // pipelined single buffer: Prog's last batch reads its amplitudes out of shared memory,
                // passes a barrier and issues the gather of the NEXT tile into the freed buffer before
                // computing and storing (to HBM) — the next load overlaps this tile's last batch
                ctx.pf_dst = sm_base;
                if (tid == 0) next_tile = atomicAdd(ctr, 1ull);
                __syncthreads();
                uint64_t t = next_tile;
                if (t < ntiles) prefetch(t, 0);
                while (t < ntiles) {
                    __syncthreads();  // every thread has read next_tile
                    if (tid == 0) next_tile = atomicAdd(ctr, 1ull);
                    ctx.base = tile_base(t);
                    if (desc.lad_count) ladder_prologue<TPB>(lad_sm, lad_k, desc.lad_count, ctx.base, tid);
                    cp_async_wait<0>();
                    __syncthreads();  // the gather of t, next_tile and lad_k are visible
                    const uint64_t tn = next_tile;
                    ctx.pf_valid = tn < ntiles;
                    ctx.nbase = ctx.pf_valid ? tile_base(tn) : 0;
                    Prog::template run<R, TPB>(ctx);  // ends with a barrier
                    t = tn;
                }
                cp_async_wait<0>();
                return;
            }
            // the index of the tile AFTER the current one is taken at the current tile's start and kept in
            // thread 0's register until the tile ends, so the atomic's latency hides under the tile's work
            // instead of sitting between tiles (the value is only published to the CTA at the end)
            if (tid == 0) next_tile = atomicAdd(ctr, 1ull);
            __syncthreads();
            uint64_t t = next_tile;
            while (t < ntiles) {
                unsigned long long nt = 0;
                if (tid == 0) nt = atomicAdd(ctr, 1ull);
                if (DIRECT & 1) {
                    ctx.base = tile_base(t);
                    if (desc.lad_count) {
                        ladder_prologue<TPB>(lad_sm, lad_k, desc.lad_count, ctx.base, tid);
                        __syncthreads();
                    }
                    Prog::template run<R, TPB>(ctx);  // ends with a barrier (the next tile reuses smem)
                    if (!(DIRECT & 2) && desc.nbatch > 0)
                        for (uint32_t j = tid; j < namp; j += TPB) stg1(a + (ctx.base | (seg_off[(j >> L) & 63] | seg_off[64 + ((j >> L) >> 6)]) | (j & lmask)), ctx.smb[swz(j)]);
                } else {
                    prefetch(t, 0);
                    ctx.base = tile_base(t);
                    if (desc.lad_count) ladder_prologue<TPB>(lad_sm, lad_k, desc.lad_count, ctx.base, tid);
                    cp_async_wait<0>();
                    __syncthreads();
                    ctx.smb = sm;
                    Prog::template run<R, TPB>(ctx);
                    if (!(DIRECT & 2))
                        for (uint32_t j = tid; j < namp; j += TPB) stg1(a + (ctx.base | (seg_off[(j >> L) & 63] | seg_off[64 + ((j >> L) >> 6)]) | (j & lmask)), ctx.smb[swz(j)]);
                }
                if (tid == 0) next_tile = nt;  // every thread read the previous value before run's barriers
                __syncthreads();                // (and the scatter above has read the buffer)
                t = next_tile;
            }
            return;
        }
    }
    uint64_t tile = blockIdx.x;
    int buf = 0;
#pragma unroll
    for (int k = 0; k < NBUF - 1; ++k) {  // always NBUF-1 committed groups ahead (possibly empty)
        const uint64_t t = tile + (uint64_t)k * gridDim.x;
        if (t < ntiles)
            prefetch(t, k);
        else
            cp_async_commit();
    }
    for (; tile < ntiles; tile += gridDim.x, buf = (buf + 1 == NBUF) ? 0 : buf + 1) {
        const uint64_t ahead = tile + (uint64_t)(NBUF - 1) * gridDim.x;
        const int abuf = buf == 0 ? NBUF - 1 : buf - 1;  // freed by the previous tile
        if (ahead < ntiles)
            prefetch(ahead, abuf);
        else
            cp_async_commit();
        ctx.base = tile_base(tile);
        if (desc.lad_count) ladder_prologue<TPB>(lad_sm, lad_k, desc.lad_count, ctx.base, tid);
        cp_async_wait<NBUF - 1>();  // the group of `tile` has landed
        __syncthreads();
        ctx.smb = sm + (size_t)buf * namp;
        Prog::template run<R, TPB>(ctx);
        for (uint32_t j = tid; j < namp; j += TPB) stg1(a + (ctx.base | (seg_off[(j >> L) & 63] | seg_off[64 + ((j >> L) >> 6)]) | (j & lmask)), ctx.smb[swz(j)]);
        __syncthreads();  // this buffer is refilled by the prefetch of the next iteration
    }
}

// one gather slice of the NEXT tile into the freed buffer (DIRECT & 4: issued by the last batch)
__device__ __forceinline__ void pf_slice(const TileCtx &c, uint32_t j) {
    cp_async16(c.pf_dst + swz(j) * 16u, c.a + (c.nbase | (c.seg_off[(j >> c.L) & 63] | c.seg_off[64 + ((j >> c.L) >> 6)]) | (j & c.lmask)));
}

}  // namespace qsb
