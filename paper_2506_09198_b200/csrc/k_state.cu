// k_state.cu — initialisation, deterministic norm, scaling and the global-qubit exchange kernels.
#include "qs_device.cuh"
#include "qs_kernels.h"

namespace qsb {

constexpr int STPB = 256;

// ------------------------------------------------------------------------------------------------
// Random state (reading R9): amplitude i = gauss2(seed, i), SplitMix64
// counter stream + Box-Muller, a function of the GLOBAL index only (sharding-invariant).  This is
// the CUDA side's own implementation of the generator; the oracle has an independent one.
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ uint64_t splitmix64(uint64_t seed, uint64_t j) {
    uint64_t z = seed + (j + 1) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ double2 gauss2(uint64_t seed, uint64_t i) {
    const uint64_t x1 = splitmix64(seed, 2 * i), x2 = splitmix64(seed, 2 * i + 1);
    const double u1 = (double)((x1 >> 11) + 1) * 0x1.0p-53;  // (0, 1]
    const double u2 = (double)(x2 >> 11) * 0x1.0p-53;        // [0, 1)
    const double rho = sqrt(-2.0 * log(u1));
    double s, c;
    sincospi(2.0 * u2, &s, &c);
    return make_double2(rho * c, rho * s);
}

__global__ void k_set_amp(double2 *a, uint64_t index, double re, double im) { a[index] = make_double2(re, im); }

int launch_set_amp(double2 *a, uint64_t index, double re, double im, cudaStream_t st) {
    k_set_amp<<<1, 1, 0, st>>>(a, index, re, im);
    return 1;
}

__global__ void __launch_bounds__(STPB) k_scale(double2 *__restrict__ a, uint64_t nunits, double s) {
    const uint64_t step = (uint64_t)gridDim.x * STPB;
    for (uint64_t v = (uint64_t)blockIdx.x * STPB + threadIdx.x; v < nunits; v += step) {
        Amp2 x = ldg2(a + 2 * v);
        x.a.x = __dmul_rn(x.a.x, s);
        x.a.y = __dmul_rn(x.a.y, s);
        x.b.x = __dmul_rn(x.b.x, s);
        x.b.y = __dmul_rn(x.b.y, s);
        stg2(a + 2 * v, x);
    }
}

int launch_scale(double2 *a, uint64_t count, double s, cudaStream_t st, int num_sms) {
    const uint64_t nunits = count / 2;
    k_scale<<<grid_for(nunits, STPB, num_sms), STPB, 0, st>>>(a, nunits, s);
    return 1;
}

// ------------------------------------------------------------------------------------------------
// Deterministic sum |a|^2: each leaf of 2^min(13, n-3)
// amplitudes is summed in a fixed per-thread order + a fixed shared-memory tree; leaf sums are
// combined by a perfect binary tree of adjacent pairs.  Leaves never span shards (P <= 8), so every
// shard count sums the same leaves in the same tree: the norm is bitwise P-invariant (the host
// finishes the tree over shards).
// ------------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(STPB) k_norm_leaf(const double2 *__restrict__ a, uint64_t leaf, uint64_t nleaf, double *out) {
    __shared__ double sh[STPB];
    const uint64_t units = leaf / 2;
    for (uint64_t L = blockIdx.x; L < nleaf; L += gridDim.x) {
        const double2 *p = a + L * leaf;
        double s = 0.0;
        for (uint64_t u = threadIdx.x; u < units; u += STPB) {
            const Amp2 x = ldg2(p + 2 * u);
            s = __fma_rn(x.a.x, x.a.x, s);
            s = __fma_rn(x.a.y, x.a.y, s);
            s = __fma_rn(x.b.x, x.b.x, s);
            s = __fma_rn(x.b.y, x.b.y, s);
        }
        sh[threadIdx.x] = s;
        __syncthreads();
        for (int w = STPB / 2; w >= 1; w >>= 1) {
            if ((int)threadIdx.x < w) sh[threadIdx.x] = sh[threadIdx.x] + sh[threadIdx.x + w];
            __syncthreads();
        }
        if (threadIdx.x == 0) out[L] = sh[0];
        __syncthreads();
    }
}

// one CTA per group of g = min(n, 512) consecutive values (n, g powers of two): perfect binary tree
__global__ void __launch_bounds__(STPB) k_tree(const double *__restrict__ in, double *__restrict__ out, uint64_t n) {
    __shared__ double b0[512], b1[512];
    const uint64_t g = n < 512 ? n : 512;
    const double *src = in + (uint64_t)blockIdx.x * g;
    for (uint64_t i = threadIdx.x; i < g; i += STPB) b0[i] = src[i];
    __syncthreads();
    double *cur = b0, *nxt = b1;
    for (uint64_t w = g / 2; w >= 1; w /= 2) {
        for (uint64_t i = threadIdx.x; i < w; i += STPB) nxt[i] = cur[2 * i] + cur[2 * i + 1];
        __syncthreads();
        double *t = cur;
        cur = nxt;
        nxt = t;
    }
    if (threadIdx.x == 0) out[blockIdx.x] = cur[0];
}

// The random state and its norm leaves in ONE pass over HBM (generation fused with k_norm_leaf): a CTA
// per leaf; thread t generates the units t, t + STPB, ... of its leaf — the order k_norm_leaf reads them —
// stores them and accumulates |a|^2 with the same FMA chain, then the same shared-memory tree.  The leaf
// sums are therefore bitwise those k_norm_leaf would compute from the stored state.
__global__ void __launch_bounds__(STPB) k_init_random_leaf(double2 *__restrict__ a, uint64_t leaf, uint64_t nleaf,
                                                           uint64_t gbase, uint64_t seed, double *out) {
    __shared__ double sh[STPB];
    const uint64_t units = leaf / 2;
    for (uint64_t L = blockIdx.x; L < nleaf; L += gridDim.x) {
        double2 *p = a + L * leaf;
        const uint64_t g0 = gbase + L * leaf;
        double s = 0.0;
        for (uint64_t u = threadIdx.x; u < units; u += STPB) {
            Amp2 x;
            x.a = gauss2(seed, g0 + 2 * u);
            x.b = gauss2(seed, g0 + 2 * u + 1);
            stg2(p + 2 * u, x);
            s = __fma_rn(x.a.x, x.a.x, s);
            s = __fma_rn(x.a.y, x.a.y, s);
            s = __fma_rn(x.b.x, x.b.x, s);
            s = __fma_rn(x.b.y, x.b.y, s);
        }
        sh[threadIdx.x] = s;
        __syncthreads();
        for (int w = STPB / 2; w >= 1; w >>= 1) {
            if ((int)threadIdx.x < w) sh[threadIdx.x] = sh[threadIdx.x] + sh[threadIdx.x + w];
            __syncthreads();
        }
        if (threadIdx.x == 0) out[L] = sh[0];
        __syncthreads();
    }
}

// the perfect binary tree over nleaf leaf sums in A (B: scratch of the same size) -> *d_out
static int norm_tree(double *A, double *B, uint64_t nleaf, double *d_out, cudaStream_t st) {
    int launches = 0;
    uint64_t n = nleaf;
    while (n > 1) {
        const uint64_t groups = n > 512 ? n / 512 : 1;
        double *dst = groups == 1 ? d_out : B;
        k_tree<<<(unsigned)groups, STPB, 0, st>>>(A, dst, n);
        ++launches;
        n = groups;
        double *t = A;
        A = B;
        B = t;
    }
    return launches;
}

int launch_norm2(const double2 *a, uint64_t count, int leaf_log2, double *scratch, double *d_out, cudaStream_t st,
                 int num_sms) {
    const uint64_t leaf = 1ull << leaf_log2;  // <= count; the same for every shard count (see qs_api.cu)
    const uint64_t nleaf = count / leaf;
    const uint64_t g = nleaf < (uint64_t)num_sms * 8 ? nleaf : (uint64_t)num_sms * 8;
    k_norm_leaf<<<(unsigned)g, STPB, 0, st>>>(a, leaf, nleaf, nleaf == 1 ? d_out : scratch);
    return 1 + norm_tree(scratch, scratch + nleaf, nleaf, d_out, st);
}

int launch_init_random_norm(double2 *a, uint64_t count, uint64_t global_base, uint64_t seed, int leaf_log2,
                            double *scratch, double *d_out, cudaStream_t st, int num_sms) {
    const uint64_t leaf = 1ull << leaf_log2;
    const uint64_t nleaf = count / leaf;
    const uint64_t g = nleaf < (uint64_t)num_sms * 8 ? nleaf : (uint64_t)num_sms * 8;
    k_init_random_leaf<<<(unsigned)g, STPB, 0, st>>>(a, leaf, nleaf, global_base, seed, nleaf == 1 ? d_out : scratch);
    return 1 + norm_tree(scratch, scratch + nleaf, nleaf, d_out, st);
}

// ------------------------------------------------------------------------------------------------
// Global-qubit exchange: fused 1q update of one received chunk.
// ------------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(STPB) k_xpair(double2 *__restrict__ a, const double2 *__restrict__ r, uint64_t nunits,
                                                uint64_t loff, int ctrl, int bit, U2 u) {
    const double2 ua = bit ? u.u[2] : u.u[0];
    const double2 ub = bit ? u.u[3] : u.u[1];
    const uint64_t step = (uint64_t)gridDim.x * STPB;
    for (uint64_t v = (uint64_t)blockIdx.x * STPB + threadIdx.x; v < nunits; v += step) {
        const Amp2 l = ldg2(a + 2 * v), x = ldg2(r + 2 * v);
        Amp2 o;
        // row `bit` of U times (a0, a1), a0 = the amplitude whose global target bit is 0
        o.a = bit ? cmac2(ua, x.a, ub, l.a) : cmac2(ua, l.a, ub, x.a);
        o.b = bit ? cmac2(ua, x.b, ub, l.b) : cmac2(ua, l.b, ub, x.b);
        if (ctrl >= 0) {
            const uint64_t i = loff + 2 * v;
            if (!((i >> ctrl) & 1)) o.a = l.a;
            if (!(((i + 1) >> ctrl) & 1)) o.b = l.b;
        }
        stg2(a + 2 * v, o);
    }
}

int launch_xpair_update(double2 *a, const double2 *r, uint64_t count, uint64_t local_offset, int ctrl, int bit,
                        const double *u2, cudaStream_t st, int num_sms) {
    U2 u;
    for (int i = 0; i < 4; ++i) u.u[i] = make_double2(u2[2 * i], u2[2 * i + 1]);
    const uint64_t nunits = count / 2;
    k_xpair<<<grid_for(nunits, STPB, num_sms), STPB, 0, st>>>(a, r, nunits, local_offset, ctrl, bit, u);
    return 1;
}

// Controlled 1q with a LOCAL control c and a GLOBAL target (§8(e)): only the control-1 half is
// exchanged, packed.  Element j of the control-1 sub-lattice is local index ins0(j, c) | 1 << c; the
// partner's element j has the same local bits.  a[i] = row `bit` of U applied to (a0, a1), where the
// amplitude with global target bit 0 is a0 (operand order of the local kernels).
__global__ void __launch_bounds__(STPB) k_xpair_packed(double2 *__restrict__ a, const double2 *__restrict__ r, int c,
                                                       uint64_t j0, uint64_t count, int bit, U2 u) {
    const double2 ua = bit ? u.u[2] : u.u[0];
    const double2 ub = bit ? u.u[3] : u.u[1];
    const uint64_t cb = 1ull << c;
    const uint64_t step = (uint64_t)gridDim.x * STPB;
    if (c >= 1) {  // pairs (j, j+1), j even, are adjacent in the state
        for (uint64_t v = (uint64_t)blockIdx.x * STPB + threadIdx.x; v < count / 2; v += step) {
            const uint64_t i = ins0(j0 + 2 * v, c) | cb;
            const Amp2 l = ldg2(a + i), x = ldg2(r + 2 * v);
            Amp2 o;
            o.a = bit ? cmac2(ua, x.a, ub, l.a) : cmac2(ua, l.a, ub, x.a);
            o.b = bit ? cmac2(ua, x.b, ub, l.b) : cmac2(ua, l.b, ub, x.b);
            stg2(a + i, o);
        }
    } else {
        for (uint64_t v = (uint64_t)blockIdx.x * STPB + threadIdx.x; v < count; v += step) {
            const uint64_t i = ((j0 + v) << 1) | 1ull;
            const double2 l = ldg1(a + i), x = ldg1(r + v);
            stg1(a + i, bit ? cmac2(ua, x, ub, l) : cmac2(ua, l, ub, x));
        }
    }
}

int launch_xpair_packed(double2 *a, const double2 *r, int c, uint64_t j0, uint64_t count, int bit, const double *u2,
                        cudaStream_t st, int num_sms) {
    U2 u;
    for (int i = 0; i < 4; ++i) u.u[i] = make_double2(u2[2 * i], u2[2 * i + 1]);
    k_xpair_packed<<<grid_for(count / 2, STPB, num_sms), STPB, 0, st>>>(a, r, c, j0, count, bit, u);
    return 1;
}

// sub-lattice {i : bit l of i == v}; element j of it is ins0(j, l) | v << l
template <bool PACK>
__global__ void __launch_bounds__(STPB) k_pack(double2 *__restrict__ a, double2 *__restrict__ buf, int l, int v,
                                               uint64_t j0, uint64_t count) {
    const uint64_t step = (uint64_t)gridDim.x * STPB;
    const uint64_t vb = (uint64_t)v << l;
    if (l >= 1) {  // pairs (j, j+1), j even, are adjacent in the state
        for (uint64_t u = (uint64_t)blockIdx.x * STPB + threadIdx.x; u < count / 2; u += step) {
            const uint64_t j = j0 + 2 * u;
            const uint64_t i = ins0(j, l) | vb;
            if (PACK)
                stg2(buf + 2 * u, ldg2(a + i));
            else
                stg2(a + i, ldg2(buf + 2 * u));
        }
    } else {
        for (uint64_t u = (uint64_t)blockIdx.x * STPB + threadIdx.x; u < count; u += step) {
            const uint64_t i = ((j0 + u) << 1) | vb;
            if (PACK)
                stg1(buf + u, ldg1(a + i));
            else
                stg1(a + i, ldg1(buf + u));
        }
    }
}

int launch_pack(const double2 *a, double2 *buf, int l, int v, uint64_t j0, uint64_t count, cudaStream_t st, int num_sms) {
    k_pack<true><<<grid_for(count / 2, STPB, num_sms), STPB, 0, st>>>(const_cast<double2 *>(a), buf, l, v, j0, count);
    return 1;
}

int launch_unpack(double2 *a, const double2 *buf, int l, int v, uint64_t j0, uint64_t count, cudaStream_t st, int num_sms) {
    k_pack<false><<<grid_for(count / 2, STPB, num_sms), STPB, 0, st>>>(a, const_cast<double2 *>(buf), l, v, j0, count);
    return 1;
}

}  // namespace qsb
