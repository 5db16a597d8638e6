/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU state-vector simulator for the hot path of
 * arXiv 2506.09198 (PAPER.md = /root/reference/PAPER.md).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  It shares no source,
 * header, helper or constant generator with the CUDA path (paper_2506_09198_b200/csrc),
 * and neither side includes or links the other.
 *
 * Build: gcc -O2 -ffp-contract=off -fopenmp -fPIC -shared (no fast-math, no intrinsics), so
 * every complex product below is rounded exactly as written (reading R7).
 *
 * Storage (O1): double a[2*2^n], amplitude i at a[2i] (re), a[2i+1] (im) — the AoS layout of
 * PAPER.md:L114 (§II-A).  Qubit t is bit t of the index (Alg. 1, "sizeHalfBlock <- 1<<t").
 *
 * What the result IS: psi_out = M_G ... M_1 psi_in, M_g the gate embedded
 * in 2^n dimensions.  Nothing is approximated, so the oracle is that definition written out,
 * gate by gate, in list order.
 *
 * Pins (tests/test_oracle_pins.py): Alg. 1 worked index example and bijection,
 * dense Kronecker products at n <= 8 (numpy kron), H^n|0> closed form, QFT|x> closed form and
 * numpy ifft, CNOT/SWAP/X/Y truth tables, norm worked examples, SplitMix64 published vector,
 * Box-Muller distribution tests, orc_gauss2_range against orc_gauss2 / orc_init_random (bitwise).
 * No function here is "parity unpinned".
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------------------------ */
/* Alg. 1 index arithmetic (§II-A, "Hadamard (Default with new layout)")   */
/* ------------------------------------------------------------------------------------------ */
void orc_pair_index(uint64_t thisTask, int targetQubit, uint64_t *indexUp, uint64_t *indexLo)
{
    uint64_t sizeHalfBlock = (uint64_t)1 << targetQubit;           /* L124 */
    uint64_t sizeBlock = 2 * sizeHalfBlock;                        /* L125 */
    uint64_t thisBlock = thisTask / sizeHalfBlock;                 /* L132 */
    *indexUp = thisBlock * sizeBlock + (thisTask % sizeHalfBlock); /* L133 */
    *indexLo = *indexUp + sizeHalfBlock;                           /* L134 */
}

/* u*x for complex u = (ur, ui), x = (xr, xi), written out: (ur*xr - ui*xi, ur*xi + ui*xr) */
static void cmul(double ur, double ui, double xr, double xi, double *cr, double *ci)
{
    *cr = ur * xr - ui * xi;
    *ci = ur * xi + ui * xr;
}

/* ------------------------------------------------------------------------------------------ */
/* O2: |x>   (SPEC.md:L44-L52 create_state, "amplitude 0 = (1, 0)" generalised to index x)     */
/* ------------------------------------------------------------------------------------------ */
void orc_init_basis(double *a, int n, uint64_t x)
{
    uint64_t N = (uint64_t)1 << n;
    memset(a, 0, sizeof(double) * 2 * N);
    a[2 * x] = 1.0;
}

/* ------------------------------------------------------------------------------------------ */
/* O8: sum_i |a_i|^2, pairwise: leaves of ORC_LEAF amplitudes summed in index order, then a    */
/* fixed binary tree over the leaf sums.  Same result for any thread count.                    */
/* (SPEC.md:L54-L62 total_probability; SURVEY.md §8(c) c.6 "Norm summation")                  */
/* ------------------------------------------------------------------------------------------ */
#define ORC_LEAF 4096

static double tree_sum(const double *v, uint64_t lo, uint64_t hi)
{
    if (hi - lo == 1) return v[lo];
    uint64_t mid = lo + (hi - lo) / 2;
    return tree_sum(v, lo, mid) + tree_sum(v, mid, hi);
}

double orc_norm2_count(const double *a, uint64_t count)
{
    if (count == 0) return 0.0;
    uint64_t nleaf = (count + ORC_LEAF - 1) / ORC_LEAF;
    double *leaf = (double *)malloc(sizeof(double) * nleaf);
    if (!leaf) return NAN;
    int64_t L;
#pragma omp parallel for schedule(static)
    for (L = 0; L < (int64_t)nleaf; ++L) {
        uint64_t lo = (uint64_t)L * ORC_LEAF;
        uint64_t hi = lo + ORC_LEAF;
        if (hi > count) hi = count;
        double s = 0.0;
        for (uint64_t i = lo; i < hi; ++i) {
            double re = a[2 * i], im = a[2 * i + 1];
            s = s + (re * re + im * im);
        }
        leaf[L] = s;
    }
    double total = tree_sum(leaf, 0, nleaf);
    free(leaf);
    return total;
}

double orc_norm2(const double *a, int n)
{
    return orc_norm2_count(a, (uint64_t)1 << n);
}

/* ------------------------------------------------------------------------------------------ */
/* O3: random normalised state, SURVEY.md §8(c) c.3 (reading R9): SplitMix64 + Box-Muller,     */
/* each amplitude a function of (seed, global index) only.  Normalised by multiplying with     */
/* 1/sqrt(sum) ("Σ|amp|² = 1").                                                    */
/* ------------------------------------------------------------------------------------------ */
static uint64_t orc_mix(uint64_t z)
{
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

uint64_t orc_splitmix64(uint64_t seed, uint64_t j)
{
    return orc_mix(seed + (j + 1) * 0x9E3779B97F4A7C15ULL);
}

void orc_gauss2(uint64_t seed, uint64_t i, double *re, double *im)
{
    uint64_t x1 = orc_splitmix64(seed, 2 * i);
    uint64_t x2 = orc_splitmix64(seed, 2 * i + 1);
    double u1 = (double)((x1 >> 11) + 1) * 0x1.0p-53; /* (0, 1] */
    double u2 = (double)(x2 >> 11) * 0x1.0p-53;       /* [0, 1) */
    double rho = sqrt(-2.0 * log(u1));
    double ang = 2.0 * M_PI * u2;
    *re = rho * cos(ang);
    *im = rho * sin(ang);
}

/* The unnormalised samples gauss2(seed, i) for i in [start, start + count), at a[2(i - start)] (re) and
 * a[2(i - start) + 1] (im): what orc_init_random draws before it normalises, for states too large
 * for host memory (the QFT(32) of a random state is checked by DFT sums over these chunks). */
void orc_gauss2_range(double *a, uint64_t seed, uint64_t start, uint64_t count)
{
    int64_t k;
#pragma omp parallel for schedule(static)
    for (k = 0; k < (int64_t)count; ++k) orc_gauss2(seed, start + (uint64_t)k, &a[2 * k], &a[2 * k + 1]);
}

void orc_init_random(double *a, int n, uint64_t seed)
{
    uint64_t N = (uint64_t)1 << n;
    int64_t i;
#pragma omp parallel for schedule(static)
    for (i = 0; i < (int64_t)N; ++i) orc_gauss2(seed, (uint64_t)i, &a[2 * i], &a[2 * i + 1]);
    double s = orc_norm2(a, n);
    double inv = 1.0 / sqrt(s);
#pragma omp parallel for schedule(static)
    for (i = 0; i < (int64_t)(2 * N); ++i) a[i] = a[i] * inv;
}

/* ------------------------------------------------------------------------------------------ */
/* O4: 1q gate, Alg. 1 form: for every task, (up, lo) from Alg. 1's index */
/* arithmetic; a[up] = u00 x + u01 y; a[lo] = u10 x + u11 y (terms summed left to right).      */
/* u = {u00r,u00i,u01r,u01i,u10r,u10i,u11r,u11i}: the gate-matrix-vector product of           */
/* PAPER.md:L179-L180 ("the core operation is a matrix-vector multiplication").                */
/* ------------------------------------------------------------------------------------------ */
static void pair_update(double *a, uint64_t up, uint64_t lo, const double *u)
{
    double xr = a[2 * up], xi = a[2 * up + 1];
    double yr = a[2 * lo], yi = a[2 * lo + 1];
    double p0r, p0i, p1r, p1i, p2r, p2i, p3r, p3i;
    cmul(u[0], u[1], xr, xi, &p0r, &p0i);
    cmul(u[2], u[3], yr, yi, &p1r, &p1i);
    cmul(u[4], u[5], xr, xi, &p2r, &p2i);
    cmul(u[6], u[7], yr, yi, &p3r, &p3i);
    a[2 * up] = p0r + p1r;
    a[2 * up + 1] = p0i + p1i;
    a[2 * lo] = p2r + p3r;
    a[2 * lo + 1] = p2i + p3i;
}

void orc_apply_1q(double *a, int n, int t, const double *u)
{
    uint64_t numTasks = ((uint64_t)1 << n) >> 1; /* Alg. 1 */
    int64_t task;
#pragma omp parallel for schedule(static)
    for (task = 0; task < (int64_t)numTasks; ++task) {
        uint64_t up, lo;
        orc_pair_index((uint64_t)task, t, &up, &lo);
        pair_update(a, up, lo, u);
    }
}

/* ------------------------------------------------------------------------------------------ */
/* O5: controlled 1q.  PAPER.md:L271 / L288: "only the amplitudes corresponding to a control   */
/* bit of 1 are updated".  Iterate-and-test over every index (deliberately unlike the GPU's    */
/* bit insertion): if bit_c(i) = 1 and bit_t(i) = 0, update the pair (i, i | 2^t).             */
/* ------------------------------------------------------------------------------------------ */
void orc_apply_ctrl_1q(double *a, int n, int c, int t, const double *u)
{
    uint64_t N = (uint64_t)1 << n;
    int64_t i;
#pragma omp parallel for schedule(static)
    for (i = 0; i < (int64_t)N; ++i) {
        uint64_t ui = (uint64_t)i;
        if (((ui >> c) & 1) == 1 && ((ui >> t) & 1) == 0) pair_update(a, ui, ui | ((uint64_t)1 << t), u);
    }
}

/* ------------------------------------------------------------------------------------------ */
/* O6: general 2q gate (BASELINE.json north_star "general 4x4"; the paper's own 2q gate is     */
/* CNOT).  For every i with bit_q0 = bit_q1 = 0: idx[s] = i | (s&1)<<q0 |      */
/* (s>>1)<<q1, v = a[idx], a[idx[r]] = sum_{s=0..3} U[r][s] v[s], s ascending.                  */
/* ------------------------------------------------------------------------------------------ */
void orc_apply_2q(double *a, int n, int q0, int q1, const double *u)
{
    uint64_t N = (uint64_t)1 << n;
    int64_t i;
#pragma omp parallel for schedule(static)
    for (i = 0; i < (int64_t)N; ++i) {
        uint64_t ui = (uint64_t)i;
        if (((ui >> q0) & 1) != 0 || ((ui >> q1) & 1) != 0) continue;
        uint64_t idx[4];
        double vr[4], vi[4];
        for (int s = 0; s < 4; ++s) {
            idx[s] = ui | ((uint64_t)(s & 1) << q0) | ((uint64_t)(s >> 1) << q1);
            vr[s] = a[2 * idx[s]];
            vi[s] = a[2 * idx[s] + 1];
        }
        for (int r = 0; r < 4; ++r) {
            double accr = 0.0, acci = 0.0;
            for (int s = 0; s < 4; ++s) {
                double pr, pi;
                const double *e = &u[2 * (4 * r + s)];
                cmul(e[0], e[1], vr[s], vi[s], &pr, &pi);
                if (s == 0) {
                    accr = pr;
                    acci = pi;
                } else {
                    accr = accr + pr;
                    acci = acci + pi;
                }
            }
            a[2 * idx[r]] = accr;
            a[2 * idx[r] + 1] = acci;
        }
    }
}

/* ------------------------------------------------------------------------------------------ */
/* O7: run an ordered gate list through O4-O6 only (no specialisation, no fusion, no reorder). */
/* kind: 0 = 1q (q0 = target), 1 = ctrl-1q (q0 = ctrl, q1 = target), 2 = 2q (q0, q1).          */
/* mats: 32 doubles per gate (1q/ctrl use the first 8).  Returns 0, or -1 on a bad gate.        */
/* ------------------------------------------------------------------------------------------ */
int orc_run(double *a, int n, const int32_t *kind, const int32_t *q0, const int32_t *q1,
            const double *mats, uint64_t G)
{
    for (uint64_t g = 0; g < G; ++g) {
        const double *m = mats + 32 * g;
        if (q0[g] < 0 || q0[g] >= n) return -1;
        if (kind[g] != 0 && (q1[g] < 0 || q1[g] >= n || q1[g] == q0[g])) return -1;
        switch (kind[g]) {
        case 0: orc_apply_1q(a, n, q0[g], m); break;
        case 1: orc_apply_ctrl_1q(a, n, q0[g], q1[g], m); break;
        case 2: orc_apply_2q(a, n, q0[g], q1[g], m); break;
        default: return -1;
        }
    }
    return 0;
}
