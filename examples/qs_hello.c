/*
 * qs_hello.c — the C-ABI of include/qs.h used from plain C (no Python, no torch): a 20-qubit state,
 * a Hadamard on every qubit (Alg. 1's example gate), then the QFT of a basis state
 * through qs_run_circuit, both checked against their closed forms (H^n|0> = uniform 2^(-n/2);
 * QFT|x> = 2^(-n/2) e^{+2 pi i x y / 2^n}, reading R5 of DESIGN.md).
 *
 *   gcc -O2 -I include examples/qs_hello.c -L paper_2506_09198_b200 -l:libqs_b200.so \
 *       -Wl,-rpath,$PWD/paper_2506_09198_b200 -lm -o qs_hello && ./qs_hello
 *
 * Exit status 0 when both checks pass; prints the library's error text otherwise.
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "qs.h"

#define CHECK(call)                                                                    \
    do {                                                                               \
        qs_status st_ = (call);                                                        \
        if (st_ != QS_OK) {                                                            \
            fprintf(stderr, "%s failed (%d): %s\n", #call, (int)st_, qs_last_error(s)); \
            return 1;                                                                  \
        }                                                                              \
    } while (0)

int main(void) {
    const int n = 20;
    const uint64_t N = (uint64_t)1 << n;
    qs_state *s = NULL;
    if (qs_create(n, 1, &s) != QS_OK) {
        fprintf(stderr, "qs_create: %s\n", qs_last_error(NULL));
        return 1;
    }
    const double h = 0.70710678118654752440;  /* 0x3FE6A09E667F3BCD, reading R6 */
    const double H[8] = {h, 0, h, 0, h, 0, -h, 0};
    for (int t = 0; t < n; ++t) CHECK(qs_apply_1q(s, t, H));
    double *amps = (double *)malloc(2 * N * sizeof(double));
    if (!amps) return 1;
    CHECK(qs_read_amps(s, 0, N, amps));
    double worst = 0.0;
    for (uint64_t i = 0; i < N; ++i) {
        const double d = hypot(amps[2 * i] - ldexp(1.0, -n / 2), amps[2 * i + 1]);
        if (d > worst) worst = d;
    }
    printf("H^%d|0>: max |a - 2^(-n/2)| = %.3e\n", n, worst);
    if (worst > 1e-12) return 2;

    /* QFT|x>: H(t), controlled R_k ladder, reversal SWAPs as one qs_run_circuit call */
    const uint64_t x = 123457 % N;
    size_t G = 0, cap = (size_t)n * (n + 1) / 2 + n;
    qs_gate *gates = (qs_gate *)calloc(cap, sizeof(qs_gate));
    if (!gates) return 1;
    for (int t = n - 1; t >= 0; --t) {
        qs_gate *g = &gates[G++];
        g->kind = QS_G_1Q;
        g->q0 = t;
        memcpy(g->m, H, sizeof H);
        for (int c = t - 1; c >= 0; --c) {
            g = &gates[G++];
            g->kind = QS_G_C1Q;
            g->q0 = c;
            g->q1 = t;
            const double th = M_PI / ldexp(1.0, t - c);
            g->m[0] = 1.0;
            g->m[6] = cos(th);
            g->m[7] = sin(th);
        }
    }
    for (int i = 0; i < n / 2; ++i) {
        qs_gate *g = &gates[G++];
        g->kind = QS_G_2Q;
        g->q0 = i;
        g->q1 = n - 1 - i;
        g->m[0] = g->m[2 * (4 * 1 + 2)] = g->m[2 * (4 * 2 + 1)] = g->m[2 * 15] = 1.0;  /* SWAP */
    }
    CHECK(qs_init_basis(s, x));
    CHECK(qs_run_circuit(s, gates, G));
    CHECK(qs_read_amps(s, 0, N, amps));
    worst = 0.0;
    for (uint64_t y = 0; y < N; ++y) {
        const double ang = M_PI * (double)((x * y) % N) / ldexp(1.0, n - 1);
        const double d = hypot(amps[2 * y] - ldexp(cos(ang), -n / 2), amps[2 * y + 1] - ldexp(sin(ang), -n / 2));
        if (d > worst) worst = d;
    }
    double norm = 0.0;
    CHECK(qs_norm2(s, &norm));
    printf("QFT(%d)|%llu> (%zu gates): max |a - closed form| = %.3e, |1 - norm| = %.1e\n", n, (unsigned long long)x, G,
           worst, fabs(1.0 - norm));
    free(gates);
    free(amps);
    qs_destroy(s);
    return worst <= 1e-12 && fabs(1.0 - norm) <= 1e-12 ? 0 : 3;
}
