// fp64_peak.cu — measured FP64 (DADD / DFMA / DMUL) throughput of one B200, the ALU ceiling of the
// FP64-bound tile passes (DESIGN.md §6 "FP64 roofline").  Standalone measurement tool, not part of the
// library:  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_peak tools/fp64_peak.cu && /tmp/fp64_peak
//
// Each thread runs 16 independent dependency chains of one FP64 operation; per configuration
// (operation x warps per SM) the kernel runs ~0.2 s.  Reported: thread-operations per clock per SM
// (cycles from clock64 on SM 0's CTAs) and per second, and the SM clock the cycles imply.
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void burn(double *out, int iters, long long *cyc) {
    double a[16], b[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        a[k] = 1.0 + 1e-9 * (threadIdx.x + k);
        b[k] = 1e-12 * (k + 1);
    }
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            if (OP == 0) a[k] = __dadd_rn(a[k], b[k]);
            else if (OP == 1) a[k] = __fma_rn(a[k], 0.999999999, b[k]);
            else a[k] = __dmul_rn(a[k], 0.9999999999);
        }
    }
    const long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) s += a[k];
    if (s == 12345.678) out[0] = s;  // keep the chains alive
    if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *out;
    long long *cyc;
    cudaMalloc(&out, 8);
    cudaMalloc(&cyc, 8);
    const char *names[3] = {"DADD", "DFMA", "DMUL"};
    for (int op = 0; op < 3; ++op)
        for (int wps : {8, 16, 32}) {  // warps per SM: 256-thread CTAs, wps / 8 per SM
            const int ctas = sms * (wps / 8), tpb = 256, iters = 20000;
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            for (int rep = 0; rep < 2; ++rep) {
                cudaEventRecord(e0);
                if (op == 0) burn<0><<<ctas, tpb>>>(out, iters, cyc);
                else if (op == 1) burn<1><<<ctas, tpb>>>(out, iters, cyc);
                else burn<2><<<ctas, tpb>>>(out, iters, cyc);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
            }
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            long long c = 0;
            cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
            const double ops = (double)ctas * tpb * iters * 16;
            const double per_sm_clk = ops / sms / (double)c;
            printf("{\"op\": \"%s\", \"warps_per_sm\": %d, \"ms\": %.3f, \"thread_ops_per_clk_per_sm\": %.2f, "
                   "\"Gops_per_s\": %.1f, \"implied_mhz\": %.0f}\n",
                   names[op], wps, ms, per_sm_clk, ops / (ms * 1e-3) / 1e9, (double)c / (ms * 1e-3) / 1e6);
        }
    return 0;
}
