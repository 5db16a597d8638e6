// k_p2p.cu — global-qubit gates fused with their exchange over PEER memory (SURVEY.md §8(e) table,
// §8(f) rank 3): one kernel per rank loads its own amplitude and the partner's (NVLink P2P load),
// applies the gate, and stores both (NVLink P2P store).  No exchange buffers, no NCCL, no separate
// update pass: every amplitude crosses HBM once each way (the same 32 B per amplitude as a local
// gate) and NVLink carries 16·2^m B per direction per rank — the bytes of the pairwise exchange.
//
// Work split of a pair of ranks (d, d' = d ^ 2^(g-m)): the pair's tasks are enumerated once; the rank
// whose global bit is 0 takes the first half, the other rank the second half, so both GPUs stream
// concurrently and each task is done by exactly one of them.  The caller orders the two kernels
// against the partner's stream (ready before, done after).  Operand order is that of the local
// kernels (cmac2(u_r0, a0, u_r1, a1), a0 = amplitude with global bit 0): results are bitwise those of
// the single-GPU path.
#include "qs_device.cuh"
#include "qs_kernels.h"

namespace qsb {

constexpr int P2P_TPB = 256;

// 1q on a global target (optionally controlled by LOCAL qubit c): tasks p in [p0, p1) of the pair;
// local index i = p (no control) or ins0(p, c) | 2^c (only control-1 amplitudes change).
__global__ void __launch_bounds__(P2P_TPB) k_p2p_pair(double2 *__restrict__ loc, double2 *__restrict__ rem, uint64_t p0,
                                                     uint64_t p1, int c, int bit, U2 u) {
    const uint64_t step = (uint64_t)gridDim.x * P2P_TPB;
    for (uint64_t p = p0 + (uint64_t)blockIdx.x * P2P_TPB + threadIdx.x; p < p1; p += step) {
        const uint64_t i = c < 0 ? p : (ins0(p, c) | (1ull << c));
        const double2 l = ldg1(loc + i), r = ldg1(rem + i);
        const double2 a0 = bit ? r : l, a1 = bit ? l : r;
        const double2 n0 = cmac2(u.u[0], a0, u.u[1], a1), n1 = cmac2(u.u[2], a0, u.u[3], a1);
        stg1(loc + i, bit ? n1 : n0);
        stg1(rem + i, bit ? n0 : n1);
    }
}

// the same without a control, two amplitudes per 256-bit access
__global__ void __launch_bounds__(P2P_TPB) k_p2p_pair2(double2 *__restrict__ loc, double2 *__restrict__ rem, uint64_t v0,
                                                      uint64_t v1, int bit, U2 u) {
    const uint64_t step = (uint64_t)gridDim.x * P2P_TPB;
    for (uint64_t v = v0 + (uint64_t)blockIdx.x * P2P_TPB + threadIdx.x; v < v1; v += step) {
        const Amp2 l = ldg2(loc + 2 * v), r = ldg2(rem + 2 * v);
        Amp2 nl, nr;
        {
            const double2 a0 = bit ? r.a : l.a, a1 = bit ? l.a : r.a;
            const double2 n0 = cmac2(u.u[0], a0, u.u[1], a1), n1 = cmac2(u.u[2], a0, u.u[3], a1);
            nl.a = bit ? n1 : n0;
            nr.a = bit ? n0 : n1;
        }
        {
            const double2 a0 = bit ? r.b : l.b, a1 = bit ? l.b : r.b;
            const double2 n0 = cmac2(u.u[0], a0, u.u[1], a1), n1 = cmac2(u.u[2], a0, u.u[3], a1);
            nl.b = bit ? n1 : n0;
            nr.b = bit ? n0 : n1;
        }
        stg2(loc + 2 * v, nl);
        stg2(rem + 2 * v, nr);
    }
}

// SWAP(local l, global g): the amplitude at local j with bit l = 1 on the bit-0 rank trades places
// with the amplitude at j ^ 2^l on the bit-1 rank.  Tasks p: bit-0 rank index ins0(p, l) | 2^l, bit-1
// rank index ins0(p, l).
__global__ void __launch_bounds__(P2P_TPB) k_p2p_swap_lg(double2 *__restrict__ loc, double2 *__restrict__ rem, uint64_t p0,
                                                        uint64_t p1, int l, int bit) {
    const uint64_t step = (uint64_t)gridDim.x * P2P_TPB;
    for (uint64_t p = p0 + (uint64_t)blockIdx.x * P2P_TPB + threadIdx.x; p < p1; p += step) {
        const uint64_t j0 = ins0(p, l);
        const uint64_t jl = bit ? j0 : (j0 | (1ull << l)), jr = bit ? (j0 | (1ull << l)) : j0;
        const double2 x = ldg1(loc + jl), y = ldg1(rem + jr);
        stg1(loc + jl, y);
        stg1(rem + jr, x);
    }
}

// SWAP of two global qubits on ranks whose two bits differ: whole shards trade places
__global__ void __launch_bounds__(P2P_TPB) k_p2p_swap_all(double2 *__restrict__ loc, double2 *__restrict__ rem, uint64_t v0,
                                                         uint64_t v1) {
    const uint64_t step = (uint64_t)gridDim.x * P2P_TPB;
    for (uint64_t v = v0 + (uint64_t)blockIdx.x * P2P_TPB + threadIdx.x; v < v1; v += step) {
        const Amp2 x = ldg2(loc + 2 * v), y = ldg2(rem + 2 * v);
        stg2(loc + 2 * v, y);
        stg2(rem + 2 * v, x);
    }
}

// Pairwise device-side barrier for the one-process-per-GPU mode (peer shards mapped with CUDA IPC):
// publish `val` into the partner's flag slot for this rank (system-scope release after a system fence,
// so this rank's earlier writes are visible), then wait until the partner published `val` into ours.
// A partner that never arrives traps after ~10 s (a CUDA error at the next qs_sync, not a hang).
__global__ void k_flag_barrier(unsigned long long *my_flags, unsigned long long *peer_flags, int me, int peer,
                               unsigned long long val) {
    if (threadIdx.x != 0) return;
    __threadfence_system();
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(peer_flags + me), "l"(val) : "memory");
    const long long t0 = clock64();
    for (;;) {
        unsigned long long v;
        asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(my_flags + peer) : "memory");
        if (v >= val) break;
        __nanosleep(200);
        if (clock64() - t0 > 20000000000ll) asm volatile("trap;");
    }
    __threadfence_system();
}

int launch_flag_barrier(unsigned long long *my_flags, unsigned long long *peer_flags, int me, int peer,
                        unsigned long long val, cudaStream_t st) {
    k_flag_barrier<<<1, 32, 0, st>>>(my_flags, peer_flags, me, peer, val);
    return 1;
}

namespace {
int p2p_grid(uint64_t work, int num_sms) {
    // one-shot grid (one work unit per thread; the loops stay grid-stride for safety): the block
    // scheduler streams the blocks, which measured faster than a persistent 8-CTAs-per-SM grid-stride
    // loop for the local gates and here (virtual shards, U2 on the global qubit at n = 30:
    // 5.77 ms persistent)
    (void)num_sms;
    uint64_t g = (work + P2P_TPB - 1) / P2P_TPB;
    if (g > 0x7fffffffull) g = 0x7fffffffull;
    return (int)(g < 1 ? 1 : g);
}
}  // namespace

int launch_p2p_exchange(int action, double2 *loc, double2 *rem, int m, int bit, int ctrl, int l, bool lower,
                        const double *u2, cudaStream_t st, int num_sms) {
    const uint64_t N = 1ull << m;
    if (action == SA_XPAIR) {
        U2 u;
        for (int i = 0; i < 4; ++i) u.u[i] = make_double2(u2[2 * i], u2[2 * i + 1]);
        if (ctrl < 0) {  // N tasks of one amplitude = N/2 units of two
            const uint64_t half = N / 4, v0 = bit ? half : 0;
            k_p2p_pair2<<<p2p_grid(half, num_sms), P2P_TPB, 0, st>>>(loc, rem, v0, v0 + half, bit, u);
        } else {         // N/2 control-1 tasks
            const uint64_t half = N / 4, p0 = bit ? half : 0;
            k_p2p_pair<<<p2p_grid(half, num_sms), P2P_TPB, 0, st>>>(loc, rem, p0, p0 + half, ctrl, bit, u);
        }
        return 1;
    }
    if (action == SA_XSWAP_LG) {  // N/2 pairs
        const uint64_t half = N / 4, p0 = bit ? half : 0;
        k_p2p_swap_lg<<<p2p_grid(half, num_sms), P2P_TPB, 0, st>>>(loc, rem, p0, p0 + half, l, bit);
        return 1;
    }
    if (action == SA_XSWAP_GG) {  // N/2 units; the lower rank of the pair takes the first half
        const uint64_t half = N / 4, v0 = lower ? 0 : half;
        k_p2p_swap_all<<<p2p_grid(half, num_sms), P2P_TPB, 0, st>>>(loc, rem, v0, v0 + half);
        return 1;
    }
    return -1;
}

}  // namespace qsb
