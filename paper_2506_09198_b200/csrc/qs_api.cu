// qs_api.cu — the C ABI of include/qs.h: device/state manager, gate dispatcher, circuit executor
// and the global-qubit exchange engine.
//
// Process models (qs.h): one process driving P devices (ncclCommInitAll), P virtual shards on one
// device (fused peer kernels, or the buffered pipeline with device copies / NCCL send-recv to self as
// the transport), or one process per GPU
// (ncclCommInitRank; torchrun).  All three run the same shard-level code: every gate is routed per
// shard by qsb::localize (qs_plan.cpp) and either launched locally or run through the chunked,
// double-buffered pairwise exchange with the gate update fused per chunk.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "qs.h"
#include "qs_kernels.h"
#include "qs_plan.h"
#include "qs_plan_abi.h"

using namespace qsb;

namespace {

enum Mode { MODE_SINGLE = 0, MODE_MULTIDEV = 1, MODE_VIRTUAL = 2, MODE_RANK = 3 };

struct Shard {
    int rank = 0;
    int device = 0;
    double2 *amps = nullptr;
    char *alloc_base = nullptr;   // amps - guard (QS_DEBUG_CANARY) or amps
    cudaStream_t st = nullptr;    // compute
    cudaStream_t comm = nullptr;  // NCCL
    bool own_streams = false;
    double2 *rbuf[2] = {nullptr, nullptr};
    double2 *sbuf[2] = {nullptr, nullptr};
    cudaEvent_t ev_recv[2] = {nullptr, nullptr}, ev_upd[2] = {nullptr, nullptr}, ev_pack[2] = {nullptr, nullptr};
    cudaEvent_t ev_ready = nullptr, ev_done = nullptr;  // peer-memory exchange: partner ordering
    bool own_events = false;
    double *d_scratch = nullptr;  // norm partials
    double *d_norm = nullptr;     // 1 double (+P for allgather)
    double *h_norm = nullptr;     // pinned
    TileDesc *d_desc = nullptr;
    TileBatch *d_bat = nullptr;
    TileOp *d_ops = nullptr;
    TileLadder *d_lad = nullptr;
    size_t desc_cap = 0, bat_cap = 0, ops_cap = 0, lad_cap = 0;
    ncclComm_t nccl = nullptr;
    // one-process-per-GPU peer mapping (QS_P2P_RANK=1): partners' shards and flag arrays via CUDA IPC
    unsigned long long *flags = nullptr;        // flags[r]: last value rank r published to this rank
    std::vector<char *> peer_base;              // IPC-mapped allocation bases (index = rank)
    std::vector<unsigned long long *> peer_flags;
    std::vector<unsigned long long> seq;        // per-partner exchange counter
};

thread_local std::string g_create_error = "no error";

struct Prepared;  // run_ops' host-side preparation of an op list (defined below)

}  // namespace

struct qs_state {
    int n = 0, P = 1, m = 0, mode = MODE_SINGLE;
    int num_sms = 148;
    std::vector<Shard> sh;
    std::string err = "no error";
    qs_status sticky = QS_OK;
    uint64_t launches = 0;
    bool fuse = true;
    int tile_b = 12;
    int tile_low = 4;             // local qubits 0..tile_low-1 are in every tile (contiguous runs)
    bool tile_low_auto = true;    // ... or tile_low-1 when that saves >= 10% of the passes
    uint64_t chunk_bytes = 256ull << 20;
    bool check_unitary = true;
    bool jit_async = false;       // compile new pass kernels in the background (interpreter meanwhile);
                                  // off by default: the interpreter is 13-27x slower than the JIT kernels
                                  // on QFT/RQC passes, more than the parallel NVRTC compile costs
    bool jit = true;              // run tile passes through NVRTC straight-line kernels (jit_tile.cu)
    bool p2p = true;              // global-qubit gates through the fused peer-memory kernels (k_p2p.cu)
    bool p2p_ok = false;          // ... when every shard can address its partners (virtual; peer access)
    bool factor = true;           // circuits: scalar factoring of monomial 1q gates (qs_plan.cpp)
    bool remap = true;            // sharded: global-qubit remapping (qs_plan.cpp remap_global)
    bool reorder = true;          // commutation-aware pass scheduling (qs_plan.cpp; 0 = gate order)
    bool perm_fuse = true;        // a permutation run joins the tile pass before it when it closes (tile pairs)
    bool perm_hoist = true;       // ... or is split over the tile passes before it (qs_plan.h hoist_permutation)
    int perm_low = 5;             // permutation passes for runs of disjoint SWAPs (0 = off), runs of 2^perm_low
    int ladder_min = 4;           // PHASE LADDER merge of >= ladder_min phase ops (0 = off: bitwise = unfused)
    int vtransport = 0;           // virtual shards, buffered exchange: 0 device copies, 1 NCCL send/recv to self
    int jit_family = 1;           // 0 specialised pass kernels only, 1 specialised else family (jit_tile.cu), 2 family
    bool graph = true;            // single-shard circuits: repeated runs replay a captured CUDA graph
    std::string jit_error;        // last JIT compile failure (the interpreter ran instead)
    uint64_t last_passes = 0, last_exchanges = 0;
    std::unordered_map<uint64_t, std::shared_ptr<Prepared>> prep_cache;  // run_ops: op-list hash -> prepared run
    size_t guard = 0;             // QS_DEBUG_CANARY: bytes of 0xA5 before and after every shard
    uint64_t chunk_amps() const {
        uint64_t c = chunk_bytes / 16, shard = 1ull << m;
        return c < shard ? c : shard;
    }
};

namespace {

// an Op back as a qs_gate (diagonal ops as diagonal matrices; SWAP as its permutation matrix)
void op_to_gate(const Op &op, qs_gate &o) {
    std::memset(&o, 0, sizeof o);
    o.q0 = op.q0;
    o.q1 = op.q1;
    switch (op.kind) {
    case OP_PAIR: o.kind = QS_G_1Q; std::memcpy(o.m, op.m, 8 * sizeof(double)); break;
    case OP_CTRL_PAIR: o.kind = QS_G_C1Q; std::memcpy(o.m, op.m, 8 * sizeof(double)); break;
    case OP_QUAD: o.kind = QS_G_2Q; std::memcpy(o.m, op.m, 32 * sizeof(double)); break;
    case OP_SWAP:
        o.kind = QS_G_2Q;
        o.m[0] = o.m[2 * (4 * 1 + 2)] = o.m[2 * (4 * 2 + 1)] = o.m[2 * 15] = 1.0;
        break;
    default:  // OP_DIAG on 1 or 2 qubits: the diagonal matrix
        if (op.q1 < 0) {
            o.kind = QS_G_1Q;
            o.m[0] = op.m[0], o.m[1] = op.m[1], o.m[6] = op.m[2], o.m[7] = op.m[3];
        } else {
            o.kind = QS_G_2Q;
            for (int k = 0; k < 4; ++k) o.m[2 * (5 * k)] = op.m[2 * k], o.m[2 * (5 * k) + 1] = op.m[2 * k + 1];
        }
        break;
    }
}

std::string fmt(const char *f, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, f);
    vsnprintf(buf, sizeof buf, f, ap);
    va_end(ap);
    return buf;
}

qs_status set_err(qs_state *s, qs_status code, const std::string &msg) {
    s->err = msg;
    if (code == QS_ERR_CUDA || code == QS_ERR_NCCL) s->sticky = code;
    return code;
}

#define QS_CUDA(s, call)                                                                                     \
    do {                                                                                                     \
        cudaError_t e_ = (call);                                                                             \
        if (e_ != cudaSuccess)                                                                               \
            return set_err((s), QS_ERR_CUDA, fmt("%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_),  \
                                                 __FILE__, __LINE__));                                       \
    } while (0)

#define QS_NCCL(s, call)                                                                                     \
    do {                                                                                                     \
        ncclResult_t r_ = (call);                                                                            \
        if (r_ != ncclSuccess)                                                                               \
            return set_err((s), QS_ERR_NCCL, fmt("%s failed: %s (%s:%d)", #call, ncclGetErrorString(r_),  \
                                                 __FILE__, __LINE__));                                       \
    } while (0)

#define QS_TRY(expr)                   \
    do {                               \
        qs_status t_ = (expr);         \
        if (t_ != QS_OK) return t_;    \
    } while (0)

qs_status check_launch(qs_state *s, int launched) {
    s->launches += (uint64_t)launched;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_err(s, QS_ERR_CUDA, fmt("kernel launch failed: %s", cudaGetErrorString(e)));
    return QS_OK;
}

qs_status guard(const qs_state *s) {
    if (!s) return QS_ERR_ARG;
    if (s->sticky != QS_OK) return QS_ERR_STATE;
    return QS_OK;
}

int log2_exact(int P) {
    int k = 0;
    while ((1 << k) < P) ++k;
    return (1 << k) == P ? k : -1;
}

// ------------------------------------------------------------------------------------------------
// allocation
// ------------------------------------------------------------------------------------------------
size_t canary_bytes() {  // bounds checking of our own (compute-sanitizer is unavailable on the pool)
    const char *e = getenv("QS_DEBUG_CANARY");
    return (e && atoi(e)) ? (size_t)1 << 20 : 0;
}

qs_status check_canaries(qs_state *s) {
    if (!s->guard) return QS_OK;
    std::vector<unsigned char> h(s->guard);
    const size_t state_bytes = (size_t)16 << s->m;
    for (auto &d : s->sh) {
        QS_CUDA(s, cudaSetDevice(d.device));
        for (int side = 0; side < 2; ++side) {
            const char *src = side == 0 ? d.alloc_base : d.alloc_base + s->guard + state_bytes;
            QS_CUDA(s, cudaMemcpy(h.data(), src, s->guard, cudaMemcpyDeviceToHost));
            for (size_t i = 0; i < s->guard; ++i)
                if (h[i] != 0xA5)
                    return set_err(s, QS_ERR_CUDA, fmt("canary %s shard %d overwritten at byte %zu", side ? "after" : "before",
                                                       d.rank, i));
        }
    }
    return QS_OK;
}

uint64_t norm_scratch_doubles(int n, int m) {  // one double per leaf + the tree levels
    const uint64_t leaves = (1ull << m) >> std::min(norm_leaf_log2(n), m);
    return leaves + leaves / 256 + 1024;
}

qs_status alloc_exchange_buffers(qs_state *s, Shard &d) {
    if (s->P == 1) return QS_OK;
    const size_t bytes = (size_t)s->chunk_amps() * 16;
    for (int i = 0; i < 2; ++i) {
        QS_CUDA(s, cudaMalloc(&d.rbuf[i], bytes));
        QS_CUDA(s, cudaMalloc(&d.sbuf[i], bytes));
    }
    return QS_OK;
}

void free_exchange_buffers(Shard &d) {
    for (int i = 0; i < 2; ++i) {
        if (d.rbuf[i]) cudaFree(d.rbuf[i]);
        if (d.sbuf[i]) cudaFree(d.sbuf[i]);
        d.rbuf[i] = d.sbuf[i] = nullptr;
    }
}

qs_status alloc_shard(qs_state *s, Shard &d, bool make_streams) {
    QS_CUDA(s, cudaSetDevice(d.device));
    // measurement knob: the L2's DRAM fetch granularity (bytes; the driver default is 64), to test
    // whether gates selecting on qubit 1 pay a 64-B read atom ("64-B granule")
    if (const char *g = getenv("QS_L2_FETCH_GRAN")) QS_CUDA(s, cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)atoi(g)));
    const size_t state_bytes = (size_t)16 << s->m;
    const size_t xbytes = s->P > 1 ? 4 * (size_t)s->chunk_amps() * 16 : 0;
    const size_t need = state_bytes + xbytes + norm_scratch_doubles(s->n, s->m) * 8 + (64ull << 20);
    size_t fr = 0, tot = 0;
    QS_CUDA(s, cudaMemGetInfo(&fr, &tot));
    if (need > fr)
        return set_err(s, QS_ERR_OOM,
                       fmt("device %d: need %zu bytes (state %zu + exchange %zu + scratch), %zu free of %zu", d.device,
                           need, state_bytes, xbytes, fr, tot));
    QS_CUDA(s, cudaMalloc(&d.alloc_base, state_bytes + 2 * s->guard));
    d.amps = reinterpret_cast<double2 *>(d.alloc_base + s->guard);
    if (s->guard) {
        QS_CUDA(s, cudaMemset(d.alloc_base, 0xA5, s->guard));
        QS_CUDA(s, cudaMemset(d.alloc_base + s->guard + state_bytes, 0xA5, s->guard));
    }
    if (make_streams) {
        QS_CUDA(s, cudaStreamCreateWithFlags(&d.st, cudaStreamNonBlocking));
        QS_CUDA(s, cudaStreamCreateWithFlags(&d.comm, cudaStreamNonBlocking));
        d.own_streams = true;
        for (int i = 0; i < 2; ++i) {
            QS_CUDA(s, cudaEventCreateWithFlags(&d.ev_recv[i], cudaEventDisableTiming));
            QS_CUDA(s, cudaEventCreateWithFlags(&d.ev_upd[i], cudaEventDisableTiming));
            QS_CUDA(s, cudaEventCreateWithFlags(&d.ev_pack[i], cudaEventDisableTiming));
        }
        QS_CUDA(s, cudaEventCreateWithFlags(&d.ev_ready, cudaEventDisableTiming));
        QS_CUDA(s, cudaEventCreateWithFlags(&d.ev_done, cudaEventDisableTiming));
        d.own_events = true;
    }
    QS_CUDA(s, cudaMalloc(&d.d_scratch, norm_scratch_doubles(s->n, s->m) * 8));
    QS_CUDA(s, cudaMalloc(&d.d_norm, 8 * (1 + 16)));
    QS_CUDA(s, cudaMallocHost(&d.h_norm, 8 * (1 + 16)));
    QS_TRY(alloc_exchange_buffers(s, d));
    return QS_OK;
}

void destroy_state(qs_state *s) {
    if (!s) return;
    for (auto &d : s->sh) {
        cudaSetDevice(d.device);
        if (d.st) cudaStreamSynchronize(d.st);
        if (d.comm) cudaStreamSynchronize(d.comm);
    }
    for (auto &d : s->sh) {
        cudaSetDevice(d.device);
        for (char *b : d.peer_base)
            if (b) cudaIpcCloseMemHandle(b);
        for (unsigned long long *f : d.peer_flags)
            if (f) cudaIpcCloseMemHandle(f);
        if (d.flags) cudaFree(d.flags);
        if (d.nccl) ncclCommDestroy(d.nccl);
        if (d.alloc_base) cudaFree(d.alloc_base);
        free_exchange_buffers(d);
        if (d.d_scratch) cudaFree(d.d_scratch);
        if (d.d_norm) cudaFree(d.d_norm);
        if (d.h_norm) cudaFreeHost(d.h_norm);
        if (d.d_desc) cudaFree(d.d_desc);
        if (d.d_bat) cudaFree(d.d_bat);
        if (d.d_ops) cudaFree(d.d_ops);
        if (d.d_lad) cudaFree(d.d_lad);
        if (d.own_events) {
            for (int i = 0; i < 2; ++i) {
                cudaEventDestroy(d.ev_recv[i]);
                cudaEventDestroy(d.ev_upd[i]);
                cudaEventDestroy(d.ev_pack[i]);
            }
            cudaEventDestroy(d.ev_ready);
            cudaEventDestroy(d.ev_done);
        }
        if (d.own_streams) {
            cudaStreamDestroy(d.st);
            cudaStreamDestroy(d.comm);
        }
    }
    delete s;
}

qs_status init_basis_impl(qs_state *s, uint64_t index);

qs_status finish_create(qs_state *s, qs_state **out) {
    qs_status r = init_basis_impl(s, 0);
    if (r != QS_OK) return r;
    *out = s;
    return QS_OK;
}

qs_status create_fail(qs_state *s, qs_status r, qs_state **out) {
    g_create_error = s ? s->err : std::string("qs_create failed");
    destroy_state(s);
    *out = nullptr;
    return r;
}

qs_status common_validate(int n, int P, qs_state **out, int &k) {
    if (!out) {
        g_create_error = "out is NULL";
        return QS_ERR_ARG;
    }
    *out = nullptr;
    k = log2_exact(P);
    if (n < 1 || n > 40) {
        g_create_error = fmt("n_qubits = %d outside [1, 40]", n);
        return QS_ERR_ARG;
    }
    if (k < 0 || P > 8) {
        g_create_error = fmt("shard count %d not in {1, 2, 4, 8}", P);
        return QS_ERR_ARG;
    }
    if (P > 1 && n - k < QS_MIN_LOCAL) {
        g_create_error = fmt("n - log2(P) = %d local qubits < QS_MIN_LOCAL = %d", n - k, QS_MIN_LOCAL);
        return QS_ERR_ARG;
    }
    return QS_OK;
}

// ------------------------------------------------------------------------------------------------
// norm, init
// ------------------------------------------------------------------------------------------------
double host_tree(std::vector<double> v) {  // perfect binary tree over adjacent pairs (size 2^k)
    while (v.size() > 1) {
        std::vector<double> w(v.size() / 2);
        for (size_t i = 0; i < w.size(); ++i) w[i] = v[2 * i] + v[2 * i + 1];
        v.swap(w);
    }
    return v.empty() ? 0.0 : v[0];
}

// Σ|a|² over every shard; partials_ready: each shard's d_norm already holds its partial (init_random)
qs_status norm_total(qs_state *s, double *out, bool partials_ready = false) {
    std::vector<double> parts(s->P, 0.0);
    for (auto &d : s->sh) {
        if (partials_ready) break;
        QS_CUDA(s, cudaSetDevice(d.device));
        QS_TRY(check_launch(s, launch_norm2(d.amps, 1ull << s->m, std::min(norm_leaf_log2(s->n), s->m), d.d_scratch, d.d_norm, d.st, s->num_sms)));
    }
    if (s->mode == MODE_RANK && s->P > 1) {
        Shard &d = s->sh[0];
        QS_NCCL(s, ncclAllGather(d.d_norm, d.d_norm + 1, 1, ncclDouble, d.nccl, d.st));
        QS_CUDA(s, cudaMemcpyAsync(d.h_norm, d.d_norm + 1, 8 * s->P, cudaMemcpyDeviceToHost, d.st));
        QS_CUDA(s, cudaStreamSynchronize(d.st));
        for (int r = 0; r < s->P; ++r) parts[r] = d.h_norm[r];
    } else {
        for (auto &d : s->sh) {
            QS_CUDA(s, cudaSetDevice(d.device));
            QS_CUDA(s, cudaMemcpyAsync(d.h_norm, d.d_norm, 8, cudaMemcpyDeviceToHost, d.st));
        }
        for (auto &d : s->sh) {
            QS_CUDA(s, cudaSetDevice(d.device));
            QS_CUDA(s, cudaStreamSynchronize(d.st));
            parts[d.rank] = d.h_norm[0];
        }
    }
    *out = host_tree(parts);
    return QS_OK;
}

qs_status init_basis_impl(qs_state *s, uint64_t index) {
    const uint64_t shard_amps = 1ull << s->m;
    for (auto &d : s->sh) {
        QS_CUDA(s, cudaSetDevice(d.device));
        QS_CUDA(s, cudaMemsetAsync(d.amps, 0, shard_amps * 16, d.st));
        if ((index >> s->m) == (uint64_t)d.rank)
            QS_TRY(check_launch(s, launch_set_amp(d.amps, index & (shard_amps - 1), 1.0, 0.0, d.st)));
    }
    return QS_OK;
}

// ------------------------------------------------------------------------------------------------
// execution of one (global) op
// ------------------------------------------------------------------------------------------------
qs_status run_local(qs_state *s, Shard &d, const Op &op) {
    QS_CUDA(s, cudaSetDevice(d.device));
    return check_launch(s, launch_op(d.amps, s->m, op, d.st, s->num_sms));
}

Shard *find_rank(qs_state *s, int rank) {
    for (auto &d : s->sh)
        if (d.rank == rank) return &d;
    return nullptr;
}

// One exchange op: every owned shard has an X* action (or SKIP).  Chunked, double-buffered.
qs_status run_exchange(qs_state *s, const Op &op) {
    std::vector<ShardStep> steps(s->sh.size());
    bool via_swap = false;
    int kind = -1;
    for (size_t i = 0; i < s->sh.size(); ++i) {
        steps[i] = localize(op, s->n, s->m, s->sh[i].rank);
        if (steps[i].action == SA_VIA_SWAP) via_swap = true;
        if (steps[i].action != SA_SKIP) kind = steps[i].action;
    }
    if (via_swap) {
        std::vector<Op> seq = decompose_via_swap(op, s->m);
        if (seq.empty()) return set_err(s, QS_ERR_UNSUPPORTED, "no free local qubit for swap-to-local");
        for (const Op &o : seq) {
            bool exch = false;
            for (auto &d : s->sh) {
                ShardStep st = localize(o, s->n, s->m, d.rank);
                if (st.action == SA_LOCAL)
                    QS_TRY(run_local(s, d, st.local));
                else if (st.action != SA_SKIP)
                    exch = true;
            }
            if (exch) QS_TRY(run_exchange(s, o));
        }
        return QS_OK;
    }
    for (size_t i = 0; i < s->sh.size(); ++i)
        if (steps[i].action == SA_LOCAL) QS_TRY(run_local(s, s->sh[i], steps[i].local));
    if (kind < SA_XPAIR) return QS_OK;
    ++s->last_exchanges;

    const uint64_t shard_amps = 1ull << s->m;
    // packed exchanges move half the shard: SWAP(local, global) sends the half that changes rank;
    // a local-control / global-target gate sends only the control-1 half
    int ctrl_l = -1;
    for (size_t i = 0; i < s->sh.size(); ++i)
        if (steps[i].action == SA_XPAIR) ctrl_l = steps[i].ctrl_local;
    const bool packed = kind == SA_XSWAP_LG || (kind == SA_XPAIR && ctrl_l >= 0);
    const uint64_t total = packed ? shard_amps / 2 : shard_amps;  // elements exchanged
    const uint64_t C = std::min<uint64_t>(s->chunk_amps(), total);
    const uint64_t nch = total / C;
    const size_t cbytes = (size_t)C * 16;

    // ---------------- peer memory: one fused kernel per rank loads/stores the partner's shard -------
    if (s->p2p && s->p2p_ok && s->mode == MODE_RANK) {
        Shard &d = s->sh[0];
        const ShardStep &st = steps[0];
        if (st.action == SA_SKIP) return QS_OK;
        QS_CUDA(s, cudaSetDevice(d.device));
        const int p = st.partner;
        const unsigned long long k = ++d.seq[p];
        QS_TRY(check_launch(s, launch_flag_barrier(d.flags, d.peer_flags[p], d.rank, p, 2 * k - 1, d.st)));
        const int lt = launch_p2p_exchange(st.action, d.amps, reinterpret_cast<double2 *>(d.peer_base[p] + s->guard),
                                           s->m, st.bit, st.ctrl_local, st.l, d.rank < p, st.local.m, d.st, s->num_sms);
        if (lt < 0) return set_err(s, QS_ERR_UNSUPPORTED, "peer-memory exchange: unknown action");
        QS_TRY(check_launch(s, lt));
        QS_TRY(check_launch(s, launch_flag_barrier(d.flags, d.peer_flags[p], d.rank, p, 2 * k, d.st)));
        return QS_OK;
    }
    if (s->p2p && s->p2p_ok && s->mode != MODE_RANK) {
        const bool multidev = s->mode == MODE_MULTIDEV;
        if (multidev)  // the partner's earlier work on its shard must be complete before we touch it
            for (size_t i = 0; i < s->sh.size(); ++i) {
                if (steps[i].action == SA_SKIP) continue;
                QS_CUDA(s, cudaSetDevice(s->sh[i].device));
                QS_CUDA(s, cudaEventRecord(s->sh[i].ev_ready, s->sh[i].st));
            }
        for (size_t i = 0; i < s->sh.size(); ++i) {
            const ShardStep &st = steps[i];
            if (st.action == SA_SKIP) continue;
            Shard &d = s->sh[i];
            Shard *p = find_rank(s, st.partner);
            QS_CUDA(s, cudaSetDevice(d.device));
            if (multidev) QS_CUDA(s, cudaStreamWaitEvent(d.st, p->ev_ready, 0));
            const int lt = launch_p2p_exchange(st.action, d.amps, p->amps, s->m, st.bit, st.ctrl_local, st.l,
                                               d.rank < p->rank, st.local.m, d.st, s->num_sms);
            if (lt < 0) return set_err(s, QS_ERR_UNSUPPORTED, "peer-memory exchange: unknown action");
            QS_TRY(check_launch(s, lt));
            if (multidev) QS_CUDA(s, cudaEventRecord(d.ev_done, d.st));
        }
        if (multidev)  // ... and must not run on until our stores into its shard are complete
            for (size_t i = 0; i < s->sh.size(); ++i) {
                if (steps[i].action == SA_SKIP) continue;
                Shard *p = find_rank(s, steps[i].partner);
                QS_CUDA(s, cudaSetDevice(s->sh[i].device));
                QS_CUDA(s, cudaStreamWaitEvent(s->sh[i].st, p->ev_done, 0));
            }
        return QS_OK;
    }

    // ---------------- buffered exchange: the comm stream moves chunk c+1 while compute updates c ----
    // One pipeline for every process model; only the transport of a chunk differs:
    //   NCCL (multi-device, one process per GPU): ncclSend(own chunk) + ncclRecv(partner's) in a group;
    //   virtual shards: device copies of the partner's chunk on the comm stream (vtransport 0), or
    //   ncclSend/ncclRecv to self on a one-rank communicator of this device (vtransport 1) — the same
    //   NCCL calls, events and double buffers as the multi-GPU path, runnable on one GPU.
    // Ordering per chunk c (buffer c&1): the comm stream waits for the pack of c (packed exchanges)
    // and for the update of chunk c-2, which read the same receive buffer; the compute stream waits
    // for the receive of c.  Virtual shards share one compute and one comm stream (and their events):
    // an event recorded after the last shard's work covers every shard's.
    auto pack_params = [&](const ShardStep &st, int &pl, int &pv) {
        pl = kind == SA_XSWAP_LG ? st.l : ctrl_l;
        pv = kind == SA_XSWAP_LG ? 1 - st.bit : 1;
    };
    const bool virt = s->mode == MODE_VIRTUAL;
    for (size_t i = 0; i < s->sh.size(); ++i) {
        Shard &d = s->sh[i];
        if (steps[i].action == SA_SKIP) continue;
        QS_CUDA(s, cudaSetDevice(d.device));
        QS_CUDA(s, cudaEventRecord(d.ev_ready, d.st));
        QS_CUDA(s, cudaStreamWaitEvent(d.comm, d.ev_ready, 0));
        if (packed)
            for (uint64_t c = 0; c < std::min<uint64_t>(2, nch); ++c) {
                int pl, pv;
                pack_params(steps[i], pl, pv);
                QS_TRY(check_launch(s, launch_pack(d.amps, d.sbuf[c & 1], pl, pv, c * C, C, d.st, s->num_sms)));
                QS_CUDA(s, cudaEventRecord(d.ev_pack[c & 1], d.st));
            }
    }
    for (uint64_t c = 0; c < nch; ++c) {
        const uint64_t off = c * C;
        const int bsel = (int)(c & 1);
        for (size_t i = 0; i < s->sh.size(); ++i) {
            Shard &d = s->sh[i];
            if (steps[i].action == SA_SKIP) continue;
            QS_CUDA(s, cudaSetDevice(d.device));
            if (packed) QS_CUDA(s, cudaStreamWaitEvent(d.comm, d.ev_pack[bsel], 0));
            if (c >= 2) QS_CUDA(s, cudaStreamWaitEvent(d.comm, d.ev_upd[bsel], 0));
        }
        if (virt && s->vtransport == 0) {
            for (size_t i = 0; i < s->sh.size(); ++i) {
                if (steps[i].action == SA_SKIP) continue;
                Shard *p = find_rank(s, steps[i].partner);
                const void *src = packed ? (const void *)p->sbuf[bsel] : (const void *)(p->amps + off);
                QS_CUDA(s, cudaMemcpyAsync(s->sh[i].rbuf[bsel], src, cbytes, cudaMemcpyDeviceToDevice, s->sh[i].comm));
            }
        } else if (virt) {
            // one-rank communicator: a send and a receive to self are matched in posting order, so
            // posting (partner's chunk, our buffer) pairs moves every partner's chunk into place
            Shard &d0 = s->sh[0];
            for (size_t i = 0; i < s->sh.size(); ++i) {
                if (steps[i].action == SA_SKIP) continue;
                Shard *p = find_rank(s, steps[i].partner);
                const void *src = packed ? (const void *)p->sbuf[bsel] : (const void *)(p->amps + off);
                QS_NCCL(s, ncclGroupStart());
                ncclResult_t r1 = ncclSend(src, 2 * C, ncclDouble, 0, d0.nccl, d0.comm);
                ncclResult_t r2 = ncclRecv(s->sh[i].rbuf[bsel], 2 * C, ncclDouble, 0, d0.nccl, d0.comm);
                QS_NCCL(s, ncclGroupEnd());
                if (r1 != ncclSuccess || r2 != ncclSuccess)
                    return set_err(s, QS_ERR_NCCL, fmt("ncclSend/ncclRecv (self) failed: %s",
                                                       ncclGetErrorString(r1 != ncclSuccess ? r1 : r2)));
            }
        } else {
            QS_NCCL(s, ncclGroupStart());
            for (size_t i = 0; i < s->sh.size(); ++i) {
                Shard &d = s->sh[i];
                if (steps[i].action == SA_SKIP) continue;
                const void *src = packed ? (const void *)d.sbuf[bsel] : (const void *)(d.amps + off);
                ncclResult_t r1 = ncclSend(src, 2 * C, ncclDouble, steps[i].partner, d.nccl, d.comm);
                ncclResult_t r2 = ncclRecv(d.rbuf[bsel], 2 * C, ncclDouble, steps[i].partner, d.nccl, d.comm);
                if (r1 != ncclSuccess || r2 != ncclSuccess) {
                    ncclGroupEnd();
                    return set_err(s, QS_ERR_NCCL, fmt("ncclSend/ncclRecv failed: %s", ncclGetErrorString(r1 != ncclSuccess ? r1 : r2)));
                }
            }
            QS_NCCL(s, ncclGroupEnd());
        }
        for (size_t i = 0; i < s->sh.size(); ++i) {
            Shard &d = s->sh[i];
            if (steps[i].action == SA_SKIP) continue;
            QS_CUDA(s, cudaSetDevice(d.device));
            QS_CUDA(s, cudaEventRecord(d.ev_recv[bsel], d.comm));
            QS_CUDA(s, cudaStreamWaitEvent(d.st, d.ev_recv[bsel], 0));
        }
        for (size_t i = 0; i < s->sh.size(); ++i) {
            Shard &d = s->sh[i];
            const ShardStep &st = steps[i];
            if (st.action == SA_SKIP) continue;
            QS_CUDA(s, cudaSetDevice(d.device));
            if (st.action == SA_XPAIR && packed)
                QS_TRY(check_launch(s, launch_xpair_packed(d.amps, d.rbuf[bsel], ctrl_l, off, C, st.bit, st.local.m, d.st,
                                                           s->num_sms)));
            else if (st.action == SA_XPAIR)
                QS_TRY(check_launch(s, launch_xpair_update(d.amps + off, d.rbuf[bsel], C, off, st.ctrl_local, st.bit,
                                                           st.local.m, d.st, s->num_sms)));
            else if (st.action == SA_XSWAP_LG)
                QS_TRY(check_launch(s, launch_unpack(d.amps, d.rbuf[bsel], st.l, 1 - st.bit, off, C, d.st, s->num_sms)));
            else
                QS_CUDA(s, cudaMemcpyAsync(d.amps + off, d.rbuf[bsel], cbytes, cudaMemcpyDeviceToDevice, d.st));
        }
        // after every shard's update of chunk c (virtual shards: their sends of chunk c+2 must not
        // overwrite a pack buffer before the partner's receive of chunk c read it — ev_recv above)
        for (size_t i = 0; i < s->sh.size(); ++i) {
            Shard &d = s->sh[i];
            const ShardStep &st = steps[i];
            if (st.action == SA_SKIP) continue;
            QS_CUDA(s, cudaSetDevice(d.device));
            QS_CUDA(s, cudaEventRecord(d.ev_upd[bsel], d.st));
            if (packed && c + 2 < nch) {
                int pl, pv;
                pack_params(st, pl, pv);
                QS_TRY(check_launch(s, launch_pack(d.amps, d.sbuf[bsel], pl, pv, (c + 2) * C, C, d.st, s->num_sms)));
                QS_CUDA(s, cudaEventRecord(d.ev_pack[bsel], d.st));
            }
        }
    }
    return QS_OK;
}

// a non-tile op: local on every shard, or an exchange
qs_status run_op(qs_state *s, const Op &op) {
    bool exch = false;
    std::vector<ShardStep> steps(s->sh.size());
    for (size_t i = 0; i < s->sh.size(); ++i) {
        steps[i] = localize(op, s->n, s->m, s->sh[i].rank);
        if (steps[i].action >= SA_XPAIR) exch = true;
    }
    if (exch) return run_exchange(s, op);
    for (size_t i = 0; i < s->sh.size(); ++i) {
        if (steps[i].action == SA_LOCAL) {
            QS_TRY(run_local(s, s->sh[i], steps[i].local));
            ++s->last_passes;
        }
    }
    return QS_OK;
}

qs_status gates_to_ops(qs_state *s, const qs_gate *gates, size_t G, std::vector<Op> &ops) {
    ops.resize(G);
    for (size_t g = 0; g < G; ++g) {
        std::string msg;
        if (gates[g].flags != 0) return set_err(s, QS_ERR_ARG, fmt("gate %zu: flags must be 0", g));
        if (!classify(s->n, gates[g].kind, gates[g].q0, gates[g].q1, gates[g].m, s->check_unitary, ops[g], msg))
            return set_err(s, QS_ERR_ARG, fmt("gate %zu: %s", g, msg.c_str()));
    }
    return QS_OK;
}

// Everything run_ops derives from an op list on the host — the executed op list (after remapping and
// scalar factoring), the pass plan, every shard's tile descriptors / batches / op records / ladder records
// and the pass kernels' sources — cached per handle by a hash of the op list and the options, so a
// repeated circuit (the benchmark, parameter sweeps) only uploads the descriptors and launches: the host
// work between the caller's enqueue and the first pass (the multi-trial scheduler, the batch partition
// search, source generation) is paid once.
struct Prepared {
    std::vector<Op> ops;
    std::vector<Pass> plan;
    std::vector<std::vector<TileDesc>> descs;
    std::vector<std::vector<TileBatch>> bats;
    std::vector<std::vector<TileOp>> tops;
    std::vector<std::vector<TileLadder>> lads;
    std::vector<std::vector<size_t>> lad_at;
    std::vector<std::vector<int>> pass_desc;
    std::vector<std::vector<std::string>> spec, fam;  // per shard and tile pass: specialised / family source
    std::vector<std::vector<char>> use_fam;
    bool jit_ok = false;
    std::vector<std::string> deferred;  // background compilations to start once the passes are queued
    // CUDA graph of the whole run (single-shard handles, option "graph"): the kernel launches and counter
    // resets captured once and replayed, with the descriptors resident in buffers this entry owns
    int g_device = -1;
    TileDesc *g_desc = nullptr;
    TileBatch *g_bat = nullptr;
    TileOp *g_ops = nullptr;
    TileLadder *g_lad = nullptr;
    cudaGraphExec_t gexec = nullptr;
    std::vector<char> g_use_fam;  // the kernel choice the graph was captured with
    uint64_t g_launches = 0, g_passes = 0;
    void drop_graph() {
        if (gexec) cudaGraphExecDestroy(gexec);
        gexec = nullptr;
    }
    ~Prepared() {
        if (g_device >= 0) {
            cudaSetDevice(g_device);
            drop_graph();
            cudaFree(g_desc);
            cudaFree(g_bat);
            cudaFree(g_ops);
            cudaFree(g_lad);
        }
    }
};

qs_status prepare_ops(qs_state *s, const std::vector<Op> &ops_in, Prepared &P) {
    // sharded: global-qubit remapping when it moves fewer bytes than exchanging gate by gate
    std::vector<Op> remapped;
    if (s->remap && s->m < s->n && ops_in.size() > 1) {
        remapped = remap_global(ops_in, s->n, s->m);
        if (exchange_cost(remapped, s->m) >= exchange_cost(ops_in, s->m)) remapped.clear();
    }
    const std::vector<Op> &ops0 = remapped.empty() ? ops_in : remapped;
    // circuits: scalar factoring of monomial 1q gates (one deferred global factor)
    std::vector<Op> factored;
    if (s->factor && s->fuse && ops0.size() > 1) factored = factor_scalars(ops0);
    P.ops = factored.empty() ? ops0 : factored;
    const std::vector<Op> &ops = P.ops;
    PlanConfig cfg;
    cfg.b = s->tile_b;
    cfg.L0 = s->tile_low;
    cfg.fuse = s->fuse;
    cfg.perm_low = s->perm_low;
    cfg.perm_fuse = s->perm_fuse;
    cfg.reorder = s->reorder;
    if (s->tile_low_auto && cfg.fuse && cfg.L0 > 2) {
        // one low qubit fewer in every tile frees a tile slot (runs of 2^(L0-1) amplitudes instead
        // of 2^L0): taken when it saves at least one tile pass in ten.  Compared without fused
        // permutations: a fused pass pair-gathers short runs and costs more than a plain pass
        // (QFT(32) measured: tile_low 3 + fused reversal 0.154 s vs tile_low 4 + k_perm 0.150 s).
        // The candidate plans are independent: scheduled on concurrent host threads.
        PlanConfig c1 = cfg, c2 = cfg, c3 = cfg;
        c1.perm_fuse = c2.perm_fuse = false;
        c2.L0 = c3.L0 = cfg.L0 - 1;
        std::vector<Pass> p0, p1, p2, p3;
        std::thread t1([&]() { p1 = cfg.perm_fuse ? plan_passes(ops, s->n, s->m, c1) : std::vector<Pass>(); });
        std::thread t2([&]() { p2 = plan_passes(ops, s->n, s->m, c2); });
        std::thread t3([&]() { p3 = cfg.perm_fuse ? plan_passes(ops, s->n, s->m, c3) : std::vector<Pass>(); });
        p0 = plan_passes(ops, s->n, s->m, cfg);
        t1.join();
        t2.join();
        t3.join();
        if (!cfg.perm_fuse) {
            p1 = p0;  // c1 == cfg
            p3 = p2;  // c3 == c2
        }
        auto tiles = [](const std::vector<Pass> &p) {
            size_t k = 0;
            for (const Pass &x : p) k += x.type == 1 || x.type == 0 || x.type == 3;
            return k;
        };
        const bool low3 = 10 * tiles(p2) <= 9 * tiles(p1);
        P.plan = low3 ? p3 : p0;
        if (low3) cfg = c3;
    } else {
        P.plan = plan_passes(ops, s->n, s->m, cfg);
    }
    if (s->perm_hoist) {
        std::vector<Op> o2;
        std::vector<Pass> p2;
        if (hoist_permutation(P.ops, P.plan, s->m, cfg, o2, p2)) {
            P.ops.swap(o2);
            P.plan.swap(p2);
        }
    }
    const std::vector<Pass> &plan = P.plan;
    const size_t S = s->sh.size();
    P.descs.assign(S, {});
    P.bats.assign(S, {});
    P.tops.assign(S, {});
    P.lads.assign(S, {});
    P.lad_at.assign(S, {});
    P.pass_desc.assign(S, std::vector<int>(plan.size(), -1));
    for (size_t i = 0; i < S; ++i)
        for (size_t p = 0; p < plan.size(); ++p) {
            if (plan[p].type != 1) continue;
            std::vector<Op> local;
            for (int oi : plan[p].ops) {
                ShardStep st = localize(ops[oi], s->n, s->m, s->sh[i].rank);
                if (st.action == SA_LOCAL) local.push_back(st.local);
            }
            if (local.empty()) continue;
            TileDesc desc;
            P.lad_at[i].push_back(P.lads[i].size());
            make_tile_pass(plan[p].tile_q.data(), (int)plan[p].tile_q.size(), plan[p].L, s->m, local.data(),
                           (int)local.size(), desc, P.bats[i], P.tops[i], P.lads[i], s->ladder_min, s->reorder);
            if (!plan[p].perm.empty() &&
                !set_tile_perm(desc, plan[p].tile_q.data(), (int)plan[p].tile_q.size(), plan[p].perm.data(), s->m))
                return set_err(s, QS_ERR_UNSUPPORTED, "fused permutation does not map the tile onto itself");
            P.pass_desc[i][p] = (int)P.descs[i].size();
            P.descs[i].push_back(desc);
        }
    // JIT: one straight-line kernel per distinct pass structure, compiled in parallel and cached
    P.spec.assign(S, {});
    P.fam.assign(S, {});
    P.use_fam.assign(S, {});
    if (s->jit) {
        std::vector<std::string> spec, fam;
        for (size_t i = 0; i < S; ++i)
            for (const TileDesc &d : P.descs[i]) {
                spec.push_back(jit_tile_source(d, P.bats[i].data(), P.tops[i].data(), tile_regs(), false));
                fam.push_back(s->jit_family ? jit_tile_source(d, P.bats[i].data(), P.tops[i].data(), tile_regs(), true)
                                            : spec.back());
            }
        std::string err;
        std::vector<int> use_fam;
        P.jit_ok = jit_tile_prepare_pair(spec, fam, s->jit_family, use_fam, err, s->jit_async, &P.deferred);
        if (!P.jit_ok) s->jit_error = err;
        size_t k = 0;
        for (size_t i = 0; i < S; ++i)
            for (size_t j = 0; j < P.descs[i].size(); ++j, ++k) {
                P.spec[i].push_back(spec[k]);
                P.fam[i].push_back(fam[k]);
                P.use_fam[i].push_back((char)use_fam[k]);
            }
    }
    return QS_OK;
}

qs_status run_ops(qs_state *s, const std::vector<Op> &ops_in) {
    s->last_passes = 0;
    s->last_exchanges = 0;
    uint64_t key = 1469598103934665603ull;
    auto mix = [&](const void *p, size_t nb) {
        const unsigned char *c = static_cast<const unsigned char *>(p);
        for (size_t i = 0; i < nb; ++i) key = (key ^ c[i]) * 1099511628211ull;
    };
    for (const Op &op : ops_in) {
        mix(&op.kind, 16);  // kind, q0, q1, touch
        mix(&op.form, 4);
        mix(op.m, sizeof op.m);
    }
    const int32_t opt[16] = {s->n, s->m, s->tile_b, s->tile_low, (int)s->fuse, s->perm_low, (int)s->reorder,
                             (int)s->tile_low_auto, (int)s->perm_fuse, (int)s->remap, (int)s->factor, s->ladder_min,
                             s->jit_family, (int)s->jit, (int)s->jit_async, (int)s->perm_hoist};
    mix(opt, sizeof opt);
    std::shared_ptr<Prepared> hit;
    auto it = s->prep_cache.find(key);
    const bool cached = it != s->prep_cache.end();
    if (cached) {
        hit = it->second;
        // the hybrid JIT: passes that ran a family kernel switch to their specialised kernel once it is
        // compiled (background process, jit_tile.cu); passes whose compile failed retry
        if (s->jit) {
            bool retry = !hit->jit_ok;
            for (size_t i = 0; i < hit->use_fam.size() && !retry; ++i)
                for (size_t j = 0; j < hit->use_fam[i].size(); ++j)
                    if (hit->use_fam[i][j] && s->jit_family == 1) retry = true;
            if (retry) {
                std::vector<std::string> spec, fam;
                for (size_t i = 0; i < hit->spec.size(); ++i)
                    for (size_t j = 0; j < hit->spec[i].size(); ++j) {
                        spec.push_back(hit->spec[i][j]);
                        fam.push_back(hit->fam[i][j]);
                    }
                std::string err;
                std::vector<int> use_fam;
                hit->jit_ok = jit_tile_prepare_pair(spec, fam, s->jit_family, use_fam, err, s->jit_async, &hit->deferred);
                if (!hit->jit_ok) s->jit_error = err;
                size_t k = 0;
                for (size_t i = 0; i < hit->spec.size(); ++i)
                    for (size_t j = 0; j < hit->spec[i].size(); ++j, ++k) hit->use_fam[i][j] = (char)use_fam[k];
            }
        }
    } else {
        hit = std::make_shared<Prepared>();
        QS_TRY(prepare_ops(s, ops_in, *hit));
        if (s->prep_cache.size() >= 16) s->prep_cache.clear();  // bounded host memory (~1-2 MB per entry)
        s->prep_cache[key] = hit;
    }
    Prepared &P = *hit;
    const std::vector<Op> &ops = P.ops;
    const std::vector<Pass> &plan = P.plan;

    // the launch sequence of the plan, reading the descriptors at ddesc/dbat/dops (per shard)
    auto launch_all = [&](const std::vector<TileDesc *> &ddesc, const std::vector<TileBatch *> &dbat,
                          const std::vector<TileOp *> &dops) -> qs_status {
        for (size_t p = 0; p < plan.size(); ++p) {
            const Pass &ps = plan[p];
            if (ps.type == 1) {
                bool any = false;
                for (size_t i = 0; i < s->sh.size(); ++i) {
                    int di = P.pass_desc[i][p];
                    if (di < 0 && ps.perm.empty()) continue;
                    Shard &d = s->sh[i];
                    QS_CUDA(s, cudaSetDevice(d.device));
                    int lt = -1;
                    if (di >= 0 && P.jit_ok && s->jit)
                        lt = launch_tile_jit(P.use_fam[i][di] ? P.fam[i][di] : P.spec[i][di], d.amps, s->m, P.descs[i][di],
                                             ddesc[i] + di, dbat[i], dops[i], d.st, s->num_sms);
                    bool permuted = lt >= 0;  // the JIT kernel of a perm pass stores permuted (tile_kernel PAIR)
                    if (lt < 0 && di >= 0) {
                        lt = launch_tile(d.amps, s->m, P.descs[i][di], ddesc[i] + di, dbat[i], dops[i], d.st, s->num_sms);
                        if (lt < 0) return set_err(s, QS_ERR_UNSUPPORTED, "tile pass with more than 27 outside qubits");
                    }
                    if (lt >= 0) QS_TRY(check_launch(s, lt));
                    if (!ps.perm.empty() && !permuted) {  // interpreter / no local op here: the permutation pass
                        lt = launch_perm(d.amps, s->m, ps.perm.data(), s->perm_low, d.st, s->num_sms);
                        if (lt < 0) return set_err(s, QS_ERR_UNSUPPORTED, "qubit permutation pass not realisable");
                        QS_TRY(check_launch(s, lt));
                    }
                    any = true;
                }
                if (any) ++s->last_passes;
            } else if (ps.type == 3) {
                for (auto &d : s->sh) {
                    QS_CUDA(s, cudaSetDevice(d.device));
                    const int lt = launch_perm(d.amps, s->m, ps.perm.data(), s->perm_low, d.st, s->num_sms);
                    if (lt < 0) return set_err(s, QS_ERR_UNSUPPORTED, "qubit permutation pass not realisable");
                    QS_TRY(check_launch(s, lt));
                }
                ++s->last_passes;
            } else {
                QS_TRY(run_op(s, ops[ps.ops[0]]));
            }
        }
        return QS_OK;
    };
    auto spawn_deferred = [&]() {
        // background compilations (hybrid JIT) start after the passes are queued: spawning the compiler
        // processes is not on the path to the first kernel
        if (!P.deferred.empty()) {
            jit_tile_background(P.deferred);
            P.deferred.clear();
        }
    };

    // CUDA graph (single-shard handles, a repeated circuit whose pass kernels are compiled, no exchange
    // steps): the first repeat captures the run — counter resets and kernel launches reading descriptors
    // that stay resident in buffers the cache entry owns — and every later one replays it with one
    // cudaGraphLaunch; a change of the hybrid JIT's kernel choice recaptures.  Same kernels, same
    // arguments: bitwise the launched run.
    bool no_exchange = true;
    for (const Pass &ps : plan) no_exchange = no_exchange && ps.type != 2;
    if (s->graph && cached && s->sh.size() == 1 && s->mode == MODE_SINGLE && s->jit && P.jit_ok &&
        no_exchange) {
        Shard &d = s->sh[0];
        QS_CUDA(s, cudaSetDevice(d.device));
        if (P.gexec && P.g_use_fam == P.use_fam[0]) {
            QS_CUDA(s, cudaGraphLaunch(P.gexec, d.st));
            s->launches += P.g_launches;
            s->last_passes = P.g_passes;
            spawn_deferred();
            return QS_OK;
        }
        P.drop_graph();
        if (P.g_device < 0 && !P.descs[0].empty()) {  // the entry's resident descriptors, uploaded once
            P.g_device = d.device;
            std::vector<TileDesc> &descs = P.descs[0];
            QS_CUDA(s, cudaMalloc(&P.g_desc, descs.size() * sizeof(TileDesc)));
            QS_CUDA(s, cudaMalloc(&P.g_bat, std::max<size_t>(1, P.bats[0].size()) * sizeof(TileBatch)));
            QS_CUDA(s, cudaMalloc(&P.g_ops, std::max<size_t>(1, P.tops[0].size()) * sizeof(TileOp)));
            QS_CUDA(s, cudaMalloc(&P.g_lad, std::max<size_t>(1, P.lads[0].size()) * sizeof(TileLadder)));
            std::vector<TileDesc> dd = descs;
            for (size_t k = 0; k < dd.size(); ++k) dd[k].lads = P.g_lad + P.lad_at[0][k];
            QS_CUDA(s, cudaMemcpyAsync(P.g_desc, dd.data(), dd.size() * sizeof(TileDesc), cudaMemcpyHostToDevice, d.st));
            if (!P.bats[0].empty())
                QS_CUDA(s, cudaMemcpyAsync(P.g_bat, P.bats[0].data(), P.bats[0].size() * sizeof(TileBatch), cudaMemcpyHostToDevice, d.st));
            if (!P.tops[0].empty())
                QS_CUDA(s, cudaMemcpyAsync(P.g_ops, P.tops[0].data(), P.tops[0].size() * sizeof(TileOp), cudaMemcpyHostToDevice, d.st));
            if (!P.lads[0].empty())
                QS_CUDA(s, cudaMemcpyAsync(P.g_lad, P.lads[0].data(), P.lads[0].size() * sizeof(TileLadder), cudaMemcpyHostToDevice, d.st));
            QS_CUDA(s, cudaStreamSynchronize(d.st));  // pageable sources: staged before capture begins
        }
        const uint64_t l0 = s->launches, p0 = s->last_passes;
        cudaGraph_t g = nullptr;
        bool captured = cudaStreamBeginCapture(d.st, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
        qs_status r = QS_OK;
        if (captured) {
            r = launch_all({P.g_desc}, {P.g_bat}, {P.g_ops});
            captured = cudaStreamEndCapture(d.st, &g) == cudaSuccess && r == QS_OK && g &&
                       cudaGraphInstantiate(&P.gexec, g, 0) == cudaSuccess;
            if (g) cudaGraphDestroy(g);
        }
        if (captured) {
            P.g_use_fam = P.use_fam[0];
            P.g_launches = s->launches - l0;
            P.g_passes = s->last_passes - p0;
            QS_CUDA(s, cudaGraphLaunch(P.gexec, d.st));
            spawn_deferred();
            return QS_OK;
        }
        // capture unavailable: clear its error state and run the plan by direct launches below
        if (r != QS_OK) return r;
        P.gexec = nullptr;
        cudaGetLastError();
        s->launches = l0;
        s->last_passes = p0;
    }

    // per-shard tile descriptors, uploaded once per run (pageable sources: staged before the call returns)
    std::vector<TileDesc *> ddesc(s->sh.size());
    std::vector<TileBatch *> dbat(s->sh.size());
    std::vector<TileOp *> dops(s->sh.size());
    for (size_t i = 0; i < s->sh.size(); ++i) {
        Shard &d = s->sh[i];
        std::vector<TileDesc> &descs = P.descs[i];
        if (descs.empty()) continue;
        const std::vector<TileBatch> &bats = P.bats[i];
        const std::vector<TileOp> &tops = P.tops[i];
        const std::vector<TileLadder> &lads = P.lads[i];
        QS_CUDA(s, cudaSetDevice(d.device));
        if (lads.size() > d.lad_cap) {
            QS_CUDA(s, cudaStreamSynchronize(d.st));
            if (d.d_lad) cudaFree(d.d_lad);
            d.lad_cap = std::max<size_t>(lads.size() * 2, 64);
            QS_CUDA(s, cudaMalloc(&d.d_lad, d.lad_cap * sizeof(TileLadder)));
        }
        for (size_t k = 0; k < descs.size(); ++k) descs[k].lads = d.d_lad + P.lad_at[i][k];
        if (!lads.empty())
            QS_CUDA(s, cudaMemcpyAsync(d.d_lad, lads.data(), lads.size() * sizeof(TileLadder), cudaMemcpyHostToDevice, d.st));
        if (descs.size() > d.desc_cap || bats.size() > d.bat_cap || tops.size() > d.ops_cap) {
            QS_CUDA(s, cudaStreamSynchronize(d.st));
            if (d.d_desc) cudaFree(d.d_desc);
            if (d.d_bat) cudaFree(d.d_bat);
            if (d.d_ops) cudaFree(d.d_ops);
            d.desc_cap = std::max<size_t>(descs.size() * 2, 64);
            d.bat_cap = std::max<size_t>(bats.size() * 2, 256);
            d.ops_cap = std::max<size_t>(tops.size() * 2, 1024);
            QS_CUDA(s, cudaMalloc(&d.d_desc, d.desc_cap * sizeof(TileDesc)));
            QS_CUDA(s, cudaMalloc(&d.d_bat, d.bat_cap * sizeof(TileBatch)));
            QS_CUDA(s, cudaMalloc(&d.d_ops, d.ops_cap * sizeof(TileOp)));
        }
        QS_CUDA(s, cudaMemcpyAsync(d.d_desc, descs.data(), descs.size() * sizeof(TileDesc), cudaMemcpyHostToDevice, d.st));
        QS_CUDA(s, cudaMemcpyAsync(d.d_bat, bats.data(), bats.size() * sizeof(TileBatch), cudaMemcpyHostToDevice, d.st));
        QS_CUDA(s, cudaMemcpyAsync(d.d_ops, tops.data(), tops.size() * sizeof(TileOp), cudaMemcpyHostToDevice, d.st));
    }
    for (size_t i = 0; i < s->sh.size(); ++i) {
        ddesc[i] = s->sh[i].d_desc;
        dbat[i] = s->sh[i].d_bat;
        dops[i] = s->sh[i].d_ops;
    }
    QS_TRY(launch_all(ddesc, dbat, dops));
    spawn_deferred();
    return QS_OK;
}

qs_status run_gates(qs_state *s, const qs_gate *gates, size_t G) {
    std::vector<Op> ops;
    QS_TRY(gates_to_ops(s, gates, G, ops));
    return run_ops(s, ops);
}

qs_status range_check(qs_state *s, uint64_t start, uint64_t count, const void *buf) {
    if (!buf && count) return set_err(s, QS_ERR_ARG, "NULL buffer");
    const uint64_t N = 1ull << s->n;
    if (start > N || count > N - start) return set_err(s, QS_ERR_RANGE, fmt("range [%llu, +%llu) outside [0, 2^%d)",
                                                                          (unsigned long long)start, (unsigned long long)count, s->n));
    if (s->mode == MODE_RANK && count) {
        const uint64_t lo = (uint64_t)s->sh[0].rank << s->m, hi = lo + (1ull << s->m);
        if (start < lo || start + count > hi) return set_err(s, QS_ERR_RANGE, "range outside this rank's shard");
    }
    return QS_OK;
}

qs_status copy_amps(qs_state *s, uint64_t start, uint64_t count, double *host, bool to_host, bool sync = true) {
    const uint64_t shard_amps = 1ull << s->m;
    for (auto &d : s->sh) {
        const uint64_t lo = (uint64_t)d.rank * shard_amps, hi = lo + shard_amps;
        const uint64_t a = std::max(lo, start), b = std::min(hi, start + count);
        if (a >= b) continue;
        QS_CUDA(s, cudaSetDevice(d.device));
        double *h = host + 2 * (a - start);
        double2 *dv = d.amps + (a - lo);
        if (to_host)
            QS_CUDA(s, cudaMemcpyAsync(h, dv, (b - a) * 16, cudaMemcpyDeviceToHost, d.st));
        else
            QS_CUDA(s, cudaMemcpyAsync(dv, h, (b - a) * 16, cudaMemcpyHostToDevice, d.st));
    }
    if (!sync) return QS_OK;
    for (auto &d : s->sh) {
        QS_CUDA(s, cudaSetDevice(d.device));
        QS_CUDA(s, cudaStreamSynchronize(d.st));
    }
    return QS_OK;
}

}  // namespace

// =================================================================================================
// C ABI
// =================================================================================================
extern "C" {

// One-process-per-GPU peer mapping (opt-in, QS_P2P_RANK=1): every rank exports its shard allocation
// and a flag array with CUDA IPC, the handles travel by ncclAllGather, every rank maps all others; the
// fused peer-memory kernels are used only if every rank succeeded (ncclAllReduce min).
qs_status setup_rank_peers(qs_state *s) {
    Shard &d = s->sh[0];
    const int world = s->P;
    struct Rec {
        cudaIpcMemHandle_t mem, flags;
        int32_t ok, pad[3];
    };
    QS_CUDA(s, cudaMalloc(&d.flags, 64 * sizeof(unsigned long long)));
    QS_CUDA(s, cudaMemset(d.flags, 0, 64 * sizeof(unsigned long long)));
    Rec mine;
    std::memset(&mine, 0, sizeof mine);
    mine.ok = cudaIpcGetMemHandle(&mine.mem, d.alloc_base) == cudaSuccess &&
              cudaIpcGetMemHandle(&mine.flags, d.flags) == cudaSuccess;
    cudaGetLastError();
    char *dbuf = nullptr;
    QS_CUDA(s, cudaMalloc(&dbuf, sizeof(Rec) * (world + 1)));
    // uploads on d.st (pageable source: staged before the call returns), ordered before the collectives
    QS_CUDA(s, cudaMemcpyAsync(dbuf, &mine, sizeof(Rec), cudaMemcpyHostToDevice, d.st));
    QS_NCCL(s, ncclAllGather(dbuf, dbuf + sizeof(Rec), sizeof(Rec), ncclUint8, d.nccl, d.st));
    std::vector<Rec> all(world);
    QS_CUDA(s, cudaStreamSynchronize(d.st));
    QS_CUDA(s, cudaMemcpyAsync(all.data(), dbuf + sizeof(Rec), sizeof(Rec) * world, cudaMemcpyDeviceToHost, d.st));
    QS_CUDA(s, cudaStreamSynchronize(d.st));
    d.peer_base.assign(world, nullptr);
    d.peer_flags.assign(world, nullptr);
    d.seq.assign(world, 0);
    int ok = 1;
    for (int r = 0; r < world && ok; ++r) {
        if (r == d.rank) continue;
        if (!all[r].ok) {
            ok = 0;
            break;
        }
        void *b = nullptr, *f = nullptr;
        if (cudaIpcOpenMemHandle(&b, all[r].mem, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess ||
            cudaIpcOpenMemHandle(&f, all[r].flags, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)
            ok = 0;
        d.peer_base[r] = static_cast<char *>(b);
        d.peer_flags[r] = static_cast<unsigned long long *>(f);
    }
    cudaGetLastError();
    int32_t *dok = reinterpret_cast<int32_t *>(dbuf);
    QS_CUDA(s, cudaMemcpyAsync(dok, &ok, sizeof ok, cudaMemcpyHostToDevice, d.st));
    QS_NCCL(s, ncclAllReduce(dok, dok, 1, ncclInt32, ncclMin, d.nccl, d.st));
    QS_CUDA(s, cudaStreamSynchronize(d.st));
    QS_CUDA(s, cudaMemcpyAsync(&ok, dok, sizeof ok, cudaMemcpyDeviceToHost, d.st));
    QS_CUDA(s, cudaStreamSynchronize(d.st));
    cudaFree(dbuf);
    s->p2p_ok = ok != 0;
    return QS_OK;
}

qs_status qs_create(int n_qubits, int n_gpus, qs_state **out) {
    int k;
    qs_status r = common_validate(n_qubits, n_gpus, out, k);
    if (r != QS_OK) return r;
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev < n_gpus) {
        g_create_error = fmt("need %d CUDA devices, found %d (%s)", n_gpus, ndev, cudaGetErrorString(e));
        return e != cudaSuccess ? QS_ERR_CUDA : QS_ERR_ARG;
    }
    qs_state *s = new qs_state();
    s->guard = canary_bytes();
    s->n = n_qubits;
    s->P = n_gpus;
    s->m = n_qubits - k;
    s->mode = n_gpus == 1 ? MODE_SINGLE : MODE_MULTIDEV;
    cudaDeviceGetAttribute(&s->num_sms, cudaDevAttrMultiProcessorCount, 0);
    s->sh.resize(n_gpus);
    for (int d = 0; d < n_gpus; ++d) {
        s->sh[d].rank = d;
        s->sh[d].device = d;
        r = alloc_shard(s, s->sh[d], true);
        if (r != QS_OK) return create_fail(s, r, out);
    }
    if (n_gpus > 1) {
        std::vector<ncclComm_t> comms(n_gpus);
        std::vector<int> devs(n_gpus);
        for (int d = 0; d < n_gpus; ++d) devs[d] = d;
        ncclResult_t nr = ncclCommInitAll(comms.data(), n_gpus, devs.data());
        if (nr != ncclSuccess) {
            set_err(s, QS_ERR_NCCL, fmt("ncclCommInitAll: %s", ncclGetErrorString(nr)));
            return create_fail(s, QS_ERR_NCCL, out);
        }
        for (int d = 0; d < n_gpus; ++d) s->sh[d].nccl = comms[d];
        // peer access between every pair (NVLink/NVSwitch): enables the fused peer-memory exchange
        bool ok = true;
        for (int a = 0; a < n_gpus && ok; ++a) {
            cudaSetDevice(a);
            for (int b = 0; b < n_gpus && ok; ++b) {
                if (a == b) continue;
                int can = 0;
                if (cudaDeviceCanAccessPeer(&can, a, b) != cudaSuccess || !can) {
                    ok = false;
                    break;
                }
                cudaError_t pe = cudaDeviceEnablePeerAccess(b, 0);
                if (pe == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
                else if (pe != cudaSuccess) ok = false;
            }
        }
        cudaGetLastError();
        s->p2p_ok = ok;
    }
    r = finish_create(s, out);
    if (r != QS_OK) return create_fail(s, r, out);
    return QS_OK;
}

qs_status qs_create_virtual(int n_qubits, int n_shards, qs_state **out) {
    int k;
    qs_status r = common_validate(n_qubits, n_shards, out, k);
    if (r != QS_OK) return r;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) {
        g_create_error = fmt("no CUDA device: %s", cudaGetErrorString(e));
        return QS_ERR_CUDA;
    }
    qs_state *s = new qs_state();
    s->guard = canary_bytes();
    s->n = n_qubits;
    s->P = n_shards;
    s->m = n_qubits - k;
    s->mode = MODE_VIRTUAL;
    s->p2p_ok = true;  // every shard is in this device's memory
    cudaDeviceGetAttribute(&s->num_sms, cudaDevAttrMultiProcessorCount, dev);
    s->sh.resize(n_shards);
    for (int d = 0; d < n_shards; ++d) {
        s->sh[d].rank = d;
        s->sh[d].device = dev;
        r = alloc_shard(s, s->sh[d], d == 0);
        if (r != QS_OK) return create_fail(s, r, out);
        if (d > 0) {  // all virtual shards run in one stream (stream order = exchange order)
            Shard &d0 = s->sh[0];
            s->sh[d].st = d0.st;
            s->sh[d].comm = d0.comm;
            for (int i = 0; i < 2; ++i) {
                s->sh[d].ev_recv[i] = d0.ev_recv[i];
                s->sh[d].ev_upd[i] = d0.ev_upd[i];
                s->sh[d].ev_pack[i] = d0.ev_pack[i];
            }
            s->sh[d].ev_ready = d0.ev_ready;
            s->sh[d].ev_done = d0.ev_done;
        }
    }
    r = finish_create(s, out);
    if (r != QS_OK) return create_fail(s, r, out);
    return QS_OK;
}

qs_status qs_get_unique_id(void *id128) {
    if (!id128) return QS_ERR_ARG;
    ncclUniqueId id;
    ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) {
        g_create_error = fmt("ncclGetUniqueId: %s", ncclGetErrorString(r));
        return QS_ERR_NCCL;
    }
    static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id is 128 bytes");
    std::memcpy(id128, &id, 128);
    return QS_OK;
}

qs_status qs_create_rank(int n_qubits, int world, int rank, int device, const void *id128, qs_state **out) {
    int k;
    qs_status r = common_validate(n_qubits, world, out, k);
    if (r != QS_OK) return r;
    if (rank < 0 || rank >= world || !id128) {
        g_create_error = fmt("rank %d outside [0, %d) or NULL id", rank, world);
        return QS_ERR_ARG;
    }
    qs_state *s = new qs_state();
    s->guard = canary_bytes();
    s->n = n_qubits;
    s->P = world;
    s->m = n_qubits - k;
    s->mode = MODE_RANK;
    s->sh.resize(1);
    s->sh[0].rank = rank;
    s->sh[0].device = device;
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) {
        set_err(s, QS_ERR_CUDA, fmt("cudaSetDevice(%d): %s", device, cudaGetErrorString(e)));
        return create_fail(s, QS_ERR_CUDA, out);
    }
    cudaDeviceGetAttribute(&s->num_sms, cudaDevAttrMultiProcessorCount, device);
    r = alloc_shard(s, s->sh[0], true);
    if (r != QS_OK) return create_fail(s, r, out);
    if (world > 1) {
        ncclUniqueId id;
        std::memcpy(&id, id128, 128);
        ncclResult_t nr = ncclCommInitRank(&s->sh[0].nccl, world, id, rank);
        if (nr != ncclSuccess) {
            set_err(s, QS_ERR_NCCL, fmt("ncclCommInitRank: %s", ncclGetErrorString(nr)));
            return create_fail(s, QS_ERR_NCCL, out);
        }
        const char *pe = getenv("QS_P2P_RANK");
        if (pe && atoi(pe)) {
            r = setup_rank_peers(s);
            if (r != QS_OK) return create_fail(s, r, out);
        }
    }
    r = finish_create(s, out);
    if (r != QS_OK) return create_fail(s, r, out);
    return QS_OK;
}

void qs_destroy(qs_state *s) { destroy_state(s); }

qs_status qs_init_basis(qs_state *s, uint64_t index) {
    QS_TRY(guard(s));
    if (index >= (1ull << s->n)) return set_err(s, QS_ERR_RANGE, fmt("basis index %llu >= 2^%d", (unsigned long long)index, s->n));
    return init_basis_impl(s, index);
}

qs_status qs_init_random(qs_state *s, uint64_t seed) {
    QS_TRY(guard(s));
    // one pass generates the state and its norm leaves, a second scales it
    for (auto &d : s->sh) {
        QS_CUDA(s, cudaSetDevice(d.device));
        QS_TRY(check_launch(s, launch_init_random_norm(d.amps, 1ull << s->m, (uint64_t)d.rank << s->m, seed,
                                                       std::min(norm_leaf_log2(s->n), s->m), d.d_scratch, d.d_norm,
                                                       d.st, s->num_sms)));
    }
    double total = 0.0;
    QS_TRY(norm_total(s, &total, true));
    const double inv = 1.0 / std::sqrt(total);
    for (auto &d : s->sh) {
        QS_CUDA(s, cudaSetDevice(d.device));
        QS_TRY(check_launch(s, launch_scale(d.amps, 1ull << s->m, inv, d.st, s->num_sms)));
    }
    return QS_OK;
}

qs_status qs_apply_1q(qs_state *s, int target, const double u2[8]) {
    QS_TRY(guard(s));
    qs_gate g{QS_G_1Q, target, -1, 0, {0}};
    if (!u2) return set_err(s, QS_ERR_ARG, "NULL matrix");
    std::memcpy(g.m, u2, 8 * sizeof(double));
    std::vector<Op> ops;
    QS_TRY(gates_to_ops(s, &g, 1, ops));
    s->last_passes = s->last_exchanges = 0;
    return run_op(s, ops[0]);
}

qs_status qs_apply_ctrl_1q(qs_state *s, int ctrl, int target, const double u2[8]) {
    QS_TRY(guard(s));
    qs_gate g{QS_G_C1Q, ctrl, target, 0, {0}};
    if (!u2) return set_err(s, QS_ERR_ARG, "NULL matrix");
    std::memcpy(g.m, u2, 8 * sizeof(double));
    std::vector<Op> ops;
    QS_TRY(gates_to_ops(s, &g, 1, ops));
    s->last_passes = s->last_exchanges = 0;
    return run_op(s, ops[0]);
}

qs_status qs_apply_2q(qs_state *s, int q0, int q1, const double u4[32]) {
    QS_TRY(guard(s));
    qs_gate g{QS_G_2Q, q0, q1, 0, {0}};
    if (!u4) return set_err(s, QS_ERR_ARG, "NULL matrix");
    std::memcpy(g.m, u4, 32 * sizeof(double));
    std::vector<Op> ops;
    QS_TRY(gates_to_ops(s, &g, 1, ops));
    s->last_passes = s->last_exchanges = 0;
    return run_op(s, ops[0]);
}

qs_status qs_run_circuit(qs_state *s, const qs_gate *gates, size_t n_gates) {
    QS_TRY(guard(s));
    if (n_gates == 0) return QS_OK;
    if (!gates) return set_err(s, QS_ERR_ARG, "NULL gate array");
    return run_gates(s, gates, n_gates);
}

qs_status qs_read_amps(qs_state *s, uint64_t start, uint64_t count, double *out) {
    QS_TRY(guard(s));
    QS_TRY(range_check(s, start, count, out));
    if (!count) return QS_OK;
    return copy_amps(s, start, count, out, true);
}

qs_status qs_write_amps(qs_state *s, uint64_t start, uint64_t count, const double *in) {
    QS_TRY(guard(s));
    QS_TRY(range_check(s, start, count, in));
    if (!count) return QS_OK;
    return copy_amps(s, start, count, const_cast<double *>(in), false);
}

qs_status qs_read_amps_async(qs_state *s, uint64_t start, uint64_t count, double *out) {
    QS_TRY(guard(s));
    QS_TRY(range_check(s, start, count, out));
    if (!count) return QS_OK;
    return copy_amps(s, start, count, out, true, false);
}

qs_status qs_write_amps_async(qs_state *s, uint64_t start, uint64_t count, const double *in) {
    QS_TRY(guard(s));
    QS_TRY(range_check(s, start, count, in));
    if (!count) return QS_OK;
    return copy_amps(s, start, count, const_cast<double *>(in), false, false);
}

qs_status qs_norm2(qs_state *s, double *out) {
    QS_TRY(guard(s));
    if (!out) return set_err(s, QS_ERR_ARG, "NULL out");
    return norm_total(s, out);
}

qs_status qs_sync(qs_state *s) {
    QS_TRY(guard(s));
    for (auto &d : s->sh) {
        QS_CUDA(s, cudaSetDevice(d.device));
        QS_CUDA(s, cudaStreamSynchronize(d.st));
        QS_CUDA(s, cudaStreamSynchronize(d.comm));
    }
    QS_CUDA(s, cudaGetLastError());
    return check_canaries(s);
}

const char *qs_last_error(const qs_state *s) { return s ? s->err.c_str() : g_create_error.c_str(); }

qs_status qs_info(const qs_state *s, int *n_qubits, int *n_shards, int *local_qubits, int *owned, int *first_rank) {
    if (!s) return QS_ERR_ARG;
    if (n_qubits) *n_qubits = s->n;
    if (n_shards) *n_shards = s->P;
    if (local_qubits) *local_qubits = s->m;
    if (owned) *owned = (int)s->sh.size();
    if (first_rank) *first_rank = s->sh.empty() ? 0 : s->sh[0].rank;
    return QS_OK;
}

uint64_t qs_launch_count(const qs_state *s) { return s ? s->launches : 0; }

void *qs_stream(const qs_state *s, int i) {
    if (!s || i < 0 || i >= (int)s->sh.size()) return nullptr;
    return (void *)s->sh[i].st;
}

qs_status qs_set_option(qs_state *s, const char *key, int64_t value) {
    QS_TRY(guard(s));
    if (!key) return set_err(s, QS_ERR_ARG, "NULL key");
    std::string k(key);
    if (k == "fuse") {
        s->fuse = value != 0;
    } else if (k == "tile_qubits") {
        if (value < 6 || value > TILE_MAX_Q) return set_err(s, QS_ERR_ARG, fmt("tile_qubits %lld outside [6, %d]", (long long)value, TILE_MAX_Q));
        s->tile_b = (int)value;
    } else if (k == "check_unitary") {
        s->check_unitary = value != 0;
    } else if (k == "jit") {
        s->jit = value != 0;
    } else if (k == "tile_low_auto") {
        s->tile_low_auto = value != 0;
    } else if (k == "jit_async") {
        s->jit_async = value != 0;
    } else if (k == "jit_wait") {  // action: wait for background kernel compilations
        jit_tile_wait();
    } else if (k == "p2p") {
        s->p2p = value != 0;
    } else if (k == "factor") {
        s->factor = value != 0;
    } else if (k == "remap") {
        s->remap = value != 0;
    } else if (k == "reorder") {
        s->reorder = value != 0;
    } else if (k == "perm_fuse") {
        s->perm_fuse = value != 0;
    } else if (k == "perm_hoist") {
        s->perm_hoist = value != 0;
    } else if (k == "perm_low") {
        if (value < 0 || value > 6) return set_err(s, QS_ERR_ARG, "perm_low outside [0, 6]");
        s->perm_low = (int)value;
    } else if (k == "ladder_min") {
        if (value < 0 || value > 1000000) return set_err(s, QS_ERR_ARG, "ladder_min outside [0, 1e6]");
        s->ladder_min = (int)value;
    } else if (k == "tile_low") {
        if (value < 1 || value > 8) return set_err(s, QS_ERR_ARG, "tile_low outside [1, 8]");
        s->tile_low = (int)value;
    } else if (k == "graph") {
        s->graph = value != 0;
    } else if (k == "jit_family") {
        if (value < 0 || value > 2) return set_err(s, QS_ERR_ARG, "jit_family must be 0, 1 or 2");
        s->jit_family = (int)value;
    } else if (k == "vtransport") {
        if (value < 0 || value > 1) return set_err(s, QS_ERR_ARG, "vtransport must be 0 or 1");
        if (value == 1 && s->mode != MODE_VIRTUAL) return set_err(s, QS_ERR_ARG, "vtransport applies to virtual shards only");
        if (value == 1 && !s->sh[0].nccl) {  // one-rank communicator on this device (send/recv to self)
            QS_CUDA(s, cudaSetDevice(s->sh[0].device));
            int dev = s->sh[0].device;
            QS_NCCL(s, ncclCommInitAll(&s->sh[0].nccl, 1, &dev));
        }
        s->vtransport = (int)value;
    } else if (k == "chunk_bytes") {
        // a power of two: every exchange moves 2^m or 2^(m-1) amplitudes, so a power-of-two chunk
        // divides it and the pipeline needs no remainder chunk
        if (value < 4096 || (value & (value - 1)))
            return set_err(s, QS_ERR_ARG, "chunk_bytes must be a power of two >= 4096");
        QS_TRY(qs_sync(s));
        s->chunk_bytes = (uint64_t)value;
        for (auto &d : s->sh) {
            QS_CUDA(s, cudaSetDevice(d.device));
            free_exchange_buffers(d);
            QS_TRY(alloc_exchange_buffers(s, d));
        }
    } else {
        return set_err(s, QS_ERR_ARG, "unknown option " + k);
    }
    return QS_OK;
}

qs_status qs_jit_stats(const qs_state *s, uint64_t *compiled, uint64_t *launched, uint64_t *failed) {
    if (!s) return QS_ERR_ARG;
    jit_tile_stats(compiled, launched, failed);
    return QS_OK;
}

qs_status qs_last_plan(const qs_state *s, uint64_t *passes, uint64_t *exchanges) {
    if (!s) return QS_ERR_ARG;
    if (passes) *passes = s->last_passes;
    if (exchanges) *exchanges = s->last_exchanges;
    return QS_OK;
}

// ---------------------------------------------------------------------------------------------
// host-only planner entry points (include/qs_plan_abi.h)
// ---------------------------------------------------------------------------------------------
qs_status qs_plan_route(int n, int m, int rank, const qs_gate *g, int check_unitary, int32_t out_step[5],
                        int32_t out_op[4], double out_m[32]) {
    if (!g || !out_step || !out_op || !out_m || m < 1 || m > n) {
        g_create_error = "qs_plan_route: bad argument";
        return QS_ERR_ARG;
    }
    Op op;
    std::string msg;
    if (!classify(n, g->kind, g->q0, g->q1, g->m, check_unitary != 0, op, msg)) {
        g_create_error = msg;
        return QS_ERR_ARG;
    }
    ShardStep st = localize(op, n, m, rank);
    out_step[0] = st.action;
    out_step[1] = st.partner;
    out_step[2] = st.bit;
    out_step[3] = st.ctrl_local;
    out_step[4] = st.l;
    out_op[0] = st.local.kind;
    out_op[1] = st.local.q0;
    out_op[2] = st.local.q1;
    out_op[3] = (int32_t)st.local.touch;
    std::memcpy(out_m, st.local.m, sizeof(st.local.m));
    return QS_OK;
}

int qs_plan_decompose(int n, int m, const qs_gate *g, qs_gate *out, int max_out) {
    if (!g || !out) return -1;
    Op op;
    std::string msg;
    if (!classify(n, g->kind, g->q0, g->q1, g->m, false, op, msg)) {
        g_create_error = msg;
        return -1;
    }
    std::vector<Op> seq = decompose_via_swap(op, m);
    if ((int)seq.size() > max_out) return -1;
    for (size_t i = 0; i < seq.size(); ++i) {
        qs_gate &o = out[i];
        std::memset(&o, 0, sizeof o);
        if (seq[i].kind == OP_SWAP) {
            o.kind = QS_G_2Q;
            o.q0 = seq[i].q0;
            o.q1 = seq[i].q1;
            o.m[0] = o.m[2 * (4 * 1 + 2)] = o.m[2 * (4 * 2 + 1)] = o.m[2 * 15] = 1.0;
        } else {
            o = *g;
            o.q0 = seq[i].q0;
            o.q1 = seq[i].q1;
        }
    }
    return (int)seq.size();
}

int qs_plan_passes(int n, int m, const qs_gate *gates, size_t n_gates, int b, int L0, int fuse, int reorder,
                   int32_t *out_type, int32_t *out_nops, int32_t *out_first, uint64_t *out_tile_mask,
                   int32_t *out_order, int max_passes) {
    if ((!gates && n_gates) || m < 1 || m > n) return -1;
    std::vector<Op> ops(n_gates);
    for (size_t i = 0; i < n_gates; ++i) {
        std::string msg;
        if (!classify(n, gates[i].kind, gates[i].q0, gates[i].q1, gates[i].m, false, ops[i], msg)) {
            g_create_error = msg;
            return -1;
        }
    }
    PlanConfig cfg;
    cfg.b = b;
    cfg.L0 = L0;
    cfg.fuse = fuse != 0;
    cfg.reorder = reorder != 0;
    std::vector<Pass> plan = plan_passes(ops, n, m, cfg);
    if ((int)plan.size() > max_passes) return -1;
    size_t at = 0;
    for (size_t p = 0; p < plan.size(); ++p) {
        if (out_type) out_type[p] = plan[p].type == 1 && !plan[p].perm.empty() ? 4 : plan[p].type;
        if (out_nops) out_nops[p] = (int32_t)(plan[p].ops.size() + plan[p].perm_ops.size());
        if (out_first) out_first[p] = plan[p].ops.empty() ? -1 : plan[p].ops[0];
        for (int oi : plan[p].ops) {
            if (out_order && at < n_gates) out_order[at] = oi;
            ++at;
        }
        for (int oi : plan[p].perm_ops) {
            if (out_order && at < n_gates) out_order[at] = oi;
            ++at;
        }
        if (out_tile_mask) {
            uint64_t mask = 0;
            for (int q : plan[p].tile_q) mask |= 1ull << q;
            out_tile_mask[p] = mask;
        }
    }
    return (int)plan.size();
}

int qs_plan_remap(int n, int m, const qs_gate *gates, size_t n_gates, qs_gate *out, int max_out, int32_t out_cost[2]) {
    if ((!gates && n_gates) || m < 1 || m > n) return -1;
    std::vector<Op> ops(n_gates);
    for (size_t i = 0; i < n_gates; ++i) {
        std::string msg;
        if (!classify(n, gates[i].kind, gates[i].q0, gates[i].q1, gates[i].m, false, ops[i], msg)) {
            g_create_error = msg;
            return -1;
        }
    }
    std::vector<Op> r = remap_global(ops, n, m);
    if (out_cost) {
        out_cost[0] = exchange_cost(ops, m);
        out_cost[1] = exchange_cost(r, m);
    }
    if ((int)r.size() > max_out) return -1;
    for (size_t i = 0; i < r.size(); ++i) op_to_gate(r[i], out[i]);
    return (int)r.size();
}

int qs_plan_hoist(int n, int m, const qs_gate *gates, size_t n_gates, int b, int L0, int reorder, qs_gate *out,
                  int max_out, int32_t out_stats[3]) {
    if ((!gates && n_gates) || m < 1 || m > n || b < 6) return -1;
    std::vector<Op> ops(n_gates);
    for (size_t i = 0; i < n_gates; ++i) {
        std::string msg;
        if (!classify(n, gates[i].kind, gates[i].q0, gates[i].q1, gates[i].m, false, ops[i], msg)) {
            g_create_error = msg;
            return -1;
        }
    }
    PlanConfig cfg;
    cfg.b = b;
    cfg.L0 = L0;
    cfg.reorder = reorder != 0;
    const std::vector<Pass> plan = plan_passes(ops, n, m, cfg);
    std::vector<Op> o2;
    std::vector<Pass> p2;
    const bool h = hoist_permutation(ops, plan, m, cfg, o2, p2);
    if (out_stats) {
        out_stats[0] = (int32_t)plan.size();
        out_stats[1] = (int32_t)(h ? p2.size() : plan.size());
        int fused = 0;
        for (const Pass &p : (h ? p2 : plan)) fused += p.type == 1 && !p.perm.empty();
        out_stats[2] = fused;
    }
    if (!h) return 0;
    if ((int)o2.size() > max_out) return -1;
    for (size_t i = 0; i < o2.size(); ++i) op_to_gate(o2[i], out[i]);
    return (int)o2.size();
}

qs_status qs_plan_tile_jit(int n, int m, int rank, const qs_gate *gates, size_t n_gates, int b, int L0, int ladder_min,
                           int compile, int32_t out_stats[10]) {
    if ((!gates && n_gates) || m < 1 || m > n || rank < 0 || rank >= (1 << (n - m)) || b < 6 || b > TILE_MAX_Q) {
        g_create_error = "qs_plan_tile_jit: bad arguments";
        return QS_ERR_ARG;
    }
    std::vector<Op> ops(n_gates);
    for (size_t i = 0; i < n_gates; ++i) {
        std::string msg;
        if (!classify(n, gates[i].kind, gates[i].q0, gates[i].q1, gates[i].m, false, ops[i], msg)) {
            g_create_error = msg;
            return QS_ERR_ARG;
        }
    }
    PlanConfig cfg;
    cfg.b = b;
    cfg.L0 = L0;
    cfg.fuse = true;
    cfg.reorder = true;  // the library defaults (qs_state::reorder, ::factor)
    if (ops.size() > 1) ops = factor_scalars(ops);
    std::vector<Pass> plan = plan_passes(ops, n, m, cfg);
    {
        std::vector<Op> o2;
        std::vector<Pass> p2;
        if (hoist_permutation(ops, plan, m, cfg, o2, p2)) {  // as qs_run_circuit (option perm_hoist)
            ops.swap(o2);
            plan.swap(p2);
        }
    }
    std::vector<TileDesc> descs;
    std::vector<TileBatch> bats;
    std::vector<TileOp> tops;
    std::vector<TileLadder> lads;
    for (const Pass &ps : plan) {
        if (ps.type != 1) continue;
        std::vector<Op> local;
        for (int oi : ps.ops) {
            ShardStep st = localize(ops[oi], n, m, rank);
            if (st.action == SA_LOCAL) local.push_back(st.local);
        }
        if (local.empty()) continue;
        TileDesc d;
        make_tile_pass(ps.tile_q.data(), (int)ps.tile_q.size(), ps.L, m, local.data(), (int)local.size(), d, bats, tops,
                       lads, ladder_min, true);
        if (!ps.perm.empty() && !set_tile_perm(d, ps.tile_q.data(), (int)ps.tile_q.size(), ps.perm.data(), m)) {
            g_create_error = "fused permutation does not map the tile onto itself";
            return QS_ERR_UNSUPPORTED;
        }
        if (tile_op_bytes(d) > (unsigned long long)TILE_OP_SMEM) {
            g_create_error = "tile pass op stream exceeds its shared-memory budget";
            return QS_ERR_UNSUPPORTED;
        }
        descs.push_back(d);
    }
    std::vector<std::string> srcs;
    for (const TileDesc &d : descs) {
        std::string src = jit_tile_source(d, bats.data(), tops.data(), tile_regs(), (compile & 2) != 0);
        if (std::find(srcs.begin(), srcs.end(), src) == srcs.end()) srcs.push_back(src);
    }
    uint64_t hash = 1469598103934665603ull;
    for (const std::string &src : srcs)
        for (unsigned char ch : src) hash = (hash ^ ch) * 1099511628211ull;
    int compiled = 0;
    if (compile & 1) {
        for (const std::string &src : srcs) {
            std::string err;
            if (!jit_tile_compile_check(src, nullptr, err)) {
                g_create_error = err;
                return QS_ERR_UNSUPPORTED;
            }
            ++compiled;
        }
    }
    if (out_stats) {
        out_stats[0] = (int32_t)plan.size();
        out_stats[1] = (int32_t)descs.size();
        out_stats[2] = (int32_t)tops.size();
        out_stats[3] = (int32_t)lads.size();
        out_stats[4] = (int32_t)srcs.size();
        out_stats[5] = compiled;
        out_stats[6] = (int32_t)bats.size();
        out_stats[7] = (int32_t)(hash & 0x7fffffffu);
        int32_t wl = 0;
        for (const TileDesc &d : descs)
            for (int bi = 0; !d.perm && bi + 1 < d.nbatch; ++bi)
                wl += warp_local_transition(bats[d.batch0 + bi].dep, bats[d.batch0 + bi + 1].dep, d.b - tile_regs(),
                                            jit_tile_threads(d.b, tile_regs()));
        int32_t gl = 0;  // transitions separated by a barrier narrower than the CTA (warp or warp group)
        for (const TileDesc &d : descs) {
            const int tpb = jit_tile_threads(d.b, tile_regs());
            int wb = 0;
            while ((1 << (wb + 1)) <= tpb) ++wb;
            const int nw = std::min(wb, d.b - tile_regs()) - 5;
            for (int bi = 0; !d.perm && bi + 1 < d.nbatch; ++bi)
                gl += transition_scope(bats[d.batch0 + bi].dep, bats[d.batch0 + bi + 1].dep, d.b - tile_regs(), tpb) < nw;
        }
        out_stats[9] = gl;
        out_stats[8] = wl;
    }
    return QS_OK;
}

}  // extern "C"
