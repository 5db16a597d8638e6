// k_tile.cu — fused tile pass (paper: cache blocking / gate fusion "traverse the
// state fewer times", blocked QFT L295): the interpreter kernel and the host side.
//
// Two-level blocking of a run of consecutive ops:
//  1. TILE (HBM <-> shared memory): a persistent CTA gathers 2^b amplitudes — local qubits 0..L-1
//     (contiguous runs of >= 512 B, coalesced) plus b-L higher qubits (qsim-style gathered tile,
//     SURVEY.md §8(f) rank 1) — into shared memory, applies the run, writes it back: one HBM
//     read + write for the whole run instead of one per gate.  The next tile is prefetched with
//     cp.async into the second of two buffers while the current one is processed.
//  2. BATCH (shared memory <-> registers): ops are grouped so that the non-diagonal ones of a batch
//     act on at most R tile positions ("register slots"); each thread loads the 2^R amplitudes of
//     one sub-cube spanned by those positions into registers, applies every op of the batch with
//     compile-time register indices, and stores them back: one shared-memory round trip per batch.
//     Diagonal ops and controls may use any bit: outside the register slots the bit is a constant
//     of the sub-cube (tile position) or of the tile (qubit outside the tile).
// The host pre-decodes every op into a dense opcode (qs_tile_opcodes.inc) and every batch into its
// 16 swizzled register offsets.  Two executors of the same descriptors: this file's interpreter
// (one jump-table switch per op) and jit_tile.cpp (NVRTC, the op sequence as straight-line code).
// Per-op arithmetic is the qs_device.cuh chain in gate order: bitwise identical to the unfused path.
#include <vector>
#include <algorithm>
#include <array>
#include <set>
#include <cstdio>
#include <cstdlib>

#include "qs_kernels.h"
#include "qs_tile_ops.cuh"

namespace qsb {

// interpreter: apply the ops of every batch of the tile, one jump-table dispatch per op
struct InterpProg {
    template <int R, int TPB>
    static __device__ __forceinline__ void run(const TileCtx &c) {
        constexpr int NV = 1 << R;
        const uint64_t base = c.base;
        for (int bi = 0; bi < c.nbatch; ++bi) {
            const TileBatch *bt = c.bats + c.batch0 + bi;
            uint32_t swo[NV];
#pragma unroll
            for (int r = 0; r < NV; ++r) swo[r] = bt->swo[r];
            const int nops = bt->nops;
            const int4 *op_rec = c.ops_sm + 5 * (bt->op0 - c.op_begin);
            for (uint32_t s = c.tid; s < c.nsub; s += TPB) {
                const uint32_t jb = sub_deposit(s, bt->dep, c.nsub_bits);
                const uint32_t sjb = swz(jb);
                double2 v[NV];
#pragma unroll
                for (int r = 0; r < NV; ++r) v[r] = c.smb[sjb ^ swo[r]];
                for (int o = 0; o < nops; ++o) {
                    const int4 *rec = op_rec + 5 * o;
                    const int4 h = rec[0];
                    double2 mm[4];
#pragma unroll
                    for (int k = 0; k < 4; ++k) mm[k] = reinterpret_cast<const double2 *>(rec + 1)[k];
                    const double2 *qm = c.quad_sm + 16 * h.w;
                    switch (h.x) {
#define QS_OPCODE(code, ...) \
    case code:               \
        __VA_ARGS__;         \
        break;
#include "qs_tile_opcodes.inc"
#undef QS_OPCODE
                    default: break;
                    }
                }
#pragma unroll
                for (int r = 0; r < NV; ++r) c.smb[sjb ^ swo[r]] = v[r];
            }
            __syncthreads();
        }
    }
};

template <int R, int TPB>
__global__ void __launch_bounds__(TPB, 1) k_tile(double2 *__restrict__ a, uint64_t ntiles, const TileDesc *__restrict__ dd,
                                                 const TileBatch *__restrict__ bats, const TileOp *__restrict__ ops) {
    tile_kernel<R, TPB, 2, InterpProg>(a, ntiles, dd, bats, ops);
}

// ------------------------------------------------------------------------------------------------
// host: batch formation and op decoding
// ------------------------------------------------------------------------------------------------
int tile_regs() {  // register slots per batch: 4 (16 amplitudes / thread, 256 threads) or 3
    static int r = getenv("QS_TILE_R") ? atoi(getenv("QS_TILE_R")) : 4;
    return r == 3 ? 3 : 4;
}

// JIT passes: bit 0 = first batch loads from HBM, bit 1 = last batch stores to HBM, bit 2 = the last batch
// issues the next tile's gather; 8 = per pass (QS_TILE_DIRECT; default 8, see jit_direct_pass)
int tile_direct_io() {
    static const int v = getenv("QS_TILE_DIRECT") ? atoi(getenv("QS_TILE_DIRECT")) & 15 : 8;
    return v;
}

// warp-local batch transitions (align_warp_bits; QS_WARP_LOCAL=0 keeps the round-2 lane layout for A/B)
int tile_warp_local() {
    static const int v = getenv("QS_WARP_LOCAL") ? atoi(getenv("QS_WARP_LOCAL")) : 1;
    return v;
}

// dense opcode of an op (tables follow qs_tile_opcodes.inc)
int tile_opcode(int kind, int s0, int s1) {
    static const int ctrl[4][4] = {{-1,4,5,6},{7,-1,8,9},{10,11,-1,12},{13,14,15,-1}};
    static const int quad[4][4] = {{-1,20,21,22},{23,-1,24,25},{26,27,-1,28},{29,30,31,-1}};
    static const int swp[4][4] = {{-1,32,33,34},{-1,-1,35,36},{-1,-1,-1,37},{-1,-1,-1,-1}};
    static const int diag[5][5] = {{-1,38,39,40,41},{42,-1,43,44,45},{46,47,-1,48,49},{50,51,52,-1,53},{54,55,56,57,58}};
    switch (kind) {
    case OP_PAIR: return s0;
    case OP_CTRL_PAIR: return s0 == 4 ? 16 + s1 : ctrl[s0][s1];
    case OP_QUAD: return quad[s0][s1];
    case OP_SWAP: return swp[std::min(s0, s1)][std::max(s0, s1)];
    default: return diag[s0][s1];
    }
}

// single-factor phase op with constrained register slots a, b (4 = none)
int tile_phase_opcode(int a, int b) {
    static const int ph[5][5] = {{-1,59,60,61,62},{59,-1,63,64,65},{60,63,-1,66,67},{61,64,66,-1,68},{62,65,67,68,69}};
    return ph[a][b];
}

bool tile_opcode_is_quad(int code) { return code >= 20 && code <= 31; }

namespace {

void needs(const Op &op, const int *pos, std::vector<int> &need) {
    need.clear();
    switch (op.kind) {
    case OP_PAIR: need.push_back(pos[op.q0]); break;
    case OP_CTRL_PAIR: need.push_back(pos[op.q1]); break;
    case OP_QUAD:
    case OP_SWAP:
        need.push_back(pos[op.q0]);
        need.push_back(pos[op.q1]);
        break;
    default: break;
    }
}

}  // namespace

namespace {

struct Cx {
    double re, im;
};
inline Cx cx_mul(Cx a, Cx b) { return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re}; }

// pure-phase form of a local op: OP_DIAG whose only factor != 1 sits at k = all constrained bits 1
bool phase_form(const Op &op, int &nq, int q[2], Cx &x) {
    if (op.kind != OP_DIAG || op.q0 < 0) return false;
    nq = op.q1 < 0 ? 1 : 2;
    const uint32_t kall = (1u << nq) - 1;
    if (op.touch != (1u << kall)) return false;
    q[0] = op.q0;
    q[1] = op.q1;
    x = {op.m[2 * kall], op.m[2 * kall + 1]};
    return true;
}

// Sub-cube bit order of a batch over its non-slot positions `free_pos`: five lane bits first, covering
// every residue mod 3 (the swizzle folds position p into column bit p mod 3); a 16-B shared access is
// served per quarter warp (8 lanes), so the three lowest lane bits cover the three residues themselves
// (lowest position of each residue), then the remaining positions in the given order.
std::vector<int> lane_first_order(const std::vector<int> &free_pos) {
    std::vector<int> lanes, rest;
    const int nl = std::min<int>(5, (int)free_pos.size());
    for (int res = 0; res < 3 && (int)lanes.size() < nl; ++res)
        for (int p : free_pos)
            if (p % 3 == res) {
                lanes.push_back(p);
                break;
            }
    for (int p : free_pos)
        if ((int)lanes.size() < nl && std::find(lanes.begin(), lanes.end(), p) == lanes.end()) lanes.push_back(p);
    std::vector<int> first, others;
    for (int res = 0; res < 3; ++res)
        for (int p : lanes)
            if (p % 3 == res && std::find(first.begin(), first.end(), p) == first.end()) {
                first.push_back(p);
                break;
            }
    for (int p : lanes)
        if (std::find(first.begin(), first.end(), p) == first.end()) others.push_back(p);
    lanes = first;
    lanes.insert(lanes.end(), others.begin(), others.end());
    for (int p : free_pos)
        if (std::find(lanes.begin(), lanes.end(), p) == lanes.end()) rest.push_back(p);
    lanes.insert(lanes.end(), rest.begin(), rest.end());
    return lanes;
}

uint64_t pack_dep(const std::vector<int> &order) {
    uint64_t d = 0;
    for (size_t i = 0; i < order.size() && i < 12; ++i) d |= (uint64_t)order[i] << (4 * i);
    return d;
}

// Warp-local batch transitions (jit_tile_source): two consecutive batches that put the same tile
// positions, in the same order, on the sub-cube bits selecting the WARP (bits 5 .. log2(TPB)-1) hand
// every amplitude from a warp to the same warp, so the kernel separates them with __syncwarp instead of
// a CTA barrier and the warps of a CTA drift apart (one warp's shared-memory phase overlaps another's
// FP64 work).  Positions only move between lane, warp and iteration bits: every amplitude still meets the
// same ops in the same order (bitwise-identical results).  A transition needs warp positions W inside
// both batches' non-slot positions such that the lane rules still hold —
// lanes cover the three swizzle residues (shared-memory batches), or, in a direct-I/O batch, stay the
// lowest non-slot positions, include every low position < L (runs of 2^L amplitudes) and keep tile
// positions 0, 1 first when they were (coalesced HBM access) — and
// a dynamic program picks the layouts with the most such transitions.
void align_warp_bits(TileBatch *bt, int nb, int b, int L, int R, int tpb, bool first_direct, bool last_direct) {
    int wb = 0;  // log2 of the threads of one CTA that share sub-cube iterations
    while ((1 << (wb + 1)) <= tpb) ++wb;
    const int nsb = b - R, whi = std::min(wb, nsb), nw = whi - 5;
    if (nw <= 0 || nb < 2) return;
    auto free_of = [&](const TileBatch &x) {
        std::vector<int> f;
        for (int p = 0; p < b; ++p) {
            bool slot = false;
            for (int i = 0; i < R; ++i) slot = slot || x.rp[i] == p;
            if (!slot) f.push_back(p);
        }
        return f;
    };
    auto warp_pos = [&](uint64_t dep) {
        std::vector<int> w;
        for (int i = 5; i < whi; ++i) w.push_back((int)((dep >> (4 * i)) & 15));
        return w;
    };
    auto has = [](const std::vector<int> &v, int p) { return std::find(v.begin(), v.end(), p) != v.end(); };
    auto is_direct = [&](int k) { return (k == 0 && first_direct) || (k == nb - 1 && last_direct); };
    // the dep of batch k with warp positions w, or 0 when the lane rules fail
    auto layout = [&](int k, const std::vector<int> &w) -> uint64_t {
        const std::vector<int> f = free_of(bt[k]);
        std::vector<int> rest;
        for (int p : f)
            if (!has(w, p)) rest.push_back(p);
        for (int p : w)
            if (!has(f, p)) return 0;
        std::vector<int> lanes;
        if (is_direct(k) && tile_warp_local() == 2) return w == warp_pos(bt[k].dep) ? bt[k].dep : 0;  // A/B
        if (is_direct(k)) {
            // HBM runs: the contiguous low positions stay lane bits (a warp moves runs of 2^L amplitudes)
            for (int p : w)
                if (p < L) return 0;
            lanes = rest;  // ascending
            const bool was_coal = (bt[k].dep & 0xFFull) == 0x10ull;
            if (was_coal && !(lanes.size() >= 2 && lanes[0] == 0 && lanes[1] == 1)) return 0;
        } else {
            int cover = 0;
            for (int p : rest) cover |= 1 << (p % 3);
            if (cover != 7 && rest.size() >= 3) return 0;
            lanes = lane_first_order(rest);
        }
        std::vector<int> order(lanes.begin(), lanes.begin() + std::min<size_t>(5, lanes.size()));
        order.insert(order.end(), w.begin(), w.end());
        if (lanes.size() > 5) order.insert(order.end(), lanes.begin() + 5, lanes.end());
        return pack_dep(order);
    };
    // candidates per batch: its current dep (index 0), then every nw-subset of its non-slot positions
    // (ascending) whose layout keeps the lane rules; a dynamic program over the batches takes the
    // candidate sequence with the most equal consecutive warp positions (ties keep current deps)
    std::vector<std::vector<uint64_t>> cand(nb);
    for (int k = 0; k < nb; ++k) {
        cand[k].push_back(bt[k].dep);
        const std::vector<int> f = free_of(bt[k]);
        const int nf = (int)f.size();
        std::vector<int> idx(nw);
        for (int i = 0; i < nw; ++i) idx[i] = i;
        while (nf >= nw) {
            std::vector<int> w;
            for (int i = 0; i < nw; ++i) w.push_back(f[idx[i]]);
            const uint64_t d = layout(k, w);
            if (d && d != bt[k].dep) cand[k].push_back(d);
            int i = nw - 1;
            while (i >= 0 && idx[i] == nf - nw + i) --i;
            if (i < 0) break;
            ++idx[i];
            for (int t = i + 1; t < nw; ++t) idx[t] = idx[t - 1] + 1;
        }
    }
    // transition score: 0 = CTA barrier, up to nw = warp-local (transition_scope: the lowest warp bits that
    // may differ between the two batches; a group of 2^scope warps then exchanges data only within itself)
    auto same_warp = [&](uint64_t a, uint64_t c) { return nw - transition_scope(a, c, nsb, tpb); };
    std::vector<std::vector<int>> score(nb), from(nb);
    score[0].assign(cand[0].size(), 0);
    from[0].assign(cand[0].size(), -1);
    for (int k = 1; k < nb; ++k) {
        score[k].assign(cand[k].size(), -1);
        from[k].assign(cand[k].size(), 0);
        for (size_t c = 0; c < cand[k].size(); ++c)
            for (size_t p = 0; p < cand[k - 1].size(); ++p) {
                const int v = score[k - 1][p] + same_warp(cand[k - 1][p], cand[k][c]);
                if (v > score[k][c]) score[k][c] = v, from[k][c] = (int)p;
            }
    }
    int c = 0;
    for (size_t x = 1; x < cand[nb - 1].size(); ++x)
        if (score[nb - 1][x] > score[nb - 1][c]) c = (int)x;
    for (int k = nb - 1; k >= 0; --k) {
        bt[k].dep = cand[k][c];
        c = from[k][c];
    }
}

}  // namespace

int transition_scope(uint64_t dep_a, uint64_t dep_b, int nsub_bits, int tpb) {
    int wb = 0;
    while ((1 << (wb + 1)) <= tpb) ++wb;
    const int whi = std::min(wb, nsub_bits);
    int k = std::max(0, whi - 5);  // warp bits 5 + k .. whi - 1 must agree
    while (k > 0 && ((dep_a >> (4 * (5 + k - 1))) & 15) == ((dep_b >> (4 * (5 + k - 1))) & 15)) --k;
    return k;
}

bool warp_local_transition(uint64_t dep_a, uint64_t dep_b, int nsub_bits, int tpb) {
    return transition_scope(dep_a, dep_b, nsub_bits, tpb) == 0;
}

bool set_tile_perm(TileDesc &desc, const int *tile_q, int b, const int *perm, int m) {
    int pos[64];
    for (int q = 0; q < 64; ++q) pos[q] = -1;
    for (int i = 0; i < b; ++i) pos[tile_q[i]] = i;
    for (int i = 0; i < b; ++i) {
        const int pq = perm[tile_q[i]];
        if (pq < 0 || pq >= m || pos[pq] < 0 || perm[pq] != tile_q[i]) return false;
    }
    for (int i = 0; i < desc.n_out; ++i) {
        const int pq = perm[desc.out_q[i]];
        if (pq < 0 || pq >= m || pos[pq] >= 0 || perm[pq] != desc.out_q[i]) return false;
    }
    // tile-index order (DRAM locality of the pairs in flight): the outside qubits below 12 that pi fixes
    // first (the tiles sharing a 4-KiB..64-KiB span, and so their partners, are neighbours), then the
    // moved qubits pair by pair (x, pi(x)), so a window of consecutive indices covers every combination of
    // the low moved bits on BOTH sides of the pairs, then the rest ascending
    {
        std::vector<int> ord, used(64, 0);
        for (int i = 0; i < desc.n_out; ++i) {
            const int q = desc.out_q[i];
            if (q < 12 && perm[q] == q) ord.push_back(q), used[q] = 1;
        }
        for (int i = 0; i < desc.n_out; ++i) {
            const int q = desc.out_q[i];
            if (used[q] || perm[q] == q) continue;
            ord.push_back(q), used[q] = 1;
            ord.push_back(perm[q]), used[perm[q]] = 1;
        }
        for (int i = 0; i < desc.n_out; ++i)
            if (!used[desc.out_q[i]]) ord.push_back(desc.out_q[i]);
        for (int i = 0; i < desc.n_out; ++i) {
            desc.out_q[i] = ord[i];
            desc.out_pq[i] = perm[ord[i]];
        }
    }
    for (int k = 0; k < 3; ++k)
        for (int x = 0; x < 16; ++x) {
            uint32_t r = 0;
            for (int i = 0; i < 4; ++i) {
                const int p = 4 * k + i;
                if (p < b && ((x >> i) & 1)) r |= 1u << pos[perm[tile_q[p]]];
            }
            desc.rho[k][x] = (uint16_t)r;
        }
    desc.perm = 1;
    return true;
}

void make_tile_pass(const int *tile_q, int b, int L, int m, const Op *local_ops, int nops, TileDesc &desc,
                    std::vector<TileBatch> &batches, std::vector<TileOp> &ops, std::vector<TileLadder> &lads,
                    int ladder_min, bool reorder_batches) {
    const int R = tile_regs();
    desc = TileDesc();
    desc.b = b;
    desc.L = L;
    desc.n_hi = b - L;
    for (int i = 0; i < b - L; ++i) desc.hi_q[i] = tile_q[L + i];
    int pos[64];
    for (int q = 0; q < 64; ++q) pos[q] = -1;
    for (int i = 0; i < b; ++i) pos[tile_q[i]] = i;
    int no = 0;
    for (int q = 0; q < m; ++q)
        if (pos[q] < 0) desc.out_q[no++] = q;
    desc.n_out = no;
    desc.batch0 = (int32_t)batches.size();
    desc.op_begin = (int32_t)ops.size();
    const size_t lad_begin = lads.size();
    int nquad = 0;
    // shared-memory budget of the op stream: the planner sized the pass for 80 B per op + 256 B per
    // QUAD; a ladder (one op record + its TileLadder) is only formed while the total still fits
    size_t op_bytes = 0;
    for (int i = 0; i < nops; ++i) op_bytes += 80 + (local_ops[i].kind == OP_QUAD ? 256 : 0);

    // greedy batches: non-diagonal ops of a batch use <= R tile positions; order kept
    std::vector<int> cur, need;
    std::vector<int> members;
    auto close = [&]() {
        if (members.empty()) return;
        std::vector<int> rp = cur;
        for (int p = b - 1; (int)rp.size() < R && p >= 0; --p)  // fill with the highest free positions
            if (std::find(rp.begin(), rp.end(), p) == rp.end()) rp.push_back(p);
        std::sort(rp.begin(), rp.end());
        TileBatch bt = TileBatch();
        for (int i = 0; i < TILE_R; ++i) bt.rp[i] = i < R ? rp[i] : 31;
        for (int r = 0; r < 16; ++r) {
            uint32_t off = 0;
            for (int i = 0; i < R; ++i) off |= (uint32_t)((r >> i) & 1) << rp[i];
            bt.swo[r] = r < (1 << R) ? swz(off) : 0;
        }
        {   // sub-cube bits -> the non-slot positions; lane bits first, covering every residue mod 3
            std::vector<int> free_pos;
            for (int p = 0; p < b; ++p)
                if (std::find(rp.begin(), rp.end(), p) == rp.end()) free_pos.push_back(p);
            bt.dep = pack_dep(lane_first_order(free_pos));
        }
        bt.op0 = (int32_t)ops.size();
        bt.nops = 0;  // set after the ladder merge below
        // slot of qubit q in this batch (0..R-1) or 4 (not a register slot) with its bit source
        auto slot_src = [&](int q, int &slot, int32_t &src) {
            slot = 4;
            src = -1;
            if (q < 0) return;
            const int p = pos[q];
            for (int i = 0; i < R; ++i)
                if (rp[i] == p) slot = i;
            if (slot == 4) src = p >= 0 ? p : -2 - q;
        };
        std::vector<TileOp> bops;
        for (int oi : members) {
            const Op &op = local_ops[oi];
            TileOp t = TileOp();
            int s0, s1;
            slot_src(op.q0, s0, t.src0);
            slot_src(op.q1, s1, t.src1);
            t.code = tile_opcode(op.kind, s0, s1);
            if (op.kind == OP_PAIR && op.m[1] == 0.0 && op.m[3] == 0.0 && op.m[5] == 0.0 && op.m[7] == 0.0)
                t.code = 150 + s0;  // real matrix (H): half the FP64 work, same values
            t.touch = op.kind == OP_QUAD ? (uint32_t)nquad++ : op.touch;
            const int nm = op.kind == OP_QUAD ? 16 : 4;
            for (int k = 0; k < nm; ++k) t.m[k] = make_double2(op.m[2 * k], op.m[2 * k + 1]);
            if (op.kind == OP_CTRL_PAIR && t.code >= 4 && t.code <= 19) {  // CNOT-like: monomial entries
                int e[4], ok = 1;
                for (int k = 0; k < 4; ++k) ok &= (e[k] = mono_code(op.m + 2 * k)) >= 0;
                if (ok) {
                    t.code = 169 + (t.code - 4);
                    t.touch = (uint32_t)(e[0] | e[1] << 4 | e[2] << 8 | e[3] << 12);
                }
            }
            if (op.kind == OP_PAIR) {  // monomial entries (after scalar factoring): additions only;
                int e[4], ok = 1;       // w(+-1+-i) entries (form 1) add one FMA per component
                double w = 0.0;
                for (int k = 0; k < 4; ++k) {
                    double wk = 0.0;
                    e[k] = op.form == 1 ? mono_code_w(op.m + 2 * k, &wk) : mono_code(op.m + 2 * k);
                    ok &= e[k] >= 0 && (wk == 0.0 || w == 0.0 || wk == w);
                    if (wk != 0.0) w = wk;
                }
                if (ok) {
                    t.code = 165 + s0;
                    t.touch = (uint32_t)(e[0] | e[1] << 4 | e[2] << 8 | e[3] << 12);
                    t.m[0] = make_double2(w, 0.0);
                }
            }
            if (op.kind == OP_DIAG) {  // single touched k with all constrained bits 1 -> phase form
                const int nq = op.q0 < 0 ? 0 : (op.q1 < 0 ? 1 : 2);
                const uint32_t kall = (1u << nq) - 1;
                if (op.touch == (1u << kall)) {
                    int a = 4, bb = 4;
                    int32_t fa = -1000, fb = -1000;
                    const int qs[2] = {op.q0, op.q1};
                    const int ss[2] = {s0, s1};
                    const int32_t srcs[2] = {t.src0, t.src1};
                    for (int j2 = 0; j2 < nq; ++j2) {
                        if (ss[j2] < 4) {
                            if (a == 4) a = ss[j2]; else bb = ss[j2];
                        } else {
                            if (fa == -1000) fa = srcs[j2]; else fb = srcs[j2];
                        }
                        (void)qs;
                    }
                    t.code = tile_phase_opcode(a, bb);
                    t.src0 = fa;
                    t.src1 = fb;
                    t.m[0] = make_double2(op.m[2 * kall], op.m[2 * kall + 1]);
                    if (op.m[2 * kall] == -1.0 && op.m[2 * kall + 1] == 0.0) t.code += 154 - 59;  // sign flip
                }
            }
            bops.push_back(t);
        }
        // PHASE LADDERS: merge runs of >= ladder_min consecutive pure-phase ops that share one
        // constrained qubit t ({c, t} -> control c, {t} -> constant), or that are all single-bit
        // phases (no t).  Longest run wins; order of the remaining ops is kept.
        const int N = (int)members.size();
        std::vector<int> nq(N, 0);
        std::vector<std::array<int, 2>> cq(N);
        std::vector<Cx> cxv(N);
        for (int j = 0; j < N; ++j) {
            int q2[2];
            if (phase_form(local_ops[members[j]], nq[j], q2, cxv[j])) cq[j] = {q2[0], q2[1]};
            else nq[j] = 0;
        }
        auto has = [&](int j, int q) { return nq[j] >= 1 && (cq[j][0] == q || (nq[j] == 2 && cq[j][1] == q)); };
        for (int i = 0; i < N;) {
            int best_len = 1, best_t = -2;
            if (ladder_min > 0 && nq[i] > 0) {
                for (int w = 0; w < nq[i]; ++w) {
                    const int t = cq[i][w];
                    int j = i;
                    while (j < N && has(j, t)) ++j;
                    if (j - i > best_len) best_len = j - i, best_t = t;
                }
                int j = i;
                while (j < N && nq[j] == 1) ++j;
                if (j - i > best_len) best_len = j - i, best_t = -1;
            }
            const size_t grow = 80 + sizeof(TileLadder), shrink = 80 * (size_t)best_len;
            const bool fits = op_bytes + grow <= (size_t)TILE_OP_SMEM + shrink;
            if (best_t == -2 || best_len < ladder_min || (int)(lads.size() - lad_begin) >= TILE_MAX_LADDERS || !fits) {
                ops.push_back(bops[i]);
                ++i;
                continue;
            }
            op_bytes = op_bytes + grow - shrink;
            // controls in first-seen order, factors multiplied in op order
            Cx k0 = {1.0, 0.0};
            std::vector<int> cl;
            std::vector<Cx> cv;
            for (int j = i; j < i + best_len; ++j) {
                int c = -1;
                if (best_t >= 0) {
                    if (nq[j] == 2) c = cq[j][0] == best_t ? cq[j][1] : cq[j][0];
                } else {
                    c = cq[j][0];
                }
                if (c < 0) {
                    k0 = cx_mul(k0, cxv[j]);
                    continue;
                }
                auto it = std::find(cl.begin(), cl.end(), c);
                if (it == cl.end()) {
                    cl.push_back(c);
                    cv.push_back(cxv[j]);
                } else {
                    cv[it - cl.begin()] = cx_mul(cv[it - cl.begin()], cxv[j]);
                }
            }
            TileLadder ld = TileLadder();
            ld.k0 = make_double2(k0.re, k0.im);
            for (int s2 = 0; s2 < 4; ++s2) ld.xs[s2] = make_double2(1.0, 0.0);
            Cx tpos[TILE_MAX_Q];
            bool tctl[TILE_MAX_Q] = {false};
            int mask = 0;
            for (size_t u = 0; u < cl.size(); ++u) {
                int slot;
                int32_t src;
                slot_src(cl[u], slot, src);
                if (slot < 4) {
                    ld.xs[slot] = make_double2(cv[u].re, cv[u].im);
                    mask |= 1 << slot;
                } else if (src >= 0) {
                    tpos[src] = cv[u];
                    tctl[src] = true;
                } else {
                    ld.bq[ld.nb] = cl[u];
                    ld.bx[ld.nb] = make_double2(cv[u].re, cv[u].im);
                    ++ld.nb;
                }
            }
            for (int k = 0; k < 3; ++k)
                for (int xv = 0; xv < 16; ++xv) {
                    Cx pr = {1.0, 0.0};
                    for (int bit = 0; bit < 4; ++bit) {
                        const int p = 4 * k + bit;
                        if (((xv >> bit) & 1) && p < TILE_MAX_Q && tctl[p]) pr = cx_mul(pr, tpos[p]);
                    }
                    ld.tj[k][xv] = make_double2(pr.re, pr.im);
                }
            TileOp t = TileOp();
            int st = 4;
            t.src0 = -1000;
            if (best_t >= 0) {
                int32_t src;
                slot_src(best_t, st, src);
                if (st == 4) t.src0 = src;
            }
            t.code = 70 + 16 * st + mask;
            t.src1 = -1000;
            t.touch = (uint32_t)(lads.size() - lad_begin);
            lads.push_back(ld);
            ops.push_back(t);
            i += best_len;
        }
        bt.nops = (int32_t)(ops.size() - (size_t)bt.op0);
        batches.push_back(bt);
        members.clear();
        cur.clear();
    };
    if (!reorder_batches) {
        for (int i = 0; i < nops; ++i) {
            needs(local_ops[i], pos, need);
            std::vector<int> u = cur;
            for (int p : need)
                if (std::find(u.begin(), u.end(), p) == u.end()) u.push_back(p);
            if ((int)u.size() > R) {
                close();
                u = need;
            }
            cur = u;
            members.push_back(i);
        }
        close();
    } else {
        // batches through the pass's dependency DAG (the planner's rule: an op waits for the previous
        // non-diagonal op on each of its qubits; a non-diagonal op also for the diagonal ops since):
        // a batch takes every ready op whose register positions are in its slot set, growing the set
        // by the position that completes the most ready ops — fewer shared-memory round trips
        std::vector<std::vector<int>> succ(nops), nd(nops);
        std::vector<int> npred(nops, 0), lastnd(64, -1);
        std::vector<std::vector<int>> dsince(64);
        auto edge = [&](int a, int c) {
            if (a < 0) return;
            succ[a].push_back(c);
            ++npred[c];
        };
        for (int k = 0; k < nops; ++k) {
            const Op &op = local_ops[k];
            needs(op, pos, nd[k]);
            const bool dg = op.kind == OP_DIAG;
            int qq[2], nq = 0;
            if (op.q0 >= 0) qq[nq++] = op.q0;
            if (op.q1 >= 0) qq[nq++] = op.q1;
            if (nq == 0) {  // whole-state scale: a barrier
                for (int a = 0; a < k; ++a) edge(a, k);
                for (int q = 0; q < 64; ++q) lastnd[q] = k, dsince[q].clear();
                continue;
            }
            for (int u = 0; u < nq; ++u) {
                edge(lastnd[qq[u]], k);
                if (dg) {
                    dsince[qq[u]].push_back(k);
                } else {
                    for (int dd : dsince[qq[u]]) edge(dd, k);
                    dsince[qq[u]].clear();
                }
            }
            if (!dg)
                for (int u = 0; u < nq; ++u) lastnd[qq[u]] = k;
        }
        // several greedy partitions (the first deterministic: grow by the position whose addition lets
        // the batch take the most ops transitively; later trials pick at random among the near-best);
        // the partition with the fewest batches is emitted (fewer shared-memory round trips)
        auto partition = [&](uint64_t seed) {
            std::vector<std::vector<int>> parts, slots;
            std::vector<int> np = npred;
            std::set<int> ready;
            for (int k = 0; k < nops; ++k)
                if (np[k] == 0) ready.insert(k);
            uint64_t rng = seed * 0x9E3779B97F4A7C15ull + 7;
            std::vector<int> mem, cs, tnp;
            std::vector<int> queue;
            int done = 0;
            while (done < nops) {
                cs.clear();
                mem.clear();
                for (;;) {
                    bool took = true;
                    while (took) {
                        took = false;
                        for (auto it = ready.begin(); it != ready.end(); ++it) {
                            const int k = *it;
                            bool fits = true;
                            for (int p : nd[k]) fits = fits && std::find(cs.begin(), cs.end(), p) != cs.end();
                            if (!fits) continue;
                            ready.erase(it);
                            mem.push_back(k);
                            ++done;
                            for (int c : succ[k])
                                if (--np[c] == 0) ready.insert(c);
                            took = true;
                            break;  // rescan from the lowest index
                        }
                    }
                    if ((int)cs.size() >= R || ready.empty()) break;
                    int best = -1, bscore = 0;
                    std::vector<int> score(b, 0);
                    for (int p = 0; p < b; ++p) {
                        if (std::find(cs.begin(), cs.end(), p) != cs.end()) continue;
                        // transitive closure of what the batch could take with p added
                        cs.push_back(p);
                        tnp = np;
                        queue.assign(ready.begin(), ready.end());
                        int sc = 0;
                        for (size_t qi = 0; qi < queue.size(); ++qi) {
                            const int k = queue[qi];
                            bool fits = true;
                            for (int q : nd[k]) fits = fits && std::find(cs.begin(), cs.end(), q) != cs.end();
                            if (!fits) continue;
                            ++sc;
                            for (int c : succ[k])
                                if (--tnp[c] == 0) queue.push_back(c);
                        }
                        cs.pop_back();
                        score[p] = sc;
                        if (sc > bscore) bscore = sc, best = p;
                    }
                    if (seed != 0 && best >= 0) {
                        int nc = 0;
                        for (int p = 0; p < b; ++p) nc += score[p] > 0 && score[p] >= bscore - 1;
                        rng = rng * 6364136223846793005ull + 1442695040888963407ull;
                        int pick = (int)((rng >> 33) % (uint64_t)nc);
                        for (int p = 0; p < b; ++p)
                            if (score[p] > 0 && score[p] >= bscore - 1 && pick-- == 0) {
                                best = p;
                                break;
                            }
                    }
                    if (best < 0) {  // an op needing two more positions
                        for (int k : ready) {
                            int miss = 0;
                            for (int q : nd[k]) miss += std::find(cs.begin(), cs.end(), q) == cs.end();
                            if (miss > 0 && (int)cs.size() + miss <= R) {
                                for (int q : nd[k])
                                    if (std::find(cs.begin(), cs.end(), q) == cs.end()) cs.push_back(q);
                                best = 0;
                                break;
                            }
                        }
                        if (best < 0) break;
                    } else {
                        cs.push_back(best);
                    }
                }
                if (mem.empty()) {  // not expected: take the lowest ready op alone
                    const int k = *ready.begin();
                    ready.erase(ready.begin());
                    mem.push_back(k);
                    ++done;
                    for (int c : succ[k])
                        if (--np[c] == 0) ready.insert(c);
                    cs = nd[k];
                }
                parts.push_back(mem);
                slots.push_back(cs);
            }
            return std::make_pair(parts, slots);
        };
        static const int trials = getenv("QS_BATCH_TRIALS") ? std::max(1, atoi(getenv("QS_BATCH_TRIALS"))) : 32;
        auto bestp = partition(0);
        for (int t = 1; t < trials; ++t) {
            auto p = partition((uint64_t)t);
            if (p.first.size() < bestp.first.size()) bestp.swap(p);
        }
        for (size_t i = 0; i < bestp.first.size(); ++i) {
            members = bestp.first[i];
            cur = bestp.second[i];
            close();
        }
    }
    desc.nbatch = (int32_t)batches.size() - desc.batch0;
    if (tile_direct_io() && desc.nbatch > 0) {
        // direct-I/O batches (the first reads HBM, the last writes it): lanes on the lowest non-slot
        // positions, so a warp's accesses cover contiguous runs (any lane order gives the same values)
        for (int k : {desc.batch0, desc.batch0 + desc.nbatch - 1}) {
            const int dio = tile_direct_io() & 8 ? 3 : tile_direct_io();
            if (!((k == desc.batch0 ? 1 : 0) & dio) && !((k == desc.batch0 + desc.nbatch - 1 ? 2 : 0) & dio)) continue;
            TileBatch &bt = batches[k];
            std::vector<int> order;
            for (int p = 0; p < b; ++p) {
                bool slot = false;
                for (int i = 0; i < R; ++i) slot = slot || bt.rp[i] == p;
                if (!slot) order.push_back(p);
            }
            bt.dep = 0;
            for (size_t i = 0; i < order.size() && i < 12; ++i) bt.dep |= (uint64_t)order[i] << (4 * i);
        }
    }
    if (tile_warp_local() && desc.nbatch > 1) {
        const int dio = tile_direct_io() & 8 ? 3 : tile_direct_io();
        align_warp_bits(batches.data() + desc.batch0, desc.nbatch, b, L, R, jit_tile_threads(b, R), (dio & 1) != 0,
                        (dio & 2) != 0);
    }
    desc.op_count = (int32_t)ops.size() - desc.op_begin;
    desc.quad_count = nquad;
    desc.lad_count = (int32_t)(lads.size() - lad_begin);
    desc.lads = nullptr;  // the caller points it at the device copy of lads[lad_begin ..)
}

int launch_tile(double2 *a, int m, const TileDesc &hdesc, const TileDesc *ddesc, const TileBatch *dbatches,
                const TileOp *dops, cudaStream_t st, int num_sms) {
    static uint64_t attr_mask = 0;  // per device
    const size_t smem = (size_t)2 * (16 << hdesc.b) + tile_op_bytes(hdesc);
    const int maxsmem = (int)((size_t)2 * (16 << TILE_MAX_Q) + TILE_OP_SMEM);
    if (tile_op_bytes(hdesc) > TILE_OP_SMEM) return -1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (!((attr_mask >> dev) & 1)) {
        cudaFuncSetAttribute(k_tile<4, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsmem);
        cudaFuncSetAttribute(k_tile<4, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsmem);
        cudaFuncSetAttribute(k_tile<3, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsmem);
        cudaFuncSetAttribute(k_tile<3, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsmem);
        attr_mask |= 1ull << dev;
    }
    if (hdesc.n_out > 27) return -1;  // tile-index deposit tables: 7 nibbles (n_out <= 27)
    const uint64_t ntiles = 1ull << (m - hdesc.b);
    uint64_t g = (uint64_t)num_sms;
    if (g > ntiles) g = ntiles;
    const int R = tile_regs();
    const int sub = 1 << (hdesc.b - R);
    if (R == 4) {
        if (sub >= 256)
            k_tile<4, 256><<<(unsigned)g, 256, smem, st>>>(a, ntiles, ddesc, dbatches, dops);
        else
            k_tile<4, 64><<<(unsigned)g, 64, smem, st>>>(a, ntiles, ddesc, dbatches, dops);
    } else {
        if (sub >= 512)
            k_tile<3, 512><<<(unsigned)g, 512, smem, st>>>(a, ntiles, ddesc, dbatches, dops);
        else
            k_tile<3, 64><<<(unsigned)g, 64, smem, st>>>(a, ntiles, ddesc, dbatches, dops);
    }
    return 1;
}

}  // namespace qsb
