// qs_plan.cpp — see qs_plan.h.  Pure host code.
#include "qs_plan.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <functional>
#include <set>
#include <thread>

namespace qsb {

namespace {

inline bool is_one(const double *c) { return c[0] == 1.0 && c[1] == 0.0; }
inline bool is_zero(const double *c) { return c[0] == 0.0 && c[1] == 0.0; }

// max |U^H U - I| for a d x d row-major interleaved complex matrix
double unitarity_defect(const double *m, int d) {
    double worst = 0.0;
    for (int i = 0; i < d; ++i)
        for (int j = 0; j < d; ++j) {
            double re = 0.0, im = 0.0;  // sum_r conj(U[r][i]) U[r][j]
            for (int r = 0; r < d; ++r) {
                const double *a = m + 2 * (d * r + i);
                const double *b = m + 2 * (d * r + j);
                re += a[0] * b[0] + a[1] * b[1];
                im += a[0] * b[1] - a[1] * b[0];
            }
            if (i == j) re -= 1.0;
            worst = std::max(worst, std::max(std::fabs(re), std::fabs(im)));
        }
    return worst;
}

void set_touch(Op &op, int nd) {
    op.touch = 0;
    for (int k = 0; k < nd; ++k)
        if (!is_one(&op.m[2 * k])) op.touch |= 1u << k;
}

}  // namespace

bool classify(int n, int32_t kind, int32_t q0, int32_t q1, const double *m, bool check_unitary, Op &out,
              std::string &msg) {
    if (!m) {
        msg = "NULL matrix";
        return false;
    }
    if (kind < 0 || kind > 2) {
        msg = "unknown gate kind " + std::to_string(kind);
        return false;
    }
    if (q0 < 0 || q0 >= n) {
        msg = "qubit " + std::to_string(q0) + " outside [0, " + std::to_string(n) + ")";
        return false;
    }
    if (kind != 0) {
        if (q1 < 0 || q1 >= n) {
            msg = "qubit " + std::to_string(q1) + " outside [0, " + std::to_string(n) + ")";
            return false;
        }
        if (q1 == q0) {
            msg = kind == 1 ? "ctrl == target" : "q0 == q1";
            return false;
        }
    }
    const int d = kind == 2 ? 4 : 2;
    for (int i = 0; i < 2 * d * d; ++i)
        if (!std::isfinite(m[i])) {
            msg = "non-finite matrix entry";
            return false;
        }
    if (check_unitary) {
        double defect = unitarity_defect(m, d);
        if (defect > 1e-10) {
            msg = "matrix is not unitary (max|U^H U - I| = " + std::to_string(defect) + ")";
            return false;
        }
    }
    out = Op();
    if (kind == 0 || kind == 1) {
        const double *u00 = m, *u01 = m + 2, *u10 = m + 4, *u11 = m + 6;
        bool diag = is_zero(u01) && is_zero(u10);
        if (kind == 0) {
            if (diag) {
                out.kind = OP_DIAG;
                out.q0 = q0;
                out.q1 = -1;
                std::memcpy(&out.m[0], u00, 16);
                std::memcpy(&out.m[2], u11, 16);
                set_touch(out, 2);
            } else {
                out.kind = OP_PAIR;
                out.q0 = q0;
                std::memcpy(out.m, m, 8 * sizeof(double));
            }
        } else {
            if (diag) {  // k = bit_c + 2 bit_t: d = {1, u00, 1, u11}
                out.kind = OP_DIAG;
                out.q0 = q0;
                out.q1 = q1;
                out.m[0] = 1.0;
                std::memcpy(&out.m[2], u00, 16);
                out.m[4] = 1.0;
                std::memcpy(&out.m[6], u11, 16);
                set_touch(out, 4);
            } else {
                out.kind = OP_CTRL_PAIR;
                out.q0 = q0;
                out.q1 = q1;
                std::memcpy(out.m, m, 8 * sizeof(double));
            }
        }
        return true;
    }
    // 2q
    bool diag = true, swap = true;
    for (int r = 0; r < 4; ++r)
        for (int c = 0; c < 4; ++c) {
            const double *e = m + 2 * (4 * r + c);
            if (r != c && !is_zero(e)) diag = false;
            int sc = (r == 1) ? 2 : (r == 2) ? 1 : r;  // SWAP permutation
            if (c == sc ? !is_one(e) : !is_zero(e)) swap = false;
        }
    out.q0 = q0;
    out.q1 = q1;
    if (diag) {
        out.kind = OP_DIAG;
        for (int k = 0; k < 4; ++k) std::memcpy(&out.m[2 * k], m + 2 * (4 * k + k), 16);
        set_touch(out, 4);
    } else if (swap) {
        out.kind = OP_SWAP;
    } else {
        out.kind = OP_QUAD;
        std::memcpy(out.m, m, 32 * sizeof(double));
    }
    return true;
}

ShardStep localize(const Op &op, int n, int m, int rank) {
    (void)n;
    ShardStep st;
    auto G = [&](int q) { return q >= m; };
    auto rb = [&](int q) { return (rank >> (q - m)) & 1; };
    switch (op.kind) {
    case OP_DIAG: {
        int nq = op.q0 < 0 ? 0 : (op.q1 < 0 ? 1 : 2);
        int slot_q[2] = {op.q0, op.q1};
        int local_slot[2], nl = 0, fixed_k = 0;
        for (int s = 0; s < nq; ++s) {
            if (G(slot_q[s]))
                fixed_k |= rb(slot_q[s]) << s;
            else
                local_slot[nl++] = s;
        }
        Op lo;
        lo.kind = OP_DIAG;
        lo.q0 = nl > 0 ? slot_q[local_slot[0]] : -1;
        lo.q1 = nl > 1 ? slot_q[local_slot[1]] : -1;
        for (int kl = 0; kl < (1 << nl); ++kl) {
            int k = fixed_k;
            for (int j = 0; j < nl; ++j) k |= ((kl >> j) & 1) << local_slot[j];
            lo.m[2 * kl] = op.m[2 * k];
            lo.m[2 * kl + 1] = op.m[2 * k + 1];
        }
        set_touch(lo, 1 << nl);
        if (lo.touch == 0) return st;
        st.action = SA_LOCAL;
        st.local = lo;
        return st;
    }
    case OP_PAIR:
        if (!G(op.q0)) {
            st.action = SA_LOCAL;
            st.local = op;
        } else {
            st.action = SA_XPAIR;
            st.partner = rank ^ (1 << (op.q0 - m));
            st.bit = rb(op.q0);
            st.local = op;
        }
        return st;
    case OP_CTRL_PAIR: {
        int c = op.q0, t = op.q1;
        if (!G(c) && !G(t)) {
            st.action = SA_LOCAL;
            st.local = op;
        } else if (G(c) && !G(t)) {
            if (!rb(c)) return st;
            st.action = SA_LOCAL;
            st.local = op;
            st.local.kind = OP_PAIR;
            st.local.q0 = t;
            st.local.q1 = -1;
        } else {
            if (G(c) && !rb(c)) return st;
            st.action = SA_XPAIR;
            st.partner = rank ^ (1 << (t - m));
            st.bit = rb(t);
            st.ctrl_local = G(c) ? -1 : c;
            st.local = op;
        }
        return st;
    }
    case OP_SWAP: {
        int a = op.q0, b = op.q1;
        if (!G(a) && !G(b)) {
            st.action = SA_LOCAL;
            st.local = op;
        } else if (G(a) && G(b)) {
            if (rb(a) == rb(b)) return st;
            st.action = SA_XSWAP_GG;
            st.partner = rank ^ (1 << (a - m)) ^ (1 << (b - m));
        } else {
            int g = G(a) ? a : b, l = G(a) ? b : a;
            st.action = SA_XSWAP_LG;
            st.partner = rank ^ (1 << (g - m));
            st.bit = rb(g);
            st.l = l;
        }
        return st;
    }
    case OP_QUAD:
    default:
        if (!G(op.q0) && !G(op.q1)) {
            st.action = SA_LOCAL;
            st.local = op;
        } else {
            st.action = SA_VIA_SWAP;
        }
        return st;
    }
}

std::vector<Op> decompose_via_swap(const Op &op, int m) {
    std::vector<Op> out;
    int qs[2] = {op.q0, op.q1};
    int nq = op.kind == OP_PAIR ? 1 : 2;
    std::vector<int> used;
    for (int i = 0; i < nq; ++i) used.push_back(qs[i]);
    Op moved = op;
    int *slots[2] = {&moved.q0, &moved.q1};
    std::vector<std::pair<int, int>> swaps;
    int f = m - 1;
    for (int i = 0; i < nq; ++i) {
        if (qs[i] < m) continue;
        while (f >= 0 && std::find(used.begin(), used.end(), f) != used.end()) --f;
        if (f < 0) return {};  // no free local qubit (cannot happen for m >= 3)
        swaps.push_back({qs[i], f});
        used.push_back(f);
        *slots[i] = f;
        --f;
    }
    for (auto &s : swaps) {
        Op sw;
        sw.kind = OP_SWAP;
        sw.q0 = s.second;  // local
        sw.q1 = s.first;   // global
        out.push_back(sw);
    }
    out.push_back(moved);
    for (auto it = swaps.rbegin(); it != swaps.rend(); ++it) {
        Op sw;
        sw.kind = OP_SWAP;
        sw.q0 = it->second;
        sw.q1 = it->first;
        out.push_back(sw);
    }
    return out;
}

int exchange_cost(const std::vector<Op> &ops, int m) {
    int c = 0;
    for (const Op &op : ops) {
        const bool g0 = op.q0 >= m, g1 = op.q1 >= m;
        switch (op.kind) {
        case OP_PAIR: c += g0 ? 2 : 0; break;
        case OP_CTRL_PAIR: c += g1 ? (g0 ? 2 : 1) : 0; break;
        case OP_QUAD: c += 2 * (int)g0 + 2 * (int)g1; break;
        case OP_SWAP: c += (g0 && g1) ? 2 : (g0 || g1) ? 1 : 0; break;
        default: break;
        }
    }
    return c;
}

// ---------------------------------------------------------------------------------------------
// Scalar factoring: see qs_plan.h.
// ---------------------------------------------------------------------------------------------
int mono_code(const double *e) {  // 0, 1, -1, i, -i -> 0..4; -1 if not one of them
    if (e[0] == 0.0 && e[1] == 0.0) return 0;
    if (e[0] == 1.0 && e[1] == 0.0) return 1;
    if (e[0] == -1.0 && e[1] == 0.0) return 2;
    if (e[0] == 0.0 && e[1] == 1.0) return 3;
    if (e[0] == 0.0 && e[1] == -1.0) return 4;
    return -1;
}

int mono_code_w(const double *e, double *w) {
    const int c = mono_code(e);
    if (c >= 0) return c;
    const double re = e[0], im = e[1];
    if (!(std::fabs(re) == std::fabs(im)) || re == 0.0 || !std::isfinite(re)) return -1;
    *w = std::fabs(re);
    return re > 0 ? (im > 0 ? 5 : 6) : (im > 0 ? 7 : 8);
}

namespace {

// U = c M with every entry of M either e*c EXACTLY for e in {0, +-1, +-i} (the products are exact),
// or c*(w a, w b) == u EXACTLY (one double complex product, a, b = +-1) with one shared real w > 0.
// c = the first nonzero entry.  Writes M to mm; form = 1 if a w entry occurs.
bool cheap_factor(const double *m, double c[2], double mm[8], int &form) {
    int f = -1;
    for (int k = 0; k < 4 && f < 0; ++k)
        if (m[2 * k] != 0.0 || m[2 * k + 1] != 0.0) f = k;
    if (f < 0) return false;
    c[0] = m[2 * f];
    c[1] = m[2 * f + 1];
    form = 0;
    double wshared = 0.0;
    for (int k = 0; k < 4; ++k) {
        const double re = m[2 * k], im = m[2 * k + 1];
        double e[2];
        if (re == 0.0 && im == 0.0) e[0] = 0.0, e[1] = 0.0;
        else if (re == c[0] && im == c[1]) e[0] = 1.0, e[1] = 0.0;
        else if (re == -c[0] && im == -c[1]) e[0] = -1.0, e[1] = 0.0;
        else if (re == -c[1] && im == c[0]) e[0] = 0.0, e[1] = 1.0;   // i c
        else if (re == c[1] && im == -c[0]) e[0] = 0.0, e[1] = -1.0;  // -i c
        else {
            bool found = false;
            for (int ab = 0; ab < 4 && !found; ++ab) {
                const double a = (ab & 1) ? -1.0 : 1.0, b = (ab & 2) ? -1.0 : 1.0;
                const double dre = a * c[0] - b * c[1], dim = a * c[1] + b * c[0];  // c (a + b i)
                const double w = dre != 0.0 ? re / dre : (dim != 0.0 ? im / dim : 0.0);
                if (!(w > 0.0) || !std::isfinite(w) || (wshared != 0.0 && w != wshared)) continue;
                const double pre = c[0] * (w * a) - c[1] * (w * b), pim = c[0] * (w * b) + c[1] * (w * a);
                if (pre == re && pim == im) {
                    found = true;
                    wshared = w;
                    e[0] = w * a;
                    e[1] = w * b;
                }
            }
            if (!found) return false;
            form = 1;
        }
        mm[2 * k] = e[0];
        mm[2 * k + 1] = e[1];
    }
    return true;
}

}  // namespace

std::vector<Op> factor_scalars(const std::vector<Op> &ops) {
    std::vector<Op> out;
    out.reserve(ops.size() + 2);
    double C[2] = {1.0, 0.0};
    double lg = 0.0;  // log2 |C|
    auto flush = [&]() {
        if (C[0] == 1.0 && C[1] == 0.0) return;
        Op sc;  // scale the whole state (DIAG over no qubit)
        sc.kind = OP_DIAG;
        sc.q0 = sc.q1 = -1;
        sc.m[0] = C[0];
        sc.m[1] = C[1];
        sc.touch = 1;
        out.push_back(sc);
        C[0] = 1.0, C[1] = 0.0;
        lg = 0.0;
    };
    for (const Op &op : ops) {
        double c[2], mm[8];
        int form = 0;
        if (op.kind == OP_PAIR && cheap_factor(op.m, c, mm, form) && !(c[0] == 1.0 && c[1] == 0.0)) {
            Op o = op;
            for (int i = 0; i < 8; ++i) o.m[i] = mm[i];
            o.form = form;
            out.push_back(o);
            const double re = C[0] * c[0] - C[1] * c[1], im = C[0] * c[1] + C[1] * c[0];
            C[0] = re, C[1] = im;
            lg += std::log2(std::hypot(c[0], c[1]));
            if (std::fabs(lg) > 400.0) flush();  // keep the deferred magnitude far from over/underflow
            continue;
        }
        out.push_back(op);
    }
    // the final factor goes right after the last non-SWAP op, so it joins that op's tile pass instead
    // of trailing SWAP runs (permutation passes / exchanges) and costing a pass of its own
    size_t at = out.size();
    while (at > 0 && out[at - 1].kind == OP_SWAP) --at;
    std::vector<Op> tail(out.begin() + at, out.end());
    out.resize(at);
    flush();
    out.insert(out.end(), tail.begin(), tail.end());
    return out;
}

// ---------------------------------------------------------------------------------------------
// Global-qubit remapping: see qs_plan.h.
// ---------------------------------------------------------------------------------------------
namespace {

// logical qubits this op needs LOCAL to run without an exchange (non-diagonal roles)
int remap_needs(const Op &op, int q[2]) {
    switch (op.kind) {
    case OP_PAIR: q[0] = op.q0; return 1;
    case OP_CTRL_PAIR: q[0] = op.q1; return 1;  // a global control is a rank predicate
    case OP_QUAD: q[0] = op.q0; q[1] = op.q1; return 2;
    default: return 0;                          // DIAG: never; SWAP: relabelled
    }
}

Op make_swap(int a, int b) {
    Op sw;
    sw.kind = OP_SWAP;
    sw.q0 = std::min(a, b);
    sw.q1 = std::max(a, b);
    return sw;
}

}  // namespace

std::vector<Op> remap_global(const std::vector<Op> &ops, int n, int m) {
    std::vector<Op> out;
    if (m >= n) return ops;
    const int G = (int)ops.size();
    // next[k][j]: for need j of op k, the next op index > k needing the same logical qubit
    std::vector<std::vector<int>> uses(n);
    for (int k = 0; k < G; ++k) {
        int q[2];
        const int c = remap_needs(ops[k], q);
        for (int j = 0; j < c; ++j) uses[q[j]].push_back(k);
    }
    std::vector<size_t> upos(n, 0);  // per logical qubit: first entry of uses[] that is >= the current op
    std::vector<int> phys(n), logi(n);
    for (int q = 0; q < n; ++q) phys[q] = logi[q] = q;
    auto next_use = [&](int lq, int k) {
        while (upos[lq] < uses[lq].size() && uses[lq][upos[lq]] < k) ++upos[lq];
        return upos[lq] < uses[lq].size() ? uses[lq][upos[lq]] : G + 1 + lq;  // never: furthest
    };
    for (int k = 0; k < G; ++k) {
        const Op &op = ops[k];
        if (op.kind == OP_SWAP) {  // a SWAP gate is a relabelling of two logical qubits
            const int pa = phys[op.q0], pb = phys[op.q1];
            phys[op.q0] = pb;
            phys[op.q1] = pa;
            logi[pa] = op.q1;
            logi[pb] = op.q0;
            continue;
        }
        int q[2];
        const int c = remap_needs(op, q);
        for (int j = 0; j < c; ++j) {
            if (phys[q[j]] < m) continue;
            // victim: the local position whose logical qubit is needed furthest in the future (Belady),
            // never a qubit of this op
            int best = -1, best_use = -1;
            for (int p = m - 1; p >= 0; --p) {
                const int lq = logi[p];
                if (lq == op.q0 || lq == op.q1) continue;
                const int u = next_use(lq, k);
                if (u > best_use) best_use = u, best = p;
            }
            const int g = phys[q[j]], lv = logi[best];
            out.push_back(make_swap(best, g));
            phys[q[j]] = best;
            logi[best] = q[j];
            phys[lv] = g;
            logi[g] = lv;
        }
        Op o = op;
        if (o.q0 >= 0) o.q0 = phys[o.q0];
        if (o.q1 >= 0) o.q1 = phys[o.q1];
        out.push_back(o);
    }
    // restore the canonical layout: logical q back at position q — global positions first (each
    // costs one exchange), then the local ones (a permutation pass, no exchange)
    for (int pass = 0; pass < 2; ++pass)
    for (int p = pass == 0 ? m : 0; p < (pass == 0 ? n : m); ++p) {
        if (logi[p] == p) continue;
        const int where = phys[p];  // position now holding logical p
        out.push_back(make_swap(p, where));
        const int lp = logi[p];
        logi[where] = lp;
        phys[lp] = where;
        logi[p] = p;
        phys[p] = p;
    }
    return out;
}

bool tile_requirements(const Op &op, int m, std::vector<int> &need) {
    need.clear();
    switch (op.kind) {
    case OP_DIAG:
        return true;
    case OP_PAIR:
        if (op.q0 >= m) return false;
        need.push_back(op.q0);
        return true;
    case OP_CTRL_PAIR:  // the control may sit outside the tile (then it is a fixed bit per tile)
        if (op.q1 >= m) return false;
        need.push_back(op.q1);
        return true;
    case OP_QUAD:
    case OP_SWAP:
    default:
        if (op.q0 >= m || op.q1 >= m) return false;
        need.push_back(op.q0);
        need.push_back(op.q1);
        return true;
    }
}

namespace {

// fraction of a full read+write pass a direct kernel for this op moves (sector-effective)
double direct_cost(const Op &op) {
    switch (op.kind) {
    case OP_PAIR:
    case OP_QUAD:
        return 1.0;
    case OP_CTRL_PAIR:
        return op.q0 == 0 ? 1.0 : 0.5;
    case OP_SWAP:
        return (op.q0 == 0 || op.q1 == 0) ? 1.0 : 0.5;
    case OP_DIAG: {
        int nq = op.q0 < 0 ? 0 : (op.q1 < 0 ? 1 : 2);
        if (nq == 0) return op.touch ? 1.0 : 0.0;
        int qs[2] = {op.q0, op.q1};
        int z = -1;
        for (int s = 0; s < nq; ++s)
            if (qs[s] == 0) z = s;
        int cells = 0;
        for (int k = 0; k < (1 << nq); ++k) {
            bool t = (op.touch >> k) & 1;
            if (z >= 0) t = t || ((op.touch >> (k ^ (1 << z))) & 1);  // sector partner
            cells += t;
        }
        return double(cells) / double(1 << nq);
    }
    }
    return 1.0;
}

}  // namespace

namespace {

// Ops that must run as their own step: non-tileable (a non-diagonal role on a global qubit).
bool is_tileable(const Op &op, int m) {
    std::vector<int> need;
    return tile_requirements(op, m, need);
}

bool is_identity(const Op &op) { return op.kind == OP_DIAG && op.touch == 0 && op.q0 >= 0; }

// A run of consecutive, pairwise disjoint local SWAPs starting at i whose qubits do not fit one tile:
// returns its end (exclusive) and the involution it applies, or i if there is none.
int perm_run(const std::vector<Op> &ops, int i, int m, int b, int L0, std::vector<int> &perm) {
    perm.assign(m, 0);
    for (int q = 0; q < m; ++q) perm[q] = q;
    std::vector<int> used;
    int j = i;
    while (j < (int)ops.size() && ops[j].kind == OP_SWAP && ops[j].q0 < m && ops[j].q1 < m &&
           std::find(used.begin(), used.end(), ops[j].q0) == used.end() &&
           std::find(used.begin(), used.end(), ops[j].q1) == used.end()) {
        used.push_back(ops[j].q0);
        used.push_back(ops[j].q1);
        std::swap(perm[ops[j].q0], perm[ops[j].q1]);
        ++j;
    }
    std::vector<int> U = used;
    for (int q = 0; q < L0; ++q)
        if (std::find(U.begin(), U.end(), q) == U.end()) U.push_back(q);
    return (j - i >= 2 && (int)U.size() > b) ? j : i;
}

// qubits of an op for dependency purposes (all roles)
int op_qubits(const Op &op, int q[2]) {
    int k = 0;
    if (op.q0 >= 0) q[k++] = op.q0;
    if (op.q1 >= 0) q[k++] = op.q1;
    return k;
}

}  // namespace

std::vector<Pass> plan_passes(const std::vector<Op> &ops, int n, int m, const PlanConfig &cfg) {
    (void)n;
    std::vector<Pass> out;
    const int b = std::min(cfg.b, m);
    const int L0 = std::min(cfg.L0, b);
    const bool fuse = cfg.fuse && b >= 6;  // tiles need >= 6 qubits (batches of 4 register slots)
    const size_t op_bytes_cap = 80 * 1024;  // k_tile stages the pass's op stream in shared memory
    auto op_bytes = [](const Op &op) -> size_t { return 80 + (op.kind == OP_QUAD ? 256 : 0); };

    // emit one group of ops (in execution order) whose non-diagonal qubits S fit a tile: a tile pass,
    // or single-op kernels when a pass would move no fewer bytes
    // emit() appends to `sink`: the result, or a trial schedule (trials run on several threads, each
    // with its own destination; everything else the schedulers capture is read-only)
    auto emit = [&](std::vector<Pass> *sink, const std::vector<int> &grp, const std::vector<int> &S) {
        if (grp.empty()) return;
        double direct = 0.0;
        for (int i : grp) direct += direct_cost(ops[i]);
        if (grp.size() == 1 || direct <= 1.0) {
            for (int i : grp) {
                Pass p;
                p.type = 0;
                p.ops.push_back(i);
                sink->push_back(p);
            }
            return;
        }
        std::vector<int> tq = S;
        for (int q = 0; q < L0; ++q)
            if (std::find(tq.begin(), tq.end(), q) == tq.end()) tq.push_back(q);
        for (int q = 0; (int)tq.size() < b && q < m; ++q)
            if (std::find(tq.begin(), tq.end(), q) == tq.end()) tq.push_back(q);
        std::sort(tq.begin(), tq.end());
        Pass cur;
        cur.type = 1;
        cur.ops = grp;
        cur.tile_q.assign(tq.begin(), tq.end());
        int L = 0;
        while (L < (int)tq.size() && tq[L] == L) ++L;
        cur.L = L;
        sink->push_back(cur);
    };

    // in gate order: greedy, a pass closes when the next op's qubits do not fit
    auto schedule_inorder = [&](const std::vector<int> &seg) {
        std::vector<int> grp, S, need;
        size_t cur_bytes = 0;
        for (int i : seg) {
            tile_requirements(ops[i], m, need);
            std::vector<int> U = S;
            for (int q : need)
                if (std::find(U.begin(), U.end(), q) == U.end()) U.push_back(q);
            int extra_low = 0;
            for (int q = 0; q < L0; ++q)
                if (std::find(U.begin(), U.end(), q) == U.end()) ++extra_low;
            if ((int)U.size() + extra_low > b || cur_bytes + op_bytes(ops[i]) > op_bytes_cap) {
                emit(&out, grp, S);
                grp.clear();
                cur_bytes = 0;
                U = need;
            }
            S = U;
            grp.push_back(i);
            cur_bytes += op_bytes(ops[i]);
        }
        emit(&out, grp, S);
    };

    // commutation-aware (cfg.reorder): the segment's dependency DAG — an op waits for the previous
    // non-diagonal op on each of its qubits, a non-diagonal op also for every diagonal op since then
    // (diagonal gates commute with each other) — scheduled greedily: a pass starts from the low
    // qubits, takes every ready op whose non-diagonal qubits are in its tile set S (in gate order),
    // and, when none is left, grows S by the qubit that unlocks the most ready ops, up to b qubits.
    auto schedule_reorder = [&](const std::vector<int> &seg, uint64_t seed, std::vector<Pass> *sink) {
        uint64_t rng = seed * 0x9E3779B97F4A7C15ull + 1;  // trial 0: deterministic greedy
        const int G = (int)seg.size();
        std::vector<std::vector<int>> succ(G);
        std::vector<int> npred(G, 0);
        int nq_all = m;  // diagonal roles and fixed controls may sit on global qubits (>= m)
        for (int k = 0; k < G; ++k) nq_all = std::max(nq_all, 1 + std::max(ops[seg[k]].q0, ops[seg[k]].q1));
        std::vector<int> lastnd(nq_all, -1);
        std::vector<std::vector<int>> diag_since(nq_all);
        auto add_edge = [&](int a, int c) {
            if (a < 0) return;
            if (!succ[a].empty() && succ[a].back() == c) return;
            succ[a].push_back(c);
            ++npred[c];
        };
        int last_barrier = -1;           // a whole-state scale op (no qubit) is a barrier: it keeps
        std::vector<int> since_barrier;  // its place, so deferred magnitudes never pile up
        for (int k = 0; k < G; ++k) {
            const Op &op = ops[seg[k]];
            int q[2];
            const int nq = op_qubits(op, q);
            const bool dg = op.kind == OP_DIAG;
            if (nq == 0) {
                for (int a : since_barrier) add_edge(a, k);
                add_edge(last_barrier, k);
                last_barrier = k;
                since_barrier.clear();
                continue;
            }
            add_edge(last_barrier, k);
            since_barrier.push_back(k);
            for (int u = 0; u < nq; ++u) {
                add_edge(lastnd[q[u]], k);
                if (dg) {
                    diag_since[q[u]].push_back(k);
                } else {
                    for (int d : diag_since[q[u]]) add_edge(d, k);
                    diag_since[q[u]].clear();
                }
            }
            if (!dg)
                for (int u = 0; u < nq; ++u) lastnd[q[u]] = k;
        }
        std::vector<std::vector<int>> needk(G);
        for (int k = 0; k < G; ++k) tile_requirements(ops[seg[k]], m, needk[k]);
        std::vector<char> tileable(G);
        for (int k = 0; k < G; ++k) tileable[k] = is_tileable(ops[seg[k]], m);
        std::set<int> ready;
        for (int k = 0; k < G; ++k)
            if (npred[k] == 0) ready.insert(k);
        int done = 0;
        while (done < G) {
            // exchange steps (non-tileable ops) run as soon as they are ready: they unlock the gates
            // waiting for a qubit to become local, so the next tile pass can take those too
            bool exch = false;
            for (auto it = ready.begin(); it != ready.end();) {
                const int k = *it;
                if (tileable[k]) {
                    ++it;
                    continue;
                }
                Pass p;
                p.type = 2;
                p.ops.push_back(seg[k]);
                sink->push_back(p);
                it = ready.erase(it);
                ++done;
                exch = true;
                for (int c : succ[k])
                    if (--npred[c] == 0) ready.insert(c);
                it = ready.begin();
            }
            if (exch) continue;
            std::vector<int> S;
            for (int q = 0; q < L0; ++q) S.push_back(q);
            std::vector<char> inS(m, 0);
            for (int q : S) inS[q] = 1;
            std::vector<int> grp;
            size_t cur_bytes = 0;
            bool full = false;
            for (;;) {
                bool progress = true;
                while (progress && !full) {
                    progress = false;
                    for (auto it = ready.begin(); it != ready.end();) {
                        const int k = *it;
                        bool fits = tileable[k];
                        for (int q : needk[k]) fits = fits && inS[q];
                        if (!fits) {
                            ++it;
                            continue;
                        }
                        if (cur_bytes + op_bytes(ops[seg[k]]) > op_bytes_cap) {
                            full = true;
                            break;
                        }
                        it = ready.erase(it);
                        grp.push_back(seg[k]);
                        cur_bytes += op_bytes(ops[seg[k]]);
                        ++done;
                        progress = true;
                        for (int c : succ[k])
                            if (--npred[c] == 0) ready.insert(c);
                        it = ready.begin();  // newly ready ops may precede: rescan in gate order
                    }
                }
                if (full || (int)S.size() >= b) break;
                // grow S by the qubit whose addition lets the pass take the most ops: for every
                // candidate (a missing qubit of a ready op) count the closure — ops that become
                // takeable, transitively, once it is in the tile (ties: the lowest qubit)
                std::vector<char> cand(m, 0);
                for (int k : ready) {
                    if (!tileable[k]) continue;
                    for (int q : needk[k])
                        if (!inS[q]) cand[q] = 1;
                }
                int best = -1, best_gain = 0;
                std::vector<int> np;
                std::vector<int> queue;
                std::vector<int> gains(m, 0);
                for (int q = 0; q < m; ++q) {
                    if (!cand[q]) continue;
                    inS[q] = 1;
                    np.assign(npred.begin(), npred.end());
                    queue.assign(ready.begin(), ready.end());
                    int gain = 0;
                    for (size_t qi = 0; qi < queue.size(); ++qi) {
                        const int k = queue[qi];
                        if (!tileable[k]) continue;
                        bool fits = true;
                        for (int x : needk[k]) fits = fits && inS[x];
                        if (!fits) continue;
                        ++gain;
                        for (int c2 : succ[k])
                            if (--np[c2] == 0) queue.push_back(c2);
                    }
                    inS[q] = 0;
                    gains[q] = gain;
                    if (gain > best_gain) best_gain = gain, best = q;
                }
                if (seed != 0 && best >= 0) {  // later trials: a random pick among the near-best
                    int nc = 0;
                    for (int q = 0; q < m; ++q) nc += cand[q] && gains[q] > 0 && gains[q] >= best_gain - 1;
                    rng = rng * 6364136223846793005ull + 1442695040888963407ull;
                    int pick = (int)((rng >> 33) % (uint64_t)nc);
                    for (int q = 0; q < m; ++q)
                        if (cand[q] && gains[q] > 0 && gains[q] >= best_gain - 1 && pick-- == 0) {
                            best = q;
                            break;
                        }
                }
                if (best < 0) {  // ops needing two more qubits
                    for (int k : ready) {
                        if (!tileable[k]) continue;
                        int nmiss = 0;
                        for (int q : needk[k]) nmiss += !inS[q];
                        if (nmiss >= 1 && (int)S.size() + nmiss <= b) {
                            for (int q : needk[k])
                                if (!inS[q]) {
                                    best = q;
                                    break;
                                }
                            break;
                        }
                    }
                }
                if (best < 0) break;
                S.push_back(best);
                inS[best] = 1;
            }
            if (grp.empty()) {  // not expected (a ready op always fits a fresh tile): run it alone
                if (ready.empty()) break;  // (cannot happen for an acyclic dependency graph)
                const int k = *ready.begin();
                ready.erase(ready.begin());
                grp.push_back(seg[k]);
                ++done;
                for (int c : succ[k])
                    if (--npred[c] == 0) ready.insert(c);
            }
            std::vector<int> Sn;  // S restricted to what the group needs (emit adds the low qubits)
            for (int i : grp) {
                std::vector<int> nd;
                tile_requirements(ops[i], m, nd);
                for (int q : nd)
                    if (std::find(Sn.begin(), Sn.end(), q) == Sn.end()) Sn.push_back(q);
            }
            emit(sink, grp, Sn);
        }
    };

    std::vector<int> perm;
    for (int i = 0; i < (int)ops.size();) {
        const Op &op = ops[i];
        if (is_identity(op)) {
            ++i;
            continue;
        }
        if (!fuse) {
            Pass p;
            p.type = is_tileable(op, m) ? 0 : 2;
            p.ops.push_back(i);
            out.push_back(p);
            ++i;
            continue;
        }
        if (cfg.perm_low > 0) {
            const int j = perm_run(ops, i, m, b, L0, perm);
            if (j > i) {
                Pass p;
                p.type = 3;
                for (int k = i; k < j; ++k) p.ops.push_back(k);
                p.perm.assign(perm.begin(), perm.end());
                out.push_back(p);
                i = j;
                continue;
            }
        }
        if (!is_tileable(op, m)) {
            Pass p;
            p.type = 2;
            p.ops.push_back(i);
            out.push_back(p);
            ++i;
            continue;
        }
        // a segment up to the next permutation run: gate order keeps tileable ops between exchange
        // steps; the DAG scheduler takes exchange steps into the segment and runs them when ready
        std::vector<int> seg;
        int j = i;
        while (j < (int)ops.size() && (cfg.reorder || is_tileable(ops[j], m))) {
            if (j > i && cfg.perm_low > 0 && perm_run(ops, j, m, b, L0, perm) > j) break;
            if (!is_identity(ops[j])) seg.push_back(j);
            ++j;
        }
        if (cfg.reorder) {
            // several greedy trials (the first deterministic, the others with random near-best picks):
            // the schedule with the fewest steps wins (grid RQC(32): 21 -> 19-20 passes)
            // The trials are independent: they run on up to 16 host threads, and the first trial (in
            // trial order) with the fewest steps is kept — the same schedule as a serial loop
            const int ntr = std::max(1, cfg.trials);
            std::vector<std::vector<Pass>> trials(ntr);
            const int nth = std::max(1, std::min(ntr, (int)std::min(16u, std::max(1u, std::thread::hardware_concurrency()))));
            if (nth == 1) {
                for (int t = 0; t < ntr; ++t) schedule_reorder(seg, (uint64_t)t, &trials[t]);
            } else {
                std::vector<std::thread> th;
                for (int w = 0; w < nth; ++w)
                    th.emplace_back([&, w]() {
                        for (int t = w; t < ntr; t += nth) schedule_reorder(seg, (uint64_t)t, &trials[t]);
                    });
                for (auto &x : th) x.join();
            }
            std::vector<Pass> best;
            for (int t = 0; t < ntr; ++t)
                if (t == 0 || trials[t].size() < best.size()) best.swap(trials[t]);
            // restarts from prefixes of the best schedule: keep its first k steps, reschedule the rest
            // (the remaining ops form a closed upper set of the DAG, so a fresh DAG over them is exact)
            for (size_t k = 1; cfg.restarts > 0 && k + 1 < best.size(); ++k) {
                std::vector<char> done(ops.size(), 0);
                for (size_t q = 0; q < k; ++q)
                    for (int oi : best[q].ops) done[oi] = 1;
                std::vector<int> rest;
                for (int oi : seg)
                    if (!done[oi]) rest.push_back(oi);
                bool improved = false;
                for (int t = 0; t < cfg.restarts && !improved; ++t) {
                    std::vector<Pass> trial;
                    schedule_reorder(rest, (uint64_t)(1000 + 97 * k + t), &trial);
                    if (k + trial.size() < best.size()) {
                        best.resize(k);
                        best.insert(best.end(), trial.begin(), trial.end());
                        improved = true;
                    }
                }
                if (improved) k = 0;  // start over on the shorter schedule
            }
            out.insert(out.end(), best.begin(), best.end());
        } else {
            schedule_inorder(seg);
        }
        i = j;
    }

    // fused permutation: a permutation run that directly follows a tile pass is applied by that pass's
    // store when the pass's needed qubits Q (its ops' tile requirements and the low qubits) close under
    // pi within perm_fuse_b qubits — the tile is Q ∪ pi(Q), so tile T lands on tile pi(T) and one CTA
    // owns each pair (tile_kernel PAIR: a cluster of two CTAs).  One HBM pass fewer (QFT: the final reversal).
    if (fuse && cfg.perm_fuse) {
        std::vector<Pass> res;
        for (Pass &p : out) {
            if (p.type == 3 && !res.empty() && res.back().type == 1 && res.back().perm.empty()) {
                Pass &t = res.back();
                std::vector<int> C, need;
                for (int q = 0; q < L0; ++q) C.push_back(q);
                for (int oi : t.ops) {
                    tile_requirements(ops[oi], m, need);
                    for (int q : need)
                        if (std::find(C.begin(), C.end(), q) == C.end()) C.push_back(q);
                }
                const size_t nq = C.size();
                for (size_t k = 0; k < nq; ++k)
                    if (std::find(C.begin(), C.end(), p.perm[C[k]]) == C.end()) C.push_back(p.perm[C[k]]);
                // tiles need >= TILE_MIN_Q qubits: add the lowest qubits with their images
                for (int q = 0; (int)C.size() < 6 && q < m; ++q)
                    if (std::find(C.begin(), C.end(), q) == C.end()) {
                        C.push_back(q);
                        if (std::find(C.begin(), C.end(), p.perm[q]) == C.end()) C.push_back(p.perm[q]);
                    }
                if ((int)C.size() <= std::min(cfg.perm_fuse_b, b) && (int)C.size() >= 6 && m - (int)C.size() <= 27) {
                    std::sort(C.begin(), C.end());
                    t.tile_q.assign(C.begin(), C.end());
                    int L = 0;
                    while (L < (int)C.size() && C[L] == L) ++L;
                    t.L = L;
                    t.perm = p.perm;
                    t.perm_ops = p.ops;
                    continue;
                }
            }
            res.push_back(std::move(p));
        }
        out.swap(res);
    }
    return out;
}

namespace {

// x with bits a and b exchanged for every transposition (a, b) selected in `sel`
uint64_t swap_bits(uint64_t x, const std::vector<std::pair<int, int>> &T, uint64_t sel) {
    for (size_t i = 0; i < T.size(); ++i) {
        if (!((sel >> i) & 1)) continue;
        const uint64_t ba = (x >> T[i].first) & 1, bb = (x >> T[i].second) & 1;
        if (ba != bb) x ^= (1ull << T[i].first) | (1ull << T[i].second);
    }
    return x;
}

int popc(uint64_t x) { return __builtin_popcountll(x); }

}  // namespace

bool hoist_permutation(const std::vector<Op> &ops, const std::vector<Pass> &plan, int m, const PlanConfig &cfg,
                       std::vector<Op> &ops_out, std::vector<Pass> &plan_out) {
    const int b = std::min(cfg.b, m), L0 = std::min(cfg.L0, b), fb = std::min(cfg.perm_fuse_b, b);
    if (!cfg.fuse || !cfg.perm_fuse || m > 63 || b < 6) return false;
    const uint64_t low = (1ull << L0) - 1;
    for (size_t z = 1; z < plan.size(); ++z) {
        if (plan[z].type != 3) continue;
        size_t s = z;
        while (s > 0 && z - s < 8 && plan[s - 1].type == 1 && plan[s - 1].perm.empty()) --s;
        if (s == z) continue;
        const std::vector<int> &pi = plan[z].perm;
        std::vector<std::pair<int, int>> T;
        for (int a = 0; a < m; ++a)
            if (pi[a] > a) T.emplace_back(a, pi[a]);
        if (T.empty() || T.size() > 32) continue;
        const int K = (int)(z - s);
        const uint64_t all = (1ull << T.size()) - 1;
        std::vector<uint64_t> need(K, 0);  // logical qubits each pass needs in its tile
        std::vector<int> nd;
        for (int k = 0; k < K; ++k)
            for (int oi : plan[s + k].ops) {
                tile_requirements(ops[oi], m, nd);
                for (int q : nd) need[k] |= 1ull << q;
            }
        // the transpositions a fused pass with needed qubits Q (physical) can take from `avail`: both
        // qubits inside Q or both outside (free), then (grow) those with one qubit inside while
        // |Q ∪ sigma(Q)| <= fb; returns the selection and C
        auto choose = [&](uint64_t Q, uint64_t avail, bool grow, uint64_t &C) {
            uint64_t sel = 0;
            C = Q;
            for (size_t i = 0; i < T.size(); ++i) {
                if (!((avail >> i) & 1)) continue;
                const bool ia = (Q >> T[i].first) & 1, ib = (Q >> T[i].second) & 1;
                if (ia == ib) sel |= 1ull << i;
            }
            if (grow)
                for (size_t i = 0; i < T.size(); ++i) {
                    if (!((avail >> i) & 1) || ((sel >> i) & 1)) continue;
                    const uint64_t c2 = C | (1ull << T[i].first) | (1ull << T[i].second);
                    if (popc(c2) <= fb) {
                        sel |= 1ull << i;
                        C = c2;
                    }
                }
            return sel;
        };
        int best = K + 1;
        std::vector<uint64_t> cur(K, 0), bestsel;
        std::function<void(int, uint64_t, int)> dfs = [&](int k, uint64_t done, int fused) {
            if (fused >= best) return;
            if (k == K) {
                if (done == all) {
                    best = fused;
                    bestsel = cur;
                }
                return;
            }
            // ops of pass k act on relabelled qubits: physical = the transpositions done so far applied
            const uint64_t Q = swap_bits(need[k], T, done) | low;
            if (popc(Q) > b) return;
            cur[k] = 0;
            dfs(k + 1, done, fused);
            uint64_t prev = 0;
            for (int grow = 0; grow < 2; ++grow) {
                uint64_t C = 0;
                const uint64_t sel = choose(Q, all & ~done, grow != 0, C);
                if (!sel || sel == prev || popc(C) > fb || popc(C) < 6 || m - popc(C) > 27) continue;
                prev = sel;
                cur[k] = sel;
                dfs(k + 1, done | sel, fused + 1);
                cur[k] = 0;
            }
        };
        dfs(0, 0, 0);
        if (best > K) continue;

        // rebuild: relabelled ops of passes s..z-1, the SWAPs of each fused pass, pass z removed
        ops_out.clear();
        plan_out.clear();
        std::vector<int> phys(m);
        for (int q = 0; q < m; ++q) phys[q] = q;
        uint64_t done = 0;
        for (size_t p = 0; p < plan.size(); ++p) {
            if (p == z) continue;
            const bool in_run = p >= s && p < z;
            Pass np = plan[p];
            np.ops.clear();
            np.perm_ops.clear();
            for (int oi : plan[p].ops) {
                Op o = ops[oi];
                if (in_run) {
                    if (o.q0 >= 0 && o.q0 < m) o.q0 = phys[o.q0];
                    if (o.q1 >= 0 && o.q1 < m) o.q1 = phys[o.q1];
                    if (o.kind == OP_SWAP && o.q0 > o.q1) std::swap(o.q0, o.q1);
                }
                np.ops.push_back((int)ops_out.size());
                ops_out.push_back(o);
            }
            for (int oi : plan[p].perm_ops) {
                np.perm_ops.push_back((int)ops_out.size());
                ops_out.push_back(ops[oi]);
            }
            if (in_run) {
                const int k = (int)(p - s);
                const uint64_t Q = swap_bits(need[k], T, done) | low;
                const uint64_t sel = bestsel[k];
                uint64_t C = Q;
                std::vector<int> perm;
                if (sel) {
                    perm.resize(m);
                    for (int q = 0; q < m; ++q) perm[q] = q;
                    for (size_t i = 0; i < T.size(); ++i) {
                        if (!((sel >> i) & 1)) continue;
                        const int a = T[i].first, c = T[i].second;
                        std::swap(perm[a], perm[c]);
                        if ((Q >> a) & 1 || (Q >> c) & 1) C |= (1ull << a) | (1ull << c);
                        Op sw;
                        sw.kind = OP_SWAP;
                        sw.q0 = a;
                        sw.q1 = c;
                        np.perm_ops.push_back((int)ops_out.size());
                        ops_out.push_back(sw);
                        // untouched so far: the logical qubits a, c sit at physical a, c
                        std::swap(phys[a], phys[c]);
                    }
                    // fill with the lowest qubits the permutation fixes (longer contiguous runs)
                    for (int q = 0; popc(C) < fb && q < m; ++q)
                        if (perm[q] == q) C |= 1ull << q;
                    done |= sel;
                } else {
                    for (int q = 0; popc(C) < b && q < m; ++q) C |= 1ull << q;
                }
                np.tile_q.clear();
                for (int q = 0; q < m; ++q)
                    if ((C >> q) & 1) np.tile_q.push_back(q);
                int L = 0;
                while (L < (int)np.tile_q.size() && np.tile_q[L] == L) ++L;
                np.L = L;
                np.perm = perm;
            }
            plan_out.push_back(std::move(np));
        }
        return true;
    }
    return false;
}

}  // namespace qsb
