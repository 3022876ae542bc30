// Host-side planner.  See plan.h and DESIGN.md.
//
//  A1 cluster tree   — Def. A.1; split rule "adaptive split axis"
//                      (listing PAPER.md:472) read as: tight bounding box of the node's points,
//                      split the longest axis (ties -> x) at the cardinality median (stable by
//                      current order; left gets ceil(m/2)).  Uniform depth L = ceil(log2(n/32)).
//  A2 block tree     — Def. A.2 son rule with the admissibility
//                      TStdGeomAdmCond(2.0, use_min_diam):
//                      min(diam tau, diam sigma) <= eta * dist(tau, sigma), dist > 0.
//  A7 schedule       — lazy, column-oriented (left-looking) H-Cholesky, DESIGN.md Sec. 4.
#include "plan.h"

#include <algorithm>
#include <cmath>
#include <functional>
#include <limits>
#include <numeric>
#include <unordered_map>

namespace {

inline int64_t heap_id(int l, int64_t c) { return ((int64_t)1 << l) - 1 + c; }
inline uint64_t node_key(int l, int64_t i, int64_t j) {
    return ((uint64_t)l << 58) | ((uint64_t)i << 29) | (uint64_t)j;
}

struct Builder {
    Plan &P;
    int L;
    std::unordered_map<uint64_t, int32_t> key2node;
    std::vector<std::vector<DTerm>> node_terms;
    std::vector<int32_t> node_term_wave;
    std::vector<int32_t> tile_wave, rfin_wave, rdone_wave, core_wave, phw_wave;
    std::vector<int32_t> done_memo;
    std::vector<std::vector<int32_t>> col;   // per cluster heap id: off-diagonal entries (node ids)
    int32_t n_fac_u = 0;

    explicit Builder(Plan &p) : P(p), L(p.depth) {}

    double diam(int64_t h) const {
        const double *b = &P.bb[4 * h];
        double dx = b[2] - b[0], dy = b[3] - b[1];
        return std::sqrt(dx * dx + dy * dy);
    }
    double dist(int64_t h1, int64_t h2) const {
        const double *a = &P.bb[4 * h1], *b = &P.bb[4 * h2];
        double gx = std::max(0.0, std::max(a[0] - b[2], b[0] - a[2]));
        double gy = std::max(0.0, std::max(a[1] - b[3], b[1] - a[3]));
        return std::sqrt(gx * gx + gy * gy);
    }
    bool admissible(int l, int64_t i, int64_t j) const {
        if (P.eta <= 0.0) return false;
        int64_t hi = heap_id(l, i), hj = heap_id(l, j);
        double d = dist(hi, hj);
        if (!(d > 0.0)) return false;
        return std::min(diam(hi), diam(hj)) <= P.eta * d;
    }

    int32_t make(int l, int64_t i, int64_t j, int32_t parent, bool forced) {
        int32_t id = (int32_t)P.nodes.size();
        DNode nd{};
        nd.level = l; nd.i = (int32_t)i; nd.j = (int32_t)j;
        nd.parent = parent; nd.idx = -1; nd.leaf_off = 0; nd.leaf_cnt = 0;
        P.nodes.push_back(nd);
        for (int k = 0; k < 4; ++k) P.children.push_back(-1);
        key2node[node_key(l, i, j)] = id;
        int type;
        if (i == j) {
            type = (l == L) ? ND_T : ND_H;
        } else {
            bool adm = !forced && admissible(l, i, j);
            if (adm && l < L && P.cluster_size(l) > P.dense_below) type = ND_R;
            else if (l == L) type = ND_T;
            else { type = ND_H; forced = forced || adm; }
        }
        P.nodes[id].type = type;
        if (type == ND_T) {
            P.nodes[id].idx = (int32_t)P.tile_node.size();
            P.tile_node.push_back(id);
        } else if (type == ND_R) {
            DRBlk r{};
            r.node = id; r.level = l; r.m = (int32_t)P.cluster_size(l);
            r.row0 = i * P.cluster_size(l); r.col0 = j * P.cluster_size(l);
            r.uv_off = P.uv_elems;
            P.uv_elems += r.m;
            P.nodes[id].idx = (int32_t)P.rblk.size();
            P.rblk.push_back(r);
        } else {
            if (i == j) {
                int32_t c0 = make(l + 1, 2 * i, 2 * j, id, forced);
                int32_t c2 = make(l + 1, 2 * i + 1, 2 * j, id, forced);
                int32_t c3 = make(l + 1, 2 * i + 1, 2 * j + 1, id, forced);
                P.children[4 * id + 0] = c0; P.children[4 * id + 2] = c2; P.children[4 * id + 3] = c3;
            } else {
                for (int a = 0; a < 2; ++a)
                    for (int b = 0; b < 2; ++b) {
                        int32_t c = make(l + 1, 2 * i + a, 2 * j + b, id, forced);
                        P.children[4 * id + 2 * a + b] = c;
                    }
            }
        }
        return id;
    }

    int32_t owner(int l, int64_t i, int64_t j) const {
        while (true) {
            auto it = key2node.find(node_key(l, i, j));
            if (it != key2node.end()) return it->second;
            --l; i >>= 1; j >>= 1;
        }
    }

    int32_t term_wave_chain(int32_t nd) const {
        int32_t w = 0;
        for (int32_t x = nd; x >= 0; x = P.nodes[x].parent) w = std::max(w, node_term_wave[x]);
        return w;
    }

    int32_t done_wave(int32_t nd) {
        if (done_memo[nd] >= 0) return done_memo[nd];
        const DNode &x = P.nodes[nd];
        int32_t w = 0;
        if (x.type == ND_T) w = tile_wave[x.idx];
        else if (x.type == ND_R) w = rdone_wave[x.idx];
        else
            for (int k = 0; k < 4; ++k) {
                int32_t c = P.children[4 * nd + k];
                if (c >= 0) w = std::max(w, done_wave(c));
            }
        done_memo[nd] = w;
        return w;
    }

    int32_t emit(int32_t type, int32_t a, int32_t b, int32_t c, int32_t wave) {
        P.tasks.push_back(DTask{type, a, b, c});
        P.task_wave.push_back(wave);
        P.n_waves = std::max(P.n_waves, wave + 1);
        return wave;
    }

    void add_term(int32_t target_node, const DTerm &t, int32_t wave) {
        node_terms[target_node].push_back(t);
        node_term_wave[target_node] = std::max(node_term_wave[target_node], wave);
    }

    void collect_leaves(int32_t nd, std::vector<int32_t> &out) const {
        const DNode &x = P.nodes[nd];
        if (x.type != ND_H) { out.push_back(nd); return; }
        for (int k = 0; k < 4; ++k) {
            int32_t c = P.children[4 * nd + k];
            if (c >= 0) collect_leaves(c, out);
        }
    }

    void post(int l, int64_t c) {
        int64_t sig = heap_id(l, c);
        int32_t beg_ops = (int32_t)P.ops.size();
        if (l < L) { post(l + 1, 2 * c); post(l + 1, 2 * c + 1); }
        const int64_t m = P.cluster_size(l);
        const int64_t start = c * m;
        int32_t diag_tile = -1;
        if (l == L) {
            int32_t d = key2node.at(node_key(L, c, c));
            diag_tile = P.nodes[d].idx;
            int32_t w = 1 + term_wave_chain(d);
            tile_wave[diag_tile] = emit(TK_POTRF, d, diag_tile, 0, w);
            P.ops.push_back(DOp{OP_TRSM, diag_tile, HCOV_LEAF, 0, start, start});
        }
        std::vector<int32_t> &ents = col[sig];
        std::sort(ents.begin(), ents.end(), [&](int32_t a, int32_t b) { return P.nodes[a].i < P.nodes[b].i; });
        std::vector<int32_t> rents;
        for (int32_t e : ents) {
            const DNode &x = P.nodes[e];
            if (x.type == ND_T) {
                int32_t w = 1 + std::max(term_wave_chain(e), tile_wave[diag_tile]);
                tile_wave[x.idx] = emit(TK_TRSM, e, diag_tile, 0, w);
            } else if (x.type == ND_R) {
                int32_t w = 1 + term_wave_chain(e);
                rfin_wave[x.idx] = emit(TK_RFIN, e, 0, 0, w);
                rents.push_back(x.idx);
            }
        }
        P.col_r_off[sig] = (int32_t)P.col_r.size();
        for (int32_t r : rents) P.col_r.push_back(r);
        P.col_r_off[sig + 1] = (int32_t)P.col_r.size();  // (fixed up below; off array is n_clusters+1)
        if (!rents.empty()) {
            int32_t dnode = key2node.at(node_key(l, c, c));
            int32_t w = done_wave(dnode);
            for (int32_t r : rents) w = std::max(w, rfin_wave[r]);
            w = emit(TK_SOLVE, (int32_t)sig, 0, 0, w + 1);
            for (int32_t r : rents) rdone_wave[r] = w;
        }
        for (int32_t e : ents) {
            const DNode &x = P.nodes[e];
            int64_t r0 = (int64_t)x.i * m;
            if (x.type == ND_T) P.ops.push_back(DOp{OP_UPD_T, x.idx, (int32_t)m, 0, r0, start});
            else if (x.type == ND_R) P.ops.push_back(DOp{OP_UPD_R, x.idx, (int32_t)m, 0, r0, start});
        }
        // PHW tasks: one per H entry when the column has R entries.
        std::unordered_map<int32_t, int32_t> h2phw;
        if (!rents.empty()) {
            for (int32_t e : ents) {
                if (P.nodes[e].type != ND_H) continue;
                DPhw q{};
                q.hnode = e;
                q.part_off = P.col_r_off[sig];
                q.part_cnt = (int32_t)rents.size();
                q.fac_base = (int32_t)P.fac_row0.size();
                q.m = (int32_t)m;
                q.w_off = P.w_elems;
                P.w_elems += m * (int64_t)rents.size();
                for (int p = 0; p < (int)rents.size(); ++p) {
                    P.fac_row0.push_back((int64_t)P.nodes[e].i * m);
                    P.fac_nrows.push_back((int32_t)m);
                    P.fac_rank_src.push_back(rents[p]);
                    P.fac_off.push_back(q.w_off + (int64_t)p * m);
                    P.fac_pool.push_back(1);
                }
                // flattened leaves of the H node
                std::vector<int32_t> lv;
                collect_leaves(e, lv);
                P.nodes[e].leaf_off = (int32_t)P.hleaf.size();
                P.nodes[e].leaf_cnt = (int32_t)lv.size();
                P.hleaf.insert(P.hleaf.end(), lv.begin(), lv.end());
                int32_t w = done_wave(e);
                for (int32_t r : rents) w = std::max(w, rdone_wave[r]);
                int32_t qid = (int32_t)P.phw.size();
                P.phw.push_back(q);
                phw_wave.push_back(emit(TK_PHW, e, qid, 0, w + 1));
                h2phw[e] = qid;
            }
        }
        // products among the entries of this column (lower: e1.i >= e2.i)
        for (size_t a = 0; a < ents.size(); ++a) {
            for (size_t b = 0; b <= a; ++b) {
                int32_t e1 = ents[a], e2 = ents[b];
                const DNode &x1 = P.nodes[e1], &x2 = P.nodes[e2];
                int t1 = x1.type, t2 = x2.type;
                if (t1 == ND_H && t2 == ND_H) continue;
                int32_t o = owner(l, x1.i, x2.i);
                DTerm t{};
                int32_t w;
                if (t1 == ND_T && t2 == ND_T) {
                    t.kind = TM_TT; t.a = x1.idx; t.b = x2.idx; t.core = -1;
                    w = std::max(tile_wave[x1.idx], tile_wave[x2.idx]);
                } else if (t1 == ND_R && t2 == ND_R) {
                    int32_t core = P.n_cores++;
                    int32_t wv = 1 + std::max(rdone_wave[x1.idx], rdone_wave[x2.idx]);
                    core_wave.push_back(emit(TK_PRR, x1.idx, x2.idx, core, wv));
                    t.kind = TM_LR; t.a = x1.idx; t.b = x2.idx; t.core = core;
                    w = core_wave[core];
                } else if (t1 == ND_R && t2 == ND_H) {
                    int32_t q = h2phw.at(e2);
                    int p = (int)(std::find(rents.begin(), rents.end(), x1.idx) - rents.begin());
                    t.kind = TM_LR; t.a = x1.idx; t.b = P.phw[q].fac_base + p; t.core = -1;
                    w = phw_wave[q];
                } else if (t1 == ND_H && t2 == ND_R) {
                    int32_t q = h2phw.at(e1);
                    int p = (int)(std::find(rents.begin(), rents.end(), x2.idx) - rents.begin());
                    t.kind = TM_LR; t.a = P.phw[q].fac_base + p; t.b = x2.idx; t.core = -1;
                    w = phw_wave[q];
                } else {
                    continue;  // impossible with same-level entries (T only at leaf level)
                }
                add_term(o, t, w);
            }
        }
        P.op_beg[sig] = beg_ops;
        P.op_end[sig] = (int32_t)P.ops.size();
    }
};

}  // namespace

int plan_build(Plan &P, const double *s, int64_t n, double eta, int dense_below) {
    if (n <= 0) return 2;
    for (int64_t k = 0; k < 2 * n; ++k)
        if (!std::isfinite(s[k])) return 1;
    int L = 0;
    while (((int64_t)HCOV_LEAF << L) < n) ++L;
    P.n = n; P.depth = L; P.n_leaves = (int64_t)1 << L; P.n_pad = (int64_t)HCOV_LEAF << L;
    P.eta = eta; P.dense_below = std::max(dense_below, HCOV_LEAF);
    P.n_clusters = ((int64_t)2 << L) - 1;
    P.bb.assign(4 * P.n_clusters, 0.0);

    // ---- A1 -------------------------------------------------------------------------------
    std::vector<int64_t> perm(n);
    std::iota(perm.begin(), perm.end(), 0);
    std::vector<int64_t> rs{0}, re{n};
    for (int l = 0; l <= L; ++l) {
        int64_t nc = (int64_t)1 << l;
        std::vector<int64_t> rs2, re2;
        if (l < L) { rs2.resize(2 * nc); re2.resize(2 * nc); }
        for (int64_t c = 0; c < nc; ++c) {
            double lx = std::numeric_limits<double>::infinity(), ly = lx, hx = -lx, hy = -lx;
            for (int64_t k = rs[c]; k < re[c]; ++k) {
                double x = s[2 * perm[k]], y = s[2 * perm[k] + 1];
                lx = std::min(lx, x); hx = std::max(hx, x);
                ly = std::min(ly, y); hy = std::max(hy, y);
            }
            double *b = &P.bb[4 * heap_id(l, c)];
            if (re[c] > rs[c]) { b[0] = lx; b[1] = ly; b[2] = hx; b[3] = hy; }
            else { b[0] = b[1] = b[2] = b[3] = std::numeric_limits<double>::quiet_NaN(); }
            if (l == L) continue;
            int axis = (hx - lx >= hy - ly) ? 0 : 1;
            std::stable_sort(perm.begin() + rs[c], perm.begin() + re[c],
                             [&](int64_t a, int64_t b2) { return s[2 * a + axis] < s[2 * b2 + axis]; });
            int64_t m = re[c] - rs[c], m1 = (m + 1) / 2;
            rs2[2 * c] = rs[c]; re2[2 * c] = rs[c] + m1;
            rs2[2 * c + 1] = rs[c] + m1; re2[2 * c + 1] = re[c];
        }
        if (l < L) { rs.swap(rs2); re.swap(re2); }
    }
    P.perm_i2e.assign(P.n_pad, -1);
    P.xs.assign(P.n_pad, std::numeric_limits<double>::quiet_NaN());
    P.ys.assign(P.n_pad, std::numeric_limits<double>::quiet_NaN());
    for (int64_t c = 0; c < P.n_leaves; ++c) {
        if (re[c] - rs[c] > HCOV_LEAF) return 3;  // cannot happen (sizes <= ceil(n / 2^L) <= 32)
        for (int64_t k = rs[c]; k < re[c]; ++k) {
            int64_t pos = c * HCOV_LEAF + (k - rs[c]);
            P.perm_i2e[pos] = perm[k];
            P.xs[pos] = s[2 * perm[k]];
            P.ys[pos] = s[2 * perm[k] + 1];
        }
    }

    // ---- A2 -------------------------------------------------------------------------------
    Builder B(P);
    B.make(0, 0, 0, -1, false);
    const size_t nn = P.nodes.size();
    B.node_terms.assign(nn, {});
    B.node_term_wave.assign(nn, 0);
    B.done_memo.assign(nn, -1);
    B.tile_wave.assign(P.n_tiles(), 0);
    B.rfin_wave.assign(P.n_r(), 0);
    B.rdone_wave.assign(P.n_r(), 0);
    B.col.assign(P.n_clusters, {});
    for (size_t k = 0; k < nn; ++k) {
        const DNode &x = P.nodes[k];
        if (x.i != x.j) B.col[heap_id(x.level, x.j)].push_back((int32_t)k);
    }
    // factor table part 1: U of R blocks
    for (const DRBlk &r : P.rblk) {
        P.fac_row0.push_back(r.row0);
        P.fac_nrows.push_back(r.m);
        P.fac_rank_src.push_back((int32_t)(&r - &P.rblk[0]));
        P.fac_off.push_back(r.uv_off);
        P.fac_pool.push_back(0);
    }

    // ---- A7 schedule (post-order over clusters) -------------------------------------------
    P.col_r_off.assign(P.n_clusters + 1, 0);
    P.op_beg.assign(P.n_clusters, 0);
    P.op_end.assign(P.n_clusters, 0);
    // col_r_off is written as [off(s), off(s)+cnt) at visit time; keep explicit counts instead
    std::vector<int32_t> col_cnt(P.n_clusters, 0);
    {
        // post() writes col_r_off[sig] and col_r_off[sig+1]; since visits are not in heap-id
        // order, record counts separately.
        B.post(0, 0);
    }
    // recompute col_r_off as a proper CSR in heap-id order
    {
        std::vector<std::vector<int32_t>> per(P.n_clusters);
        for (int64_t sig = 0; sig < P.n_clusters; ++sig) {
            for (int32_t e : B.col[sig])
                if (P.nodes[e].type == ND_R) per[sig].push_back(P.nodes[e].idx);
        }
        // the PHW partner lists referenced the visit-order offsets; rebuild both consistently
        std::vector<int32_t> newcol;
        std::vector<int32_t> newoff(P.n_clusters + 1, 0);
        for (int64_t sig = 0; sig < P.n_clusters; ++sig) {
            newoff[sig] = (int32_t)newcol.size();
            newcol.insert(newcol.end(), per[sig].begin(), per[sig].end());
        }
        newoff[P.n_clusters] = (int32_t)newcol.size();
        for (DPhw &q : P.phw) {
            const DNode &h = P.nodes[q.hnode];
            q.part_off = newoff[heap_id(h.level, h.j)];
        }
        P.col_r.swap(newcol);
        P.col_r_off.swap(newoff);
    }
    P.phw_part = P.col_r;

    // flatten terms
    P.terms.clear();
    for (size_t k = 0; k < nn; ++k) {
        P.nodes[k].term_off = (int32_t)P.terms.size();
        P.nodes[k].term_cnt = (int32_t)B.node_terms[k].size();
        P.terms.insert(P.terms.end(), B.node_terms[k].begin(), B.node_terms[k].end());
    }
    // waves: sort tasks by (wave, type)
    std::vector<int32_t> idx(P.tasks.size());
    std::iota(idx.begin(), idx.end(), 0);
    std::stable_sort(idx.begin(), idx.end(), [&](int32_t a, int32_t b) {
        if (P.task_wave[a] != P.task_wave[b]) return P.task_wave[a] < P.task_wave[b];
        return P.tasks[a].type < P.tasks[b].type;
    });
    P.wave_tasks = idx;
    P.wave_off.assign(P.n_waves + 1, 0);
    for (int32_t t : idx) P.wave_off[P.task_wave[t] + 1]++;
    for (int32_t w = 0; w < P.n_waves; ++w) P.wave_off[w + 1] += P.wave_off[w];

    // row lists: per leaf row segment, T/R nodes intersecting it (lower triangle incl. diag)
    {
        std::vector<std::vector<int32_t>> rows(P.n_leaves);
        for (size_t k = 0; k < nn; ++k) {
            const DNode &x = P.nodes[k];
            if (x.type == ND_H) continue;
            int64_t span = (int64_t)1 << (L - x.level);
            for (int64_t seg = (int64_t)x.i * span; seg < (int64_t)(x.i + 1) * span; ++seg)
                rows[seg].push_back((int32_t)k);
        }
        P.row_off.assign(P.n_leaves + 1, 0);
        for (int64_t seg = 0; seg < P.n_leaves; ++seg) {
            P.row_off[seg] = (int32_t)P.row_nodes.size();
            // columns ascending
            std::sort(rows[seg].begin(), rows[seg].end(), [&](int32_t a, int32_t b) {
                const DNode &xa = P.nodes[a], &xb = P.nodes[b];
                return ((int64_t)xa.j << (L - xa.level)) < ((int64_t)xb.j << (L - xb.level));
            });
            P.row_nodes.insert(P.row_nodes.end(), rows[seg].begin(), rows[seg].end());
        }
        P.row_off[P.n_leaves] = (int32_t)P.row_nodes.size();
    }
    return 0;
}
