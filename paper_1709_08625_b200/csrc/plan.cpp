// Host-side planner.  See plan.h and DESIGN.md.
//
//  A1 cluster tree   — Def. A.1; split rule "adaptive split axis"
//                      (listing PAPER.md:472) read as: tight bounding box of the node's points,
//                      split the longest axis (ties -> x) at the cardinality median (stable by
//                      current order; left gets ceil(m/2)).  Uniform depth L = ceil(log2(n/32)).
//  A2 block tree     — Def. A.2 son rule with the admissibility
//                      TStdGeomAdmCond(2.0, use_min_diam):
//                      min(diam tau, diam sigma) <= eta * dist(tau, sigma), dist > 0.
//  A3-A9 task DAG    — assembly, lazy column-oriented (left-looking) H-Cholesky and forward
//                      H-solve as a dependency graph of small tasks.
#include "plan.h"

#include <algorithm>
#include <cmath>
#include <functional>
#include <limits>
#include <numeric>
#include <unordered_map>

namespace {

// blocks below this size (and >= HCOV_GANG_MIN) are "gangs" of one CTA (PlanOpts.gang1_below)
thread_local int64_t t_gang1_below = 0;
// gang shape (PlanOpts): rows per member, largest gang below m = 65,536, RAPP gang of m = 512
thread_local int64_t t_gang_rows = 256;
thread_local int32_t t_gang_max_small = 4, t_rapp512 = 4;
// largest low-rank block whose RAPP is one dense-mode task on a single CTA (PlanOpts.big_m)
thread_local int64_t t_big_m = 256;

// gang size of an ACA / RAPP task of a low-rank block of size m (0 = a single CTA, queue 0)
inline int32_t gang_of(int64_t m)
{
    if (m < HCOV_GANG_MIN) return 0;
    if (m < t_gang1_below) return 1;
    // gangs of up to 4 CTAs (faster to form, fewer idle members in the serial phases); 8 only for
    // the largest blocks, which bounds a member's rows (and the per-CTA scratch) at m/8
    const int64_t gmax = m >= 65536 ? HCOV_GANG : t_gang_max_small;
    return (int32_t)std::min<int64_t>(gmax, std::max<int64_t>(2, m / t_gang_rows));
}
// RAPP gangs of blocks below 65,536 rows are side-split (DTask.pad = 1): half the members factor
// the X panel, half the Y panel (one QR per member instead of two; engine.cuh gang_compress_split)
inline bool rapp_split(int64_t m) { return m >= HCOV_GANG_MIN && m >= t_gang1_below && m < 65536 && m > t_big_m; }
inline int32_t rapp_gang_of(int64_t m)
{
    if (m <= t_big_m) return 0;
    if (!rapp_split(m)) return gang_of(m);
    return m <= 512 ? t_rapp512 : HCOV_GANG;
}

inline int64_t heap_id(int l, int64_t c) { return ((int64_t)1 << l) - 1 + c; }
inline uint64_t node_key(int l, int64_t i, int64_t j)
{
    return ((uint64_t)l << 58) | ((uint64_t)i << 29) | (uint64_t)j;
}

struct Builder {
    Plan &P;
    const PlanOpts &O;
    int L;
    std::unordered_map<uint64_t, int8_t> geo_type;   // device-built block tree (PlanGeo), if given
    bool use_geo = false, geo_miss = false;
    std::unordered_map<uint64_t, int32_t> key2node;
    std::vector<std::vector<int32_t>> node_terms;   // term ids per node
    std::vector<std::vector<int32_t>> col;          // per cluster heap id: off-diagonal entries
    std::vector<std::vector<int32_t>> rows;         // per leaf row: T/R nodes intersecting it (cols asc)
    std::vector<std::vector<int32_t>> deps;         // per task
    std::vector<int32_t> tile_fill, fin_tile, aca_task, rfin, rdone;
    std::vector<int32_t> term_p0, term_p1;
    int32_t root_solve = -1;
    bool too_many_partners = false;

    Builder(Plan &p, const PlanOpts &o) : P(p), O(o), L(p.depth) {}

    // ---------------------------------------------------------------- A2 geometry
    // box of cluster h: lo[d] = b[d], hi[d] = b[D + d] (D = dim)
    double diam(int64_t h) const
    {
        const int D = P.dim;
        const double *b = &P.bb[2 * D * h];
        double s2 = 0.0;
        for (int d = 0; d < D; ++d) {
            const double e = b[D + d] - b[d];
            s2 = (d == 0) ? e * e : s2 + e * e;
        }
        return std::sqrt(s2);
    }
    double dist(int64_t h1, int64_t h2) const
    {
        const int D = P.dim;
        const double *a = &P.bb[2 * D * h1], *b = &P.bb[2 * D * h2];
        double s2 = 0.0;
        for (int d = 0; d < D; ++d) {
            const double g = std::max(0.0, std::max(a[d] - b[D + d], b[d] - a[D + d]));
            s2 = (d == 0) ? g * g : s2 + g * g;
        }
        return std::sqrt(s2);
    }
    bool admissible(int l, int64_t i, int64_t j) const
    {
        if (O.eta <= 0.0) return false;
        int64_t hi = heap_id(l, i), hj = heap_id(l, j);
        double d = dist(hi, hj);
        if (!(d > 0.0)) return false;
        return std::min(diam(hi), diam(hj)) <= O.eta * d;
    }

    int32_t make(int l, int64_t i, int64_t j, int32_t parent, bool forced)
    {
        int32_t id = (int32_t)P.nodes.size();
        DNode nd{};
        nd.level = l; nd.i = (int32_t)i; nd.j = (int32_t)j;
        nd.parent = parent; nd.idx = -1;
        P.nodes.push_back(nd);
        for (int k = 0; k < 4; ++k) P.children.push_back(-1);
        key2node[node_key(l, i, j)] = id;
        int type;
        if (use_geo) {
            auto it = geo_type.find(node_key(l, i, j));
            if (it == geo_type.end()) { geo_miss = true; type = ND_T; }
            else type = it->second;
            if (type == ND_T && l != L && i == j) geo_miss = true;
        } else if (i == j) {
            type = (l == L) ? ND_T : ND_H;
        } else {
            bool adm = !forced && admissible(l, i, j);
            if (adm && l < L && P.cluster_size(l) > O.dense_below) type = ND_R;
            else if (l == L) type = ND_T;
            else { type = ND_H; forced = forced || adm; }
        }
        P.nodes[id].type = type;
        if (type == ND_T) {
            P.nodes[id].idx = (int32_t)P.tile_node.size();
            P.tile_node.push_back(id);
            if (i == j) P.diag_tile[i] = P.nodes[id].idx;
        } else if (type == ND_R) {
            DRBlk r{};
            r.node = id; r.level = l; r.m = (int32_t)P.cluster_size(l); r.solve = -1;
            r.row0 = i * P.cluster_size(l); r.col0 = j * P.cluster_size(l);
            r.uv_off = P.uv_elems;
            // capacity: kcap columns; 2 kcap for blocks recompressed in chunks (intermediate states)
            P.uv_elems += (int64_t)r.m * (r.m > O.big_m ? 2 : 1);
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

    int32_t owner(int l, int64_t i, int64_t j) const
    {
        while (true) {
            auto it = key2node.find(node_key(l, i, j));
            if (it != key2node.end()) return it->second;
            --l; i >>= 1; j >>= 1;
        }
    }

    void collect_leaves(int32_t nd, std::vector<int32_t> &out) const
    {
        const DNode &x = P.nodes[nd];
        if (x.type != ND_H) { out.push_back(nd); return; }
        for (int k = 0; k < 4; ++k) {
            int32_t c = P.children[4 * nd + k];
            if (c >= 0) collect_leaves(c, out);
        }
    }

    int64_t col_start(int32_t nd) const { return (int64_t)P.nodes[nd].j * P.cluster_size(P.nodes[nd].level); }

    // ---------------------------------------------------------------- DAG helpers
    int32_t task(int32_t type, int32_t a, int32_t b, int32_t c, int32_t d, int32_t qcls, std::vector<int32_t> dp)
    {
        int32_t id = (int32_t)P.tasks.size();
        P.tasks.push_back(DTask{type, a, b, c, d, qcls, 0, 0});
        std::sort(dp.begin(), dp.end());
        dp.erase(std::unique(dp.begin(), dp.end()), dp.end());
        if (!dp.empty() && dp[0] < 0) dp.erase(dp.begin(), std::upper_bound(dp.begin(), dp.end(), -1));
        deps.push_back(std::move(dp));
        return id;
    }
    void add_term_prods(std::vector<int32_t> &dp, int32_t t) const
    {
        if (term_p0[t] >= 0) dp.push_back(term_p0[t]);
        if (term_p1[t] >= 0) dp.push_back(term_p1[t]);
    }
    std::vector<int32_t> merged_terms(int32_t nd) const
    {
        std::vector<int32_t> v;
        for (int32_t y = nd; y >= 0; y = P.nodes[y].parent)
            v.insert(v.end(), node_terms[y].begin(), node_terms[y].end());
        std::sort(v.begin(), v.end());
        return v;
    }
    // Chunked chain over the merged term list of a leaf node; the last chunk is `fin_type`.
    int32_t chain(int32_t nd, int32_t first_dep, int32_t app_type, int32_t fin_type, int32_t a, int32_t d,
                  int32_t extra_dep, int32_t qcls)
    {
        std::vector<int32_t> tl = merged_terms(nd);
        const int32_t base = (int32_t)P.xterm.size();
        P.xterm.insert(P.xterm.end(), tl.begin(), tl.end());
        const int k = (int)tl.size();
        if (k == 0 && fin_type < 0) return first_dep;
        // tiles: chunks of O.chunk terms (exact updates); small low-rank blocks: one task (exact
        // dense accumulation); large low-rank blocks: chunks of O.rchunk terms, intermediate states
        // kept near-losslessly at capacity 2 kcap, the last chunk truncates to (eps, kmax)
        int nch = std::max(1, (k + O.chunk - 1) / O.chunk);
        if (app_type == TK_RAPP)
            nch = (P.rblk[a].m <= O.big_m) ? 1 : std::max(1, (k + O.rchunk - 1) / O.rchunk);
        int32_t prev = first_dep;
        for (int q = 0; q < nch; ++q) {
            int b = (int)((int64_t)k * q / nch), e = (int)((int64_t)k * (q + 1) / nch);
            const bool last = (q == nch - 1);
            std::vector<int32_t> dp{prev};
            for (int z = b; z < e; ++z) add_term_prods(dp, tl[z]);
            int32_t ty = app_type;
            if (last && fin_type >= 0) { ty = fin_type; dp.push_back(extra_dep); }
            const int32_t dd = (app_type == TK_RAPP) ? (last ? (O.factor_trunc ? 2 : 1) : 0) : d;
            prev = task(ty, a, base + b, base + e, dd, qcls, dp);
            if (app_type == TK_RAPP && rapp_split(P.rblk[a].m)) P.tasks[prev].pad = 1;
        }
        return prev;
    }

    // ---------------------------------------------------------------- solves
    struct SolveCtx {
        int32_t s;
        int64_t a, b;   // leaf range
        std::vector<int32_t> seg;   // per leaf (local)
        std::unordered_map<int64_t, int32_t> join;   // cluster heap id -> task
        std::unordered_map<int32_t, int32_t> proj;   // R id -> task
    };
    int32_t join(SolveCtx &S, int lv, int64_t c)
    {
        if (lv == L) return S.seg[c - S.a];
        int64_t h = heap_id(lv, c);
        auto it = S.join.find(h);
        if (it != S.join.end()) return it->second;
        int32_t j0 = join(S, lv + 1, 2 * c), j1 = join(S, lv + 1, 2 * c + 1);
        int32_t t = task(TK_NOP, 0, 0, 0, 0, 0, {j0, j1});
        S.join[h] = t;
        return t;
    }
    int32_t proj_task(SolveCtx &S, int32_t r)
    {
        auto it = S.proj.find(r);
        if (it != S.proj.end()) return it->second;
        const DRBlk &b = P.rblk[r];
        const DSolve &sv = P.solves[S.s];
        DSlot sl{P.slot_a, P.slot_b};
        if (sv.rhs_cnt > 0) P.slot_a += sv.rhs_cnt; else P.slot_b += 1;
        int32_t slot = (int32_t)P.slots.size();
        P.slots.push_back(sl);
        const int32_t tau = P.nodes[b.node].j;
        int32_t t = task(TK_PROJ, S.s, r, slot, 0, 0, {rdone[r], rfin[r], join(S, b.level, tau)});
        S.proj[r] = t;
        return t;
    }
    // Y <- L_ss^{-1} Y on the diagonal block of cluster (l, c); returns the task after which Y is final.
    int32_t build_solve(int l, int64_t c, const std::vector<int32_t> &rhs)
    {
        DSolve sv{};
        sv.level = l; sv.c = (int32_t)c;
        sv.rhs_off = (int32_t)P.solve_rhs.size();
        sv.rhs_cnt = (int32_t)rhs.size();
        sv.m = P.cluster_size(l);
        sv.row0 = c * sv.m;
        P.solve_rhs.insert(P.solve_rhs.end(), rhs.begin(), rhs.end());
        SolveCtx S;
        S.s = (int32_t)P.solves.size();
        P.solves.push_back(sv);
        S.a = c << (L - l);
        S.b = (c + 1) << (L - l);
        S.seg.assign(S.b - S.a, -1);
        std::vector<int32_t> rhs_deps;
        for (int32_t r : rhs) rhs_deps.push_back(rfin[r]);
        for (int64_t i = S.a; i < S.b; ++i) {
            std::vector<int32_t> dp(rhs_deps);
            dp.push_back(fin_tile[P.diag_tile[i]]);
            const int32_t cb = (int32_t)P.ctr.size();
            for (int32_t nd : rows[i]) {
                const DNode &x = P.nodes[nd];
                if (x.type == ND_T) {
                    if (x.j >= S.a && x.j < i) {
                        P.ctr.push_back(DCtr{0, x.idx, x.j, 0});
                        dp.push_back(fin_tile[x.idx]);
                        dp.push_back(S.seg[x.j - S.a]);
                    }
                } else if (col_start(nd) >= S.a * HCOV_LEAF) {
                    const int32_t r = x.idx;
                    int32_t pt = proj_task(S, r);
                    int32_t slot = P.tasks[pt].c;
                    P.ctr.push_back(DCtr{1, r, slot, 0});
                    dp.push_back(pt);
                }
            }
            const int32_t ce = (int32_t)P.ctr.size();
            S.seg[i - S.a] = task(TK_SEG, S.s, (int32_t)i, cb, ce, 0, dp);
        }
        return join(S, l, c);
    }

    // Root back-solve u = L~^{-T} v (transpose of the root forward solve; NEXT (f1), listing
    // PAPER.md:550-555): leaf segments from the last to the first; segment i subtracts, for every
    // strictly-lower leaf (rho, sigma) whose column range holds i, its transpose applied to the final
    // u of its rows: tiles T^T u_rho (kind 0, aux = row segment), low-rank blocks V_b[rows of i] t_b
    // with t_b = U_b^T u[rows of b] from a BPROJ task (kind 1), which waits for all of b's row segments.
    void build_backsolve(const std::vector<std::vector<int32_t>> &colsv)
    {
        const int64_t nl = P.n_leaves;
        std::vector<int32_t> bseg(nl, -1);
        std::unordered_map<int64_t, int32_t> bj, bproj;
        std::function<int32_t(int, int64_t)> bjoin = [&](int lv, int64_t c) -> int32_t {
            if (lv == L) return bseg[c];
            const int64_t h = heap_id(lv, c);
            auto it = bj.find(h);
            if (it != bj.end()) return it->second;
            const int32_t t = task(TK_NOP, 0, 0, 0, 0, 0, {bjoin(lv + 1, 2 * c), bjoin(lv + 1, 2 * c + 1)});
            bj[h] = t;
            return t;
        };
        for (int64_t i = nl - 1; i >= 0; --i) {
            std::vector<int32_t> dp;
            const int32_t cb = (int32_t)P.ctr.size();
            for (int32_t nd : colsv[i]) {
                const DNode &x = P.nodes[nd];
                if (x.type == ND_T) {
                    P.ctr.push_back(DCtr{0, x.idx, x.i, 0});
                    dp.push_back(bseg[x.i]);
                } else {
                    const int32_t r = x.idx;
                    auto it = bproj.find(r);
                    int32_t pt;
                    if (it != bproj.end()) pt = it->second;
                    else {
                        pt = task(TK_BPROJ, 0, r, 0, 0, 0, {bjoin(x.level, x.i)});
                        bproj[r] = pt;
                    }
                    P.ctr.push_back(DCtr{1, r, 0, 0});
                    dp.push_back(pt);
                }
            }
            const int32_t ce = (int32_t)P.ctr.size();
            bseg[i] = task(TK_BSEG, 0, (int32_t)i, cb, ce, 0, dp);
        }
    }

    // W = H_e * [V of partners]: PHWP per low-rank leaf of H_e, PHWR per leaf row of H_e.
    int32_t build_phw(int32_t e, const std::vector<int32_t> &rents, int32_t col_off, int32_t solve_done)
    {
        const DNode h = P.nodes[e];
        const int64_t m = P.cluster_size(h.level);
        DPhw q{};
        q.hnode = e;
        q.part_off = col_off;
        q.part_cnt = (int32_t)rents.size();
        q.fac_base = (int32_t)P.fac_row0.size();
        q.m = (int32_t)m;
        q.w_off = P.w_elems;
        P.w_elems += m * (int64_t)rents.size();
        const int32_t qid = (int32_t)P.phw.size();
        if (rents.size() >= ((size_t)1 << 20)) too_many_partners = true;   // fac_off packs p in 20 bits
        for (int p = 0; p < (int)rents.size(); ++p) {
            P.fac_row0.push_back((int64_t)h.i * m);
            P.fac_nrows.push_back((int32_t)m);
            P.fac_rank_src.push_back(rents[p]);
            P.fac_off.push_back(((int64_t)qid << 20) | p);  // W slice: (phw id, partner index < 2^20), offset at run time
            P.fac_pool.push_back(1);
        }
        P.phw.push_back(q);
        std::vector<int32_t> lv;
        collect_leaves(e, lv);
        std::unordered_map<int32_t, std::pair<int32_t, int32_t>> rq;   // R id -> (task, slot)
        for (int32_t nd : lv) {
            const DNode &x = P.nodes[nd];
            if (x.type != ND_R) continue;
            DSlot sl{P.slot_a, P.slot_b};
            P.slot_a += (int64_t)rents.size();
            int32_t slot = (int32_t)P.slots.size();
            P.slots.push_back(sl);
            int32_t t = task(TK_PHWP, qid, x.idx, slot, 0, 0, {rdone[x.idx], rfin[x.idx], solve_done});
            rq[x.idx] = {t, slot};
        }
        const int64_t rho0 = (int64_t)h.i * m, sig0 = (int64_t)h.j * m;
        std::vector<int32_t> rowt;
        for (int64_t i = rho0 / HCOV_LEAF; i < (rho0 + m) / HCOV_LEAF; ++i) {
            std::vector<int32_t> dp{solve_done};
            const int32_t cb = (int32_t)P.ctr.size();
            for (int32_t nd : rows[i]) {
                const int64_t cs = col_start(nd);
                if (cs < sig0 || cs >= sig0 + m) continue;
                const DNode &x = P.nodes[nd];
                if (x.type == ND_T) {
                    P.ctr.push_back(DCtr{0, x.idx, x.j, 0});
                    dp.push_back(fin_tile[x.idx]);
                } else {
                    auto pr = rq.at(x.idx);
                    P.ctr.push_back(DCtr{1, x.idx, pr.second, 0});
                    dp.push_back(pr.first);
                }
            }
            const int32_t ce = (int32_t)P.ctr.size();
            rowt.push_back(task(TK_PHWR, qid, (int32_t)i, cb, ce, 0, dp));
        }
        return task(TK_NOP, 0, 0, 0, 0, 0, rowt);
    }

    int32_t new_term(int32_t kind, int32_t a, int32_t b, int32_t core, int32_t p0, int32_t p1, int32_t owner_node)
    {
        int32_t id = (int32_t)P.terms.size();
        P.terms.push_back(DTerm{kind, a, b, core});
        term_p0.push_back(p0);
        term_p1.push_back(p1);
        node_terms[owner_node].push_back(id);
        return id;
    }

    // ---------------------------------------------------------------- column processing
    void post(int l, int64_t c)
    {
        if (l < L) { post(l + 1, 2 * c); post(l + 1, 2 * c + 1); }
        const int64_t sig = heap_id(l, c);
        if (l == L) {
            const int32_t d = key2node.at(node_key(L, c, c));
            const int32_t t = P.nodes[d].idx;
            fin_tile[t] = chain(d, tile_fill[t], TK_TAPP, TK_POTRF, t, -1, -1, 0);
        }
        std::vector<int32_t> &ents = col[sig];
        std::sort(ents.begin(), ents.end(), [&](int32_t a, int32_t b) { return P.nodes[a].i < P.nodes[b].i; });
        std::vector<int32_t> rents;
        for (int32_t e : ents) {
            const DNode &x = P.nodes[e];
            if (x.type == ND_T) {
                const int32_t dt = P.diag_tile[c];
                fin_tile[x.idx] = chain(e, tile_fill[x.idx], TK_TAPP, TK_TRSM, x.idx, dt, fin_tile[dt], 0);
            } else if (x.type == ND_R) {
                const int32_t qc = rapp_gang_of(P.rblk[x.idx].m);
                rfin[x.idx] = chain(e, aca_task[x.idx], TK_RAPP, -1, x.idx, 0, -1, qc);
                rents.push_back(x.idx);
            }
        }
        const int32_t col_off = (int32_t)P.col_r_off[sig];
        std::unordered_map<int32_t, int32_t> h2phw, h2done;
        if (!rents.empty()) {
            const int32_t s_id = (int32_t)P.solves.size();
            for (int32_t r : rents) P.rblk[r].solve = s_id;
            const int32_t done = build_solve(l, c, rents);
            int32_t pdone = done;
            if (O.factor_trunc) {
                // SPD-preserving mode: truncate every factor block L_21 = U (L_ss^{-1} V)^T of the
                // column once its solve is done; the products use the truncated blocks
                std::vector<int32_t> tt;
                for (int32_t r : rents) {
                    const int32_t base = (int32_t)P.xterm.size();
                    const int32_t t = task(TK_RAPP, r, base, base, 1, rapp_gang_of(P.rblk[r].m), {done});
                    if (rapp_split(P.rblk[r].m)) P.tasks[t].pad = 1;
                    rdone[r] = t;
                    tt.push_back(t);
                }
                pdone = task(TK_NOP, 0, 0, 0, 0, 0, tt);
            } else {
                for (int32_t r : rents) rdone[r] = done;
            }
            for (int32_t e : ents) {
                if (P.nodes[e].type != ND_H) continue;
                h2phw[e] = (int32_t)P.phw.size();
                h2done[e] = build_phw(e, rents, col_off, pdone);
            }
        }
        // Schur-complement terms L_{e1} L_{e2}^T (e1.i >= e2.i) onto the owner of (e1.i, e2.i)
        for (size_t a = 0; a < ents.size(); ++a) {
            for (size_t b = 0; b <= a; ++b) {
                const int32_t e1 = ents[a], e2 = ents[b];
                const DNode &x1 = P.nodes[e1], &x2 = P.nodes[e2];
                const int t1 = x1.type, t2 = x2.type;
                if (t1 == ND_H && t2 == ND_H) continue;   // resolved at the children's columns
                const int32_t o = owner(l, x1.i, x2.i);
                if (t1 == ND_T && t2 == ND_T) {
                    new_term(TM_TT, x1.idx, x2.idx, -1, fin_tile[x1.idx], fin_tile[x2.idx], o);
                } else if (t1 == ND_R && t2 == ND_R) {
                    const int32_t core = P.n_cores++;
                    int32_t pt = task(TK_PRR, x1.idx, x2.idx, core, 0, 0, {rdone[x1.idx], rdone[x2.idx]});
                    new_term(TM_LR, x1.idx, x2.idx, core, pt, -1, o);
                } else if (t1 == ND_R && t2 == ND_H) {
                    const int32_t q = h2phw.at(e2);
                    const int p = (int)(std::find(rents.begin(), rents.end(), x1.idx) - rents.begin());
                    new_term(TM_LR, x1.idx, P.phw[q].fac_base + p, -1, h2done.at(e2), -1, o);
                } else if (t1 == ND_H && t2 == ND_R) {
                    const int32_t q = h2phw.at(e1);
                    const int p = (int)(std::find(rents.begin(), rents.end(), x2.idx) - rents.begin());
                    new_term(TM_LR, P.phw[q].fac_base + p, x2.idx, -1, h2done.at(e1), -1, o);
                }
                // T x R, R x T cannot occur: entries of one column share the level, T only at level L
            }
        }
    }
};

}  // namespace

int plan_build(Plan &P, const double *s, int64_t n, const PlanOpts &opt, const PlanGeo *geo)
{
    if (n <= 0) return 2;
    if (opt.dim != 2 && opt.dim != 3) return 1;
    const int D = opt.dim;
    if (!geo)
        for (int64_t k = 0; k < D * n; ++k)
            if (!std::isfinite(s[k])) return 1;
    P.opt = opt;
    t_gang1_below = opt.gang1_below;
    t_gang_rows = std::max<int64_t>(32, opt.gang_rows);
    t_gang_max_small = std::max(2, std::min(HCOV_GANG, opt.gang_max_small));
    t_rapp512 = std::max(2, std::min(HCOV_GANG, opt.rapp512)) & ~1;
    P.opt.dense_below = std::max(opt.dense_below, HCOV_LEAF);
    P.opt.chunk = std::max(1, opt.chunk);
    P.opt.fill_tiles = std::max(1, opt.fill_tiles);
    P.opt.big_m = std::max<int64_t>(32, std::min<int64_t>(HCOV_DENSE_MAX, opt.big_m));
    t_big_m = P.opt.big_m;
    int L = 0;
    while (((int64_t)HCOV_LEAF << L) < n) ++L;
    P.n = n; P.depth = L; P.n_leaves = (int64_t)1 << L; P.n_pad = (int64_t)HCOV_LEAF << L;
    P.n_clusters = ((int64_t)2 << L) - 1;
    P.dim = D;
    P.bb.assign(2 * D * P.n_clusters, 0.0);

    if (geo) {   // A1 done on the device (tree.cu K1)
        if (geo->depth != L || (int64_t)geo->perm_i2e.size() != P.n_pad || (int64_t)geo->xs.size() != P.n_pad ||
            (int64_t)geo->ys.size() != P.n_pad || (int64_t)geo->bb.size() != 2 * D * P.n_clusters ||
            (D == 3 && (int64_t)geo->zs.size() != P.n_pad))
            return 3;
        P.perm_i2e = geo->perm_i2e;
        P.xs = geo->xs;
        P.ys = geo->ys;
        if (D == 3) P.zs = geo->zs;
        P.bb = geo->bb;
    }
    // ---- A1 -------------------------------------------------------------------------------
    std::vector<int64_t> perm(geo ? 0 : n);
    if (!geo) {
    std::iota(perm.begin(), perm.end(), 0);
    std::vector<int64_t> rs{0}, re{n};
    for (int l = 0; l <= L; ++l) {
        int64_t nc = (int64_t)1 << l;
        std::vector<int64_t> rs2, re2;
        if (l < L) { rs2.resize(2 * nc); re2.resize(2 * nc); }
        for (int64_t c = 0; c < nc; ++c) {
            double lo[3], hi[3];
            for (int d = 0; d < D; ++d) { lo[d] = std::numeric_limits<double>::infinity(); hi[d] = -lo[d]; }
            for (int64_t k = rs[c]; k < re[c]; ++k)
                for (int d = 0; d < D; ++d) {
                    const double x = s[D * perm[k] + d];
                    lo[d] = std::min(lo[d], x); hi[d] = std::max(hi[d], x);
                }
            double *b = &P.bb[2 * D * heap_id(l, c)];
            for (int d = 0; d < D; ++d) {
                b[d] = (re[c] > rs[c]) ? lo[d] : std::numeric_limits<double>::quiet_NaN();
                b[D + d] = (re[c] > rs[c]) ? hi[d] : std::numeric_limits<double>::quiet_NaN();
            }
            if (l == L) continue;
            // longest extent, ties -> lowest axis (x, then y)
            int axis = 0;
            for (int d = 1; d < D; ++d)
                if (hi[d] - lo[d] > hi[axis] - lo[axis]) axis = d;
            std::stable_sort(perm.begin() + rs[c], perm.begin() + re[c],
                             [&](int64_t a, int64_t b2) { return s[D * a + axis] < s[D * b2 + axis]; });
            int64_t m = re[c] - rs[c], m1 = (m + 1) / 2;
            rs2[2 * c] = rs[c]; re2[2 * c] = rs[c] + m1;
            rs2[2 * c + 1] = rs[c] + m1; re2[2 * c + 1] = re[c];
        }
        if (l < L) { rs.swap(rs2); re.swap(re2); }
    }
    P.perm_i2e.assign(P.n_pad, -1);
    P.xs.assign(P.n_pad, std::numeric_limits<double>::quiet_NaN());
    P.ys.assign(P.n_pad, std::numeric_limits<double>::quiet_NaN());
    if (D == 3) P.zs.assign(P.n_pad, std::numeric_limits<double>::quiet_NaN());
    for (int64_t c = 0; c < P.n_leaves; ++c) {
        if (re[c] - rs[c] > HCOV_LEAF) return 3;  // cannot happen (sizes <= ceil(n / 2^L) <= 32)
        for (int64_t k = rs[c]; k < re[c]; ++k) {
            int64_t pos = c * HCOV_LEAF + (k - rs[c]);
            P.perm_i2e[pos] = perm[k];
            P.xs[pos] = s[D * perm[k]];
            P.ys[pos] = s[D * perm[k] + 1];
            if (D == 3) P.zs[pos] = s[D * perm[k] + 2];
        }
    }
    }   // !geo

    // ---- A2 -------------------------------------------------------------------------------
    Builder B(P, P.opt);
    if (geo) {   // A2 done on the device (tree.cu K2): the recursion below only reads its node types
        B.use_geo = true;
        size_t cnt = 0;
        for (const auto &v : geo->level_pairs) cnt += v.size();
        B.geo_type.reserve(cnt);
        for (int l = 0; l < (int)geo->level_pairs.size(); ++l) {
            if (geo->level_types[l].size() != geo->level_pairs[l].size()) return 3;
            for (size_t p = 0; p < geo->level_pairs[l].size(); ++p)
                B.geo_type[node_key(l, geo->level_pairs[l][p].first, geo->level_pairs[l][p].second)] =
                    geo->level_types[l][p];
        }
    }
    P.diag_tile.assign(P.n_leaves, -1);
    B.make(0, 0, 0, -1, false);
    if (B.use_geo && (B.geo_miss || P.nodes.size() != B.geo_type.size())) return 3;
    const size_t nn = P.nodes.size();
    B.node_terms.assign(nn, {});
    B.col.assign(P.n_clusters, {});
    B.rows.assign(P.n_leaves, {});
    for (size_t k = 0; k < nn; ++k) {
        const DNode &x = P.nodes[k];
        if (x.i != x.j) B.col[heap_id(x.level, x.j)].push_back((int32_t)k);
        if (x.type == ND_H) continue;
        int64_t span = (int64_t)1 << (L - x.level);
        for (int64_t seg = (int64_t)x.i * span; seg < (int64_t)(x.i + 1) * span; ++seg)
            B.rows[seg].push_back((int32_t)k);
    }
    for (auto &rw : B.rows)
        std::sort(rw.begin(), rw.end(), [&](int32_t a, int32_t b) { return B.col_start(a) < B.col_start(b); });
    // column R lists (CSR by heap id, rows ascending)
    P.col_r_off.assign(P.n_clusters + 1, 0);
    for (int64_t sig = 0; sig < P.n_clusters; ++sig) {
        std::vector<int32_t> &e = B.col[sig];
        std::sort(e.begin(), e.end(), [&](int32_t a, int32_t b) { return P.nodes[a].i < P.nodes[b].i; });
        P.col_r_off[sig] = (int32_t)P.col_r.size();
        for (int32_t k : e)
            if (P.nodes[k].type == ND_R) P.col_r.push_back(P.nodes[k].idx);
    }
    P.col_r_off[P.n_clusters] = (int32_t)P.col_r.size();
    // factor table part 1: U of R blocks
    for (size_t r = 0; r < P.rblk.size(); ++r) {
        P.fac_row0.push_back(P.rblk[r].row0);
        P.fac_nrows.push_back(P.rblk[r].m);
        P.fac_rank_src.push_back((int32_t)r);
        P.fac_off.push_back(P.rblk[r].uv_off);
        P.fac_pool.push_back(0);
    }

    // ---- A3-A6: assembly tasks (roots) ------------------------------------------------------
    const int64_t nt = P.n_tiles(), nr = P.n_r();
    B.tile_fill.assign(nt, -1);
    B.fin_tile.assign(nt, -1);
    B.aca_task.assign(nr, -1);
    B.rfin.assign(nr, -1);
    B.rdone.assign(nr, -1);
    for (int64_t t0 = 0; t0 < nt; t0 += P.opt.fill_tiles) {
        int32_t cnt = (int32_t)std::min<int64_t>(P.opt.fill_tiles, nt - t0);
        int32_t id = B.task(TK_FILL, (int32_t)t0, cnt, 0, 0, 0, {});
        for (int64_t t = t0; t < t0 + cnt; ++t) B.tile_fill[t] = id;
    }
    for (int64_t r = 0; r < nr; ++r)
        B.aca_task[r] = B.task(TK_ACA, (int32_t)r, 0, 0, 0, gang_of(P.rblk[r].m), {});

    // ---- A7: lazy column H-Cholesky; A9: root forward solve --------------------------------
    B.post(0, 0);
    const int32_t first_root_task = (int32_t)P.tasks.size();
    B.root_solve = (int32_t)P.solves.size();
    B.build_solve(0, 0, {});
    if (B.too_many_partners) return 1;
    // columns (transpose of rows[]): strictly-lower leaves over each leaf column, rows ascending
    std::vector<std::vector<int32_t>> colsv(P.n_leaves);
    for (size_t k = 0; k < P.nodes.size(); ++k) {
        const DNode &x = P.nodes[k];
        if (x.type == ND_H || x.i == x.j) continue;
        const int64_t span = (int64_t)1 << (L - x.level);
        for (int64_t seg = (int64_t)x.j * span; seg < (int64_t)(x.j + 1) * span; ++seg) colsv[seg].push_back((int32_t)k);
    }
    for (auto &cv : colsv)
        std::sort(cv.begin(), cv.end(), [&](int32_t a, int32_t b) {
            const int64_t ra = (int64_t)P.nodes[a].i * P.cluster_size(P.nodes[a].level);
            const int64_t rb = (int64_t)P.nodes[b].i * P.cluster_size(P.nodes[b].level);
            return ra < rb;
        });
    P.col_off.assign(P.n_leaves + 1, 0);
    P.col_nodes.clear();
    for (int64_t seg = 0; seg < P.n_leaves; ++seg) {
        P.col_off[seg] = (int32_t)P.col_nodes.size();
        P.col_nodes.insert(P.col_nodes.end(), colsv[seg].begin(), colsv[seg].end());
    }
    P.col_off[P.n_leaves] = (int32_t)P.col_nodes.size();
    const int32_t first_back_task = (int32_t)P.tasks.size();
    B.build_backsolve(colsv);

    // ---- DAG: phases, successors, per-mode in-degrees and roots, critical path ------------
    const int32_t ntk = (int32_t)P.tasks.size();
    P.root_solve = B.root_solve;
    P.phase.assign(ntk, 1);
    for (int32_t t = 0; t < ntk; ++t) {
        const int ty = P.tasks[t].type;
        if (ty == TK_FILL || ty == TK_ACA) P.phase[t] = 0;
        else if (t >= first_back_task) P.phase[t] = 3;
        else if (t >= first_root_task) P.phase[t] = 2;
    }
    P.succ_off.assign(ntk + 1, 0);
    for (int32_t t = 0; t < ntk; ++t)
        for (int32_t d : B.deps[t]) P.succ_off[d + 1]++;
    for (int32_t t = 0; t < ntk; ++t) P.succ_off[t + 1] += P.succ_off[t];
    P.succ.assign(P.succ_off[ntk], 0);
    {
        std::vector<int32_t> fillp(P.succ_off.begin(), P.succ_off.end() - 1);
        for (int32_t t = 0; t < ntk; ++t)
            for (int32_t d : B.deps[t]) P.succ[fillp[d]++] = t;
    }
    std::vector<int32_t> len(ntk, 0);
    std::vector<int64_t> key(ntk, 0);
    P.crit_len = 0;
    for (int32_t t = 0; t < ntk; ++t) {
        const DTask &k = P.tasks[t];
        int32_t lmax = 0;
        for (int32_t d : B.deps[t]) lmax = std::max(lmax, len[d]);
        len[t] = lmax + (k.type == TK_NOP ? 0 : 1);
        if (P.phase[t] <= 2) P.crit_len = std::max(P.crit_len, len[t]);   // the evaluation's chain
        if (k.type == TK_FILL) {
            int64_t cmin = INT64_MAX;
            for (int32_t q = k.a; q < k.a + k.b; ++q) cmin = std::min<int64_t>(cmin, P.nodes[P.tile_node[q]].j);
            key[t] = cmin * HCOV_LEAF;
        } else if (k.type == TK_ACA) {
            key[t] = P.rblk[k.a].col0;
        } else {
            key[t] = (int64_t)1 << 40;   // non-assembly roots keep generation order
        }
    }
    // priority bands of queue 0: bottom level (longest remaining path, weighted by a rough
    // per-type cost in units of ~25 us) quantised into HCOV_BANDS bands
    {
        std::vector<double> w(ntk, 1.0), bl(ntk, 0.0);
        for (int32_t t = 0; t < ntk; ++t) {
            const DTask &k = P.tasks[t];
            if (k.type == TK_NOP) w[t] = 0.0;
            else if (k.type == TK_RAPP || k.type == TK_ACA) {
                const double m = (double)P.rblk[k.a].m;
                if (k.type == TK_RAPP && m <= P.opt.big_m) w[t] = 40.0 * std::max(1.0, m * m / 65536.0);   // dense mode
                else w[t] = (m <= 256) ? 40.0 : 40.0 + m / (64.0 * std::max(1, k.qcls));
            } else if (k.type == TK_SEG || k.type == TK_PHWR || k.type == TK_BSEG) w[t] = 3.0;
        }
        double bmax = 0.0;
        for (int32_t t = ntk - 1; t >= 0; --t) {
            double mx = 0.0;
            for (int32_t z = P.succ_off[t]; z < P.succ_off[t + 1]; ++z) mx = std::max(mx, bl[P.succ[z]]);
            bl[t] = w[t] + mx;
            bmax = std::max(bmax, bl[t]);
        }
        std::vector<int32_t> cnt(HCOV_BANDS, 0);
        for (int32_t t = 0; t < ntk; ++t) {
            int b = (int)std::floor(HCOV_BANDS * bl[t] / (bmax + 1e-9));
            b = std::min(HCOV_BANDS - 1, std::max(0, b));
            P.tasks[t].band = b;
            if (P.tasks[t].type != TK_NOP) cnt[b] += std::max(1, P.tasks[t].qcls);
        }
        P.band_off.assign(HCOV_BANDS + 1, 0);
        for (int b = 0; b < HCOV_BANDS; ++b) P.band_off[b + 1] = P.band_off[b] + std::max(1, cnt[b]);
    }
    static const int mask[HCOV_MODES] = {7, 1, 2, 4, 8};
    for (int md = 0; md < HCOV_MODES; ++md) {
        P.indeg[md].assign(ntk, 0);
        std::vector<std::pair<int64_t, int32_t>> rk[2];
        for (int32_t t = 0; t < ntk; ++t) {
            if (!(mask[md] & (1 << P.phase[t]))) continue;
            int32_t cnt = 0;
            for (int32_t d : B.deps[t])
                if (mask[md] & (1 << P.phase[d])) ++cnt;
            P.indeg[md][t] = cnt;
            const DTask &k = P.tasks[t];
            // one queue: a gang task of G CTAs occupies G consecutive entries (task * 32 + member)
            if (k.type != TK_NOP) P.n_q[md][0] += 1;
            if (cnt == 0) rk[0].push_back({key[t], t});   // (a NOP always has a dependency)
        }
        {
            // queue 0: roots placed in their bands in key order
            std::stable_sort(rk[0].begin(), rk[0].end());
            P.q0init[md].assign(P.band_off[HCOV_BANDS], -1);
            P.q0tail[md].assign(HCOV_BANDS, 0);
            for (auto &pr : rk[0]) {
                const int b = P.tasks[pr.second].band;
                const int G = std::max(1, P.tasks[pr.second].qcls);
                for (int g = 0; g < G; ++g) P.q0init[md][P.band_off[b] + P.q0tail[md][b]++] = pr.second * 32 + g;
            }
        }
        for (int c = 0; c < 2; ++c) {
            std::stable_sort(rk[c].begin(), rk[c].end());
            P.roots[md][c].clear();
            for (auto &pr : rk[c]) {
                if (c == 0) P.roots[md][c].push_back(pr.second);
                else
                    for (int g = 0; g < P.tasks[pr.second].qcls; ++g) P.roots[md][c].push_back(pr.second * 32 + g);
            }
        }
    }
    for (const DRBlk &r : P.rblk) {
        P.max_rm = std::max<int64_t>(P.max_rm, r.m);
        const int32_t g = gang_of(r.m);
        if (g > 0) P.max_mq = std::max<int64_t>(P.max_mq, r.m - (int64_t)(g - 1) * (r.m / g));   // last member
        if (rapp_split(r.m)) {   // side-split RAPP gang: G/2 members per side
            const int64_t gs = rapp_gang_of(r.m) / 2;
            P.max_mq = std::max<int64_t>(P.max_mq, r.m - (gs - 1) * (r.m / gs));
        }
    }
    return 0;
}
