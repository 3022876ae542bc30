// Host-side planner: cluster tree (A1), block tree (A2) and the theta-independent
// lazy-column H-Cholesky task schedule (A7), see DESIGN.md "H-Cholesky formulation".
#pragma once
#include <cstdint>
#include <vector>

#include "hcov_internal.h"

struct Plan {
    // ---- A1: cluster tree -------------------------------------------------------------
    int64_t n = 0, n_pad = 0;
    int depth = 0;                  // L; leaves = 2^L clusters of 32 (padded) positions
    int64_t n_leaves = 0;
    double eta = 2.0;
    int dense_below = 32;
    std::vector<int64_t> perm_i2e;  // n_pad, -1 for phantom positions
    std::vector<double> xs, ys;     // n_pad internal coordinates (NaN for phantom)
    std::vector<double> bb;         // 4 per cluster heap id: lo_x, lo_y, hi_x, hi_y
    int64_t n_clusters = 0;         // 2^(L+1) - 1 (heap ids: id = 2^l - 1 + c)

    // ---- A2: block tree (lower triangle incl. diagonal) ------------------------------
    std::vector<DNode> nodes;
    std::vector<int32_t> tile_node;  // tile id -> node id
    std::vector<DRBlk> rblk;         // R id -> block
    std::vector<int32_t> children;   // 4 per node (-1 where absent); H nodes only

    // ---- A7: schedule ------------------------------------------------------------------
    std::vector<DTerm> terms;        // flattened by node (DNode::term_off/cnt)
    std::vector<DTask> tasks;        // in generation (post-order) order
    std::vector<int32_t> task_wave;  // wave (topological level) of each task
    int32_t n_waves = 0;
    std::vector<int32_t> wave_off;   // tasks sorted by (wave, type): wave w = [wave_off[w], wave_off[w+1])
    std::vector<int32_t> wave_tasks; // task ids sorted by (wave, type, generation)
    std::vector<int32_t> col_r_off, col_r;   // per cluster heap id: R ids of its column entries
    std::vector<DPhw> phw;
    std::vector<int32_t> phw_part;   // partner R ids
    std::vector<int32_t> hleaf;      // flattened leaf node lists of H nodes used by PHW
    int64_t w_elems = 0;             // W pool size in elements (per unit kcap: multiply by kcap)
    int32_t n_cores = 0;
    std::vector<int32_t> core_fac;   // unused placeholder (core dims come from factors)
    // factors: [0, nR) = U of R blocks, [nR, nR + nW) = W slices
    std::vector<int64_t> fac_row0;
    std::vector<int32_t> fac_nrows;
    std::vector<int32_t> fac_rank_src;  // R id whose rank is the factor's column count
    std::vector<int64_t> fac_off;       // element offset in its pool (per unit kcap for W: col offset)
    std::vector<int8_t> fac_pool;       // 0 = U pool, 1 = W pool
    // forward-solve program
    std::vector<DOp> ops;
    std::vector<int32_t> op_beg, op_end;  // per cluster heap id
    // row lists for the parallel forward solve / sampling: per leaf row, T/R nodes intersecting it
    std::vector<int32_t> row_off, row_nodes;
    // low-rank blocks in element units
    int64_t uv_elems = 0;            // per unit kcap
    int32_t max_m_rfin_small = 0;

    int64_t n_tiles() const { return (int64_t)tile_node.size(); }
    int64_t n_r() const { return (int64_t)rblk.size(); }
    int64_t cluster_size(int level) const { return (int64_t)HCOV_LEAF << (depth - level); }
};

// Build everything from host coordinates s (n x 2 row-major, external order).
// Returns 0 on success, nonzero on invalid input.
int plan_build(Plan &P, const double *s_host, int64_t n, double eta, int dense_below);
