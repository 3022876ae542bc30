// Host-side planner: cluster tree (A1), block tree (A2) and the theta-independent task DAG of
// the assembly (A3-A6), the lazy left-looking H-Cholesky (A7) and the forward H-solve (A9).
// See DESIGN.md "H-Cholesky formulation" and "Engine".
#pragma once
#include <cstdint>
#include <utility>
#include <vector>

#include "hcov_internal.h"

struct PlanOpts {
    double eta = 2.0;
    int dense_below = 32;   // admissible blocks of cluster size <= dense_below are dense tiles
    int chunk = 4;          // pending terms applied per TAPP task
    int rchunk = 4;         // pending terms appended per RAPP task of a large low-rank block (4 since the
                            // terms enter with min(rank A, rank B) columns; 3 before)
    int fill_tiles = 8;     // tiles per FILL task
    int64_t big_m = 256;    // low-rank blocks up to this size: one dense-mode RAPP task (a single CTA);
                            // larger ones: chunked recompression (gangs), capacity 2 kcap (<= HCOV_DENSE_MAX)
    int dim = 2;            // 2-D locations, or 3 (the 3-D variant)
    int64_t gang_rows = 256;   // rows per gang member (ACA / non-split RAPP gangs: G = m / gang_rows)
    int gang_max_small = 4;    // largest such gang below m = 65,536
    int rapp512 = 4;           // side-split RAPP gang of the m = 512 blocks (even)
    int64_t gang1_below = 0;   // low-rank blocks with HCOV_GANG_MIN <= m < gang1_below run their ACA /
                               // RAPP tasks as one-CTA gangs (in-CTA TSQR, no inter-CTA barriers)
    bool factor_trunc = false;  // SPD-preserving mode (R27): per low-rank block, the last
                                // update chunk keeps the block near-lossless (d = 2), the block's
                                // forward solve runs on that, then a TRUNC task (a RAPP without terms,
                                // d = 1) truncates the factor block L_21 to (eps, kmax)
};

struct Plan {
    PlanOpts opt;
    // ---- A1: cluster tree -------------------------------------------------------------
    int64_t n = 0, n_pad = 0;
    int depth = 0;                  // L; leaves = 2^L clusters of 32 (padded) positions
    int64_t n_leaves = 0;
    std::vector<int64_t> perm_i2e;  // n_pad, -1 for phantom positions
    int dim = 2;                    // 2 or 3
    std::vector<double> xs, ys, zs; // n_pad internal coordinates (NaN for phantom); zs only for dim 3
    std::vector<double> bb;         // 2 dim per cluster heap id: lo_x, lo_y[, lo_z], hi_x, hi_y[, hi_z]
    int64_t n_clusters = 0;         // 2^(L+1) - 1 (heap ids: id = 2^l - 1 + c)

    // ---- A2: block tree (lower triangle incl. diagonal) ------------------------------
    std::vector<DNode> nodes;
    std::vector<int32_t> tile_node;  // tile id -> node id
    std::vector<DRBlk> rblk;         // R id -> block
    std::vector<int32_t> children;   // 4 per node (-1 where absent); H nodes only
    std::vector<int32_t> diag_tile;  // per leaf: tile id of its diagonal block
    int64_t uv_elems = 0;            // U / V pool size per unit kcap

    // ---- A7 / A9: terms, factors, products ---------------------------------------------
    std::vector<DTerm> terms;
    std::vector<int32_t> xterm_off;  // per tile (t) then per R (n_tiles + r): range in xterm[]
    std::vector<int32_t> xterm;      // term ids (merged own + ancestor terms, generation order)
    std::vector<int32_t> col_r_off, col_r;   // per cluster heap id: R ids of its column entries
    std::vector<DPhw> phw;
    int64_t w_elems = 0;             // W pool size per unit kcap
    int32_t n_cores = 0;
    std::vector<int64_t> fac_row0;   // factors: [0, nR) = U of R blocks, then W slices
    std::vector<int32_t> fac_nrows;
    std::vector<int32_t> fac_rank_src;  // R id whose rank is the factor's column count
    std::vector<int64_t> fac_off;       // element offset per unit kcap in its pool
    std::vector<int8_t> fac_pool;       // 0 = U pool, 1 = W pool
    std::vector<DSolve> solves;      // [0] = root forward solve
    std::vector<int32_t> solve_rhs;
    std::vector<DSlot> slots;        // PROJ / PHWP product slots
    int64_t slot_a = 0, slot_b = 0;  // pool size = slot_a * kcap^2 + slot_b * kcap
    std::vector<DCtr> ctr;           // SEG / PHWR contribution lists

    // ---- DAG ---------------------------------------------------------------------------
    // Engine modes: 0 = phases 0-2 (hcov_eval), 1 = assembly (A3-A6), 2 = H-Cholesky (A7),
    // 3 = forward solve (A8-A9), 4 = back-solve u = L~^{-T} v (NEXT (f1)).  Phase of a task:
    // 0 assembly, 1 Cholesky, 2 root forward solve, 3 root back-solve.
    std::vector<DTask> tasks;
    std::vector<int8_t> phase;
    std::vector<int32_t> succ_off, succ;
    std::vector<int32_t> indeg[HCOV_MODES];       // dependencies inside the mode, per task
    std::vector<int32_t> roots[HCOV_MODES][2];    // initial ready tasks per mode and queue class
    std::vector<int32_t> band_off;                // queue 0: HCOV_BANDS + 1 offsets of the bands' rings
    std::vector<int32_t> q0init[HCOV_MODES];      // queue 0 initial content per mode (-1 = empty slot)
    std::vector<int32_t> q0tail[HCOV_MODES];      // per mode: initial tail of each band
    int32_t n_q[HCOV_MODES][2] = {};              // non-NOP tasks per mode and queue class
    int32_t crit_len = 0;                // longest dependency chain (tasks, NOPs excluded)
    int64_t max_rm = 0;                  // largest low-rank block
    int64_t max_mq = 0;                  // largest rows-per-member of a gang task
    int32_t root_solve = -1;
    std::vector<int32_t> col_off, col_nodes;   // per leaf column segment: strictly-lower T/R leaves over it

    int64_t n_tiles() const { return (int64_t)tile_node.size(); }
    int64_t n_r() const { return (int64_t)rblk.size(); }
    int64_t cluster_size(int level) const { return (int64_t)HCOV_LEAF << (depth - level); }
};

// Cluster tree and block tree built on the device (tree.cu, kernels K1 / K2): the internal order,
// the cluster bounding boxes, and every block-tree node per level with its type (NodeType).
struct PlanGeo {
    int depth = 0;
    std::vector<int64_t> perm_i2e;   // n_pad
    std::vector<double> xs, ys, zs;  // n_pad (zs: dim 3 only)
    std::vector<double> bb;          // 2 dim per cluster heap id
    std::vector<std::vector<std::pair<int32_t, int32_t>>> level_pairs;   // (i, j) per level
    std::vector<std::vector<int8_t>> level_types;                        // NodeType per pair
};

// Build everything from host coordinates s (n x 2 row-major, external order), or, when geo is
// given, from the device-built trees (s_host is then unused and may be null).
// Returns 0 on success, 1 invalid input, 2 empty input, 3 inconsistent geo.
int plan_build(Plan &P, const double *s_host, int64_t n, const PlanOpts &opt, const PlanGeo *geo = nullptr);

#ifdef __CUDACC__
#include <cuda_runtime.h>
// K1 + K2 on the device (tree.cu).  0 ok, 1 invalid input, 2 empty input, -1 CUDA error.
int tree_geo_device(const double *s_dev, int64_t n, const PlanOpts &opt, cudaStream_t st, PlanGeo &g);
#endif
