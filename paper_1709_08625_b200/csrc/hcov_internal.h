// Internal data structures shared by the host planner (plan.cpp) and the device engine
// (engine.cuh, hcov.cu).  POD only; the device arrays are copies of the host vectors.
#pragma once
#include <stdint.h>

#define HCOV_LEAF 32
#define HCOV_TILE (HCOV_LEAF * HCOV_LEAF)
#define HCOV_GANG 8           // largest gang (CTAs cooperating on one task); HCOV_BANDS * (HCOV_GANG - 1)
                              // must stay below the number of engine CTAs (at most one partially
                              // formed gang per band can hold CTAs, so every gang eventually forms)
#define HCOV_DENSE_MAX 512    // largest low-rank block the dense-mode RAPP supports (PlanOpts.big_m picks the split)
#define HCOV_SMEM_DBL 28160 // dynamic shared memory of the engine CTA (220 KB + static <= 227 KB; one 512-thread CTA per SM)
#define HCOV_BIG_MQ 8192      // gang members with more rows use a big-member scratch slot (hcov.cu)
#define HCOV_BIG_GROUPS 4     // big-member groups (HCOV_GANG slots each)
#define HCOV_MAX_BATCH 8      // H-matrices (theta candidates) per engine launch in hcov_mle_batch
#define HCOV_GANG_MIN 512     // low-rank blocks from this size on are processed by gangs of min(8, m/256) CTAs

// Block-tree node types (lower triangle incl. diagonal).
enum NodeType : int32_t { ND_H = 0, ND_R = 1, ND_T = 2 };

struct DNode {
    int32_t level, i, j;   // row / column cluster index at `level` (cluster size 32 << (depth-level))
    int32_t type;          // NodeType
    int32_t parent;        // node id of the parent, -1 for the root
    int32_t idx;           // tile id (ND_T) or low-rank block id (ND_R); -1 for ND_H
};

// A pending Schur-complement term (lazy left-looking H-Cholesky):
//   TT: tile_a * tile_b^T (32 x 32 dense product);
//   LR: A * K * B^T with A, B factors (fac ids) and K a core (or I if core < 0).
// Rows of A / B are global internal indices starting at fac_row0.
enum TermKind : int32_t { TM_TT = 0, TM_LR = 1 };
struct DTerm {
    int32_t kind;
    int32_t a, b;
    int32_t core;
};

// Tasks of the DAG executed by the persistent engine (one CTA per task).
enum TaskType : int32_t {
    TK_FILL = 0,   // a = first tile, b = count: dense tiles of C~ (A4)
    TK_ACA = 1,    // a = R id: ACA + truncation of an admissible block of C~ (A5, A6)
    TK_TAPP = 2,   // a = tile, [b, c) = range of xterm[]: apply pending terms to the tile
    TK_POTRF = 3,  // a = diag tile, [b, c) terms: apply, then Cholesky + L^{-1} + log det partial (A7, A8)
    TK_TRSM = 4,   // a = tile, [b, c) terms, d = diag tile of its column: apply, then X <- X L^{-T}
    TK_RAPP = 5,   // a = R id, [b, c) terms, d = 1 on the last chunk: append the terms' factors, recompress
    TK_SEG = 6,    // a = solve id, b = leaf row segment, [c, d) = ctr[] contributions: forward solve rows
    TK_PROJ = 7,   // a = solve id, b = R id, c = proj slot: P = V_b^T Y[cols of b]
    TK_PRR = 8,    // a, b = R ids, c = core id: K = V_a^T V_b
    TK_PHWP = 9,   // a = phw id, b = R id (leaf of the H block), c = q slot: Q = V_x^T V_partners[cols of x]
    TK_PHWR = 10,  // a = phw id, b = leaf row segment, [c, d) = ctr[]: W rows = H(rows, :) V_partners
    TK_NOP = 11,   // join (completed inline by the engine, never occupies a CTA)
    TK_BSEG = 12,  // b = leaf segment, [c, d) = ctr[]: back-solve rows u_i = L_ii^{-T} (v_i - sum L_ri^T u_r)
    TK_BPROJ = 13, // b = R id: t_b = U_b^T u[rows of b] (back-solve projection into tbuf)
    TK_NTYPES = 14
};
#define HCOV_MODES 5   // engine modes (plan.h)
struct DTask {
    int32_t type;
    int32_t a, b, c, d;
    int32_t qcls;      // 0 = one CTA; G > 1 = gang task of G CTAs (G consecutive queue entries)
    int32_t band;      // queue 0 priority band (HCOV_BANDS - 1 = most urgent), by the task's bottom level
    int32_t pad;       // RAPP gang: 1 = side-split (members 0..G/2-1 hold X rows, G/2..G-1 Y rows)
};
#define HCOV_BANDS 16

// Contribution of one block-tree leaf to a row segment in a SEG / PHWR task.
//   kind 0: dense tile `id` (column segment aux);  kind 1: low-rank block `id`, product slot aux.
struct DCtr {
    int32_t kind, id, aux, pad;
};

// A forward-solve problem  Y <- L_ss^{-1} Y  on the diagonal block of cluster s.  The right-hand
// sides are the V factors of the low-rank entries of column s (rhs_cnt R ids in solve_rhs[]),
// or the permuted data vector z for the root solve (rhs_cnt = 0).
struct DSolve {
    int32_t level, c;        // cluster
    int32_t rhs_off, rhs_cnt;
    int64_t row0, m;
};

// Product slots (PROJ / PHWP results): doubles at  offa * kcap * kcap + offb * kcap.
struct DSlot {
    int64_t offa, offb;
};

// Low-rank block static description.
struct DRBlk {
    int32_t node;      // node id
    int32_t level;
    int32_t m;         // block size (rows = cols)
    int32_t solve;     // solve id of its column (the solve that finalises V)
    int64_t row0, col0;
    int64_t uv_off;    // offset (elements per unit kcap) of U and V in the pools; m x kcap (m x 2 kcap if
                       // m > HCOV_DENSE_MAX) col-major
};

// W = H * [V_partners] bookkeeping for an H entry of a column with low-rank entries.
struct DPhw {
    int32_t hnode;               // H node id (rows rho, cols sigma)
    int32_t part_off, part_cnt;  // partner R ids in col_r[]
    int32_t fac_base;            // factor ids fac_base .. fac_base+part_cnt-1 are its W slices
    int64_t w_off;               // offset (elements per unit kcap) of W: m x (kcap * part_cnt)
    int32_t m;
    int32_t pad;
};
