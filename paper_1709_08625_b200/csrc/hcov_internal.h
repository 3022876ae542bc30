// Internal data structures shared by the host planner (plan.cpp) and the device kernels.
// POD only; device arrays are copies of the host vectors built in plan.cpp.
#pragma once
#include <stdint.h>

#define HCOV_LEAF 32
#define HCOV_TILE (HCOV_LEAF * HCOV_LEAF)

// Block-tree node types (lower triangle incl. diagonal).
enum NodeType : int32_t { ND_H = 0, ND_R = 1, ND_T = 2 };

struct DNode {
    int32_t level, i, j;   // row / column cluster index at `level` (cluster size 32 << (depth-level))
    int32_t type;          // NodeType
    int32_t parent;        // node id of the parent, -1 for the root
    int32_t idx;           // tile id (ND_T) or low-rank block id (ND_R); -1 for ND_H
    int32_t term_off, term_cnt;  // pending-update terms attached to this node (lazy Schur updates)
    int32_t leaf_off, leaf_cnt;  // ND_H only: flattened list of leaf nodes (T/R) inside, for H x X
};

// A pending Schur-complement term  A * K * B^T  (K = I if core < 0) or a dense tile product
// A * B^T (kind TT).  Rows of A / B are global internal indices starting at fac_row0.
enum TermKind : int32_t { TM_TT = 0, TM_LR = 1 };
struct DTerm {
    int32_t kind;
    int32_t a, b;   // TT: tile ids.  LR: factor ids.
    int32_t core;   // LR: core id or -1
};

enum TaskType : int32_t {
    TK_POTRF = 0,  // a = diag T node: finalise (apply terms) + dense Cholesky + log det partial
    TK_TRSM = 1,   // a = off-diag T node, b = diag tile id of its column: finalise + X <- S L^-T
    TK_RFIN = 2,   // a = R node: finalise S = U V^T - terms, recompress to (eps, kmax)
    TK_SOLVE = 3,  // a = cluster heap id s: V <- L_ss^-1 V for all R entries of column s
    TK_PRR = 4,    // a, b = R nodes (same column), c = core id:  K = V_a^T V_b
    TK_PHW = 5,    // a = H node, b = phw id: W = H * [V of partners]
    TK_NOP = 6
};
struct DTask {
    int32_t type;
    int32_t a, b, c;
};

// Forward-solve program op (post-order over the cluster tree).
enum OpKind : int32_t { OP_TRSM = 0, OP_UPD_T = 1, OP_UPD_R = 2 };
struct DOp {
    int32_t kind;
    int32_t id;        // tile id (TRSM, UPD_T) or R id (UPD_R)
    int32_t m;         // rows / cols of the block (32 for tiles)
    int32_t pad;
    int64_t row0;      // first internal row of the block
    int64_t col0;      // first internal column of the block
};

// Low-rank block static description.
struct DRBlk {
    int32_t node;      // node id
    int32_t level;
    int32_t m;         // block size (rows = cols)
    int32_t pad;
    int64_t row0, col0;
    int64_t uv_off;    // offset (elements) of U and V in the U / V pools; each m x kcap col-major
};

// Product H x [V_partners] bookkeeping.
struct DPhw {
    int32_t hnode;     // H node id (rows rho, cols sigma)
    int32_t part_off, part_cnt;  // partner R ids in phw_part[]
    int32_t fac_base;  // factor ids fac_base .. fac_base+part_cnt-1 are its W slices
    int64_t w_off;     // offset (elements) of W in the W pool, m x (kcap * part_cnt)
    int32_t m;
    int32_t pad;
};
