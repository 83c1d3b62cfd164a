// aux_kernels.cuh -- O(n+m) and O(n*ell^2) helper kernels around the tile passes.
// Every reduction is deterministic: fixed per-block ranges, fixed in-block
// trees, and a "last block" (ticket counter) that merges the block partials
// in block order. No floating-point atomics.
#pragma once
#include "internal.h"

namespace sknr {

constexpr int AUX_NT = 256;

// ------------------------------------------------------------------ packing
// A_i = L64*(lw_i + v_i*inv_eps - kc*sq_i) and scaled coordinates; optional
// statistics of (v - ref) for the bound shift (LSE passes only).
struct PrepInArgs {
    int64_t count = 0;
    int d = 0, pk = 1;
    const double* v = nullptr;    // potential on the input side (nullable)
    const double* lw = nullptr;   // log weight term (nullable)
    const double* sq = nullptr;   // squared norms (points; nullable)
    const double* coords = nullptr;
    double inv_eps = 1, kc = 0, sigma = 0;
    double* pack = nullptr;
    // LSE statistics
    const double* ref = nullptr;  // previous input of this direction (nullable => no stats)
    int dir = 0;
    double* part = nullptr;       // 2*gridDim doubles
    double exact_spread = 600.0;  // (max-min)(v-ref)/eps above which the exact path is forced
    DevState* st = nullptr;
    unsigned guard = 0;
};

__global__ void k_prep_in(PrepInArgs a);

enum { SHIFT_NONE = 0, SHIFT_BOUND = 1 };

struct PrepOutArgs {
    int64_t count = 0;
    int d = 0, pk = 1;
    const double* v = nullptr;
    const double* lw = nullptr;
    const double* sq = nullptr;
    const double* coords = nullptr;
    double inv_eps = 1, kc = 0, sigma = 0;
    int shift_mode = SHIFT_NONE;
    const double* Lref = nullptr;  // bound shift: previous LSE of this direction
    double* shift = nullptr;       // written (natural log units)
    double* pack = nullptr;
    int dir = 0;
    DevState* st = nullptr;
    unsigned guard = 0;
};

__global__ void k_prep_out(PrepOutArgs a);

struct FinalizeArgs {
    const double* partial = nullptr;
    int64_t nb = 0, n_out = 0;
    double* shift = nullptr;
    double* pack = nullptr;   // max-finalize rewrites B in place
    int pk = 1;
    const double* sq = nullptr;
    double kc = 0;
    double eps = 1;
    double* L = nullptr;
    double* pot = nullptr;
    int dir = 0;
    int retry_phase = 0;
    DevState* st = nullptr;
    unsigned guard = 0;
    double lo_ok = 0x1p-900;  // lse: a sum below this means the bound shift was too loose
    double* S = nullptr;      // lse (row-sharded column transform): the local sums S_o
};

// Culling bounds: over permuted positions, the maximum of pack[i*pk] + lskc*sq[i]
// (- LS sub[i] when given), i = perm[p], per group of gs (gs divides AUX_NT).
// Optionally zeroes a work-queue counter for the pass that follows.
__global__ void k_group_max(const double* pack, int pk, const double* sq, double lskc, const int* perm,
                            int64_t count, int gs, double* out, const DevState* st, unsigned guard,
                            unsigned* zero_counter, const double* sub = nullptr);

__global__ void k_max_finalize(FinalizeArgs a);
// Row-sharded column LSE: merge the gathered rank rows X[r] = [shift (m) | S (m)] in rank
// order: L_j = M_j + log(sum_r S_rj exp(shift_rj - M_j)), M_j = max_r shift_rj; pot = -eps L.
__global__ void k_lse_merge(const double* X, int world, int64_t m, double eps, double* L, double* pot,
                            const DevState* st, unsigned guard);
__global__ void k_lse_finalize(FinalizeArgs a);
__global__ void k_rsum_finalize(const double* rsum, int64_t n_tiles, int64_t n, double* out, const DevState* st,
                                unsigned guard);
__global__ void k_sum_finalize(const double* partial, int64_t nb, int64_t n_out, const double* scale,
                               double* out, DevState* st, unsigned guard);
__global__ void k_lse_commit(const double* in_vec, double* ref, int64_t count, int dir, DevState* st,
                             unsigned guard);
__global__ void k_block_finalize(const double* partial, int64_t nb, int kt, int k, int64_t n_out,
                                 const double* scale, double* out, int64_t ld, DevState* st,
                                 unsigned guard, int64_t blk_rows);
// out[q] = scale * sum_b part[b*Q + q] (column fold of split partial rows, deterministic)
__global__ void k_fold_sum(const double* part, int64_t nb, int64_t Q, double scale, double* out,
                           const DevState* st, unsigned guard);
// grid for the column-fold finalize kernels: one block per 32 outputs
inline int fold_grid(int64_t Q) {
    int64_t g = (Q + 31) / 32;
    if (g < 1) g = 1;
    if (g > 148 * 8) g = 148 * 8;
    return static_cast<int>(g);
}
__global__ void k_pack_w(const double* X, int64_t n, int64_t ldx, int k, int kt, const double* rowscale,
                         double* W);

// ------------------------------------------------------------------ Gram
// G[a + b*ka] = sum_t w_t U[t + a*ldu] V[t + b*ldv]  (V==nullptr -> V=U; w nullable)
struct GramArgs {
    int64_t T = 0;
    int ka = 1, kb = 1;
    const double* U = nullptr;
    int64_t ldu = 0;
    const double* V = nullptr;
    int64_t ldv = 0;
    const double* w = nullptr;
    int diag_only = 0;
    double* part = nullptr;     // gridDim * ka*kb
    double* out = nullptr;
    double out_scale = 1.0;
    unsigned* counter = nullptr;
    DevState* st = nullptr;
    unsigned guard = 0;
};
__global__ void k_gram(GramArgs a);
int gram_blocks(int64_t T);

// Fused deterministic scalar reductions over one or two index segments:
// term t reduces over segment seg[t] either sum x*y (y == nullptr: sum x),
// sum x*x, or max |x|. Results land in out[t]; the last block merges block
// partials in block order, then runs an optional epilogue on DevState.
enum { RED_DOT = 0, RED_SQ = 1, RED_MAXABS = 2 };
enum { EPI_NONE = 0, EPI_GAUGE = 1, EPI_CHECK = 2, EPI_ACCEPT = 3, EPI_STEP = 4, EPI_ACCEPT_DQ = 5 };
constexpr int RED_MAX_TERMS = 6;
constexpr int RED_PER_BLOCK = AUX_NT * 2;  // elements per k_reduce block (up to 296 blocks)
struct RedArgs {
    int64_t T[2] = {0, 0};
    int nterms = 0;
    const double* x[RED_MAX_TERMS] = {};
    const double* y[RED_MAX_TERMS] = {};
    int op[RED_MAX_TERMS] = {};
    int seg[RED_MAX_TERMS] = {};
    double* out = nullptr;   // nterms results
    double* part = nullptr;  // gridDim * nterms
    unsigned* counter = nullptr;
    int epilogue = EPI_NONE;
    int newton = 0;
    DevState* st = nullptr;
    unsigned guard = 0;
};
__global__ void k_reduce(RedArgs a);
__global__ void k_epilogue(DevState* st, int epilogue, int newton, const double* r, unsigned guard);
int reduce_blocks(int64_t T);

}  // namespace sknr
