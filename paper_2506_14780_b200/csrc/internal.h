// internal.h -- declarations shared by the CUDA translation units of libsknr_b200.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "sknr_device.cuh"

namespace sknr {

// MODE_BLOCK_RS: block pass that also emits the transposed weighted sums
// rsum[out_tile][in] = sum_{o in tile} e(o, in) * out_w[o] (points d <= 4 only).
// MODE_SUM_CULL: sum pass over spatially sorted point clouds that skips (output
// group, input group) pairs whose every term is provably below e^-T of the
// output's total (points d <= 4, opt-in; see pts_cull_kernel).
// MODE_SUM_F32: opt-in fp32 sum pass (sknr_problem_set_precision(p, 32); points d <= 4):
// the same partial sums with the cell exponent in fp32 and exp2 on the MUFU unit.
// MODE_SUM_CULL_F32: both (the culled pass with the fp32 arithmetic on its kept groups).
enum { MODE_SUM = 0, MODE_MAX = 1, MODE_BLOCK = 2, MODE_BLOCK_RS = 3, MODE_SUM_CULL = 4, MODE_BLOCK_CULL = 5,
       MODE_SUM_F32 = 6, MODE_SUM_CULL_F32 = 7 };

// Group sizes of the culling bounds (permuted positions): the sum pass tests input
// groups of CULL_GI against output groups of CULL_GO (one warp's 32 x 4 outputs);
// the block pass uses 32 x 32 (CULL_GB in tile_kernels.cu).
constexpr int CULL_GI = 32, CULL_GO = 128;

// Arguments of the persistent tile kernels (tile_kernels.cu).
struct TileArgs {
    int64_t n_out = 0, n_in = 0;
    int64_t in_block = 0, n_out_tiles = 0, n_in_blocks = 0, n_tiles = 0;
    const double* out_pack = nullptr;  // points: [n_out][PK] (B, Y...); dense: B [n_out]
    const double* in_pack = nullptr;   // points: [n_in][PK] (A, X...);  dense: A [n_in]
    const double* C = nullptr;         // dense: element (o, in) at C[o + in*ldc]
    int64_t ldc = 0;
    double kappa = 0.0;                // dense: u = A + B - kappa*C
    const double* W = nullptr;         // block: W[in*KT + c]
    double* partial = nullptr;         // sum/max: [ib][n_out]; block: [ib][KT][n_out]
    const double* out_w = nullptr;     // block_rs: weights of the outputs (n_out)
    double* rsum = nullptr;            // block_rs: [n_out_tiles][n_in]
    const DevState* st = nullptr;
    unsigned guard = 0;
    // MODE_SUM_CULL
    const int* perm_in = nullptr;      // permuted position -> input index
    const int* perm_out = nullptr;     // permuted position -> output index
    const double* box_gi = nullptr;    // [input group][2D] lo..., hi... (centred coordinates)
    const double* box_go = nullptr;    // [output group][2D]
    const double* f_gi = nullptr;      // group max of F_in = A_in + LS kc |x_in|^2
    const double* s_go = nullptr;      // group max of S_out = B_out + LS kc |y_out|^2 (- LS log-total)
    double lskc = 0.0;                 // LS * kappa / eps
    double cull_t = 60.0;              // skip terms below e^-T of the output's total
    double inv_eps = 1.0;
    int dir = 0;
    int retry_phase = 0;
    unsigned* sched = nullptr;         // dynamic tile counter (zeroed by the preceding k_group_max)
    // tensor-core (int8 slice) block pass, i8_kernels.cu
    const uint8_t* vsl = nullptr;      // V digit tiles, 7168 bytes per 32-input chunk
    const unsigned* vexp = nullptr;    // per column: 2048 + largest exponent (0: zero column)
    int kt = 0;                        // columns of W (<= 32)
    // pts_i8w_kernel work units: i8_og output tiles x i8_ig input blocks of the
    // i8_out_tiles x i8_in_blocks tiling (n_out_tiles / n_in_blocks then count unit rows)
    int64_t i8_og = 1, i8_ig = 1, i8_out_tiles = 0, i8_in_blocks = 0;
};

struct TilePlan {
    const void* fn = nullptr;
    bool i8 = false;                   // pts_i8_kernel: needs launch_i8_vprep on W first
    int grid = 0, smem = 0, occ = 0, nt = 128;
    int64_t out_tile = 0, in_block = 0, n_out_tiles = 0, n_in_blocks = 0, n_tiles = 0;
    int64_t i8_og = 1, i8_ig = 1, i8_out_tiles = 0, i8_in_blocks = 0;  // pts_i8w_kernel work units
};

// dim: 0 = stored cost, 1..4 = point-cloud dimension. kt: block width (8..64) for MODE_BLOCK.
TilePlan plan_tiles(int dim, int mode, int kt, int64_t n_out, int64_t n_in, int64_t max_in_blocks,
                    int variant = -1);
void launch_tiles(const TilePlan& p, TileArgs a, cudaStream_t s);
int block_kt_for(int k);
int chunk_inputs(int mode, int kt);

// Newton block pass S = V^T P~ / r = P~ beta on the tensor cores (i8_kernels.cu)
const void* i8_block_kernel(int d);
bool i8_block_enabled();
void set_i8_block_enabled(bool on);
int i8_block_smem();
int i8_block_threads();
int i8_block_out_tile();
int i8_max_in_block();
int64_t i8_vslice_bytes(int64_t n_in);
void launch_i8_vprep(const double* W, int kt, int64_t n_in, uint8_t* vsl, unsigned* vexp, const DevState* st,
                     unsigned guard, cudaStream_t s);

void count_launch();
int64_t launch_count();

// Small-problem batch (sknr_solve_small_batch): a group of CTAs (one CTA when the batch
// fills the GPU) runs a whole SK solve of one point-cloud problem (n, m <=
// small_max_count(d), d <= 4) inside one kernel.
constexpr int kSmallMax = 8192;
// largest n, m for the small-problem kernel at dimension d: every CTA stages one side's
// points (d + 1 doubles each) next to the 32 KiB exp2 table in <= 227 KiB of shared memory
inline int small_max_count(int d) {
    const int words = 232448 / 8 - (256 * 16) - 64;
    const int c = words / (d + 1);
    return c < kSmallMax ? c : kSmallMax;
}
struct SmallProbDev {
    const double *x = nullptr, *y = nullptr, *a = nullptr, *b = nullptr;  // col-major coords, weights
    double *f = nullptr, *g = nullptr, *h = nullptr;                     // potentials (f, g in/out), scratch
    int n = 0, m = 0;
    double eps = 1.0, kappa = 1.0;
    long long iters = 0;
    int conv = 0;
};
// Launches the small-problem kernel for `count` problems whose largest side is max_nm;
// returns the CTAs per problem used (G). gpart: count*G*4 doubles, gbar: 2*count zeroed
// unsigneds (only touched when G > 1); allocate them for G = small_group_size(...).
int small_group_size(int d, int count, int max_nm);
void launch_sk_small(int d, SmallProbDev* probs, int count, int max_nm, double tol, long long max_iter,
                     int warm_g, int G, double* gpart, unsigned* gbar, cudaStream_t s);

}  // namespace sknr
