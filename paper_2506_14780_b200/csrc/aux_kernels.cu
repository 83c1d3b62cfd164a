// aux_kernels.cu -- packing, finalize and Gram kernels (see aux_kernels.cuh).
#include "aux_kernels.cuh"

namespace sknr {

namespace {

constexpr double kInf = __builtin_huge_val();

template <typename T, typename Op>
__device__ __forceinline__ T block_reduce(T v, T* sh, Op op) {
    // fixed tree over AUX_NT threads: deterministic
    const int tid = threadIdx.x;
    sh[tid] = v;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (tid < s) sh[tid] = op(sh[tid], sh[tid + s]);
        __syncthreads();
    }
    const T r = sh[0];
    __syncthreads();
    return r;
}

struct MaxOp {
    __device__ double operator()(double a, double b) const { return fmax(a, b); }
};
struct MinOp {
    __device__ double operator()(double a, double b) const { return fmin(a, b); }
};

// Returns true in exactly one block: the last one to finish (all partials visible).
__device__ __forceinline__ bool last_block(unsigned* counter) {
    __shared__ bool is_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned ticket = atomicAdd(counter, 1u);
        is_last = (ticket == gridDim.x - 1);
    }
    __syncthreads();
    if (is_last) __threadfence();
    return is_last;
}

}  // namespace

// ------------------------------------------------------------------ prep
__global__ void __launch_bounds__(AUX_NT) k_prep_in(PrepInArgs a) {
    SKNR_PDL_ENTRY();
    if (guard_skip(a.st, a.guard)) return;
    __shared__ double sh[AUX_NT];
    double lmax = -kInf, lmin = kInf;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < a.count;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        double e = 0.0;
        if (a.lw) e = a.lw[i];
        if (a.v) e += a.v[i] * a.inv_eps;
        if (a.sq) e -= a.kc * a.sq[i];
        a.pack[i * a.pk] = kLS * e;
        for (int c = 0; c < a.d; ++c) a.pack[i * a.pk + 1 + c] = a.sigma * a.coords[i + c * a.count];
        for (int c = a.d + 1; c < a.pk; ++c) a.pack[i * a.pk + c] = 0.0;
        if (a.ref) {
            const double dv = a.v[i] - a.ref[i];
            lmax = fmax(lmax, dv);
            lmin = fmin(lmin, dv);
        }
    }
    if (!a.ref) return;
    const double bmax = block_reduce(lmax, sh, MaxOp());
    const double bmin = block_reduce(lmin, sh, MinOp());
    if (threadIdx.x == 0) {
        a.part[2 * blockIdx.x] = bmax;
        a.part[2 * blockIdx.x + 1] = bmin;
    }
    if (!last_block(&a.st->counters[a.dir])) return;
    double mx = -kInf, mn = kInf;
    for (unsigned b = threadIdx.x; b < gridDim.x; b += blockDim.x) {
        mx = fmax(mx, a.part[2 * b]);
        mn = fmin(mn, a.part[2 * b + 1]);
    }
    mx = block_reduce(mx, sh, MaxOp());
    mn = block_reduce(mn, sh, MinOp());
    if (threadIdx.x == 0) {
        a.st->dmax[a.dir] = mx;
        a.st->dmin[a.dir] = mn;
        const bool ok = a.st->ref_valid[a.dir] && (mx - mn) * a.inv_eps <= a.exact_spread &&
                        isfinite(mx) && isfinite(mn);
        a.st->need_exact[a.dir] = ok ? 0 : 1;
        a.st->retry[a.dir] = 0;
        if (!ok) a.st->n_exact[a.dir] += 1;
        a.st->counters[a.dir] = 0u;
    }
}

__global__ void __launch_bounds__(AUX_NT) k_prep_out(PrepOutArgs a) {
    SKNR_PDL_ENTRY();
    if (guard_skip(a.st, a.guard)) return;
    const bool bound = a.shift_mode == SHIFT_BOUND && !a.st->need_exact[a.dir];
    const double dshift = bound ? a.st->dmax[a.dir] * a.inv_eps : 0.0;
    for (int64_t o = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; o < a.count;
         o += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        double e = 0.0;
        if (a.lw) e = a.lw[o];
        if (a.v) e += a.v[o] * a.inv_eps;
        if (a.sq) e -= a.kc * a.sq[o];
        double s = 0.0;
        if (a.shift_mode == SHIFT_BOUND) {
            s = bound ? a.Lref[o] + dshift : 0.0;
            a.shift[o] = s;
        }
        a.pack[o * a.pk] = kLS * (e - s);
        for (int c = 0; c < a.d; ++c) a.pack[o * a.pk + 1 + c] = a.sigma * a.coords[o + c * a.count];
        for (int c = a.d + 1; c < a.pk; ++c) a.pack[o * a.pk + c] = 0.0;
    }
}

// ------------------------------------------------------------------ culling bounds
__global__ void __launch_bounds__(AUX_NT) k_group_max(const double* pack, int pk, const double* sq, double lskc,
                                                      const int* perm, int64_t count, int gs, double* out,
                                                      const DevState* st, unsigned guard, unsigned* zero_counter,
                                                      const double* sub) {
    SKNR_PDL_ENTRY();
    if (guard_skip(st, guard)) return;
    if (zero_counter && blockIdx.x == 0 && threadIdx.x == 0) *zero_counter = 0u;
    __shared__ double vals[AUX_NT];
    const int64_t p = static_cast<int64_t>(blockIdx.x) * AUX_NT + threadIdx.x;
    double v = -kInf;
    if (p < count) {
        const int64_t i = perm[p];
        v = pack[i * pk] + lskc * sq[i];
        if (sub) v -= kLS * sub[i];
    }
    vals[threadIdx.x] = v;
    __syncthreads();
    // tree max within each group of gs consecutive positions (gs a power of two <= AUX_NT)
    for (int s = gs / 2; s > 0; s >>= 1) {
        if ((threadIdx.x % gs) < s) vals[threadIdx.x] = fmax(vals[threadIdx.x], vals[threadIdx.x + s]);
        __syncthreads();
    }
    if (threadIdx.x % gs == 0 && p < count) out[p / gs] = vals[threadIdx.x];
}

// ------------------------------------------------------------------ finalize
// Split-K partials are folded column-wise: a block owns 32 consecutive output
// entries q (one per lane) and its 8 warps take the partial rows b = w, w+8, ...
// in increasing order; warp 0 then adds the 8 warp sums in warp order. Every
// load of a warp is one 256-byte row segment, each thread issues nb/8 independent
// loads, and the summation order is fixed by (nb, layout) alone: deterministic.
constexpr int FOLD_W = AUX_NT / 32;

template <bool MAX>
__device__ __forceinline__ double fold_rows(const double* __restrict__ p, int64_t nb, int64_t stride,
                                            int64_t q, bool valid, double (*sh)[32]) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double s = MAX ? -kInf : 0.0;
    if (valid) {
        const double* col = p + q;
#pragma unroll 4
        for (int64_t b = w; b < nb; b += FOLD_W) {
            const double v = col[b * stride];
            s = MAX ? fmax(s, v) : s + v;
        }
    }
    sh[w][lane] = s;
    __syncthreads();
    if (w == 0) {
        s = sh[0][lane];
#pragma unroll
        for (int k = 1; k < FOLD_W; ++k) s = MAX ? fmax(s, sh[k][lane]) : s + sh[k][lane];
    }
    __syncthreads();
    return s;  // valid in warp 0
}

#define FOLD_LOOP(Q)                                                                      \
    for (int64_t q0 = static_cast<int64_t>(blockIdx.x) * 32; q0 < (Q);                  \
         q0 += static_cast<int64_t>(gridDim.x) * 32)

// Exact shift: shift_o += max_u / L64, B_o recomputed from it.
__global__ void __launch_bounds__(AUX_NT) k_max_finalize(FinalizeArgs a) {
    SKNR_PDL_ENTRY();
    if (guard_skip(a.st, a.guard)) return;
    __shared__ double sh[FOLD_W][32];
    FOLD_LOOP(a.n_out) {
        const int64_t o = q0 + (threadIdx.x & 31);
        const double M = fold_rows<true>(a.partial, a.nb, a.n_out, o, o < a.n_out, sh);
        if (threadIdx.x < 32 && o < a.n_out) {
            const double s = a.shift[o] + M * kInvLS;
            a.shift[o] = s;
            double e = 0.0;
            if (a.sq) e -= a.kc * a.sq[o];
            a.pack[o * a.pk] = kLS * (e - s);
        }
    }
}

// L_o = shift_o + log(sum_b partial[b][o]); pot_o = -eps L_o. A sum outside
// [2^-900, 2^900] means the bound shift was too loose: request the exact path
// (n_retry counts the 32-output chunks that saw such a sum).
__global__ void __launch_bounds__(AUX_NT) k_lse_finalize(FinalizeArgs a) {
    SKNR_PDL_ENTRY();
    if (guard_skip(a.st, a.guard)) return;
    __shared__ double sh[FOLD_W][32];
    FOLD_LOOP(a.n_out) {
        const int64_t o = q0 + (threadIdx.x & 31);
        const bool valid = o < a.n_out;
        const double S = fold_rows<false>(a.partial, a.nb, a.n_out, o, valid, sh);
        if (threadIdx.x < 32) {
            bool bad = false;
            if (valid) {
                bad = !(S >= a.lo_ok && S <= 0x1p900);
                const double L = a.shift[o] + log(S);
                if (a.L) a.L[o] = L;
                if (a.S) a.S[o] = S;
                if (a.pot) a.pot[o] = -a.eps * L;
            }
            if (__any_sync(0xffffffffu, bad) && threadIdx.x == 0 && !a.retry_phase &&
                !a.st->need_exact[a.dir]) {
                a.st->retry[a.dir] = 1;
                atomicAdd(&a.st->n_retry[a.dir], 1ull);
            }
        }
    }
}

__global__ void __launch_bounds__(AUX_NT) k_lse_merge(const double* X, int world, int64_t m, double eps,
                                                      double* L, double* pot, const DevState* st, unsigned guard) {
    SKNR_PDL_ENTRY();
    if (guard_skip(st, guard)) return;
    for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < m;
         j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        double M = X[j];
        for (int r = 1; r < world; ++r) M = fmax(M, X[r * 2 * m + j]);
        double T = 0.0;
        for (int r = 0; r < world; ++r) T += X[r * 2 * m + m + j] * exp(X[r * 2 * m + j] - M);
        const double v = M + log(T);
        L[j] = v;
        if (pot) pot[j] = -eps * v;
    }
}

// out[i] = sum over output tiles t (in order) of rsum[t][i]: the fused block pass's
// transposed sums (r = P~ beta), deterministic.
__global__ void __launch_bounds__(AUX_NT) k_rsum_finalize(const double* rsum, int64_t n_tiles, int64_t n,
                                                          double* out, const DevState* st, unsigned guard) {
    SKNR_PDL_ENTRY();
    if (guard_skip(st, guard)) return;
    __shared__ double sh[FOLD_W][32];
    FOLD_LOOP(n) {
        const int64_t i = q0 + (threadIdx.x & 31);
        const double s = fold_rows<false>(rsum, n_tiles, n, i, i < n, sh);
        if (threadIdx.x < 32 && i < n) out[i] = s;
    }
}

__global__ void __launch_bounds__(AUX_NT) k_sum_finalize(const double* partial, int64_t nb,
                                                         int64_t n_out, const double* scale,
                                                         double* out, DevState* st, unsigned guard) {
    SKNR_PDL_ENTRY();
    if (guard_skip(st, guard)) return;
    __shared__ double sh[FOLD_W][32];
    FOLD_LOOP(n_out) {
        const int64_t o = q0 + (threadIdx.x & 31);
        const double S = fold_rows<false>(partial, nb, n_out, o, o < n_out, sh);
        if (threadIdx.x < 32 && o < n_out) out[o] = scale ? scale[o] * S : S;
    }
}

__global__ void __launch_bounds__(AUX_NT) k_lse_commit(const double* in_vec, double* ref, int64_t count,
                                                       int dir, DevState* st, unsigned guard) {
    SKNR_PDL_ENTRY();
    if (guard_skip(st, guard)) return;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        ref[i] = in_vec[i];
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        st->ref_valid[dir] = 1;
        st->need_exact[dir] = 0;
        st->retry[dir] = 0;
    }
}

// partial layout [b][c][o] (c < kt): entry q = c*n_out + o of the first k columns
// is the contiguous range q < k*n_out of each row b (row stride kt*n_out).
__global__ void __launch_bounds__(AUX_NT) k_block_finalize(const double* partial, int64_t nb, int kt,
                                                           int k, int64_t n_out, const double* scale,
                                                           double* out, int64_t ld, DevState* st,
                                                           unsigned guard, int64_t blk_rows) {
    SKNR_PDL_ENTRY();
    if (guard_skip(st, guard)) return;
    __shared__ double sh[FOLD_W][32];
    const int64_t total = n_out * k;
    FOLD_LOOP(total) {
        const int64_t e = q0 + (threadIdx.x & 31);
        const double S = fold_rows<false>(partial, nb, kt * n_out, e, e < total, sh);
        if (threadIdx.x < 32 && e < total) {
            const int64_t o = e % n_out;
            const int64_t c = e / n_out;
            // blk_rows > 0: rank-blocked layout for a reduce-scatter -- block q = rows
            // [q * blk_rows, (q + 1) * blk_rows), its k columns contiguous (ld = blk_rows)
            const int64_t at = blk_rows > 0 ? (o / blk_rows) * (k * blk_rows) + c * blk_rows + o % blk_rows
                                            : o + c * ld;
            out[at] = scale ? scale[o] * S : S;
        }
    }
}

// Column fold of gram partials: out[q] = scale * sum_b part[b*Q + q].
__global__ void __launch_bounds__(AUX_NT) k_fold_sum(const double* part, int64_t nb, int64_t Q, double scale,
                                                     double* out, const DevState* st, unsigned guard) {
    SKNR_PDL_ENTRY();
    if (guard_skip(st, guard)) return;
    __shared__ double sh[FOLD_W][32];
    FOLD_LOOP(Q) {
        const int64_t q = q0 + (threadIdx.x & 31);
        const double S = fold_rows<false>(part, nb, Q, q, q < Q, sh);
        if (threadIdx.x < 32 && q < Q) out[q] = scale * S;
    }
}

// W[i*kt + c] = rowscale_i * X[i + c*ldx] for c < k, 0 for k <= c < kt.
__global__ void __launch_bounds__(AUX_NT) k_pack_w(const double* X, int64_t n, int64_t ldx, int k,
                                                   int kt, const double* rowscale, double* W) {
    SKNR_PDL_ENTRY();
    const int64_t total = n * kt;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = e / kt;
        const int c = static_cast<int>(e % kt);
        double v = 0.0;
        if (c < k) v = X[i + c * ldx] * (rowscale ? rowscale[i] : 1.0);
        W[e] = v;
    }
}

// ------------------------------------------------------------------ Gram
int gram_blocks(int64_t T) {  // >= 64 rows per block, up to two CTAs per SM
    int64_t b = (T + 63) / 64;
    if (b < 1) b = 1;
    if (b > 296) b = 296;
    return static_cast<int>(b);
}

// Each block owns a contiguous t-range; rows are staged 32 at a time in shared
// memory (w folded into U); thread owns pairs p = tid + q*AUX_NT.
__global__ void __launch_bounds__(AUX_NT) k_gram(GramArgs a) {
    SKNR_PDL_ENTRY();
    if (guard_skip(a.st, a.guard)) return;
    constexpr int RB = 32;
    constexpr int KMAXP = 64;
    __shared__ double su[RB * KMAXP];
    __shared__ double sv[RB * KMAXP];
    const int ka = a.ka, kb = a.kb;
    const int npairs = a.diag_only ? ka : ka * kb;
    constexpr int QMAX = (KMAXP * KMAXP + AUX_NT - 1) / AUX_NT;
    double acc[QMAX];
#pragma unroll
    for (int q = 0; q < QMAX; ++q) acc[q] = 0.0;
    const int64_t per = (a.T + gridDim.x - 1) / gridDim.x;
    const int64_t t0 = blockIdx.x * per;
    const int64_t t1 = (t0 + per < a.T) ? t0 + per : a.T;
    const double* V = a.V ? a.V : a.U;
    const int64_t ldv = a.V ? a.ldv : a.ldu;
    for (int64_t tb = t0; tb < t1; tb += RB) {
        const int cnt = static_cast<int>((t1 - tb) < RB ? (t1 - tb) : RB);
        __syncthreads();
        for (int e = threadIdx.x; e < cnt * ka; e += blockDim.x) {
            const int r = e % cnt, c = e / cnt;
            const double w = a.w ? a.w[tb + r] : 1.0;
            su[r * KMAXP + c] = w * a.U[tb + r + c * a.ldu];
        }
        for (int e = threadIdx.x; e < cnt * kb; e += blockDim.x) {
            const int r = e % cnt, c = e / cnt;
            sv[r * KMAXP + c] = V[tb + r + c * ldv];
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < QMAX; ++q) {
            const int p = threadIdx.x + q * AUX_NT;
            if (p >= npairs) break;
            const int ia = a.diag_only ? p : p % ka;
            const int ib = a.diag_only ? p : p / ka;
            double s = acc[q];
            for (int r = 0; r < cnt; ++r) s = fma(su[r * KMAXP + ia], sv[r * KMAXP + ib], s);
            acc[q] = s;
        }
    }
    // one block: the result directly; several: rows of partials for k_fold_sum
    double* dst = gridDim.x == 1 ? a.out : a.part + static_cast<int64_t>(blockIdx.x) * npairs;
    const double sc = gridDim.x == 1 ? a.out_scale : 1.0;
#pragma unroll
    for (int q = 0; q < QMAX; ++q) {
        const int p = threadIdx.x + q * AUX_NT;
        if (p < npairs) dst[p] = sc * acc[q];
    }
    // several blocks: the host folds the partial rows with k_fold_sum
}

int reduce_blocks(int64_t T) {
    int64_t b = (T + RED_PER_BLOCK - 1) / RED_PER_BLOCK;
    if (b < 1) b = 1;
    if (b > 296) b = 296;
    return static_cast<int>(b);
}

// r layout (EPI_CHECK): |row-a|^2, a.f, max|row-a|, |col-b|^2, max|col-b|, b.h
__device__ void run_epilogue(DevState* st, int epilogue, int newton, const double* r) {
    if (epilogue == EPI_GAUGE) {
        st->c_gauge = r[0];
    } else if (epilogue == EPI_CHECK) {
        // marginal_gap (core.cpp:145-150) and Q0 = a.f + b.h; stopping test (solver.cpp:123)
        if (st->done) return;
        st->gap_l2 = sqrt(r[0]) + sqrt(r[3]);
        st->gap_inf = r[2] + r[4];
        st->q0 = r[1] + r[5];
        if (st->gap_l2 < st->tol) {
            st->conv = 1;
            st->done = 1;
        } else if (newton) {
            st->newton_ok = 1;
            st->attempted = 1;
        }
    } else if (epilogue == EPI_ACCEPT) {
        // Q1 = a.f' + b.h'; accept iff Q1 > Q0 (solver.cpp:46-47)
        if (st->done || !st->newton_ok) return;
        st->q1 = r[0] + r[1];
        st->accept = st->q1 > st->q0 ? 1 : 0;
    } else if (epilogue == EPI_STEP) {
        // stable accept test, first half: r = (a.d, max|d|), d = f' - f
        if (st->done || !st->newton_ok) return;
        st->adq = r[0];
        st->lit = r[1] <= st->lit_dmax ? 0 : 1;
    } else if (epilogue == EPI_ACCEPT_DQ) {
        // dQ = a.d + b.(h' - h) > 0: the predicate Q1 > Q0 of solver.cpp:46-47 evaluated
        // as a difference whose rounding scales with the step, not with |Q|
        if (st->done || !st->newton_ok || st->lit) return;
        const double dq = st->adq + r[0];
        st->q1 = st->q0 + dq;
        st->accept = dq > 0.0 ? 1 : 0;
    }
}

__global__ void __launch_bounds__(AUX_NT) k_reduce(RedArgs a) {
    SKNR_PDL_ENTRY();
    if (guard_skip(a.st, a.guard)) return;
    __shared__ double sh[RED_MAX_TERMS][AUX_NT / 32];
    double acc[RED_MAX_TERMS];
#pragma unroll
    for (int t = 0; t < RED_MAX_TERMS; ++t) acc[t] = 0.0;
    // Each segment has its own element-to-thread layout: segment 1 (the m-long, replicated
    // side when rows are sharded) is reduced by its own fixed number of blocks, so its sums
    // round identically on every rank whatever the length of the rank's segment 0.
    for (int seg = 0; seg < 2; ++seg) {
        const int64_t T = a.T[seg];
        int64_t g = gridDim.x;
        if (seg == 1) {
            g = (T + RED_PER_BLOCK - 1) / RED_PER_BLOCK;  // reduce_blocks(T[1])
            g = g < 1 ? 1 : (g > 296 ? 296 : g);
            g = g < gridDim.x ? g : gridDim.x;
            if (blockIdx.x >= g) continue;
        }
        for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < T;
             i += g * blockDim.x) {
#pragma unroll
            for (int t = 0; t < RED_MAX_TERMS; ++t) {
                if (t >= a.nterms || a.seg[t] != seg) continue;
                const double x = a.x[t][i];
                if (a.op[t] == RED_DOT)
                    acc[t] = a.y[t] ? fma(x, a.y[t][i], acc[t]) : acc[t] + x;
                else if (a.op[t] == RED_SQ)
                    acc[t] = fma(x, x, acc[t]);
                else
                    acc[t] = fmax(acc[t], fabs(x));
            }
        }
    }
    // warp tree then fixed cross-warp order
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int t = 0; t < RED_MAX_TERMS; ++t) {
        double v = acc[t];
        for (int o = 16; o > 0; o >>= 1) {
            const double w = __shfl_down_sync(0xffffffffu, v, o);
            v = a.op[t] == RED_MAXABS ? fmax(v, w) : v + w;
        }
        if (lane == 0) sh[t][warp] = v;
    }
    __syncthreads();
    __shared__ bool is_last;
    if (threadIdx.x == 0) {
        for (int t = 0; t < a.nterms; ++t) {
            double v = sh[t][0];
            for (int w = 1; w < AUX_NT / 32; ++w) v = a.op[t] == RED_MAXABS ? fmax(v, sh[t][w]) : v + sh[t][w];
            a.part[static_cast<int64_t>(blockIdx.x) * a.nterms + t] = v;
        }
        __threadfence();
        is_last = atomicAdd(a.counter, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    // last block: warp t folds term t's block partials, lane l taking blocks l, l+32, ...
    // in order, then a fixed shuffle tree (the same order whatever the timing)
    __shared__ double rs[RED_MAX_TERMS];
    if (warp < a.nterms) {
        const int t = warp;
        const bool mx = a.op[t] == RED_MAXABS;
        double v = 0.0;
        for (unsigned b = lane; b < gridDim.x; b += 32) {
            const double w = a.part[static_cast<int64_t>(b) * a.nterms + t];
            v = mx ? fmax(v, w) : v + w;
        }
        for (int o = 16; o > 0; o >>= 1) {
            const double w = __shfl_down_sync(0xffffffffu, v, o);
            v = mx ? fmax(v, w) : v + w;
        }
        if (lane == 0) rs[t] = v;
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    double r[RED_MAX_TERMS] = {};
    for (int t = 0; t < a.nterms; ++t) {
        r[t] = rs[t];
        a.out[t] = rs[t];
    }
    *a.counter = 0u;
    run_epilogue(a.st, a.epilogue, a.newton, r);
}

__global__ void k_epilogue(DevState* st, int epilogue, int newton, const double* r, unsigned guard) {
    SKNR_PDL_ENTRY();
    if (guard_skip(st, guard)) return;
    if (threadIdx.x == 0 && blockIdx.x == 0) run_epilogue(st, epilogue, newton, r);
}

}  // namespace sknr
