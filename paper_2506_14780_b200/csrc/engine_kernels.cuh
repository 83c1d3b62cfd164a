// engine_kernels.cuh -- O(n+m) and O(k^2) helper kernels of the solver, spectral and coupling code
// Part of the libsknr_b200 translation unit: included once, in order, by engine.cu
// (shares its types, static helpers and kernels; not a standalone header).
#pragma once

// ============================================================ small kernels
__global__ void k_fill(double* x, int64_t n, double v) {
    SKNR_PDL_ENTRY();
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        x[i] = v;
}

__global__ void k_copy(double* dst, const double* src, int64_t n, DevState* st, unsigned guard) {
    SKNR_PDL_ENTRY();
    if (guard_skip(st, guard)) return;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        dst[i] = src[i];
}

__global__ void k_state_init(DevState* st, long long max_iter, double tol, double lit_dmax = 0.0) {
    SKNR_PDL_ENTRY();
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    st->lit = 0;
    st->lit_dmax = lit_dmax;
    st->trace_base = 0;
    st->done = 0;
    st->iter_active = 0;
    st->conv = 0;
    st->newton_ok = 0;
    st->accept = 0;
    st->attempted = 0;
    st->iter = 0;
    st->max_iter = max_iter;
    st->tol = tol;
    for (int d = 0; d < 2; ++d) {
        st->need_exact[d] = 1;
        st->retry[d] = 0;
        st->ref_valid[d] = 0;
    }
    for (int c = 0; c < 32; ++c) st->counters[c] = 0u;
}

__global__ void k_invalidate_refs(DevState* st) {
    SKNR_PDL_ENTRY();
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        st->ref_valid[0] = st->ref_valid[1] = 0;
        st->done = 0;
        st->newton_ok = 0;
    }
}

__global__ void k_iter_begin(DevState* st) {
    SKNR_PDL_ENTRY();
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    if (st->done) {
        st->iter_active = 0;
        return;
    }
    st->iter += 1;
    st->iter_active = 1;
    st->newton_ok = 0;
    st->accept = 0;
    st->attempted = 0;
    st->t_iter0 = globaltimer_ns();
}

// f = f_pre - c ; rowres_i = a_i expm1(f_pre_i/eps + L_i) ; g += c
__global__ void k_gauge_apply(double* f, const double* L, const double* a, int64_t n, double* g,
                              int64_t m, double inv_eps, double* rowres, DevState* st) {
    SKNR_PDL_ENTRY();
    if (st->done) return;
    const double c = st->c_gauge;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n + m;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        if (i < n) {
            const double fp = f[i];
            rowres[i] = a[i] * expm1(fp * inv_eps + L[i]);
            f[i] = fp - c;
        } else {
            g[i - n] += c;
        }
    }
}

// colres_j = b_j expm1((g_j - h_j)/eps)
__global__ void k_colres(const double* g, const double* h, const double* b, int64_t m, double inv_eps,
                         double* colres, DevState* st, unsigned guard) {
    SKNR_PDL_ENTRY();
    if (guard_skip(st, guard)) return;
    for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < m;
         j += static_cast<int64_t>(gridDim.x) * blockDim.x)
        colres[j] = b[j] * expm1((g[j] - h[j]) * inv_eps);
}

// alpha - r = -a_i expm1(f_i/eps + L_i(h)) ; r = a - (alpha - r)
__global__ void k_newton_r(const double* f, const double* L, const double* a, int64_t n, double inv_eps,
                           double* am, double* r, DevState* st, unsigned guard) {
    SKNR_PDL_ENTRY();
    if (guard_skip(st, guard)) return;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double d = -a[i] * expm1(f[i] * inv_eps + L[i]);
        am[i] = d;
        r[i] = a[i] - d;
    }
}

// try_newton's ell x ell algebra on one CTA (solver.cpp:37-44, objective.cpp:138-140):
// H = -(1/eps)(G1 - cross); H = (H+H^T)/2; LLT(-H) (fails iff a pivot <= 0, as
// Eigen's llt_inplace::unblocked); delta = LLT.solve(grad).
__global__ void k_newton_solve(const double* G1, const double* cross, const double* grad, int ell,
                               double inv_eps, double* delta, DevState* st, unsigned guard) {
    SKNR_PDL_ENTRY();
    if (guard_skip(st, guard)) return;
    extern __shared__ double sA[];  // ell*ell
    __shared__ int fail;
    __shared__ double piv;
    const int tid = threadIdx.x;
    if (tid == 0) fail = 0;
    for (int e = tid; e < ell * ell; e += blockDim.x) {
        const int r = e % ell, c = e / ell;
        const double h_rc = -inv_eps * (G1[r + c * ell] - cross[r + c * ell]);
        const double h_cr = -inv_eps * (G1[c + r * ell] - cross[c + r * ell]);
        sA[e] = -(0.5 * (h_rc + h_cr));
    }
    __syncthreads();
    // Right-looking factorisation. Every entry sees the same scalar operations in the
    // same order as the oracle's left-looking loop (A_rc -= L_rt L_ct for t = 0, 1, ...,
    // then / L_cc), so the factor is the oracle's, but each column costs three barriers
    // instead of a serial dot product. Eigen itself differs at the rounding level: its
    // LLT::compute runs llt_inplace::blocked, which is the unblocked loop only below 32
    // columns (and even then with SIMD dot products); for ell >= 32 (C4: 32, C5: 24 -> no)
    // it factors in blocks with GEMM trailing updates. The reference's Cholesky order is
    // therefore parity-unpinned; only the oracle's is matched.
    for (int c = 0; c < ell; ++c) {
        if (tid == 0) {
            const double x = sA[c + c * ell];
            if (!(x > 0.0)) fail = 1;
            piv = sqrt(x);
            sA[c + c * ell] = piv;
        }
        __syncthreads();
        if (fail) break;
        for (int r = c + 1 + tid; r < ell; r += blockDim.x) sA[r + c * ell] = sA[r + c * ell] / piv;
        __syncthreads();
        const int rs = ell - c - 1;
        for (int e = tid; e < rs * rs; e += blockDim.x) {
            const int r = c + 1 + e % rs, q = c + 1 + e / rs;
            if (r >= q) sA[r + q * ell] -= sA[r + c * ell] * sA[q + c * ell];
        }
        __syncthreads();
    }
    if (fail) {
        if (tid == 0) st->newton_ok = 0;
        return;
    }
    // L y = grad, then L^T delta = y, column-oriented on warp 0 (2 rows per lane)
    __shared__ double sy[64];
    if (tid >= 32) return;
    for (int r = tid; r < ell; r += 32) sy[r] = grad[r];
    __syncwarp();
    for (int t = 0; t < ell; ++t) {
        const double yt = sy[t] / sA[t + t * ell];
        for (int r = t + 1 + tid; r < ell; r += 32) sy[r] -= sA[r + t * ell] * yt;
        __syncwarp();
        if (tid == 0) sy[t] = yt;
        __syncwarp();
    }
    for (int t = ell - 1; t >= 0; --t) {
        const double yt = sy[t] / sA[t + t * ell];
        for (int r = tid; r < t; r += 32) sy[r] -= sA[t + r * ell] * yt;
        __syncwarp();
        if (tid == 0) sy[t] = yt;
        __syncwarp();
    }
    for (int r = tid; r < ell; r += 32) delta[r] = sy[r];
}

// candidate = f + V delta (solver.cpp:45)
__global__ void k_fcand(const double* f, const double* V, int64_t n, int ell, const double* delta,
                        double* out, DevState* st, unsigned guard) {
    SKNR_PDL_ENTRY();
    if (guard_skip(st, guard)) return;
    __shared__ double sd[64];
    if (threadIdx.x < ell) sd[threadIdx.x] = delta[threadIdx.x];
    __syncthreads();
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        double s = 0.0;
        for (int c = 0; c < ell; ++c) s += V[i + c * n] * sd[c];
        out[i] = f[i] + s;
    }
}

// Stable accept test, per row: candidate f' = f + V delta, d = f' - f (exact: f' and f
// are close), and the block-pass weights W[i] = (1, expm1(d_i/eps), exp(d_i/eps), 0, ...)
// of the anchor pass s_j = sum_i P~_ij, t_j = sum_i P~_ij expm1(d_i/eps),
// u_j = sum_i P~_ij exp(d_i/eps) (|d|/eps <= 600 here: the larger steps take the literal test).
__global__ void k_fcand_step(const double* f, const double* V, int64_t n, int ell, const double* delta,
                             double inv_eps, double* out, double* dvec, double* W, int kt, DevState* st,
                             unsigned guard) {
    SKNR_PDL_ENTRY();
    if (guard_skip(st, guard)) return;
    __shared__ double sd[64];
    if (threadIdx.x < ell) sd[threadIdx.x] = delta[threadIdx.x];
    __syncthreads();
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        double s = 0.0;
        for (int c = 0; c < ell; ++c) s += V[i + c * n] * sd[c];
        const double fc = f[i] + s;
        const double d = fc - f[i];
        out[i] = fc;
        dvec[i] = d;
        W[i * kt] = 1.0;
        W[i * kt + 1] = expm1(fmin(d * inv_eps, 700.0));
        W[i * kt + 2] = exp(fmin(d * inv_eps, 700.0));
    }
}

// h'_j - h_j = -eps log(u_j / s_j) from the anchor pass (ST = [s | t | u], m x 3), and
// the candidate's transform h' = h + (h' - h) (the next sweep's g if accepted). The ratio
// u/s = 1 + t/s is taken as log1p(t/s) when |t/s| <= 1/2 (small steps: u - s would cancel)
// and as log(u/s) otherwise (t/s -> -1 would cancel: a column whose mass the step moves
// away); both forms are accurate to rounding on their side of the switch (kDhSwitch).
constexpr double kDhSwitch = 0.5;
__global__ void k_dh(const double* ST, const double* h, int64_t m, double eps, double* dh, double* hcand,
                     DevState* st, unsigned guard) {
    SKNR_PDL_ENTRY();
    if (guard_skip(st, guard)) return;
    for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < m;
         j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double ts = ST[m + j] / ST[j];
        const double v = -eps * (fabs(ts) <= kDhSwitch ? log1p(ts) : log(ST[2 * m + j] / ST[j]));
        dh[j] = v;
        hcand[j] = h[j] + v;
    }
}

// accepted: f <- candidate, next g <- h(candidate); otherwise next g <- h.
__global__ void k_select(double* f, const double* fcand, int64_t n, double* gnext, const double* h,
                         const double* hcand, int64_t m, DevState* st) {
    SKNR_PDL_ENTRY();
    if (st->done) return;
    const bool acc = st->newton_ok && st->accept;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n + m;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        if (i < n) {
            if (acc) f[i] = fcand[i];
        } else {
            gnext[i - n] = acc ? hcand[i - n] : h[i - n];
        }
    }
}

// End of an iteration: trace record, max_iter stop and -- when the solve runs as a
// device-side WHILE loop (conditional graph node) -- the loop condition. The device
// trace holds `cap` records starting at iteration trace_base + 1; when it is full the
// loop pauses (condition 0 without `done`) so the host can drain it and relaunch.
__global__ void k_record(DevState* st, sknr_record* trace, long long cap, int trace_enabled,
                         cudaGraphConditionalHandle loop) {
    SKNR_PDL_ENTRY();
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    if (!st->iter_active) {
        if (loop) cudaGraphSetConditional(loop, 0);
        return;
    }
    st->iter_active = 0;
    const long long k = st->iter;
    const long long slot = k - 1 - st->trace_base;
    if (trace_enabled && slot >= 0 && slot < cap) {
        sknr_record r;
        r.index = k;
        r.marginal_error = st->gap_l2;
        r.marginal_error_inf = st->gap_inf;
        const bool acc = st->attempted && st->newton_ok && st->accept;
        r.semi_dual_value = acc ? st->q1 : st->q0;
        r.newton_attempted = st->attempted;
        r.newton_accepted = acc ? 1 : 0;
        r.wall_time_ms = static_cast<double>(globaltimer_ns() - st->t_iter0) * 1e-6;
        trace[slot] = r;
    }
    if (k >= st->max_iter) st->done = 1;
    const bool full = trace_enabled && slot + 1 >= cap;
    if (loop) cudaGraphSetConditional(loop, (st->done || full) ? 0 : 1);
}

__global__ void k_trace_rebase(DevState* st) {
    if (threadIdx.x == 0 && blockIdx.x == 0) st->trace_base = st->iter;
}

__global__ void k_axpby(const double* x, const double* y, int64_t n, double a, double b, double* out) {
    SKNR_PDL_ENTRY();
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        out[i] = a * x[i] + b * y[i];
}

// ---- top_modes helpers
// Y[:,c] -= u0 * s_c
__global__ void k_deflate(double* Y, int64_t n, int k, const double* u0, const double* s) {
    SKNR_PDL_ENTRY();
    const int64_t total = n * k;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = e % n;
        const int c = static_cast<int>(e / n);
        Y[e] -= u0[i] * s[c];
    }
}

// out (n x l) = X (n x k) * W (k x l), W col-major
__global__ void k_small_gemm(const double* X, int64_t n, int k, const double* W, int l, double* out) {
    SKNR_PDL_ENTRY();
    extern __shared__ double sW[];
    for (int e = threadIdx.x; e < k * l; e += blockDim.x) sW[e] = W[e];
    __syncthreads();
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        for (int a = 0; a < l; ++a) {
            double s = 0.0;
            for (int r = 0; r < k; ++r) s += X[i + r * n] * sW[r + a * k];
            out[i + a * n] = s;
        }
    }
}

// out (n x l) += sgn * X (n x k) * W (k x l), W col-major
__global__ void k_small_gemm_acc(const double* X, int64_t n, int k, const double* W, int l, double sgn,
                                 double* out) {
    SKNR_PDL_ENTRY();
    extern __shared__ double sW[];
    for (int e = threadIdx.x; e < k * l; e += blockDim.x) sW[e] = W[e];
    __syncthreads();
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        for (int a = 0; a < l; ++a) {
            double s = 0.0;
            for (int r = 0; r < k; ++r) s += X[i + r * n] * sW[r + a * k];
            out[i + a * n] += sgn * s;
        }
    }
}

// R = YW - theta_a XW
__global__ void k_resid(const double* YW, const double* XW, const double* theta, int64_t n, int l,
                        double* R) {
    SKNR_PDL_ENTRY();
    const int64_t total = n * l;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int a = static_cast<int>(e / n);
        R[e] = YW[e] - theta[a] * XW[e];
    }
}

__global__ void k_div_rows(const double* X, const double* s, int64_t n, int l, double* out) {
    SKNR_PDL_ENTRY();
    const int64_t total = n * l;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x)
        out[e] = X[e] / s[e % n];
}

// SplitMix64 start block (spectral.cpp:138-142): draw t = c*n + i of the
// stream seeded 0x73706563 is state seed + (t+1)*gamma -- computed in parallel.
__global__ void k_splitmix_block(double* X, int64_t n, int k, unsigned long long seed, int64_t n_global,
                                 int64_t row_begin) {
    SKNR_PDL_ENTRY();
    const int64_t total = n * k;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t t = (e / n) * n_global + row_begin + e % n;  // draw index of (row, column)
        unsigned long long z = seed + static_cast<unsigned long long>(t + 1) * 0x9E3779B97F4A7C15ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z = z ^ (z >> 31);
        const double u01 = static_cast<double>(z >> 11) * 0x1.0p-53;
        X[e] = -1.0 + 2.0 * u01;
    }
}

// ---- Householder QR with Eigen's conventions (makeHouseholder /
// applyHouseholderOnTheLeft, HouseholderQR + householderQ()*Identity):
// hh[4c..4c+3] = {tau, beta, 1/(c0-beta), zero_tail}
__global__ void k_hh_norm(double* X, int64_t n, int c, double* part, double* hh, unsigned* counter) {
    SKNR_PDL_ENTRY();
    __shared__ double sh[AUX_NT];
    double s = 0.0;
    const double* col = X + static_cast<int64_t>(c) * n;
    for (int64_t r = c + 1 + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < n;
         r += static_cast<int64_t>(gridDim.x) * blockDim.x)
        s = fma(col[r], col[r], s);
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int k = blockDim.x / 2; k > 0; k >>= 1) {
        if (threadIdx.x < k) sh[threadIdx.x] += sh[threadIdx.x + k];
        __syncthreads();
    }
    __shared__ bool is_last;
    if (threadIdx.x == 0) {
        part[blockIdx.x] = sh[0];
        __threadfence();
        is_last = atomicAdd(counter, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!is_last || threadIdx.x != 0) return;
    __threadfence();
    double tail = 0.0;
    for (unsigned b = 0; b < gridDim.x; ++b) tail += part[b];
    const double c0 = col[c];
    double tau, beta, zero;
    if (tail <= 2.2250738585072014e-308) {
        tau = 0.0;
        beta = c0;
        zero = 1.0;
    } else {
        beta = sqrt(c0 * c0 + tail);
        if (c0 >= 0.0) beta = -beta;
        tau = (beta - c0) / beta;
        zero = 0.0;
    }
    hh[4 * c] = tau;
    hh[4 * c + 1] = beta;
    hh[4 * c + 2] = c0 - beta;
    hh[4 * c + 3] = zero;
    X[c + static_cast<int64_t>(c) * n] = beta;
    *counter = 0u;
}

// v_r = X[r,c]/(c0-beta) (written back); w_c2 = X[c,c2] + sum_{r>c} v_r X[r,c2]
// for c2 in [c2lo, k) of matrix M (M==X for the factorisation, Q for forming Q).
__global__ void k_hh_w(double* X, const double* M, int64_t n, int k, int c, int c2lo, int scale_v,
                       const double* hh, double* part, double* w, unsigned* counter) {
    SKNR_PDL_ENTRY();
    constexpr int KM = 64;
    __shared__ double sh[AUX_NT];
    __shared__ double sw[KM];
    const double denom = hh[4 * c + 2];
    const bool zero = hh[4 * c + 3] != 0.0;
    double acc[KM];
    const int nw = k - c2lo;
    for (int q = 0; q < nw; ++q) acc[q] = 0.0;
    double* colc = X + static_cast<int64_t>(c) * n;
    for (int64_t r = c + 1 + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < n;
         r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        double v = colc[r];
        if (scale_v) {
            v = zero ? 0.0 : v / denom;
            colc[r] = v;
        }
        for (int q = 0; q < nw; ++q) acc[q] = fma(v, M[r + static_cast<int64_t>(c2lo + q) * n], acc[q]);
    }
    for (int q = 0; q < nw; ++q) {
        sh[threadIdx.x] = acc[q];
        __syncthreads();
        for (int s = blockDim.x / 2; s > 0; s >>= 1) {
            if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
            __syncthreads();
        }
        if (threadIdx.x == 0) sw[q] = sh[0];
        __syncthreads();
    }
    __shared__ bool is_last;
    if (threadIdx.x == 0) {
        for (int q = 0; q < nw; ++q) part[static_cast<int64_t>(blockIdx.x) * KM + q] = sw[q];
        __threadfence();
        is_last = atomicAdd(counter, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    for (int q = threadIdx.x; q < nw; q += blockDim.x) {
        double s = 0.0;
        for (unsigned b = 0; b < gridDim.x; ++b) s += part[static_cast<int64_t>(b) * KM + q];
        w[q] = M[c + static_cast<int64_t>(c2lo + q) * n] + s;
    }
    if (threadIdx.x == 0) *counter = 0u;
}

// M[r,c2] -= tau w_c2 v_r for r >= c (v_c = 1), c2 in [c2lo, k)
__global__ void k_hh_update(const double* X, double* M, int64_t n, int k, int c, int c2lo,
                            const double* hh, const double* w) {
    SKNR_PDL_ENTRY();
    const double tau = hh[4 * c];
    if (tau == 0.0) return;
    const int nw = k - c2lo;
    const int64_t rows = n - c;
    const int64_t total = rows * nw;
    const double* v = X + static_cast<int64_t>(c) * n;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = c + e % rows;
        const int q = static_cast<int>(e / rows);
        const double vr = (r == c) ? 1.0 : v[r];
        M[r + static_cast<int64_t>(c2lo + q) * n] -= tau * w[q] * vr;
    }
}

__global__ void k_eye(double* Q, int64_t n, int k) {
    SKNR_PDL_ENTRY();
    const int64_t total = n * k;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x)
        Q[e] = (e % n == e / n) ? 1.0 : 0.0;
}

// plan_ij = a_i b_j exp((f_i + g_j - C_ij)/eps)  (coupling_from, core.cpp:84-103) for the
// rows [r0, r0 + rows), col-major with leading dimension rows; f is indexed globally.
__global__ void k_coupling(const double* C, const double* x, const double* y, int64_t n, int64_t m,
                           int64_t r0, int64_t rows, int d, double kappa, const double* a,
                           const double* b, const double* f, const double* g, double inv_eps,
                           double* plan) {
    SKNR_PDL_ENTRY();
    const int64_t total = rows * m;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = r0 + e % rows, j = e / rows;
        double c;
        if (C) {
            c = C[i + j * n];
        } else {
            double s = 0.0;
            for (int q = 0; q < d; ++q) {
                const double t = x[i + q * n] - y[j + q * m];
                s += t * t;
            }
            c = kappa * s;
        }
        plan[e] = a[i] * b[j] * exp((f[i] + g[j] - c) * inv_eps);
    }
}

// Stored cost built on device from points (direct difference, generators.cpp:101),
// written in both layouts.
__global__ void k_build_cost(const double* x, const double* y, int64_t n, int64_t m, int d,
                             double kappa, double* C, double* CT) {
    SKNR_PDL_ENTRY();
    const int64_t total = n * m;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = e % n, j = e / n;
        double s = 0.0;
        for (int q = 0; q < d; ++q) {
            const double t = x[i + q * n] - y[j + q * m];
            s += t * t;
        }
        const double c = kappa * s;
        C[e] = c;
        if (CT) CT[j + i * m] = c;
    }
}

// transpose n x m col-major -> m x n col-major
// full_semi_dual_hessian (objective.cpp:150-171) on a materialised plan (col-major n x m,
// plan_ij = P~_ij b_j): out_ik = sum_j plan_ij plan_kj / b_j (= P~ diag(b) P~^T), j ascending
// within each 32-wide chunk, chunks in order. 32 x 32 output tiles, 256 threads, 4 outputs each.
__global__ void __launch_bounds__(256) k_plan_outer(const double* plan, int64_t n, int64_t m, const double* b,
                                                    double* out) {
    SKNR_PDL_ENTRY();
    __shared__ double sa[32][33], sb[32][33];
    const int64_t i0 = static_cast<int64_t>(blockIdx.x) * 32, k0 = static_cast<int64_t>(blockIdx.y) * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // ty: 0..7
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int64_t j0 = 0; j0 < m; j0 += 32) {
        __syncthreads();
        for (int q = ty; q < 32; q += 8) {
            const int64_t j = j0 + q;
            const bool jv = j < m;
            const double ib = jv ? 1.0 / b[j] : 0.0;
            sa[q][tx] = (jv && i0 + tx < n) ? plan[i0 + tx + j * n] : 0.0;
            sb[q][tx] = (jv && k0 + tx < n) ? plan[k0 + tx + j * n] * ib : 0.0;
        }
        __syncthreads();
#pragma unroll 8
        for (int q = 0; q < 32; ++q) {
            const double av = sa[q][tx];
#pragma unroll
            for (int t = 0; t < 4; ++t) acc[t] = fma(av, sb[q][ty + 8 * t], acc[t]);
        }
    }
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        const int64_t i = i0 + tx, k = k0 + ty + 8 * t;
        if (i < n && k < n) out[i + k * n] = acc[t];
    }
}

// row sums of a col-major n x m matrix, j ascending
__global__ void k_row_sums(const double* A, int64_t n, int64_t m, double* out) {
    SKNR_PDL_ENTRY();
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        double s = 0.0;
        for (int64_t j = 0; j < m; ++j) s += A[i + j * n];
        out[i] = s;
    }
}

__global__ void k_transpose(const double* A, int64_t n, int64_t m, double* AT) {
    SKNR_PDL_ENTRY();
    __shared__ double tile[32][33];
    for (int64_t bj = blockIdx.y * 32; bj < m; bj += static_cast<int64_t>(gridDim.y) * 32)
        for (int64_t bi = blockIdx.x * 32; bi < n; bi += static_cast<int64_t>(gridDim.x) * 32) {
            for (int r = threadIdx.y; r < 32; r += blockDim.y) {
                const int64_t i = bi + threadIdx.x, j = bj + r;
                if (i < n && j < m) tile[r][threadIdx.x] = A[i + j * n];
            }
            __syncthreads();
            for (int r = threadIdx.y; r < 32; r += blockDim.y) {
                const int64_t j = bj + threadIdx.x, i = bi + r;
                if (i < n && j < m) AT[j + i * m] = tile[threadIdx.x][r];
            }
            __syncthreads();
        }
}

