// engine_spectral.cuh -- top_modes on the device: QR helpers, Chebyshev / subspace / block-Lanczos iterations
// Part of the libsknr_b200 translation unit: included once, in order, by engine.cu
// (shares its types, static helpers and kernels; not a standalone header).
#pragma once

// ============================================================ top_modes
// Symmetric eigen-decomposition (stands in for Eigen::SelfAdjointEigenSolver,
// spectral.cpp:156): Householder tridiagonalisation followed by implicit QL
// with Wilkinson-type shifts (the classic tred2/tql2 pair), ascending
// eigenvalues, orthonormal eigenvectors in columns. O(k^3) for the k x k
// Rayleigh-Ritz matrix.
static bool symeig_tql(const double* Ain, int k, double* evals, double* evecs) {
    std::vector<double> a(static_cast<size_t>(k) * k), d(k), e(k);
    auto A = [&](int i, int j) -> double& { return a[static_cast<size_t>(i) * k + j]; };
    for (int i = 0; i < k; ++i)
        for (int j = 0; j < k; ++j) A(i, j) = Ain[i + j * k];
    for (int i = k - 1; i > 0; --i) {
        const int l = i - 1;
        double h = 0.0, scale = 0.0;
        if (l > 0) {
            for (int q = 0; q <= l; ++q) scale += std::abs(A(i, q));
            if (scale == 0.0) {
                e[i] = A(i, l);
            } else {
                for (int q = 0; q <= l; ++q) {
                    A(i, q) /= scale;
                    h += A(i, q) * A(i, q);
                }
                double f = A(i, l);
                double g = f >= 0.0 ? -std::sqrt(h) : std::sqrt(h);
                e[i] = scale * g;
                h -= f * g;
                A(i, l) = f - g;
                f = 0.0;
                for (int j = 0; j <= l; ++j) {
                    A(j, i) = A(i, j) / h;
                    g = 0.0;
                    for (int q = 0; q <= j; ++q) g += A(j, q) * A(i, q);
                    for (int q = j + 1; q <= l; ++q) g += A(q, j) * A(i, q);
                    e[j] = g / h;
                    f += e[j] * A(i, j);
                }
                const double hh = f / (h + h);
                for (int j = 0; j <= l; ++j) {
                    f = A(i, j);
                    e[j] = g = e[j] - hh * f;
                    for (int q = 0; q <= j; ++q) A(j, q) -= (f * e[q] + g * A(i, q));
                }
            }
        } else {
            e[i] = A(i, l);
        }
        d[i] = h;
    }
    d[0] = 0.0;
    e[0] = 0.0;
    for (int i = 0; i < k; ++i) {
        const int l = i - 1;
        if (d[i] != 0.0) {
            for (int j = 0; j <= l; ++j) {
                double g = 0.0;
                for (int q = 0; q <= l; ++q) g += A(i, q) * A(q, j);
                for (int q = 0; q <= l; ++q) A(q, j) -= g * A(q, i);
            }
        }
        d[i] = A(i, i);
        A(i, i) = 1.0;
        for (int j = 0; j <= l; ++j) A(j, i) = A(i, j) = 0.0;
    }
    for (int i = 1; i < k; ++i) e[i - 1] = e[i];
    e[k - 1] = 0.0;
    for (int l = 0; l < k; ++l) {
        int iter = 0, m;
        do {
            for (m = l; m < k - 1; ++m) {
                const double dd = std::abs(d[m]) + std::abs(d[m + 1]);
                if (std::abs(e[m]) <= 0x1p-53 * dd) break;
            }
            if (m != l) {
                if (iter++ == 100) return false;
                double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
                double r = std::hypot(g, 1.0);
                g = d[m] - d[l] + e[l] / (g + std::copysign(r, g));
                double s = 1.0, c = 1.0, p = 0.0;
                int i;
                for (i = m - 1; i >= l; --i) {
                    double f = s * e[i];
                    const double b = c * e[i];
                    e[i + 1] = (r = std::hypot(f, g));
                    if (r == 0.0) {
                        d[i + 1] -= p;
                        e[m] = 0.0;
                        break;
                    }
                    s = f / r;
                    c = g / r;
                    g = d[i + 1] - p;
                    r = (d[i] - g) * s + 2.0 * c * b;
                    d[i + 1] = g + (p = s * r);
                    g = c * r - b;
                    for (int q = 0; q < k; ++q) {
                        f = A(q, i + 1);
                        A(q, i + 1) = s * A(q, i) + c * f;
                        A(q, i) = c * A(q, i) - s * f;
                    }
                }
                if (r == 0.0 && i >= l) continue;
                d[l] -= p;
                e[l] = g;
                e[m] = 0.0;
            }
        } while (m != l);
    }
    std::vector<int> order(k);
    for (int i = 0; i < k; ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(), [&](int u, int v) { return d[u] < d[v]; });
    for (int c = 0; c < k; ++c) {
        evals[c] = d[order[c]];
        for (int r = 0; r < k; ++r) evecs[r + c * k] = A(r, order[c]);
    }
    return true;
}

static void host_sym_eig(const std::vector<double>& A, int k, std::vector<double>& evals,
                         std::vector<double>& evecs) {
    evals.assign(k, 0.0);
    evecs.assign(static_cast<size_t>(k) * k, 0.0);
    if (!symeig_tql(A.data(), k, evals.data(), evecs.data()))
        throw EigenFailure("top_modes: dense Ritz solve failed", std::numeric_limits<double>::infinity());
}

struct QrWork {
    DBuf hh, w, part, Q, backup, flag, full;
    // SKNR_FORCE_HOUSEHOLDER=1: every round takes the Householder path (tests of the
    // fallback, sharded and not)
    bool force_householder = std::getenv("SKNR_FORCE_HOUSEHOLDER") != nullptr;
};

// Cholesky G + shift*I = L L^T (shift = coef * trace(G)), then Rinv = L^{-T}
// (upper). One CTA; k <= 64. *fail = 1 if a pivot is not positive.
__global__ void k_chol_inv(const double* G, int k, double coef, double* Rinv, int* fail) {
    SKNR_PDL_ENTRY();
    extern __shared__ double sL[];  // k*k
    __shared__ double piv;
    __shared__ int bad;
    const int tid = threadIdx.x;
    if (tid == 0) {
        bad = 0;
        double tr = 0.0;
        for (int c = 0; c < k; ++c) tr += G[c + c * k];
        piv = coef * tr;
    }
    __syncthreads();
    const double shift = piv;
    for (int e = tid; e < k * k; e += blockDim.x) {
        const int r = e % k, c = e / k;
        sL[e] = G[e] + (r == c ? shift : 0.0);
    }
    __syncthreads();
    for (int c = 0; c < k; ++c) {
        if (tid == 0) {
            double x = sL[c + c * k];
            for (int t = 0; t < c; ++t) x -= sL[c + t * k] * sL[c + t * k];
            if (!(x > 0.0)) bad = 1;
            piv = sqrt(x);
            sL[c + c * k] = piv;
        }
        __syncthreads();
        if (bad) break;
        for (int r = c + 1 + tid; r < k; r += blockDim.x) {
            double v = sL[r + c * k];
            for (int t = 0; t < c; ++t) v -= sL[r + t * k] * sL[c + t * k];
            sL[r + c * k] = v / piv;
        }
        __syncthreads();
    }
    if (bad) {
        if (tid == 0) *fail = 1;
        return;
    }
    // column j of L^{-1} by forward substitution; Rinv = (L^{-1})^T
    for (int j = tid; j < k; j += blockDim.x) {
        double x[64];
        for (int r = 0; r < k; ++r) {
            double v = (r == j) ? 1.0 : 0.0;
            for (int t = j; t < r; ++t) v -= sL[r + t * k] * x[t];
            x[r] = r < j ? 0.0 : v / sL[r + r * k];
        }
        for (int r = 0; r < k; ++r) Rinv[j + r * k] = x[r];  // Rinv(j, r) = Linv(r, j)
    }
}

// Thin Householder Q of X (n x k) in place (spectral.cpp:116-117 conventions).
static void device_householder_q(Problem& P, double* X, int64_t n, int k, QrWork& qw) {
    cudaStream_t s = P.stream;
    qw.hh.ensure(4 * 64);
    qw.w.ensure(64);
    qw.part.ensure(148 * 64);
    qw.Q.ensure(static_cast<size_t>(n) * k);
    unsigned* ctr = &P.st->counters[8];
    const int kk = static_cast<int>(std::min<int64_t>(k, n));
    const int gb = std::max(1, std::min(148, static_cast<int>((n + 4095) / 4096)));
    for (int c = 0; c < kk; ++c) {
        count_launch();
        k_hh_norm<<<gb, AUX_NT, 0, s>>>(X, n, c, qw.part.p, qw.hh.p, ctr);
        count_launch();
        k_hh_w<<<gb, AUX_NT, 0, s>>>(X, X, n, k, c, c + 1, 1, qw.hh.p, qw.part.p, qw.w.p, ctr);
        if (c + 1 < k) {
            count_launch();
            k_hh_update<<<grid_for((n - c) * (k - c - 1)), AUX_NT, 0, s>>>(X, X, n, k, c, c + 1, qw.hh.p,
                                                                          qw.w.p);
        }
    }
    count_launch();
    k_eye<<<grid_for(n * k), AUX_NT, 0, s>>>(qw.Q.p, n, k);
    for (int c = kk - 1; c >= 0; --c) {
        count_launch();
        k_hh_w<<<gb, AUX_NT, 0, s>>>(X, qw.Q.p, n, k, c, c, 0, qw.hh.p, qw.part.p, qw.w.p, ctr);
        count_launch();
        k_hh_update<<<grid_for((n - c) * (k - c)), AUX_NT, 0, s>>>(X, qw.Q.p, n, k, c, c, qw.hh.p,
                                                                   qw.w.p);
    }
    CK(cudaMemcpyAsync(X, qw.Q.p, sizeof(double) * n * k, cudaMemcpyDeviceToDevice, s));
    CK(cudaGetLastError());
}

// CholeskyQR step: X <- X R^{-1} with R^T R = X^T X (+ shift I). The shifted
// first pass makes the factorisation succeed for cond(X) up to ~1/u (shifted
// CholeskyQR3); a failed Cholesky sets *fail and the caller falls back to
// Householder.
static void device_cholqr_step(Problem& P, double* X, int64_t n, int k, bool shifted, QrWork& qw,
                               int* fail) {
    qw.Q.ensure(static_cast<size_t>(n) * k);
    qw.w.ensure(64 * 64 * 2);
    double* G = qw.w.p;
    double* Rinv = qw.w.p + 64 * 64;
    gram_all(P, n, k, k, X, n, X, n, nullptr, G, 0);
    const double shift_coef = shifted ? 11.0 * (static_cast<double>(n) * k + k * (k + 1.0)) * 0x1p-53 : 0.0;
    count_launch();
    k_chol_inv<<<1, 64, sizeof(double) * k * k, P.stream>>>(G, k, shift_coef, Rinv, fail);
    count_launch();
    k_small_gemm<<<grid_for(n), AUX_NT, sizeof(double) * k * k, P.stream>>>(X, n, k, Rinv, k, qw.Q.p);
    CK(cudaMemcpyAsync(X, qw.Q.p, sizeof(double) * n * k, cudaMemcpyDeviceToDevice, P.stream));
}

// orthonormalize_deflated (spectral.cpp:113-121): same deflation rounds and
// stopping test; the QR is shifted CholeskyQR3 (same column space as the
// reference's Householder Q; columns may differ in sign, which neither the
// Rayleigh-Ritz step nor the Newton step sees) with a device Householder
// fallback (Eigen's reflector convention) when the Gram is numerically singular.
static void device_orth_deflated(Problem& P, double* X, int64_t n, int k, const double* u0,
                                 QrWork& qw) {
    double* s = P.misc.p;  // k dots
    qw.flag.ensure(1);
    int* fail = reinterpret_cast<int*>(qw.flag.p);
    for (int round = 0; round < 3; ++round) {
        gram_all(P, n, k, 1, X, n, u0, n, nullptr, s, 0);
        count_launch();
        k_deflate<<<grid_for(n * k), AUX_NT, 0, P.stream>>>(X, n, k, u0, s);
        bool use_householder = qw.force_householder;
        if (!use_householder) {
            CK(cudaMemcpyAsync(qw.backup.p, X, sizeof(double) * n * k, cudaMemcpyDeviceToDevice, P.stream));
            CK(cudaMemsetAsync(fail, 0, sizeof(int), P.stream));
            device_cholqr_step(P, X, n, k, true, qw, fail);
            device_cholqr_step(P, X, n, k, false, qw, fail);
            device_cholqr_step(P, X, n, k, false, qw, fail);
            int hfail = 0;
            CK(cudaMemcpyAsync(&hfail, fail, sizeof(int), cudaMemcpyDeviceToHost, P.stream));
            CK(cudaStreamSynchronize(P.stream));
            if (hfail) {  // restore the deflated block and redo this round with Householder
                CK(cudaMemcpyAsync(X, qw.backup.p, sizeof(double) * n * k, cudaMemcpyDeviceToDevice, P.stream));
                use_householder = true;
            }
        }
        if (use_householder) {
            if (P.shard) {
                // row-sharded: every rank gathers the whole n x k block, runs the same
                // device Householder QR on it (identical inputs -> identical Q on every
                // rank) and keeps its own rows
                qw.full.ensure(static_cast<size_t>(P.n_global) * k);
                gather_row_block(P, X, k, qw.full.p);
                device_householder_q(P, qw.full.p, P.n_global, k, qw);
                CK(cudaMemcpy2DAsync(X, sizeof(double) * n, qw.full.p + P.row_begin, sizeof(double) * P.n_global,
                                     sizeof(double) * n, k, cudaMemcpyDeviceToDevice, P.stream));
            } else {
                device_householder_q(P, X, n, k, qw);
            }
        }
        gram_all(P, n, k, 1, X, n, u0, n, nullptr, s, 0);
        std::vector<double> hs(k + 1);
        download(hs.data(), s, k, P.stream);
        CK(cudaStreamSynchronize(P.stream));
        double worst = 0.0;
        for (int c = 0; c < k; ++c) worst = std::max(worst, std::abs(hs[c]));
        if (worst < 1e-13) break;
    }
}

struct Basis {
    std::vector<double> vectors, vectors_sym, rhos;
    int64_t sweeps = 0;
};

// Y = R~ R~^T X with the Perron direction sqrt(alpha) deflated (spectral.cpp:150-151):
// two DMMA block passes (column then row direction) and a rank-one correction.
struct OpWork {
    DBuf Z, W;
    // culling of the operator passes (opt-in): per-output lower bounds of log(sum of
    // terms) for the two directions, from the anchor's own transforms
    bool cull = false;
    DBuf sub0, sub1, tmp;
};

// sub = (v - vt)/eps (+ lw): log-total lower bound of an operator pass's outputs
__global__ void k_cull_sub(const double* v, const double* vt, const double* lw, double inv_eps, int64_t count,
                           double* sub) {
    SKNR_PDL_ENTRY();
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        sub[i] = (v[i] - vt[i]) * inv_eps + (lw ? lw[i] : 0.0);
}

static void lse(Problem& P, int dir, const double* in_vec, double* pot, unsigned guard);

// Operator passes of R~ R~^T at the anchor (f, g): column pass terms sqrt(a_i) e^{(f_i+g_j-C_ij)/eps}
// sum to >= e^{(g_j - g~_j)/eps} (g~ = f^{C,eps}), row pass terms to >= sqrt(a_i) e^{(f_i - f~_i)/eps}
// (f~ = g^{C,eps}); these lower bounds normalise the culling test (pts_mma_cull_kernel).
static void prepare_op_culling(Problem& P, const double* f, const double* g, OpWork& ow) {
    ow.cull = cull_block_active(P, 0) && cull_block_active(P, 1) && cull_active(P, 0) && cull_active(P, 1);
    if (!ow.cull) return;
    const int64_t n = P.n, m = P.m;
    ow.sub0.ensure(m);
    ow.sub1.ensure(n);
    ow.tmp.ensure(std::max(n, m));
    cudaStream_t s = P.stream;
    lse(P, 0, f, ow.tmp.p, G_NONE);  // g~
    count_launch();
    k_cull_sub<<<grid_for(m), AUX_NT, 0, s>>>(g, ow.tmp.p, nullptr, P.inv_eps(), m, ow.sub0.p);
    lse(P, 1, g, ow.tmp.p, G_NONE);  // f~
    count_launch();
    k_cull_sub<<<grid_for(n), AUX_NT, 0, s>>>(f, ow.tmp.p, P.src.lsw.p, P.inv_eps(), n, ow.sub1.p);
}

static void apply_sym_sym(Problem& P, const double* f, const double* g, const double* X, double* Y,
                          int block, int kt, OpWork& ow) {
    const int64_t n = P.n, m = P.m;
    cudaStream_t s = P.stream;
    ow.Z.ensure(m * block);
    ow.W.ensure(std::max(n, m) * kt);
    // Z = R~^T X : z_j = sqrt(b_j) sum_i sqrt(a_i) e^{(f_i+g_j-C_ij)/eps} X_i
    count_launch();
    k_pack_w<<<grid_for(n * kt), AUX_NT, 0, s>>>(X, n, n, block, kt, nullptr, ow.W.p);
    PassSpec zt;
    zt.dir = 0;
    zt.in_v = f;
    zt.in_lw = P.src.lsw.p;
    zt.out_v = g;
    zt.W = ow.W.p;
    zt.k = block;
    zt.kt = kt;
    zt.out_scale = P.tgt.sw.p;
    zt.out = ow.Z.p;
    zt.cull = ow.cull;
    zt.cull_logtot = ow.sub0.p;
    plan_pass(P, zt);
    // Y = R~ Z : y_i = sum_j sqrt(a_i) e^{..} sqrt(b_j) z_j
    count_launch();
    k_pack_w<<<grid_for(m * kt), AUX_NT, 0, s>>>(ow.Z.p, m, m, block, kt, P.tgt.sw.p, ow.W.p);
    PassSpec yr;
    yr.dir = 1;
    yr.in_v = g;
    yr.out_v = f;
    yr.out_lw = P.src.lsw.p;
    yr.W = ow.W.p;
    yr.k = block;
    yr.kt = kt;
    yr.out = Y;
    yr.cull = ow.cull;
    yr.cull_logtot = ow.sub1.p;
    plan_pass(P, yr);
    // Y -= sqrt(a) (sqrt(a)^T Y)
    gram_all(P, n, block, 1, Y, n, P.src.sw.p, n, nullptr, P.misc.p, 0);
    count_launch();
    k_deflate<<<grid_for(n * block), AUX_NT, 0, s>>>(Y, n, block, P.src.sw.p, P.misc.p);
}

// Chebyshev three-term step: out = a * (AY - c * Y) - b * Yprev
__global__ void k_cheb_step(const double* AY, const double* Y, const double* Yprev, int64_t count, double a,
                            double c, double b, double* out) {
    SKNR_PDL_ENTRY();
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        out[i] = a * (AY[i] - c * Y[i]) - (Yprev ? b * Yprev[i] : 0.0);
}

// top_modes (spectral.cpp:125-193) on device; f, g are device vectors.
// method 0: the reference's block subspace iteration (one operator application
// per sweep; `sweeps` counts them). method 1 (opt-in, not in the reference):
// Chebyshev-filtered subspace iteration -- each outer step applies a degree-q
// Chebyshev polynomial of R~R~^T that damps the unwanted interval [0, theta_k]
// (theta_k = smallest Ritz value of the block) before the same Rayleigh-Ritz
// and the same residual test; `sweeps` then counts operator applications.
// Host Cholesky (upper factor R with G = R^T R) of a k x k SPD matrix; false on breakdown.
static bool host_chol_upper(const std::vector<double>& G, int k, std::vector<double>& R) {
    R.assign(static_cast<size_t>(k) * k, 0.0);
    for (int j = 0; j < k; ++j) {
        double d = G[j + j * k];
        for (int t = 0; t < j; ++t) d -= R[t + j * k] * R[t + j * k];
        if (!(d > 0.0)) return false;
        const double rjj = std::sqrt(d);
        R[j + j * k] = rjj;
        for (int c = j + 1; c < k; ++c) {
            double v = G[j + c * k];
            for (int t = 0; t < j; ++t) v -= R[t + j * k] * R[t + c * k];
            R[j + c * k] = v / rjj;
        }
    }
    return true;
}
// Inverse of an upper-triangular k x k matrix (col-major).
static std::vector<double> host_upper_inv(const std::vector<double>& R, int k) {
    std::vector<double> X(static_cast<size_t>(k) * k, 0.0);
    for (int c = 0; c < k; ++c) {
        X[c + c * k] = 1.0 / R[c + c * k];
        for (int r = c - 1; r >= 0; --r) {
            double s = 0.0;
            for (int t = r + 1; t <= c; ++t) s += R[r + t * k] * X[t + c * k];
            X[r + c * k] = -s / R[r + r * k];
        }
    }
    return X;
}

// top_modes, method 2 (opt-in, not in the reference; the north star's "device-side
// Lanczos/Krylov estimate"): restarted block Lanczos on the same operator R~R~^T with
// sqrt(alpha) deflated. Each cycle builds s (12..16) blocks of b = ell+5 Krylov vectors with full
// (two-pass) block reorthogonalisation and CholeskyQR2 for the next block, Rayleigh-Ritz
// on the block-tridiagonal projection (host), and restarts from the top b Ritz vectors.
// Convergence is declared with the reference's own criterion: the explicit residuals
// ||R~R~^T x_a - theta_a x_a|| of the top ell Ritz pairs (one extra application) <= tol.
// `sweeps` counts operator applications.
static Basis top_modes_lanczos(Problem& P, const double* f, const double* g, int64_t ell, double tol,
                               int64_t max_apps, int b, int steps) {
    const int64_t n = P.n;
    const int kt = block_kt_for(b);
    const int s = std::max(12, std::min(steps, 16));  // shorter cycles restart too often (C4: 8 -> 423 apps)
    cudaStream_t st = P.stream;
    DBuf Qs, W, Xr, AX, R, dC, th;
    Qs.ensure(static_cast<size_t>(s + 1) * n * b);
    W.ensure(static_cast<size_t>(n) * b);
    Xr.ensure(static_cast<size_t>(n) * b);
    AX.ensure(static_cast<size_t>(n) * b);
    R.ensure(static_cast<size_t>(n) * b);
    dC.ensure(static_cast<size_t>(64) * 64 * 2);
    th.ensure(64);
    P.misc.ensure(256);
    QrWork qw;
    OpWork ow;
    prepare_op_culling(P, f, g, ow);
    qw.backup.ensure(static_cast<size_t>(n) * b);
    auto Q = [&](int j) { return Qs.p + static_cast<size_t>(j) * n * b; };
    count_launch();
    k_splitmix_block<<<grid_for(n * b), AUX_NT, 0, st>>>(Q(0), n, b, 0x73706563ull, P.n_global, P.row_begin);
    device_orth_deflated(P, Q(0), n, b, P.src.sw.p, qw);
    auto host_gram = [&](const double* U, const double* V) {
        gram_all(P, n, b, b, U, n, V, n, nullptr, dC.p, 0);
        std::vector<double> h(static_cast<size_t>(b) * b);
        download(h.data(), dC.p, static_cast<size_t>(b) * b, st);
        CK(cudaStreamSynchronize(st));
        return h;
    };
    auto gemm_acc = [&](const double* X, const std::vector<double>& M, int l, double sgn, double* out) {
        upload(dC.p, M.data(), M.size(), st);
        count_launch();
        k_small_gemm_acc<<<grid_for(n), AUX_NT, sizeof(double) * b * l, st>>>(X, n, b, dC.p, l, sgn, out);
    };
    // W (n x b) -> Q_next R with CholeskyQR2; false when W is numerically rank deficient
    auto cholqr2 = [&](double* Wp, double* Qnext, std::vector<double>& Bout) {
        std::vector<double> R1, R2;
        if (!host_chol_upper(host_gram(Wp, Wp), b, R1)) return false;
        CK(cudaMemsetAsync(Qnext, 0, sizeof(double) * n * b, st));
        gemm_acc(Wp, host_upper_inv(R1, b), b, 1.0, Qnext);
        if (!host_chol_upper(host_gram(Qnext, Qnext), b, R2)) return false;
        CK(cudaMemcpyAsync(Wp, Qnext, sizeof(double) * n * b, cudaMemcpyDeviceToDevice, st));
        CK(cudaMemsetAsync(Qnext, 0, sizeof(double) * n * b, st));
        gemm_acc(Wp, host_upper_inv(R2, b), b, 1.0, Qnext);
        Bout.assign(static_cast<size_t>(b) * b, 0.0);  // B = R2 R1
        for (int c = 0; c < b; ++c)
            for (int r = 0; r <= c; ++r) {
                double v = 0.0;
                for (int t = r; t <= c; ++t) v += R2[r + t * b] * R1[t + c * b];
                Bout[r + c * b] = v;
            }
        return true;
    };

    Basis out;
    int64_t apps = 0;
    double best = std::numeric_limits<double>::infinity();
    std::vector<double> theta(ell);
    while (apps < max_apps) {
        const int K1 = (s + 1) * b;
        std::vector<double> T(static_cast<size_t>(K1) * K1, 0.0), Blast;
        int jmax = 0;
        bool broke = false;
        for (int j = 0; j < s && apps < max_apps; ++j) {
            apply_sym_sym(P, f, g, Q(j), W.p, b, kt, ow);  // W = A Q_j (deflated)
            ++apps;
            for (int pass = 0; pass < 2; ++pass)
                for (int i = 0; i <= j; ++i) {
                    const std::vector<double> C = host_gram(Q(i), W.p);  // Q_i^T W
                    gemm_acc(Q(i), C, b, -1.0, W.p);
                    for (int c = 0; c < b; ++c)
                        for (int r = 0; r < b; ++r) T[(i * b + r) + static_cast<size_t>(j * b + c) * K1] += C[r + c * b];
                }
            jmax = j + 1;
            std::vector<double> B;
            if (!cholqr2(W.p, Q(j + 1), B)) {  // invariant subspace reached
                broke = true;
                break;
            }
            for (int c = 0; c < b; ++c)
                for (int r = 0; r < b; ++r) T[((j + 1) * b + r) + static_cast<size_t>(j * b + c) * K1] = B[r + c * b];
            Blast = B;
        }
        // Rayleigh-Ritz on the symmetrised K x K projection
        const int K = jmax * b;
        std::vector<double> Ts(static_cast<size_t>(K) * K), ev, evec;
        for (int c = 0; c < K; ++c)
            for (int r = 0; r < K; ++r)
                Ts[r + static_cast<size_t>(c) * K] =
                    0.5 * (T[r + static_cast<size_t>(c) * K1] + T[c + static_cast<size_t>(r) * K1]);
        host_sym_eig(Ts, K, ev, evec);  // ascending
        // top b Ritz vectors: X = sum_i Q_i Y_i
        CK(cudaMemsetAsync(Xr.p, 0, sizeof(double) * n * b, st));
        for (int i = 0; i < jmax; ++i) {
            std::vector<double> Yi(static_cast<size_t>(b) * b);
            for (int a = 0; a < b; ++a)
                for (int r = 0; r < b; ++r) Yi[r + a * b] = evec[(i * b + r) + static_cast<size_t>(K - 1 - a) * K];
            gemm_acc(Q(i), Yi, b, 1.0, Xr.p);
        }
        for (int a = 0; a < ell; ++a) theta[a] = ev[K - 1 - a];
        // cheap estimate ||B_last y_a(last block)||, then the explicit residual test
        double est = 0.0;
        if (!broke && !Blast.empty()) {
            for (int a = 0; a < ell; ++a) {
                double s2 = 0.0;
                for (int r = 0; r < b; ++r) {
                    double v = 0.0;
                    for (int t = 0; t < b; ++t)
                        v += Blast[r + t * b] * evec[((jmax - 1) * b + t) + static_cast<size_t>(K - 1 - a) * K];
                    s2 += v * v;
                }
                est = std::max(est, std::sqrt(s2));
            }
        }
        (void)est;  // the cheap bound is kept for diagnostics; the test below is the reference's
        {
            apply_sym_sym(P, f, g, Xr.p, AX.p, b, kt, ow);
            ++apps;
            upload(th.p, theta.data(), ell, st);
            count_launch();
            k_resid<<<grid_for(n * ell), AUX_NT, 0, st>>>(AX.p, Xr.p, th.p, n, static_cast<int>(ell), R.p);
            gram_all(P, n, static_cast<int>(ell), static_cast<int>(ell), R.p, n, R.p, n, nullptr, P.misc.p, 0, 1);
            std::vector<double> hres(ell);
            download(hres.data(), P.misc.p, ell, st);
            CK(cudaStreamSynchronize(st));
            double max_res = 0.0;
            for (int a = 0; a < ell; ++a) max_res = std::max(max_res, std::sqrt(hres[a]));
            best = std::min(best, max_res);
            if (max_res <= tol) break;
        }
        // restart from the top b Ritz vectors
        CK(cudaMemcpyAsync(Q(0), Xr.p, sizeof(double) * n * b, cudaMemcpyDeviceToDevice, st));
        device_orth_deflated(P, Q(0), n, b, P.src.sw.p, qw);
        if (apps >= max_apps) break;
    }
    out.sweeps = apps;
    if (!(best <= tol))
        throw EigenFailure("top_modes: no convergence within max_power_iters, best residual " + std::to_string(best),
                           best);
    // vectors_sym = orth(top ell Ritz vectors); rhos = sqrt(max(theta,0)); vectors = vectors_sym ./ sqrt(alpha)
    device_orth_deflated(P, Xr.p, n, static_cast<int>(ell), P.src.sw.p, qw);
    count_launch();
    k_div_rows<<<grid_for(n * ell), AUX_NT, 0, st>>>(Xr.p, P.src.sw.p, n, static_cast<int>(ell), R.p);
    const int64_t ng = P.n_global;
    out.vectors_sym.resize(ng * ell);
    out.vectors.resize(ng * ell);
    for (int64_t c = 0; c < ell; ++c) {
        gather_rows(P, Xr.p + c * n, out.vectors_sym.data() + c * ng);
        gather_rows(P, R.p + c * n, out.vectors.data() + c * ng);
    }
    out.rhos.resize(ell);
    for (int a = 0; a < ell; ++a) out.rhos[a] = std::sqrt(std::max(theta[a], 0.0));
    return out;
}

static Basis top_modes_device(Problem& P, const double* f, const double* g, int64_t ell, double tol,
                              int64_t max_power_iters, int method = 0, int degree = 8) {
    const int64_t n = P.n;
    if (ell < 1) throw InvalidArgument("top_modes: ell must be >= 1");
    if (ell >= P.n_global) throw InvalidArgument("top_modes: ell must be < n");
    if (max_power_iters < 0) max_power_iters = 500 * ell;
    const int block = static_cast<int>(std::min<int64_t>(ell + 5, P.n_global - 1));
    if (block > 64) throw InvalidArgument("top_modes: ell + 5 > 64 is not supported by sknr_b200");
    if (degree < 1) degree = 1;
    if (method == 2) return top_modes_lanczos(P, f, g, ell, tol, max_power_iters, block, degree);
    const int kt = block_kt_for(block);
    cudaStream_t s = P.stream;
    DBuf X, Y, Y2, XW, YW, R, Wd, th, Wfull;
    X.ensure(n * block);
    Y.ensure(n * block);
    Y2.ensure(n * block);
    XW.ensure(n * ell);
    YW.ensure(n * ell);
    R.ensure(n * ell);
    Wd.ensure(block * ell);
    Wfull.ensure(block * block);
    th.ensure(ell);
    P.misc.ensure(256);
    QrWork qw;
    OpWork ow;
    prepare_op_culling(P, f, g, ow);
    qw.backup.ensure(static_cast<size_t>(n) * block);
    count_launch();
    k_splitmix_block<<<grid_for(n * block), AUX_NT, 0, s>>>(X.p, n, block, 0x73706563ull, P.n_global,
                                                            P.row_begin);
    device_orth_deflated(P, X.p, n, block, P.src.sw.p, qw);

    DBuf T;
    T.ensure(block * block);
    std::vector<double> hT(block * block), ts(block * block), evals, evecs, hres(ell);
    double best = std::numeric_limits<double>::infinity();
    bool ok = false;
    Basis out;
    std::vector<double> theta(ell), w(block * ell);
    int64_t applications = 0;
    while (applications < max_power_iters) {
        apply_sym_sym(P, f, g, X.p, Y.p, block, kt, ow);  // Y = A X
        ++applications;
        // Rayleigh-Ritz on the current orthonormal block
        gram_all(P, n, block, block, X.p, n, Y.p, n, nullptr, T.p, 0);
        download(hT.data(), T.p, block * block, s);
        CK(cudaStreamSynchronize(s));
        for (int a = 0; a < block; ++a)
            for (int b = 0; b < block; ++b) ts[a + b * block] = 0.5 * (hT[a + b * block] + hT[b + a * block]);
        host_sym_eig(ts, block, evals, evecs);
        for (int a = 0; a < ell; ++a) {
            for (int r = 0; r < block; ++r) w[r + a * block] = evecs[r + (block - 1 - a) * block];
            theta[a] = evals[block - 1 - a];
        }
        upload(Wd.p, w.data(), block * ell, s);
        upload(th.p, theta.data(), ell, s);
        count_launch();
        k_small_gemm<<<grid_for(n), AUX_NT, sizeof(double) * block * ell, s>>>(X.p, n, block, Wd.p,
                                                                              static_cast<int>(ell), XW.p);
        count_launch();
        k_small_gemm<<<grid_for(n), AUX_NT, sizeof(double) * block * ell, s>>>(Y.p, n, block, Wd.p,
                                                                              static_cast<int>(ell), YW.p);
        count_launch();
        k_resid<<<grid_for(n * ell), AUX_NT, 0, s>>>(YW.p, XW.p, th.p, n, static_cast<int>(ell), R.p);
        gram_all(P, n, static_cast<int>(ell), static_cast<int>(ell), R.p, n, R.p, n, nullptr, P.misc.p, 0, 1);
        download(hres.data(), P.misc.p, ell, s);
        CK(cudaStreamSynchronize(s));
        double max_res = 0.0;
        for (int a = 0; a < ell; ++a) max_res = std::max(max_res, std::sqrt(hres[a]));
        best = std::min(best, max_res);
        if (max_res <= tol) {
            ok = true;
            break;
        }
        const bool tiny_gap = evals[0] < 1e-3 * evals[block - 1];  // fast decay: plain steps suffice
        if (method == 0 || tiny_gap || applications + degree > max_power_iters) {
            CK(cudaMemcpyAsync(X.p, Y.p, sizeof(double) * n * block, cudaMemcpyDeviceToDevice, s));
        } else {
            // rotate to the full Ritz basis, then filter with T_q on [0, theta_min]
            upload(Wfull.p, evecs.data(), block * block, s);
            count_launch();
            k_small_gemm<<<grid_for(n), AUX_NT, sizeof(double) * block * block, s>>>(X.p, n, block, Wfull.p,
                                                                                    block, Y2.p);
            count_launch();
            k_small_gemm<<<grid_for(n), AUX_NT, sizeof(double) * block * block, s>>>(Y.p, n, block, Wfull.p,
                                                                                    block, X.p);
            // now Y2 = X W (basis), X = A X W (its image)
            const double lo = 0.0, hi = std::max(evals[0], 0.0);
            const double e = 0.5 * (hi - lo), c = 0.5 * (hi + lo);
            double* Yprev = Y2.p;   // T_0 term
            double* Ycur = Y.p;     // T_1 term
            count_launch();
            k_cheb_step<<<grid_for(n * block), AUX_NT, 0, s>>>(X.p, Y2.p, nullptr, n * block, 1.0 / e, c, 0.0,
                                                               Ycur);
            double* spare = X.p;
            for (int q = 2; q <= degree; ++q) {
                apply_sym_sym(P, f, g, Ycur, spare, block, kt, ow);  // spare = A Ycur
                ++applications;
                count_launch();
                k_cheb_step<<<grid_for(n * block), AUX_NT, 0, s>>>(spare, Ycur, Yprev, n * block, 2.0 / e, c, 1.0,
                                                                   spare);
                std::swap(Yprev, Ycur);
                std::swap(Ycur, spare);
            }
            if (Ycur != X.p)
                CK(cudaMemcpyAsync(X.p, Ycur, sizeof(double) * n * block, cudaMemcpyDeviceToDevice, s));
        }
        device_orth_deflated(P, X.p, n, block, P.src.sw.p, qw);
    }
    out.sweeps = applications;
    if (!ok)
        throw EigenFailure(
            "top_modes: no convergence within max_power_iters, best residual " + std::to_string(best),
            best);
    // vectors_sym = orth(XW); rhos = sqrt(max(theta,0)); vectors = vectors_sym ./ sqrt(alpha)
    device_orth_deflated(P, XW.p, n, static_cast<int>(ell), P.src.sw.p, qw);
    count_launch();
    k_div_rows<<<grid_for(n * ell), AUX_NT, 0, s>>>(XW.p, P.src.sw.p, n, static_cast<int>(ell), R.p);
    const int64_t ng = P.n_global;
    out.vectors_sym.resize(ng * ell);
    out.vectors.resize(ng * ell);
    for (int64_t c = 0; c < ell; ++c) {
        gather_rows(P, XW.p + c * n, out.vectors_sym.data() + c * ng);
        gather_rows(P, R.p + c * n, out.vectors.data() + c * ng);
    }
    out.rhos.resize(ell);
    for (int a = 0; a < ell; ++a) out.rhos[a] = std::sqrt(std::max(theta[a], 0.0));
    return out;
}

