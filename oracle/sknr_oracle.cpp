// =============================================================================
// sknr_oracle.cpp -- CPU ORACLE. TEST INFRASTRUCTURE ONLY.
//
// A plain C++20 restatement (no Eigen, which is absent from this image) of the
// reference SK-NR(ell) path in /root/reference/proj. It is the checker for the
// B200 library: only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference leg may load it. The product path
// (paper_2506_14780_b200/) never links or calls it.
//
// Parity status: the restatement keeps the reference's per-cell formulas and
// loop orders verbatim (file:line cited per function). It is pinned against
// every known-answer value the reference's own tests hold for this path
// (tests/test_oracle_kat.py: test_core.cpp:13-46, :66-76, :101-128;
// test_solver.cpp:25-73/187-202 trajectory pin; support.hpp:87-101 closed-form
// 2x2 optimum; test_spectral.cpp top_modes-vs-dense-SVD). The reference itself
// cannot be compiled here (Eigen3 REQUIRED, proj/CMakeLists.txt:13), so where
// the reference calls Eigen (.norm/.dot reductions, GEMM, LLT, HouseholderQR,
// SelfAdjointEigenSolver) only the tolerances are pinned, not bitwise order.
//
// Output-parallel (std::thread): the O(nm) transforms parallelise over their OUTPUT
// index only (columns for the column LSE, rows for the row LSE); each output's
// reduction runs in the reference's sequential order, so results are
// bitwise-identical to the single-thread run for any thread count.
// =============================================================================
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

#include <thread>

namespace oracle {

using Index = long;
using Vec = std::vector<double>;

// ---------------------------------------------------------------- problem
// Cost accessor. kind 0: dense column-major n x m (reference CostMatrix,
// types.hpp:36-45). kind 1: squared-Euclidean cost of two column-major point
// clouds evaluated on the fly in direct-difference form, exactly the formula of
// sq_euclidean_cost (generators.cpp:94-103, :101), optionally divided by
// cost_div (C2's max-normalisation).
struct Problem {
    int kind = 0;
    const double* cost = nullptr;
    const double* x = nullptr;  // n x d col-major
    const double* y = nullptr;  // m x d col-major
    Index n = 0, m = 0, d = 0;
    double cost_div = 1.0;
    Vec a, b, la, lb;
    double eps = 1.0;

    inline double C(Index i, Index j) const {
        if (kind == 0) return cost[i + j * n];
        double s = 0.0;
        for (Index k = 0; k < d; ++k) {
            const double t = x[i + k * n] - y[j + k * m];
            s += t * t;
        }
        return cost_div == 1.0 ? s : s / cost_div;
    }
};

static int g_threads = 1;

// Static contiguous split of [0, count) over g_threads std::threads (the
// "output-parallel" restatement; libgomp is not usable in this image).
template <typename F>
static void par_for(Index count, F&& body) {
    const int t = std::max(1, std::min<int>(g_threads, static_cast<int>(count)));
    if (t == 1) {
        for (Index i = 0; i < count; ++i) body(i);
        return;
    }
    std::vector<std::thread> pool;
    const Index chunk = (count + t - 1) / t;
    for (int w = 0; w < t; ++w) {
        const Index lo = w * chunk, hi = std::min(count, lo + chunk);
        if (lo >= hi) break;
        pool.emplace_back([lo, hi, &body] {
            for (Index i = lo; i < hi; ++i) body(i);
        });
    }
    for (auto& th : pool) th.join();
}

// DiscreteMeasure (types.cpp:7-24): validate and cache scalar std::log.
static void make_measure(const double* w, Index len, Vec& out, Vec& lout) {
    if (len == 0) throw std::invalid_argument("DiscreteMeasure: empty weight vector");
    out.assign(w, w + len);
    double total = 0.0;
    for (Index i = 0; i < len; ++i) {
        if (!std::isfinite(w[i]) || w[i] <= 0.0)
            throw std::invalid_argument(
                "DiscreteMeasure: weights must be strictly positive and finite");
        total += w[i];
    }
    if (std::abs(total - 1.0) > 1e-12)
        throw std::invalid_argument("DiscreteMeasure: weights must sum to 1");
    lout.resize(len);
    for (Index i = 0; i < len; ++i) lout[i] = std::log(out[i]);
}

static double dot(const Vec& a, const Vec& b) {
    double s = 0.0;
    for (size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
    return s;
}

static void check_finite(const double* v, Index len, const char* what) {
    for (Index i = 0; i < len; ++i)
        if (!std::isfinite(v[i]))
            throw std::invalid_argument(std::string(what) + ": entries must be finite");
}

// ---------------------------------------------------------------- core.cpp
// log_sum_exp (core.cpp:9-22)
double log_sum_exp(const double* values, const double* lw, Index len) {
    if (len == 0) throw std::invalid_argument("log_sum_exp: empty reduction");
    double shift = -std::numeric_limits<double>::infinity();
    for (Index i = 0; i < len; ++i) shift = std::max(shift, values[i] + lw[i]);
    double total = 0.0;
    for (Index i = 0; i < len; ++i) total += std::exp(values[i] + lw[i] - shift);
    return shift + std::log(total);
}

// ctransform_of_f = column LSE (core.cpp:35-54)
Vec ctransform_of_f(const Problem& p, const Vec& f) {
    check_finite(f.data(), p.n, "ctransform_of_f");
    const double inv_eps = 1.0 / p.eps;
    const Index n = p.n, m = p.m;
    Vec g(m);
    par_for(m, [&](Index j) {
        double shift = -std::numeric_limits<double>::infinity();
        for (Index i = 0; i < n; ++i)
            shift = std::max(shift, p.la[i] + (f[i] - p.C(i, j)) * inv_eps);
        double total = 0.0;
        for (Index i = 0; i < n; ++i)
            total += std::exp(p.la[i] + (f[i] - p.C(i, j)) * inv_eps - shift);
        g[j] = -p.eps * (shift + std::log(total));
    });
    return g;
}

// ctransform_of_g = row LSE (core.cpp:56-82). The reference runs two j-outer
// sweeps with per-row accumulators; each row's max and sum are taken in
// increasing j, which is what the row-parallel loop below does.
Vec ctransform_of_g(const Problem& p, const Vec& g) {
    check_finite(g.data(), p.m, "ctransform_of_g");
    const double inv_eps = 1.0 / p.eps;
    const Index n = p.n, m = p.m;
    Vec base(m);
    for (Index j = 0; j < m; ++j) base[j] = p.lb[j] + g[j] * inv_eps;
    Vec f(n);
    par_for(n, [&](Index i) {
        double shift = -std::numeric_limits<double>::infinity();
        for (Index j = 0; j < m; ++j) shift = std::max(shift, base[j] - p.C(i, j) * inv_eps);
        double total = 0.0;
        for (Index j = 0; j < m; ++j) total += std::exp(base[j] - p.C(i, j) * inv_eps - shift);
        f[i] = -p.eps * (shift + std::log(total));
    });
    return f;
}

// coupling_from (core.cpp:84-103)
Vec coupling_from(const Problem& p, const Vec& f, const Vec& g) {
    const double inv_eps = 1.0 / p.eps;
    Vec plan(static_cast<size_t>(p.n) * p.m);
    par_for(p.m, [&](Index j) {
        for (Index i = 0; i < p.n; ++i)
            plan[i + j * p.n] = p.a[i] * p.b[j] * std::exp((f[i] + g[j] - p.C(i, j)) * inv_eps);
    });
    return plan;
}

// plan_marginals (core.cpp:120-143): row sums accumulate in j order, column
// sums in i order.
void plan_marginals(const Problem& p, const Vec& f, const Vec& g, Vec& row, Vec& col) {
    const double inv_eps = 1.0 / p.eps;
    const Index n = p.n, m = p.m;
    row.assign(n, 0.0);
    col.assign(m, 0.0);
    par_for(m, [&](Index j) {
        double colsum = 0.0;
        for (Index i = 0; i < n; ++i)
            colsum += p.a[i] * p.b[j] * std::exp((f[i] + g[j] - p.C(i, j)) * inv_eps);
        col[j] = colsum;
    });
    par_for(n, [&](Index i) {
        double r = 0.0;
        for (Index j = 0; j < m; ++j)
            r += p.a[i] * p.b[j] * std::exp((f[i] + g[j] - p.C(i, j)) * inv_eps);
        row[i] = r;
    });
}

// marginal_gap (core.cpp:145-150)
void marginal_gap(const Problem& p, const Vec& row, const Vec& col, double& l2, double& inf) {
    double sr = 0.0, sc = 0.0, mr = 0.0, mc = 0.0;
    for (Index i = 0; i < p.n; ++i) {
        const double d = row[i] - p.a[i];
        sr += d * d;
        mr = std::max(mr, std::abs(d));
    }
    for (Index j = 0; j < p.m; ++j) {
        const double d = col[j] - p.b[j];
        sc += d * d;
        mc = std::max(mc, std::abs(d));
    }
    l2 = std::sqrt(sr) + std::sqrt(sc);
    inf = mr + mc;
}

// ---------------------------------------------------------------- objective.cpp
// semi_dual_value (objective.cpp:42-45)
double semi_dual_value(const Problem& p, const Vec& f, Vec* g_out = nullptr) {
    Vec g = ctransform_of_f(p, f);
    const double v = dot(p.a, f) + dot(p.b, g);
    if (g_out) *g_out = std::move(g);
    return v;
}

// restricted_derivatives_with_transform (objective.cpp:110-142) with the
// conditional chunks of for_each_conditional_chunk (objective.cpp:81-106):
// P~_ij = a_i exp((f_i + g_j - C_ij)/eps), chunks of 128 columns.
void restricted_derivatives(const Problem& p, const Vec& f, const Vec& g, const double* V,
                            Index ell, Vec& grad, Vec& hess) {
    const Index n = p.n, m = p.m;
    const double inv_eps = 1.0 / p.eps;
    constexpr Index kChunk = 128;
    // S = V^T P~ (ell x m), computed column by column.
    Vec S(static_cast<size_t>(ell) * m, 0.0);
    Vec Vr(static_cast<size_t>(n) * ell);  // row-major copy: contiguous per i (same arithmetic)
    for (Index c = 0; c < ell; ++c)
        for (Index i = 0; i < n; ++i) Vr[i * ell + c] = V[i + c * n];
    // Columns in blocks of kJB per task: each V row is read once per block instead of
    // once per column (the n x ell V streams from memory otherwise); every S[c, j] still
    // accumulates over i in ascending order, so the result is unchanged.
    constexpr Index kJB = 16;
    par_for((m + kJB - 1) / kJB, [&](Index jb) {
        const Index j0 = jb * kJB, jn = std::min(kJB, m - j0);
        std::vector<double> s(static_cast<size_t>(ell) * kJB, 0.0);
        for (Index i = 0; i < n; ++i) {
            const double* vr = &Vr[i * ell];
            for (Index q = 0; q < jn; ++q) {
                const Index j = j0 + q;
                const double w = p.a[i] * std::exp((f[i] + g[j] - p.C(i, j)) * inv_eps);
                double* sq = &s[q * ell];
                for (Index c = 0; c < ell; ++c) sq[c] += vr[c] * w;
            }
        }
        for (Index q = 0; q < jn; ++q)
            for (Index c = 0; c < ell; ++c) S[c + (j0 + q) * ell] = s[q * ell + c];
    });
    // row marginal r += chunk * b_seg, chunk by chunk (objective.cpp:127-128)
    Vec r(n, 0.0);
    par_for(n, [&](Index i) {
        double acc = 0.0;
        for (Index j0 = 0; j0 < m; j0 += kChunk) {
            const Index width = std::min(kChunk, m - j0);
            double t = 0.0;
            for (Index c = 0; c < width; ++c) {
                const Index j = j0 + c;
                t += p.a[i] * std::exp((f[i] + g[j] - p.C(i, j)) * inv_eps) * p.b[j];
            }
            acc += t;
        }
        r[i] = acc;
    });
    // cross += s diag(b_seg) s^T per chunk (objective.cpp:130-133)
    Vec cross(static_cast<size_t>(ell) * ell, 0.0);
    for (Index j0 = 0; j0 < m; j0 += kChunk) {
        const Index width = std::min(kChunk, m - j0);
        for (Index a = 0; a < ell; ++a)
            for (Index bb = 0; bb < ell; ++bb) {
                double t = 0.0;
                for (Index c = 0; c < width; ++c) {
                    const Index j = j0 + c;
                    t += S[a + j * ell] * p.b[j] * S[bb + j * ell];
                }
                cross[a + bb * ell] += t;
            }
    }
    // grad = V^T (alpha - r); hess = -(1/eps)(V^T diag(r) V - cross), symmetrised
    // (objective.cpp:137-140)
    grad.assign(ell, 0.0);
    for (Index c = 0; c < ell; ++c) {
        double t = 0.0;
        for (Index i = 0; i < n; ++i) t += V[i + c * n] * (p.a[i] - r[i]);
        grad[c] = t;
    }
    Vec h(static_cast<size_t>(ell) * ell);
    for (Index a = 0; a < ell; ++a)
        for (Index bb = 0; bb < ell; ++bb) {
            double t = 0.0;
            for (Index i = 0; i < n; ++i) t += V[i + a * n] * r[i] * V[i + bb * n];
            h[a + bb * ell] = (-1.0 / p.eps) * (t - cross[a + bb * ell]);
        }
    hess.resize(static_cast<size_t>(ell) * ell);
    for (Index a = 0; a < ell; ++a)
        for (Index bb = 0; bb < ell; ++bb)
            hess[a + bb * ell] = 0.5 * (h[a + bb * ell] + h[bb + a * ell]);
}

// ---------------------------------------------------------------- dense helpers
// Eigen LLT (llt_inplace::unblocked): fails iff a pivot x <= 0.
static bool cholesky(Vec& A, Index k) {
    for (Index c = 0; c < k; ++c) {
        double x = A[c + c * k];
        for (Index t = 0; t < c; ++t) x -= A[c + t * k] * A[c + t * k];
        if (!(x > 0.0)) return false;
        x = std::sqrt(x);
        A[c + c * k] = x;
        for (Index r = c + 1; r < k; ++r) {
            double v = A[r + c * k];
            for (Index t = 0; t < c; ++t) v -= A[r + t * k] * A[c + t * k];
            A[r + c * k] = v / x;
        }
    }
    return true;
}

static Vec chol_solve(const Vec& L, Index k, const Vec& rhs) {
    Vec y(rhs);
    for (Index r = 0; r < k; ++r) {
        double v = y[r];
        for (Index t = 0; t < r; ++t) v -= L[r + t * k] * y[t];
        y[r] = v / L[r + r * k];
    }
    for (Index r = k - 1; r >= 0; --r) {
        double v = y[r];
        for (Index t = r + 1; t < k; ++t) v -= L[t + r * k] * y[t];
        y[r] = v / L[r + r * k];
    }
    return y;
}

// Symmetric eigen-decomposition (stands in for Eigen::SelfAdjointEigenSolver,
// spectral.cpp:156): Householder tridiagonalisation followed by implicit QL
// with Wilkinson-type shifts (the classic tred2/tql2 pair), ascending
// eigenvalues, orthonormal eigenvectors in columns. O(k^3) for the k x k
// Rayleigh-Ritz matrix.
bool symeig_tql(const double* Ain, int k, double* evals, double* evecs) {
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

void sym_eig(const double* A, Index k, double* evals, double* evecs) {
    if (!symeig_tql(A, static_cast<int>(k), evals, evecs))
        throw std::runtime_error("top_modes: dense Ritz solve failed");
}

// Householder QR with Eigen's reflector convention (makeHouseholder: beta =
// -sign(c0) * norm, tau = (beta - c0)/beta), returning the thin Q
// (householderQ() * Identity(n, k)), spectral.cpp:116-117.
static void householder_thin_q(Vec& X, Index n, Index k) {
    Vec taus(k, 0.0);
    for (Index c = 0; c < k && c < n; ++c) {
        double* col = &X[c * n];
        double tail = 0.0;
        for (Index r = c + 1; r < n; ++r) tail += col[r] * col[r];
        const double c0 = col[c];
        double tau, beta;
        if (tail <= std::numeric_limits<double>::min()) {
            tau = 0.0;
            beta = c0;
            for (Index r = c + 1; r < n; ++r) col[r] = 0.0;
        } else {
            beta = std::sqrt(c0 * c0 + tail);
            if (c0 >= 0.0) beta = -beta;
            const double denom = c0 - beta;
            for (Index r = c + 1; r < n; ++r) col[r] /= denom;
            tau = (beta - c0) / beta;
        }
        col[c] = beta;
        taus[c] = tau;
        if (tau != 0.0)
            for (Index c2 = c + 1; c2 < k; ++c2) {
                double* o = &X[c2 * n];
                double w = o[c];
                for (Index r = c + 1; r < n; ++r) w += col[r] * o[r];
                o[c] -= tau * w;
                for (Index r = c + 1; r < n; ++r) o[r] -= tau * w * col[r];
            }
    }
    Vec Q(static_cast<size_t>(n) * k, 0.0);
    for (Index c = 0; c < k; ++c) Q[c + c * n] = 1.0;
    for (Index c = std::min(k, n) - 1; c >= 0; --c) {
        const double tau = taus[c];
        if (tau == 0.0) continue;
        const double* v = &X[c * n];
        for (Index c2 = 0; c2 < k; ++c2) {
            double* o = &Q[c2 * n];
            double w = o[c];
            for (Index r = c + 1; r < n; ++r) w += v[r] * o[r];
            o[c] -= tau * w;
            for (Index r = c + 1; r < n; ++r) o[r] -= tau * w * v[r];
        }
    }
    X.swap(Q);
}

// orthonormalize_deflated (spectral.cpp:113-121)
static void orthonormalize_deflated(Vec& X, Index n, Index k, const Vec& u0) {
    for (int round = 0; round < 3; ++round) {
        for (Index c = 0; c < k; ++c) {
            double t = 0.0;
            for (Index i = 0; i < n; ++i) t += u0[i] * X[i + c * n];
            for (Index i = 0; i < n; ++i) X[i + c * n] -= u0[i] * t;
        }
        householder_thin_q(X, n, k);
        double worst = 0.0;
        for (Index c = 0; c < k; ++c) {
            double t = 0.0;
            for (Index i = 0; i < n; ++i) t += u0[i] * X[i + c * n];
            worst = std::max(worst, std::abs(t));
        }
        if (worst < 1e-13) break;
    }
}

// ---------------------------------------------------------------- spectral.cpp
// apply_sym_t_block (spectral.cpp:86-102): out(j,:) = sqrt(b_j) (w^T U), w_i =
// sqrt(a_i) exp((f_i + g_j - C_ij)/eps).
Vec apply_sym_t_block(const Problem& p, const Vec& f, const Vec& g, const Vec& U, Index k) {
    const double inv_eps = 1.0 / p.eps;
    const Index n = p.n, m = p.m;
    Vec sa(n), out(static_cast<size_t>(m) * k);
    for (Index i = 0; i < n; ++i) sa[i] = std::sqrt(p.a[i]);
    Vec Ur(static_cast<size_t>(n) * k);  // row-major copy: contiguous per i (same arithmetic)
    for (Index c = 0; c < k; ++c)
        for (Index i = 0; i < n; ++i) Ur[i * k + c] = U[i + c * n];
    par_for(m, [&](Index j) {
        std::vector<double> acc(k, 0.0);
        const double sb = std::sqrt(p.b[j]);
        for (Index i = 0; i < n; ++i) {
            const double w = sa[i] * std::exp((f[i] + g[j] - p.C(i, j)) * inv_eps);
            const double* ur = &Ur[i * k];
            for (Index c = 0; c < k; ++c) acc[c] += w * ur[c];
        }
        for (Index c = 0; c < k; ++c) out[j + c * m] = sb * acc[c];
    });
    return out;
}

// apply_sym_block (spectral.cpp:68-84): out += w (sqrt(b_j) V.row(j)) over j.
Vec apply_sym_block(const Problem& p, const Vec& f, const Vec& g, const Vec& V, Index k) {
    const double inv_eps = 1.0 / p.eps;
    const Index n = p.n, m = p.m;
    Vec sa(n), sb(m), out(static_cast<size_t>(n) * k);
    for (Index i = 0; i < n; ++i) sa[i] = std::sqrt(p.a[i]);
    for (Index j = 0; j < m; ++j) sb[j] = std::sqrt(p.b[j]);
    Vec Vr(static_cast<size_t>(m) * k);  // row-major copy: contiguous per j (same arithmetic)
    for (Index c = 0; c < k; ++c)
        for (Index j = 0; j < m; ++j) Vr[j * k + c] = V[j + c * m];
    par_for(n, [&](Index i) {
        std::vector<double> acc(k, 0.0);
        for (Index j = 0; j < m; ++j) {
            const double w = sa[i] * std::exp((f[i] + g[j] - p.C(i, j)) * inv_eps);
            const double* vr = &Vr[j * k];
            for (Index c = 0; c < k; ++c) acc[c] += w * (sb[j] * vr[c]);
        }
        for (Index c = 0; c < k; ++c) out[i + c * n] = acc[c];
    });
    return out;
}

// apply_R / apply_Rt (spectral.cpp:29-62)
Vec apply_R(const Problem& p, const Vec& f, const Vec& g, const Vec& g1) {
    const double inv_eps = 1.0 / p.eps;
    Vec out(p.n);
    par_for(p.n, [&](Index i) {
        double acc = 0.0;
        for (Index j = 0; j < p.m; ++j)
            acc += std::exp((f[i] + g[j] - p.C(i, j)) * inv_eps) * (p.b[j] * g1[j]);
        out[i] = acc;
    });
    return out;
}

Vec apply_Rt(const Problem& p, const Vec& f, const Vec& g, const Vec& f1) {
    const double inv_eps = 1.0 / p.eps;
    Vec out(p.m);
    par_for(p.m, [&](Index j) {
        double acc = 0.0;
        for (Index i = 0; i < p.n; ++i)
            acc += std::exp((f[i] + g[j] - p.C(i, j)) * inv_eps) * p.a[i] * f1[i];
        out[j] = acc;
    });
    return out;
}

// SplitMix64 (harness/rng.hpp:13-50)
struct SplitMix64 {
    uint64_t s;
    bool have_spare = false;
    double spare = 0.0;
    explicit SplitMix64(uint64_t seed) : s(seed) {}
    uint64_t next_u64() {
        uint64_t z = (s += 0x9E3779B97F4A7C15ull);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    }
    double uniform01() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
    double uniform(double lo, double hi) { return lo + (hi - lo) * uniform01(); }
    double normal() {
        if (have_spare) {
            have_spare = false;
            return spare;
        }
        double u, v, q;
        do {
            u = uniform(-1.0, 1.0);
            v = uniform(-1.0, 1.0);
            q = u * u + v * v;
        } while (q >= 1.0 || q == 0.0);
        const double scale = std::sqrt(-2.0 * std::log(q) / q);
        spare = v * scale;
        have_spare = true;
        return u * scale;
    }
};

struct TopModesResult {
    Vec vectors, vectors_sym, rhos;
    double best_residual = 0.0;
    long sweeps = 0;
    bool ok = false;
};

// top_modes (spectral.cpp:125-193)
TopModesResult top_modes(const Problem& p, const Vec& f, const Vec& g, Index ell, double tol,
                         Index max_power_iters) {
    const Index n = p.n;
    if (ell < 1) throw std::invalid_argument("top_modes: ell must be >= 1");
    if (ell >= n) throw std::invalid_argument("top_modes: ell must be < n");
    if (max_power_iters < 0) max_power_iters = 500 * ell;
    Vec sqrt_alpha(n);
    for (Index i = 0; i < n; ++i) sqrt_alpha[i] = std::sqrt(p.a[i]);
    const Index block = std::min<Index>(ell + 5, n - 1);

    SplitMix64 rng(0x73706563u);
    Vec x(static_cast<size_t>(n) * block);
    for (Index c = 0; c < block; ++c)
        for (Index i = 0; i < n; ++i) x[i + c * n] = rng.uniform(-1.0, 1.0);
    orthonormalize_deflated(x, n, block, sqrt_alpha);

    TopModesResult res;
    Vec ritz_vectors, ritz_values;
    double best = std::numeric_limits<double>::infinity();
    Vec evals(block), evecs(static_cast<size_t>(block) * block), t(static_cast<size_t>(block) * block);
    for (Index sweep = 0; sweep < max_power_iters; ++sweep) {
        res.sweeps = sweep + 1;
        Vec z = apply_sym_t_block(p, f, g, x, block);
        Vec y = apply_sym_block(p, f, g, z, block);
        for (Index c = 0; c < block; ++c) {
            double s = 0.0;
            for (Index i = 0; i < n; ++i) s += sqrt_alpha[i] * y[i + c * n];
            for (Index i = 0; i < n; ++i) y[i + c * n] -= sqrt_alpha[i] * s;
        }
        for (Index a = 0; a < block; ++a)
            for (Index b = 0; b < block; ++b) {
                double s = 0.0;
                for (Index i = 0; i < n; ++i) s += x[i + a * n] * y[i + b * n];
                t[a + b * block] = s;
            }
        Vec ts(t.size());
        for (Index a = 0; a < block; ++a)
            for (Index b = 0; b < block; ++b)
                ts[a + b * block] = 0.5 * (t[a + b * block] + t[b + a * block]);
        sym_eig(ts.data(), block, evals.data(), evecs.data());
        Vec w(static_cast<size_t>(block) * ell), theta(ell);
        for (Index a = 0; a < ell; ++a) {
            for (Index r = 0; r < block; ++r) w[r + a * block] = evecs[r + (block - 1 - a) * block];
            theta[a] = evals[block - 1 - a];
        }
        Vec xw(static_cast<size_t>(n) * ell, 0.0), yw(static_cast<size_t>(n) * ell, 0.0);
        for (Index a = 0; a < ell; ++a)
            for (Index r = 0; r < block; ++r) {
                const double wr = w[r + a * block];
                for (Index i = 0; i < n; ++i) {
                    xw[i + a * n] += x[i + r * n] * wr;
                    yw[i + a * n] += y[i + r * n] * wr;
                }
            }
        double max_res = 0.0;
        for (Index a = 0; a < ell; ++a) {
            double s = 0.0;
            for (Index i = 0; i < n; ++i) {
                const double d = yw[i + a * n] - theta[a] * xw[i + a * n];
                s += d * d;
            }
            max_res = std::max(max_res, std::sqrt(s));
        }
        best = std::min(best, max_res);
        if (max_res <= tol) {
            ritz_vectors = std::move(xw);
            ritz_values = std::move(theta);
            break;
        }
        x = std::move(y);
        orthonormalize_deflated(x, n, block, sqrt_alpha);
    }
    res.best_residual = best;
    if (ritz_vectors.empty()) return res;
    orthonormalize_deflated(ritz_vectors, n, ell, sqrt_alpha);
    res.vectors_sym = ritz_vectors;
    res.rhos.resize(ell);
    for (Index a = 0; a < ell; ++a) res.rhos[a] = std::sqrt(std::max(ritz_values[a], 0.0));
    res.vectors.resize(static_cast<size_t>(n) * ell);
    for (Index a = 0; a < ell; ++a)
        for (Index i = 0; i < n; ++i)
            res.vectors[i + a * n] = res.vectors_sym[i + a * n] / sqrt_alpha[i];
    res.ok = true;
    return res;
}

// ---------------------------------------------------------------- solver.cpp
struct Record {
    double marginal_error, marginal_error_inf, semi_dual_value;
    int newton_attempted, newton_accepted;
    double newton_gain, newton_step_max;  // diagnostics: Q(f') - Q(f) as tested, max_i |f'_i - f_i|
};

// diagnostics of the last try_newton (copied into the trace record)
static thread_local double g_last_gain = 0.0, g_last_step_max = 0.0;

struct SolveOut {
    Vec f, g;
    long iterations = 0;
    bool converged = false;
    std::vector<Record> trace;
};

// dual_value (objective.cpp:10-40): one global max shift over all cells, then
// one global sum, both j-outer / i-inner like the reference loops.
double dual_value(const Problem& p, const Vec& f, const Vec& g) {
    check_finite(f.data(), p.n, "dual_value");
    check_finite(g.data(), p.m, "dual_value");
    const double inv_eps = 1.0 / p.eps;
    // per-column partials in parallel, combined in column order (the reference's
    // running max is order independent; its running sum is j-major, i-minor)
    Vec colmax(p.m);
    par_for(p.m, [&](Index j) {
        const double base = p.lb[j] + g[j] * inv_eps;
        double s = -std::numeric_limits<double>::infinity();
        for (Index i = 0; i < p.n; ++i) s = std::max(s, p.la[i] + base + (f[i] - p.C(i, j)) * inv_eps);
        colmax[j] = s;
    });
    double shift = -std::numeric_limits<double>::infinity();
    for (Index j = 0; j < p.m; ++j) shift = std::max(shift, colmax[j]);
    double total = 0.0;
    for (Index j = 0; j < p.m; ++j) {
        const double base = p.lb[j] + g[j] * inv_eps;
        for (Index i = 0; i < p.n; ++i) total += std::exp(p.la[i] + base + (f[i] - p.C(i, j)) * inv_eps - shift);
    }
    const double log_mass = shift + std::log(total);
    return dot(p.a, f) + dot(p.b, g) - p.eps * std::expm1(log_mass);
}

// semi_dual_hessian_quadform (objective.cpp:53-77)
double semi_dual_hessian_quadform(const Problem& p, const Vec& f, const Vec& u) {
    if (static_cast<Index>(u.size()) != p.n)
        throw std::invalid_argument("semi_dual_hessian_quadform: length mismatch");
    const Vec g = ctransform_of_f(p, f);
    const double inv_eps = 1.0 / p.eps;
    Vec term(p.m);
    par_for(p.m, [&](Index j) {
        double m1 = 0.0, m2 = 0.0;
        for (Index i = 0; i < p.n; ++i) {
            const double w = p.a[i] * std::exp((f[i] + g[j] - p.C(i, j)) * inv_eps);
            m1 += w * u[i];
            m2 += w * u[i] * u[i];
        }
        term[j] = p.b[j] * (m2 - m1 * m1);
    });
    double acc = 0.0;
    for (Index j = 0; j < p.m; ++j) acc += term[j];
    return -acc * inv_eps;
}

// Accept test of try_newton. 0 (literal, the reference): Q(f') > Q(f) with both
// values evaluated in full (solver.cpp:46-47, objective.cpp:42-45). 1 (stable): the
// same predicate as Q(f') - Q(f) > 0, with the difference evaluated directly so its
// rounding scales with the step, not with |Q|:
//   d = f' - f,  P~_ij = a_i exp((f_i + h_j - C_ij)/eps)   (h = f^{C,eps}, the anchor)
//   h'_j - h_j = -eps log(u_j / s_j) = -eps log1p(t_j / s_j),
//   s_j = sum_i P~_ij,  t_j = sum_i P~_ij expm1(d_i/eps),  u_j = sum_i P~_ij exp(d_i/eps)
//   dQ = a.d + b.(h' - h)
// log1p(t/s) when |t/s| <= 1/2 (u - s would cancel for small steps), log(u/s) otherwise
// (1 + t/s cancels when the step moves a column's mass away: t/s -> -1).
// (exact algebra: sum_i a_i e^{(f'_i - C_ij)/eps} = e^{-h_j/eps} (s_j + t_j)). Steps with
// max|d|/eps > kStableSpan fall back to the literal test (expm1 would overflow; such
// steps are never rounding-decided).
static int g_accept_mode = 0;
constexpr double kStableSpan = 600.0;
constexpr double kDhSwitch = 0.5;

static bool stable_delta_q(const Problem& p, const Vec& f, const Vec& h, const Vec& cand, double& dq) {
    const Index n = p.n, m = p.m;
    const double inv_eps = 1.0 / p.eps;
    Vec dv(n), ev(n), xv(n);
    double dmax = 0.0;
    for (Index i = 0; i < n; ++i) {
        dv[i] = cand[i] - f[i];
        dmax = std::max(dmax, std::abs(dv[i]));
        ev[i] = std::expm1(dv[i] * inv_eps);
        xv[i] = std::exp(dv[i] * inv_eps);
    }
    if (!(dmax <= kStableSpan * p.eps)) return false;  // as the GPU (lit_dmax = 600 eps)
    Vec dh(m);
    par_for(m, [&](Index j) {
        double s = 0.0, t = 0.0, u = 0.0;
        for (Index i = 0; i < n; ++i) {
            const double w = p.a[i] * std::exp((f[i] + h[j] - p.C(i, j)) * inv_eps);
            s += w;
            t += w * ev[i];
            u += w * xv[i];
        }
        const double ts = t / s;
        dh[j] = -p.eps * (std::abs(ts) <= kDhSwitch ? std::log1p(ts) : std::log(u / s));
    });
    dq = dot(p.a, dv) + dot(p.b, dh);
    return true;
}

// try_newton (solver.cpp:30-56)
static bool try_newton(const Problem& p, Vec& f, const Vec& h, double value_at_f,
                       const double* V, Index ell, double& value_out, Vec* g_cand) {
    Vec grad, hess;
    restricted_derivatives(p, f, h, V, ell, grad, hess);
    Vec L(hess.size());
    for (size_t t = 0; t < hess.size(); ++t) L[t] = -hess[t];
    if (!cholesky(L, ell)) {
        value_out = value_at_f;
        return false;
    }
    const Vec delta = chol_solve(L, ell, grad);
    Vec cand(f);
    for (Index i = 0; i < p.n; ++i) {
        double s = 0.0;
        for (Index c = 0; c < ell; ++c) s += V[i + c * p.n] * delta[c];
        cand[i] = f[i] + s;
    }
    double dq = 0.0;
    g_last_step_max = 0.0;
    for (Index i = 0; i < p.n; ++i) g_last_step_max = std::max(g_last_step_max, std::abs(cand[i] - f[i]));
    if (g_accept_mode == 1 && !g_cand && stable_delta_q(p, f, h, cand, dq)) {
        g_last_gain = dq;
        if (dq > 0.0) {
            f = std::move(cand);
            value_out = value_at_f + dq;
            return true;
        }
        value_out = value_at_f;
        return false;
    }
    const double cv = semi_dual_value(p, cand, g_cand);
    g_last_gain = cv - value_at_f;
    if (cv > value_at_f) {
        f = std::move(cand);
        value_out = cv;
        return true;
    }
    value_out = value_at_f;
    return false;
}

// solve (solver.cpp:71-156); the final coupling_from (:154) is left to the
// caller (oracle_coupling) because it is n x m.
SolveOut solve(const Problem& p, double tol, long max_iter, Index ell, const double* V,
               const double* init_f, const double* init_g, bool trace_enabled) {
    if (!(tol > 0.0)) throw std::invalid_argument("solve: tol_omega must be positive");
    if (max_iter < 1) throw std::invalid_argument("solve: max_iter must be >= 1");
    const bool use_newton = ell > 0;
    if (use_newton && V == nullptr) throw std::invalid_argument("solve: ell > 0 requires a basis");
    SolveOut out;
    if (init_f) {
        out.f.assign(init_f, init_f + p.n);
        out.g.assign(init_g, init_g + p.m);
    } else {
        out.f.assign(p.n, 0.0);
        out.g.assign(p.m, 0.0);
    }
    for (long k = 1; k <= max_iter; ++k) {
        out.g = ctransform_of_f(p, out.f);           // sk_sweep (solver.cpp:12-17)
        out.f = ctransform_of_g(p, out.g);
        const double c = dot(p.a, out.f);            // gauge (solver.cpp:108-112)
        for (auto& v : out.f) v -= c;
        for (auto& v : out.g) v += c;
        Vec row, col;
        plan_marginals(p, out.f, out.g, row, col);
        Record rec{};
        marginal_gap(p, row, col, rec.marginal_error, rec.marginal_error_inf);
        out.iterations = k;
        if (rec.marginal_error < tol) {
            if (trace_enabled) {
                rec.semi_dual_value = semi_dual_value(p, out.f);
                out.trace.push_back(rec);
            }
            out.converged = true;
            break;
        }
        if (use_newton) {
            const Vec h = ctransform_of_f(p, out.f);
            const double value_sweep = dot(p.a, out.f) + dot(p.b, h);
            rec.newton_attempted = 1;
            double value;
            g_last_gain = g_last_step_max = 0.0;
            rec.newton_accepted = try_newton(p, out.f, h, value_sweep, V, ell, value, nullptr);
            rec.newton_gain = g_last_gain;
            rec.newton_step_max = g_last_step_max;
            rec.semi_dual_value = value;
        } else if (trace_enabled) {
            rec.semi_dual_value = semi_dual_value(p, out.f);
        }
        if (trace_enabled) out.trace.push_back(rec);
    }
    return out;
}

}  // namespace oracle

// ============================================================================
// C ABI for the Python test harness (ctypes). Status: 0 ok, 1 invalid argument,
// 2 eigensolver failure, 9 other error. Message via oracle_last_error().
// ============================================================================
using namespace oracle;

extern "C" {

typedef struct {
    int kind;
    const double* cost;
    const double* x;
    const double* y;
    long n, m, d;
    double cost_div;
    const double* alpha;
    const double* beta;
    double eps;
} oracle_problem;

static thread_local std::string g_err;

const char* oracle_last_error(void) { return g_err.c_str(); }

void oracle_set_threads(int t) {
    g_threads = t > 0 ? t : static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
}

/* Accept test of try_newton: 0 literal Q(f') > Q(f) (the reference), 1 stable dQ > 0. */
void oracle_set_accept_mode(int mode) { g_accept_mode = mode == 1 ? 1 : 0; }

int oracle_max_threads(void) {
    return static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
}

static Problem build(const oracle_problem* q) {
    Problem p;
    p.kind = q->kind;
    p.cost = q->cost;
    p.x = q->x;
    p.y = q->y;
    p.n = q->n;
    p.m = q->m;
    p.d = q->d;
    p.cost_div = q->cost_div;
    p.eps = q->eps;
    if (q->n < 1 || q->m < 1) throw std::invalid_argument("CostMatrix: need at least a 1x1 matrix");
    if (q->kind == 0) check_finite(q->cost, q->n * q->m, "CostMatrix");
    make_measure(q->alpha, q->n, p.a, p.la);
    make_measure(q->beta, q->m, p.b, p.lb);
    if (!(q->eps > 0.0) || !std::isfinite(q->eps))
        throw std::invalid_argument("EotProblem: epsilon must be positive");
    return p;
}

#define ORACLE_TRY(...)                                    \
    try {                                                  \
        __VA_ARGS__;                                       \
        return 0;                                          \
    } catch (const std::invalid_argument& e) {             \
        g_err = e.what();                                  \
        return 1;                                          \
    } catch (const std::exception& e) {                    \
        g_err = e.what();                                  \
        return 9;                                          \
    }

int oracle_log_sum_exp(const double* v, const double* lw, long len, double* out) {
    ORACLE_TRY(*out = log_sum_exp(v, lw, len))
}

int oracle_ctransform_f(const oracle_problem* q, const double* f, double* g) {
    ORACLE_TRY({
        Problem p = build(q);
        Vec ff(f, f + p.n);
        Vec gg = ctransform_of_f(p, ff);
        std::memcpy(g, gg.data(), sizeof(double) * p.m);
    })
}

int oracle_ctransform_g(const oracle_problem* q, const double* g, double* f) {
    ORACLE_TRY({
        Problem p = build(q);
        Vec gg(g, g + p.m);
        Vec ff = ctransform_of_g(p, gg);
        std::memcpy(f, ff.data(), sizeof(double) * p.n);
    })
}

int oracle_plan_marginals(const oracle_problem* q, const double* f, const double* g,
                          double* row, double* col, double* l2, double* inf) {
    ORACLE_TRY({
        Problem p = build(q);
        Vec ff(f, f + p.n), gg(g, g + p.m), r, c;
        plan_marginals(p, ff, gg, r, c);
        std::memcpy(row, r.data(), sizeof(double) * p.n);
        std::memcpy(col, c.data(), sizeof(double) * p.m);
        marginal_gap(p, r, c, *l2, *inf);
    })
}

int oracle_coupling(const oracle_problem* q, const double* f, const double* g, double* plan) {
    ORACLE_TRY({
        Problem p = build(q);
        Vec ff(f, f + p.n), gg(g, g + p.m);
        Vec pl = coupling_from(p, ff, gg);
        std::memcpy(plan, pl.data(), sizeof(double) * pl.size());
    })
}

int oracle_semi_dual_value(const oracle_problem* q, const double* f, double* out) {
    ORACLE_TRY({
        Problem p = build(q);
        Vec ff(f, f + p.n);
        *out = semi_dual_value(p, ff);
    })
}

int oracle_restricted_derivatives(const oracle_problem* q, const double* f, const double* g,
                                  const double* V, long ell, double* grad, double* hess) {
    ORACLE_TRY({
        Problem p = build(q);
        Vec ff(f, f + p.n), gg(g, g + p.m), gr, he;
        restricted_derivatives(p, ff, gg, V, ell, gr, he);
        std::memcpy(grad, gr.data(), sizeof(double) * ell);
        std::memcpy(hess, he.data(), sizeof(double) * ell * ell);
    })
}

int oracle_dual_value(const oracle_problem* q, const double* f, const double* g, double* out) {
    ORACLE_TRY({
        Problem p = build(q);
        Vec ff(f, f + p.n), gg(g, g + p.m);
        *out = dual_value(p, ff, gg);
    })
}

int oracle_semi_dual_hessian_quadform(const oracle_problem* q, const double* f, const double* u, double* out) {
    ORACLE_TRY({
        Problem p = build(q);
        Vec ff(f, f + p.n), uu(u, u + p.n);
        *out = semi_dual_hessian_quadform(p, ff, uu);
    })
}

// newton_step (solver.cpp:59-69)
int oracle_newton_step(const oracle_problem* q, const double* f, const double* V, long ell, double* f_out,
                       int* accepted, int* factorization_failed) {
    ORACLE_TRY({
        Problem p = build(q);
        if (ell < 1) throw std::invalid_argument("newton_step: empty basis");
        Vec ff(f, f + p.n);
        const Vec g = ctransform_of_f(p, ff);
        const double value = dot(p.a, ff) + dot(p.b, g);
        // factorization failure leaves f unchanged and is reported separately
        Vec grad, hess;
        restricted_derivatives(p, ff, g, V, ell, grad, hess);
        Vec L(hess.size());
        for (size_t t2 = 0; t2 < hess.size(); ++t2) L[t2] = -hess[t2];
        *factorization_failed = cholesky(L, ell) ? 0 : 1;
        double vout = value;
        *accepted = 0;
        if (!*factorization_failed) *accepted = try_newton(p, ff, g, value, V, ell, vout, nullptr) ? 1 : 0;
        std::memcpy(f_out, ff.data(), sizeof(double) * p.n);
    })
}

int oracle_apply_sym_block(const oracle_problem* q, const double* f, const double* g,
                           const double* V, long k, double* out) {
    ORACLE_TRY({
        Problem p = build(q);
        Vec ff(f, f + p.n), gg(g, g + p.m), vv(V, V + p.m * k);
        Vec o = apply_sym_block(p, ff, gg, vv, k);
        std::memcpy(out, o.data(), sizeof(double) * o.size());
    })
}

int oracle_apply_sym_t_block(const oracle_problem* q, const double* f, const double* g,
                             const double* U, long k, double* out) {
    ORACLE_TRY({
        Problem p = build(q);
        Vec ff(f, f + p.n), gg(g, g + p.m), uu(U, U + p.n * k);
        Vec o = apply_sym_t_block(p, ff, gg, uu, k);
        std::memcpy(out, o.data(), sizeof(double) * o.size());
    })
}

int oracle_apply_R(const oracle_problem* q, const double* f, const double* g, const double* g1,
                   double* out) {
    ORACLE_TRY({
        Problem p = build(q);
        Vec ff(f, f + p.n), gg(g, g + p.m), v(g1, g1 + p.m);
        Vec o = apply_R(p, ff, gg, v);
        std::memcpy(out, o.data(), sizeof(double) * p.n);
    })
}

int oracle_apply_Rt(const oracle_problem* q, const double* f, const double* g, const double* f1,
                    double* out) {
    ORACLE_TRY({
        Problem p = build(q);
        Vec ff(f, f + p.n), gg(g, g + p.m), v(f1, f1 + p.n);
        Vec o = apply_Rt(p, ff, gg, v);
        std::memcpy(out, o.data(), sizeof(double) * p.m);
    })
}

int oracle_sym_eig(const double* A, long k, double* evals, double* evecs) {
    ORACLE_TRY(sym_eig(A, k, evals, evecs))
}

// top_modes: status 2 when the residual target is not met (EigensolverError).
int oracle_top_modes(const oracle_problem* q, const double* f, const double* g, long ell,
                     double tol, long max_power_iters, double* vectors, double* vectors_sym,
                     double* rhos, double* best_residual, long* sweeps) {
    try {
        Problem p = build(q);
        Vec ff(f, f + p.n), gg(g, g + p.m);
        TopModesResult r = top_modes(p, ff, gg, ell, tol, max_power_iters);
        *best_residual = r.best_residual;
        *sweeps = r.sweeps;
        if (!r.ok) {
            g_err = "top_modes: no convergence within max_power_iters, best residual " +
                    std::to_string(r.best_residual);
            return 2;
        }
        std::memcpy(vectors, r.vectors.data(), sizeof(double) * p.n * ell);
        std::memcpy(vectors_sym, r.vectors_sym.data(), sizeof(double) * p.n * ell);
        std::memcpy(rhos, r.rhos.data(), sizeof(double) * ell);
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 9;
    }
}

typedef struct {
    double marginal_error;
    double marginal_error_inf;
    double semi_dual_value;
    int newton_attempted;
    int newton_accepted;
    double newton_gain;     /* Q(f') - Q(f) as the accept test evaluated it (0 if no candidate) */
    double newton_step_max; /* max_i |f'_i - f_i| of the candidate */
} oracle_record;

int oracle_solve(const oracle_problem* q, double tol, long max_iter, long ell, const double* V,
                 const double* init_f, const double* init_g, int trace_enabled, double* f_out,
                 double* g_out, long* iterations, int* converged, oracle_record* trace,
                 long trace_cap, long* trace_len) {
    ORACLE_TRY({
        Problem p = build(q);
        SolveOut o = solve(p, tol, max_iter, ell, V, init_f, init_g, trace_enabled != 0);
        std::memcpy(f_out, o.f.data(), sizeof(double) * p.n);
        std::memcpy(g_out, o.g.data(), sizeof(double) * p.m);
        *iterations = o.iterations;
        *converged = o.converged ? 1 : 0;
        long len = static_cast<long>(o.trace.size());
        *trace_len = len;
        for (long t = 0; t < len && t < trace_cap; ++t) {
            trace[t].marginal_error = o.trace[t].marginal_error;
            trace[t].marginal_error_inf = o.trace[t].marginal_error_inf;
            trace[t].semi_dual_value = o.trace[t].semi_dual_value;
            trace[t].newton_attempted = o.trace[t].newton_attempted;
            trace[t].newton_accepted = o.trace[t].newton_accepted;
            trace[t].newton_gain = o.trace[t].newton_gain;
            trace[t].newton_step_max = o.trace[t].newton_step_max;
        }
    })
}

// SplitMix64 draws for cross-checking the product's input generators.
void oracle_splitmix_uniform01(uint64_t seed, long count, double* out) {
    SplitMix64 r(seed);
    for (long t = 0; t < count; ++t) out[t] = r.uniform01();
}

void oracle_splitmix_normal(uint64_t seed, long count, double* out) {
    SplitMix64 r(seed);
    for (long t = 0; t < count; ++t) out[t] = r.normal();
}

}  // extern "C"
