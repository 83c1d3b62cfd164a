// engine_capi.cuh -- the extern "C" boundary declared in include/sknr_gpu.h
// Part of the libsknr_b200 translation unit: included once, in order, by engine.cu
// (shares its types, static helpers and kernels; not a standalone header).
#pragma once

// ============================================================ C ABI
using namespace sknr;

struct sknr_problem_s {
    std::unique_ptr<Problem> p;
};

static thread_local std::string g_err;
static thread_local double g_best_residual = 0.0;

#define SKNR_API_BEGIN try {
#define SKNR_API_END                        \
    return SKNR_OK;                         \
    }                                       \
    catch (const InvalidArgument& e) {      \
        g_err = e.what();                   \
        return SKNR_EINVAL;                 \
    }                                       \
    catch (const EigenFailure& e) {         \
        g_err = e.what();                   \
        g_best_residual = e.best;           \
        return SKNR_EEIGEN;                 \
    }                                       \
    catch (const CudaFailure& e) {          \
        g_err = e.what();                   \
        return SKNR_ECUDA;                  \
    }                                       \
    catch (const RuntimeFailure& e) {       \
        g_err = e.what();                   \
        return SKNR_ERUNTIME;               \
    }                                       \
    catch (const NcclFailure& e) {          \
        g_err = e.what();                   \
        return SKNR_ENCCL;                  \
    }                                       \
    catch (const std::exception& e) {       \
        g_err = e.what();                   \
        return SKNR_EINTERNAL;              \
    }

static Problem& get(sknr_problem h) {
    if (!h || !h->p) throw InvalidArgument("sknr: null problem handle");
    own_stream(h->p->stream);  // this call's buffers free stream-ordered on the problem's stream
    return *h->p;
}

static void check_finite_vec(const double* v, int64_t len, const char* what) {
    if (!v) throw InvalidArgument(std::string(what) + ": null pointer");
    for (int64_t i = 0; i < len; ++i)
        if (!std::isfinite(v[i])) throw InvalidArgument(std::string(what) + ": entries must be finite");
}

extern "C" {

const char* sknr_last_error(void) { return g_err.c_str(); }
double sknr_last_best_residual(void) { return g_best_residual; }
int64_t sknr_kernel_launch_count(void) { return launch_count(); }

int sknr_version(char* buf, int cap) {
    SKNR_API_BEGIN
    std::string v = "sknr_b200 0.1.0 sm_100a";
    int dev = 0, count = 0;
    if (cudaGetDeviceCount(&count) == cudaSuccess && count > 0) {
        cudaDeviceProp prop;
        cudaGetDevice(&dev);
        if (cudaGetDeviceProperties(&prop, dev) == cudaSuccess)
            v += std::string(" (") + prop.name + ", " + std::to_string(prop.multiProcessorCount) + " SMs)";
    } else {
        v += " (no CUDA device)";
    }
    if (buf && cap > 0) {
        std::strncpy(buf, v.c_str(), cap - 1);
        buf[cap - 1] = 0;
    }
    SKNR_API_END
}

void sknr_config_default(sknr_config* c) {
    c->tol_omega = 1e-9;
    c->max_iter = 100000;
    c->ell = 0;
    c->newton_enabled = 1;
    c->trace_enabled = 1;
    c->exact_marginals = 0;
    c->accept_test = 0;
}

int sknr_problem_create_dense(const double* cost, int64_t n, int64_t m, const double* alpha,
                              const double* beta, double epsilon, sknr_problem* out) {
    SKNR_API_BEGIN
    *out = nullptr;
    std::unique_ptr<Problem> p(new_problem(n, m, alpha, beta, epsilon));
    finish_dense(p.get(), cost);
    *out = new sknr_problem_s{std::move(p)};
    SKNR_API_END
}

int sknr_problem_create_points_ex(const double* x, const double* y, int64_t n, int64_t m, int64_t d,
                                  double cost_scale, const double* alpha, const double* beta, double epsilon,
                                  int cost_mode, sknr_problem* out);

int sknr_problem_create_points(const double* x, const double* y, int64_t n, int64_t m, int64_t d,
                               double cost_scale, const double* alpha, const double* beta, double epsilon,
                               sknr_problem* out) {
    return sknr_problem_create_points_ex(x, y, n, m, d, cost_scale, alpha, beta, epsilon, 0, out);
}

int sknr_problem_create_points_ex(const double* x, const double* y, int64_t n, int64_t m, int64_t d,
                                  double cost_scale, const double* alpha, const double* beta, double epsilon,
                                  int cost_mode, sknr_problem* out) {
    SKNR_API_BEGIN
    if (cost_mode < 0 || cost_mode > 2) throw InvalidArgument("sknr_problem_create_points: cost_mode must be 0, 1 or 2");
    *out = nullptr;
    if (d < 1) throw InvalidArgument("sq_euclidean_cost: dimension must be >= 1");
    check_finite_vec(x, n * d, "PointCloud(x)");
    check_finite_vec(y, m * d, "PointCloud(y)");
    if (!(cost_scale > 0.0) || !std::isfinite(cost_scale))
        throw InvalidArgument("sq_euclidean_cost: cost_scale must be positive");
    std::unique_ptr<Problem> p(new_problem(n, m, alpha, beta, epsilon));
    finish_points(p.get(), x, y, d, cost_scale, cost_mode);
    *out = new sknr_problem_s{std::move(p)};
    SKNR_API_END
}

int sknr_problem_set_epsilon(sknr_problem h, double epsilon) {
    SKNR_API_BEGIN
    Problem& P = get(h);
    if (!(epsilon > 0.0) || !std::isfinite(epsilon)) throw InvalidArgument("EotProblem: epsilon must be positive");
    P.eps = epsilon;
    count_launch();
    k_invalidate_refs<<<1, 32, 0, P.stream>>>(P.st);
    CK(cudaStreamSynchronize(P.stream));
    SKNR_API_END
}

int sknr_problem_info(sknr_problem h, int64_t* n, int64_t* m, int64_t* d, double* epsilon, int* kind) {
    SKNR_API_BEGIN
    Problem& P = get(h);
    // kind: 0 stored cost (given or materialised), 1 on the fly (registers), 2 on the fly (DMMA contraction)
    if (n) *n = P.n;
    if (m) *m = P.m;
    if (d) *d = P.d;
    if (epsilon) *epsilon = P.eps;
    if (kind) *kind = P.dim > 0 ? 1 : (P.dim < 0 ? 2 : 0);
    SKNR_API_END
}

// Morton order of a point set (centred coordinates, col-major count x d) in the
// bounding box of both clouds; ties keep index order.
static std::vector<int> morton_perm(const std::vector<double>& c, int64_t count, int d, const double* lo,
                                    const double* hi) {
    const int bits = std::min(21, 63 / d);
    const double scale = static_cast<double>((1ull << bits) - 1);
    std::vector<std::pair<uint64_t, int>> key(static_cast<size_t>(count));
    for (int64_t i = 0; i < count; ++i) {
        uint64_t q[4] = {0, 0, 0, 0};
        for (int k = 0; k < d; ++k) {
            const double span = hi[k] > lo[k] ? hi[k] - lo[k] : 1.0;
            double v = (c[i + k * count] - lo[k]) / span * scale;
            v = std::min(std::max(v, 0.0), scale);
            q[k] = static_cast<uint64_t>(v);
        }
        uint64_t code = 0;
        for (int b = bits - 1; b >= 0; --b)
            for (int k = 0; k < d; ++k) code = (code << 1) | ((q[k] >> b) & 1ull);
        key[static_cast<size_t>(i)] = {code, static_cast<int>(i)};
    }
    std::sort(key.begin(), key.end());
    std::vector<int> perm(static_cast<size_t>(count));
    for (int64_t i = 0; i < count; ++i) perm[static_cast<size_t>(i)] = key[static_cast<size_t>(i)].second;
    return perm;
}

static void group_boxes(const std::vector<double>& c, int64_t count, int d, const std::vector<int>& perm, int g,
                        DBuf& out) {
    const int64_t ng = (count + g - 1) / g;
    std::vector<double> box(static_cast<size_t>(ng) * 2 * d);
    for (int64_t q = 0; q < ng; ++q)
        for (int k = 0; k < d; ++k) {
            double lo = std::numeric_limits<double>::infinity(), hi = -lo;
            for (int64_t p = q * g; p < std::min(count, (q + 1) * g); ++p) {
                const double v = c[perm[static_cast<size_t>(p)] + k * count];
                lo = std::min(lo, v);
                hi = std::max(hi, v);
            }
            box[q * 2 * d + k] = lo;
            box[q * 2 * d + d + k] = hi;
        }
    out.ensure(box.size());
    CK(cudaMemcpy(out.p, box.data(), box.size() * sizeof(double), cudaMemcpyHostToDevice));
}

static void prepare_culling(Problem& P) {
    if (P.cull_ready) return;
    const int d = static_cast<int>(P.d);
    std::vector<double> xc(static_cast<size_t>(P.n * d)), yc(static_cast<size_t>(P.m * d));
    CK(cudaMemcpy(xc.data(), P.src.coords.p, xc.size() * sizeof(double), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(yc.data(), P.tgt.coords.p, yc.size() * sizeof(double), cudaMemcpyDeviceToHost));
    double lo[4], hi[4];
    for (int k = 0; k < d; ++k) {
        lo[k] = std::numeric_limits<double>::infinity();
        hi[k] = -lo[k];
        for (int64_t i = 0; i < P.n; ++i) {
            lo[k] = std::min(lo[k], xc[i + k * P.n]);
            hi[k] = std::max(hi[k], xc[i + k * P.n]);
        }
        for (int64_t j = 0; j < P.m; ++j) {
            lo[k] = std::min(lo[k], yc[j + k * P.m]);
            hi[k] = std::max(hi[k], yc[j + k * P.m]);
        }
    }
    const std::vector<int> px = morton_perm(xc, P.n, d, lo, hi), py = morton_perm(yc, P.m, d, lo, hi);
    P.src.perm.assign(px);
    P.tgt.perm.assign(py);
    group_boxes(xc, P.n, d, px, 16, P.src.box16);
    group_boxes(yc, P.m, d, py, 16, P.tgt.box16);
    group_boxes(xc, P.n, d, px, 32, P.src.box32);
    group_boxes(yc, P.m, d, py, 32, P.tgt.box32);
    group_boxes(xc, P.n, d, px, 64, P.src.box64);
    group_boxes(xc, P.n, d, px, 128, P.src.box128);
    group_boxes(yc, P.m, d, py, 64, P.tgt.box64);
    group_boxes(yc, P.m, d, py, 128, P.tgt.box128);
    for (int dir = 0; dir < 2; ++dir) {
        const int64_t nin = dir == 0 ? P.n : P.m, nout = dir == 0 ? P.m : P.n;
        P.f_gi[dir].ensure((nin + CULL_GI - 1) / CULL_GI);
        P.s_go[dir].ensure((nout + CULL_GO - 1) / CULL_GO);
        P.f_g32[dir].ensure((nin + 31) / 32);
        P.s_g16[dir].ensure((nout + 15) / 16);
    }
    P.cull_ready = true;
}

int sknr_problem_set_culling(sknr_problem h, double threshold) {
    SKNR_API_BEGIN
    Problem& P = get(h);
    std::lock_guard<std::mutex> lk(P.mu);
    if (!(threshold >= 0.0) || !std::isfinite(threshold))
        throw InvalidArgument("set_culling: threshold must be finite and >= 0");
    if (threshold > 0.0) {
        if (threshold < 40.0) throw InvalidArgument("set_culling: threshold below 40 would perturb the sums");
        if (P.dim < 1 || P.dim > 4)
            throw InvalidArgument("set_culling: needs a point-cloud problem with d <= 4");
        prepare_culling(P);
    }
    P.cull_t = threshold;
    SKNR_API_END
}

int sknr_problem_set_precision(sknr_problem h, int bits) {
    SKNR_API_BEGIN
    Problem& P = get(h);
    std::lock_guard<std::mutex> lk(P.mu);
    if (bits != 32 && bits != 64) throw InvalidArgument("set_precision: bits must be 32 or 64");
    if (bits == 32 && (P.dim < 1 || P.dim > 4))
        throw InvalidArgument("set_precision: fp32 needs a point-cloud problem with d <= 4");
    P.precision = bits;
    SKNR_API_END
}

int sknr_problem_destroy(sknr_problem h) {
    SKNR_API_BEGIN
    delete h;
    SKNR_API_END
}

static void reset_for_primitive(Problem& P) {
    count_launch();
    k_invalidate_refs<<<1, 32, 0, P.stream>>>(P.st);
}

int sknr_ctransform_of_f(sknr_problem h, const double* f, double* g) {
    SKNR_API_BEGIN
    Problem& P = get(h);
    std::lock_guard<std::mutex> lk(P.mu);
    check_finite_vec(f, P.n_global, "ctransform_of_f");
    DBuf df, dg;
    df.ensure(P.n);
    dg.ensure(P.m);
    upload_rows(P, df.p, f);
    reset_for_primitive(P);
    plan_for(P, 0, MODE_SUM, 0);
    plan_for(P, 0, MODE_MAX, 0);
    lse(P, 0, df.p, dg.p, G_NONE);
    download(g, dg.p, P.m, P.stream);
    CK(cudaStreamSynchronize(P.stream));
    SKNR_API_END
}

int sknr_ctransform_of_g(sknr_problem h, const double* g, double* f) {
    SKNR_API_BEGIN
    Problem& P = get(h);
    std::lock_guard<std::mutex> lk(P.mu);
    check_finite_vec(g, P.m, "ctransform_of_g");
    DBuf df, dg;
    df.ensure(P.n);
    dg.ensure(P.m);
    upload(dg.p, g, P.m, P.stream);
    reset_for_primitive(P);
    lse(P, 1, dg.p, df.p, G_NONE);
    gather_rows(P, df.p, f);
    SKNR_API_END
}

int sknr_plan_marginals(sknr_problem h, const double* f, const double* g, double* row, double* col,
                        double* gap_l2, double* gap_inf) {
    SKNR_API_BEGIN
    Problem& P = get(h);
    std::lock_guard<std::mutex> lk(P.mu);
    check_finite_vec(f, P.n_global, "plan_marginals(f)");
    check_finite_vec(g, P.m, "plan_marginals(g)");
    DBuf df, dg, dr, dc;
    df.ensure(P.n);
    dg.ensure(P.m);
    dr.ensure(P.n);
    dc.ensure(P.m);
    upload_rows(P, df.p, f);
    upload(dg.p, g, P.m, P.stream);
    // row_i = sum_j a_i b_j e^{..}: dir 1 (out i), column sums: dir 0 (out j)
    PassSpec pr;
    pr.dir = 1;
    pr.in_v = dg.p;
    pr.in_lw = P.tgt.lw.p;
    pr.out_v = df.p;
    pr.out_lw = P.src.lw.p;
    pr.out = dr.p;
    plan_pass(P, pr);
    PassSpec pc;
    pc.dir = 0;
    pc.in_v = df.p;
    pc.in_lw = P.src.lw.p;
    pc.out_v = dg.p;
    pc.out_lw = P.tgt.lw.p;
    pc.out = dc.p;
    plan_pass(P, pc);
    std::vector<double> hr(P.n_global), hc(P.m);
    gather_rows(P, dr.p, hr.data());
    download(hc.data(), dc.p, P.m, P.stream);
    CK(cudaStreamSynchronize(P.stream));
    const std::vector<double>& ha = P.h_alpha;
    const std::vector<double>& hb = P.h_beta;
    double sr = 0, sc = 0, mr = 0, mc = 0;
    for (int64_t i = 0; i < P.n_global; ++i) {
        const double d = hr[i] - ha[i];
        sr += d * d;
        mr = std::max(mr, std::abs(d));
    }
    for (int64_t j = 0; j < P.m; ++j) {
        const double d = hc[j] - hb[j];
        sc += d * d;
        mc = std::max(mc, std::abs(d));
    }
    if (row) std::memcpy(row, hr.data(), sizeof(double) * P.n_global);
    if (col) std::memcpy(col, hc.data(), sizeof(double) * P.m);
    if (gap_l2) *gap_l2 = std::sqrt(sr) + std::sqrt(sc);
    if (gap_inf) *gap_inf = mr + mc;
    SKNR_API_END
}

int sknr_coupling_rows(sknr_problem h, const double* f, const double* g, int64_t row_begin, int64_t row_end,
                       double* plan_rows) {
    SKNR_API_BEGIN
    Problem& P = get(h);
    std::lock_guard<std::mutex> lk(P.mu);
    // row-sharded: global row indices inside this rank's block [P.row_begin, P.row_begin + n);
    // each rank materialises its own rows of the plan (the n x m output is never gathered)
    if (row_begin < P.row_begin || row_end > P.row_begin + P.n || row_begin > row_end)
        throw InvalidArgument(P.shard ? "coupling_rows: row range outside this rank's row block"
                                      : "coupling_rows: row range out of bounds");
    check_finite_vec(f, P.n_global, "coupling_from(f)");
    check_finite_vec(g, P.m, "coupling_from(g)");
    const int64_t rows = row_end - row_begin;
    if (rows == 0) return SKNR_OK;
    row_begin -= P.row_begin;  // local from here on
    row_end -= P.row_begin;
    // host-side block size bounded to 1 GiB of device scratch per launch
    const int64_t m = P.m;
    const int64_t cap_rows = std::max<int64_t>(1, (int64_t(1) << 27) / std::max<int64_t>(m, 1));
    DBuf df, dg, dp;
    df.ensure(P.n);
    dg.ensure(m);
    upload_rows(P, df.p, f);
    upload(dg.p, g, m, P.stream);
    const bool whole = rows <= cap_rows;
    dp.ensure((whole ? rows : cap_rows) * m);
    std::vector<double> tmp;
    for (int64_t r = row_begin; r < row_end; r += cap_rows) {
        const int64_t cnt = std::min(cap_rows, row_end - r);
        count_launch();
        k_coupling<<<grid_for(cnt * m), AUX_NT, 0, P.stream>>>(
            P.kind == 0 || P.C.p ? P.C.p : nullptr, P.src.coords.p, P.tgt.coords.p, P.n, m, r, cnt,
            static_cast<int>(P.d), P.kappa, P.src.w.p, P.tgt.w.p, df.p, dg.p, P.inv_eps(), dp.p);
        if (whole) {
            download(plan_rows, dp.p, cnt * m, P.stream);
        } else {  // scatter the cnt-row block into the rows-leading-dimension output
            tmp.resize(cnt * m);
            download(tmp.data(), dp.p, cnt * m, P.stream);
            CK(cudaStreamSynchronize(P.stream));
            for (int64_t j = 0; j < m; ++j)
                std::memcpy(plan_rows + (r - row_begin) + j * rows, tmp.data() + j * cnt, sizeof(double) * cnt);
        }
    }
    CK(cudaStreamSynchronize(P.stream));
    SKNR_API_END
}

int sknr_coupling(sknr_problem h, const double* f, const double* g, double* plan) {
    const int64_t b = h && h->p ? h->p->row_begin : 0;
    return sknr_coupling_rows(h, f, g, b, b + (h && h->p ? h->p->n : 0), plan);
}

// full_semi_dual_hessian (objective.cpp:150-171): H = -(1/eps)(diag(r) - P~ diag(b) P~^T),
// symmetrised, with g = f^{C,eps}. The plan and the O(n^2 m) product run on the device.
int sknr_full_semi_dual_hessian(sknr_problem h, const double* f, int64_t dense_limit, double* hess) {
    SKNR_API_BEGIN
    Problem& P0 = get(h);
    if (P0.n_global > dense_limit) throw InvalidArgument("full_semi_dual_hessian: dense Hessian too large");
    if (P0.shard) throw RuntimeFailure("full_semi_dual_hessian: not available on a row-sharded problem");
    std::vector<double> g(P0.m);
    int rc = sknr_ctransform_of_f(h, f, g.data());
    if (rc != SKNR_OK) return rc;
    Problem& P = get(h);
    std::lock_guard<std::mutex> lk(P.mu);
    const int64_t n = P.n, m = P.m;
    DBuf df, dg, dp, dr, dout;
    df.ensure(n);
    dg.ensure(m);
    dp.ensure(n * m);
    dr.ensure(n);
    dout.ensure(n * n);
    upload(df.p, f, n, P.stream);
    upload(dg.p, g.data(), m, P.stream);
    count_launch();
    k_coupling<<<grid_for(n * m), AUX_NT, 0, P.stream>>>(P.kind == 0 || P.C.p ? P.C.p : nullptr, P.src.coords.p,
                                                         P.tgt.coords.p, n, m, 0, n, static_cast<int>(P.d), P.kappa,
                                                         P.src.w.p, P.tgt.w.p, df.p, dg.p, P.inv_eps(), dp.p);
    count_launch();
    k_row_sums<<<grid_for(n), AUX_NT, 0, P.stream>>>(dp.p, n, m, dr.p);
    count_launch();
    k_plan_outer<<<dim3(static_cast<unsigned>((n + 31) / 32), static_cast<unsigned>((n + 31) / 32)), 256, 0,
                   P.stream>>>(dp.p, n, m, P.tgt.w.p, dout.p);
    CK(cudaGetLastError());
    std::vector<double> outer(static_cast<size_t>(n * n)), r(n);
    download(outer.data(), dout.p, n * n, P.stream);
    download(r.data(), dr.p, n, P.stream);
    CK(cudaStreamSynchronize(P.stream));
    const double c = -1.0 / P.eps;
    for (int64_t k = 0; k < n; ++k)
        for (int64_t i = 0; i < n; ++i) {
            const double hik = c * ((i == k ? r[i] : 0.0) - outer[i + k * n]);
            const double hki = c * ((i == k ? r[i] : 0.0) - outer[k + i * n]);
            hess[i + k * n] = 0.5 * (hik + hki);
        }
    SKNR_API_END
}

int sknr_semi_dual_value(sknr_problem h, const double* f, double* value) {
    SKNR_API_BEGIN
    std::vector<double> g(get(h).m);  // f^{C,eps}, then Q = a.f + b.g (objective.cpp:42-45)
    int rc = sknr_ctransform_of_f(h, f, g.data());
    if (rc != SKNR_OK) return rc;
    Problem& P = get(h);
    const std::vector<double>& a = P.h_alpha;
    const std::vector<double>& b = P.h_beta;
    double s1 = 0, s2 = 0;
    for (int64_t i = 0; i < P.n_global; ++i) s1 += a[i] * f[i];
    for (int64_t j = 0; j < P.m; ++j) s2 += b[j] * g[j];
    *value = s1 + s2;
    SKNR_API_END
}

int sknr_restricted_derivatives(sknr_problem h, const double* f, const double* g, const double* vectors,
                                int64_t ell, double* grad, double* hess) {
    SKNR_API_BEGIN
    Problem& P = get(h);
    std::lock_guard<std::mutex> lk(P.mu);
    if (ell < 1) throw InvalidArgument("restricted_derivatives: empty basis");
    if (ell > 64) throw InvalidArgument("restricted_derivatives: ell > 64 is not supported by sknr_b200");
    check_finite_vec(f, P.n_global, "restricted_derivatives(f)");
    check_finite_vec(g, P.m, "restricted_derivatives(g)");
    const int64_t n = P.n, m = P.m;
    const int l = static_cast<int>(ell), kt = block_kt_for(l);
    DBuf df, dg, V, Wv, Sm, am, r, G;
    df.ensure(n);
    dg.ensure(m);
    V.ensure(n * ell);
    Wv.ensure(n * kt);
    Sm.ensure(m * ell);
    am.ensure(n);
    r.ensure(n);
    G.ensure(3 * 64 * 64);
    upload_rows(P, df.p, f);
    upload(dg.p, g, m, P.stream);
    upload_rows(P, V.p, vectors, ell);
    count_launch();
    k_pack_w<<<grid_for(n * kt), AUX_NT, 0, P.stream>>>(V.p, n, n, l, kt, nullptr, Wv.p);
    // r_i = a_i sum_j b_j e^{(f_i+g_j-C_ij)/eps} (objective.cpp:127-128): fused into the
    // block pass for point clouds, else a plan-sum pass
    const bool fuse_r = block_rs_fusable(P);
    if (!fuse_r) {
        PassSpec pr;
        pr.dir = 1;
        pr.in_v = dg.p;
        pr.in_lw = P.tgt.lw.p;
        pr.out_v = df.p;
        pr.out_lw = P.src.lw.p;
        pr.out = r.p;
        plan_pass(P, pr);
    }
    PassSpec sp;
    sp.dir = 0;
    sp.in_v = df.p;
    sp.in_lw = P.src.lw.p;
    sp.out_v = dg.p;
    sp.W = Wv.p;
    sp.k = l;
    sp.kt = kt;
    sp.out = Sm.p;
    sp.rsum_out = fuse_r ? r.p : nullptr;
    plan_pass(P, sp);
    // am = a - r
    count_launch();
    k_axpby<<<grid_for(n), AUX_NT, 0, P.stream>>>(P.src.w.p, r.p, n, 1.0, -1.0, am.p);
    double* G1 = G.p;
    double* cross = G1 + l * l;
    double* gr = cross + l * l;
    gram(P, n, l, l, V.p, n, V.p, n, r.p, G1, 0);
    gram(P, m, l, l, Sm.p, m, Sm.p, m, P.tgt.w.p, cross, 0);
    gram(P, n, l, 1, V.p, n, am.p, n, nullptr, gr, 0);
    allreduce(P, G1, static_cast<size_t>(l) * l, ncclSum);
    allreduce(P, gr, l, ncclSum);
    std::vector<double> hG1(l * l), hC(l * l);
    download(hG1.data(), G1, l * l, P.stream);
    download(hC.data(), cross, l * l, P.stream);
    download(grad, gr, l, P.stream);
    CK(cudaStreamSynchronize(P.stream));
    std::vector<double> H(l * l);
    for (int a = 0; a < l; ++a)
        for (int b = 0; b < l; ++b) H[a + b * l] = (-1.0 / P.eps) * (hG1[a + b * l] - hC[a + b * l]);
    for (int a = 0; a < l; ++a)
        for (int b = 0; b < l; ++b) hess[a + b * l] = 0.5 * (H[a + b * l] + H[b + a * l]);
    SKNR_API_END
}

int sknr_apply_sym_t_block(sknr_problem h, const double* f, const double* g, const double* u, int64_t k,
                           double* out) {
    SKNR_API_BEGIN
    Problem& P = get(h);
    std::lock_guard<std::mutex> lk(P.mu);
    if (k < 1 || k > 64) throw InvalidArgument("apply_sym_t_block: 1 <= k <= 64 required");
    const int64_t n = P.n, m = P.m;
    const int kt = block_kt_for(static_cast<int>(k));
    DBuf df, dg, U, W, O;
    df.ensure(n);
    dg.ensure(m);
    U.ensure(n * k);
    W.ensure(n * kt);
    O.ensure(m * k);
    upload_rows(P, df.p, f);
    upload(dg.p, g, m, P.stream);
    upload_rows(P, U.p, u, k);
    count_launch();
    k_pack_w<<<grid_for(n * kt), AUX_NT, 0, P.stream>>>(U.p, n, n, static_cast<int>(k), kt, nullptr, W.p);
    PassSpec zt;
    zt.dir = 0;
    zt.in_v = df.p;
    zt.in_lw = P.src.lsw.p;
    zt.out_v = dg.p;
    zt.W = W.p;
    zt.k = static_cast<int>(k);
    zt.kt = kt;
    zt.out_scale = P.tgt.sw.p;
    zt.out = O.p;
    plan_pass(P, zt);
    download(out, O.p, m * k, P.stream);
    CK(cudaStreamSynchronize(P.stream));
    SKNR_API_END
}

int sknr_apply_sym_block(sknr_problem h, const double* f, const double* g, const double* v, int64_t k,
                         double* out) {
    SKNR_API_BEGIN
    Problem& P = get(h);
    std::lock_guard<std::mutex> lk(P.mu);
    if (k < 1 || k > 64) throw InvalidArgument("apply_sym_block: 1 <= k <= 64 required");
    const int64_t n = P.n, m = P.m;
    const int kt = block_kt_for(static_cast<int>(k));
    DBuf df, dg, Vv, W, O;
    df.ensure(n);
    dg.ensure(m);
    Vv.ensure(m * k);
    W.ensure(m * kt);
    O.ensure(n * k);
    upload_rows(P, df.p, f);
    upload(dg.p, g, m, P.stream);
    upload(Vv.p, v, m * k, P.stream);
    count_launch();
    k_pack_w<<<grid_for(m * kt), AUX_NT, 0, P.stream>>>(Vv.p, m, m, static_cast<int>(k), kt, P.tgt.sw.p,
                                                        W.p);
    PassSpec yr;
    yr.dir = 1;
    yr.in_v = dg.p;
    yr.out_v = df.p;
    yr.out_lw = P.src.lsw.p;
    yr.W = W.p;
    yr.k = static_cast<int>(k);
    yr.kt = kt;
    yr.out = O.p;
    plan_pass(P, yr);
    for (int64_t c = 0; c < k; ++c) gather_rows(P, O.p + c * n, out + c * P.n_global);
    SKNR_API_END
}

int sknr_top_modes_ex(sknr_problem h, const double* f, const double* g, int64_t ell, double tol,
                      int64_t max_power_iters, int method, int degree, double* vectors, double* vectors_sym,
                      double* rhos, int64_t* sweeps);

// ---- SinkhornOperator::apply_R / apply_Rt (spectral.cpp:29-62): one k=1 block pass each.
// dir 1: (R g1)_i = sum_j e^{(f_i+g_j-C_ij)/eps} (b_j g1_j); dir 0: (Rt f1)_j = sum_i e^{..} (a_i f1_i)
static void apply_R_dir(sknr_problem h, int dir, const double* f, const double* g, const double* v, double* out,
                        const char* what) {
    Problem& P = get(h);
    std::lock_guard<std::mutex> lk(P.mu);
    check_finite_vec(f, P.n_global, "SinkhornOperator(f)");
    check_finite_vec(g, P.m, "SinkhornOperator(g)");
    const int64_t n = P.n, m = P.m;
    const int64_t nv = dir == 0 ? n : m, nout = dir == 0 ? m : n;
    if (!v) throw InvalidArgument(std::string(what) + ": null pointer");
    const int kt = block_kt_for(1);
    DBuf df, dg, dv, W, O;
    df.ensure(n);
    dg.ensure(m);
    dv.ensure(nv);
    W.ensure(nv * kt);
    O.ensure(nout);
    upload_rows(P, df.p, f);
    upload(dg.p, g, m, P.stream);
    if (dir == 0)
        upload_rows(P, dv.p, v);
    else
        upload(dv.p, v, m, P.stream);
    count_launch();
    k_pack_w<<<grid_for(nv * kt), AUX_NT, 0, P.stream>>>(dv.p, nv, nv, 1, kt, dir == 0 ? P.src.w.p : P.tgt.w.p,
                                                         W.p);
    PassSpec ps;
    ps.dir = dir;
    ps.in_v = dir == 0 ? df.p : dg.p;
    ps.out_v = dir == 0 ? dg.p : df.p;
    ps.W = W.p;
    ps.k = 1;
    ps.kt = kt;
    ps.out = O.p;
    plan_pass(P, ps);
    if (dir == 0)
        download(out, O.p, m, P.stream);
    else
        gather_rows(P, O.p, out);
    CK(cudaStreamSynchronize(P.stream));
}

int sknr_apply_R(sknr_problem h, const double* f, const double* g, const double* g1, double* out) {
    SKNR_API_BEGIN
    apply_R_dir(h, 1, f, g, g1, out, "apply_R");
    SKNR_API_END
}

int sknr_apply_Rt(sknr_problem h, const double* f, const double* g, const double* f1, double* out) {
    SKNR_API_BEGIN
    apply_R_dir(h, 0, f, g, f1, out, "apply_Rt");
    SKNR_API_END
}

// ---- dual_value (objective.cpp:10-40): a.f + b.g - eps expm1(log sum_ij a_i b_j e^{(f_i+g_j-C_ij)/eps}).
// The double sum is taken as sum_i a_i e^{(f_i - f~_i)/eps} with f~ = g^{C,eps} (one row-LSE pass),
// max-shifted on the host.
int sknr_dual_value(sknr_problem h, const double* f, const double* g, double* value) {
    SKNR_API_BEGIN
    Problem& P = get(h);
    const int64_t n = P.n_global, m = P.m;
    if (!f || !g || !value) throw InvalidArgument("dual_value: null pointer");
    for (int64_t i = 0; i < n; ++i)
        if (!std::isfinite(f[i])) throw InvalidArgument("dual_value: potentials must be finite");
    for (int64_t j = 0; j < m; ++j)
        if (!std::isfinite(g[j])) throw InvalidArgument("dual_value: potentials must be finite");
    std::vector<double> ft(n);
    const int rc = sknr_ctransform_of_g(h, g, ft.data());
    if (rc != SKNR_OK) return rc;
    const double inv_eps = 1.0 / P.eps;
    double shift = -std::numeric_limits<double>::infinity();
    std::vector<double> t(n);
    for (int64_t i = 0; i < n; ++i) {
        t[i] = std::log(P.h_alpha[i]) + (f[i] - ft[i]) * inv_eps;
        shift = std::max(shift, t[i]);
    }
    double total = 0.0;
    for (int64_t i = 0; i < n; ++i) total += std::exp(t[i] - shift);
    const double log_mass = shift + std::log(total);
    double af = 0.0, bg = 0.0;
    for (int64_t i = 0; i < n; ++i) af += P.h_alpha[i] * f[i];
    for (int64_t j = 0; j < m; ++j) bg += P.h_beta[j] * g[j];
    *value = af + bg - P.eps * std::expm1(log_mass);
    SKNR_API_END
}

// ---- semi_dual_hessian_quadform (objective.cpp:53-77): -(1/eps) sum_j b_j (m2_j - m1_j^2) with
// m1_j = sum_i P~_ij u_i, m2_j = sum_i P~_ij u_i^2 at g = f^{C,eps}: one k=2 block pass.
int sknr_semi_dual_hessian_quadform(sknr_problem h, const double* f, const double* u, double* value) {
    SKNR_API_BEGIN
    Problem& P = get(h);
    const int64_t n = P.n_global, m = P.m;
    if (!u || !value) throw InvalidArgument("semi_dual_hessian_quadform: null pointer");
    std::vector<double> g(m);
    int rc = sknr_ctransform_of_f(h, f, g.data());
    if (rc != SKNR_OK) return rc;
    std::vector<double> U(2 * n);
    for (int64_t i = 0; i < n; ++i) {
        U[i] = u[i];
        U[n + i] = u[i] * u[i];
    }
    std::vector<double> M(2 * m);
    {
        std::lock_guard<std::mutex> lk(P.mu);
        const int kt = block_kt_for(2);
        DBuf df, dg, dU, W, O;
        df.ensure(P.n);
        dg.ensure(m);
        dU.ensure(2 * P.n);
        W.ensure(P.n * kt);
        O.ensure(2 * m);
        upload_rows(P, df.p, f);
        upload(dg.p, g.data(), m, P.stream);
        upload_rows(P, dU.p, U.data(), 2);
        count_launch();
        k_pack_w<<<grid_for(P.n * kt), AUX_NT, 0, P.stream>>>(dU.p, P.n, P.n, 2, kt, nullptr, W.p);
        PassSpec ps;
        ps.dir = 0;
        ps.in_v = df.p;
        ps.in_lw = P.src.lw.p;
        ps.out_v = dg.p;
        ps.W = W.p;
        ps.k = 2;
        ps.kt = kt;
        ps.out = O.p;
        plan_pass(P, ps);
        download(M.data(), O.p, 2 * m, P.stream);
        CK(cudaStreamSynchronize(P.stream));
    }
    double acc = 0.0;
    for (int64_t j = 0; j < m; ++j) acc += P.h_beta[j] * (M[m + j] - M[j] * M[j]);
    *value = -acc / P.eps;
    SKNR_API_END
}

// Eigen::LLT<Matrix>(A) convention (llt_inplace::unblocked): fails iff a pivot is <= 0 or NaN.
static bool host_llt_solve(std::vector<double> A, int l, const double* b, double* x) {
    for (int k = 0; k < l; ++k) {
        double piv = A[k + k * l];
        for (int j = 0; j < k; ++j) piv -= A[k + j * l] * A[k + j * l];
        if (!(piv > 0.0)) return false;
        const double d = std::sqrt(piv);
        A[k + k * l] = d;
        for (int i = k + 1; i < l; ++i) {
            double s = A[i + k * l];
            for (int j = 0; j < k; ++j) s -= A[i + j * l] * A[k + j * l];
            A[i + k * l] = s / d;
        }
    }
    std::vector<double> y(l);
    for (int i = 0; i < l; ++i) {
        double s = b[i];
        for (int j = 0; j < i; ++j) s -= A[i + j * l] * y[j];
        y[i] = s / A[i + i * l];
    }
    for (int i = l - 1; i >= 0; --i) {
        double s = y[i];
        for (int j = i + 1; j < l; ++j) s -= A[j + i * l] * x[j];
        x[i] = s / A[i + i * l];
    }
    return true;
}

// ---- newton_step (solver.cpp:59-69 with try_newton :30-56): g = f^{C,eps}, Q0 = a.f + b.g,
// restricted derivatives, LLT(-H) (reject on failure), delta, f' = f + V delta, accept iff Q(f') > Q0
// (accept_test 0) or dQ > 0 (accept_test 1, see sknr_config): s = R^T(1), t = R^T(expm1(d/eps))
// at the anchor (f, g), h' - h = -eps log1p(t/s).
int sknr_newton_step_ex(sknr_problem h, const double* f, const double* vectors, int64_t ell, int accept_test,
                        double* f_out, int* accepted, int* factorization_failed) {
    SKNR_API_BEGIN
    Problem& P = get(h);
    if (ell < 1) throw InvalidArgument("newton_step: empty basis");
    if (!vectors || !f_out || !accepted || !factorization_failed)
        throw InvalidArgument("newton_step: null pointer");
    if (accept_test != 0 && accept_test != 1)
        throw InvalidArgument("newton_step: accept_test must be 0 (literal) or 1 (stable)");
    const int64_t n = P.n_global, m = P.m;
    const int l = static_cast<int>(ell);
    std::vector<double> g(m), grad(l), hess(static_cast<size_t>(l) * l);
    int rc = sknr_ctransform_of_f(h, f, g.data());
    if (rc != SKNR_OK) return rc;
    double af = 0.0, bg = 0.0;
    for (int64_t i = 0; i < n; ++i) af += P.h_alpha[i] * f[i];
    for (int64_t j = 0; j < m; ++j) bg += P.h_beta[j] * g[j];
    const double value = af + bg;
    rc = sknr_restricted_derivatives(h, f, g.data(), vectors, ell, grad.data(), hess.data());
    if (rc != SKNR_OK) return rc;
    std::vector<double> negH(hess.size()), delta(l);
    for (size_t e = 0; e < hess.size(); ++e) negH[e] = -hess[e];
    *accepted = 0;
    *factorization_failed = 0;
    std::memcpy(f_out, f, sizeof(double) * n);
    if (!host_llt_solve(negH, l, grad.data(), delta.data())) {
        *factorization_failed = 1;
        return SKNR_OK;
    }
    std::vector<double> cand(n);
    for (int64_t i = 0; i < n; ++i) {
        double s = 0.0;
        for (int c = 0; c < l; ++c) s += vectors[i + c * n] * delta[c];
        cand[i] = f[i] + s;
    }
    const double inv_eps = 1.0 / P.eps;
    double dmax = 0.0;
    std::vector<double> dv(n), ev(n), xv(n);
    for (int64_t i = 0; i < n; ++i) {
        dv[i] = cand[i] - f[i];
        dmax = std::max(dmax, std::abs(dv[i]));
        ev[i] = std::expm1(dv[i] * inv_eps);
        xv[i] = std::exp(std::min(dv[i] * inv_eps, 700.0));
    }
    bool acc = false;
    if (accept_test == 1 && dmax <= kStableSpan * P.eps) {
        std::vector<double> ones(n, 1.0), sv(m), tv(m), uv(m);
        rc = sknr_apply_Rt(h, f, g.data(), ones.data(), sv.data());
        if (rc != SKNR_OK) return rc;
        rc = sknr_apply_Rt(h, f, g.data(), ev.data(), tv.data());
        if (rc != SKNR_OK) return rc;
        rc = sknr_apply_Rt(h, f, g.data(), xv.data(), uv.data());
        if (rc != SKNR_OK) return rc;
        double dq = 0.0, bdh = 0.0;
        for (int64_t i = 0; i < n; ++i) dq += P.h_alpha[i] * dv[i];
        for (int64_t j = 0; j < m; ++j) {
            const double ts = tv[j] / sv[j];  // as k_dh
            bdh += P.h_beta[j] * (-P.eps * (std::abs(ts) <= kDhSwitch ? std::log1p(ts) : std::log(uv[j] / sv[j])));
        }
        acc = dq + bdh > 0.0;
    } else {
        double q1 = 0.0;
        rc = sknr_semi_dual_value(h, cand.data(), &q1);
        if (rc != SKNR_OK) return rc;
        acc = q1 > value;
    }
    if (acc) {
        std::memcpy(f_out, cand.data(), sizeof(double) * n);
        *accepted = 1;
    }
    SKNR_API_END
}

int sknr_newton_step(sknr_problem h, const double* f, const double* vectors, int64_t ell, double* f_out,
                     int* accepted, int* factorization_failed) {
    return sknr_newton_step_ex(h, f, vectors, ell, 0, f_out, accepted, factorization_failed);
}

// ---- projector_distance (spectral.cpp:230-242): ||(I - A A^T) B||_2 for n x k column blocks,
// via the largest eigenvalue of R^T R, R = B - A (A^T B); clamped to [0, 1]. Host arithmetic
// (O(n k^2), a diagnostic off the solve path).
int sknr_projector_distance(int64_t n, int64_t k, const double* a_sym, const double* b_sym, double* out) {
    SKNR_API_BEGIN
    if (n < 1 || k < 1 || !a_sym || !b_sym || !out) throw InvalidArgument("projector_distance: dimension mismatch");
    std::vector<double> AtB(static_cast<size_t>(k) * k, 0.0), R(static_cast<size_t>(n) * k);
    for (int64_t c = 0; c < k; ++c)
        for (int64_t a = 0; a < k; ++a) {
            double s = 0.0;
            for (int64_t i = 0; i < n; ++i) s += a_sym[i + a * n] * b_sym[i + c * n];
            AtB[a + c * k] = s;
        }
    for (int64_t c = 0; c < k; ++c)
        for (int64_t i = 0; i < n; ++i) {
            double s = 0.0;
            for (int64_t a = 0; a < k; ++a) s += a_sym[i + a * n] * AtB[a + c * k];
            R[i + c * n] = b_sym[i + c * n] - s;
        }
    std::vector<double> G(static_cast<size_t>(k) * k);
    for (int64_t c = 0; c < k; ++c)
        for (int64_t a = 0; a <= c; ++a) {
            double s = 0.0;
            for (int64_t i = 0; i < n; ++i) s += R[i + a * n] * R[i + c * n];
            G[a + c * k] = G[c + a * k] = s;
        }
    std::vector<double> ev, evec;
    host_sym_eig(G, static_cast<int>(k), ev, evec);
    double lmax = 0.0;
    for (double e : ev) lmax = std::max(lmax, e);
    *out = std::clamp(std::sqrt(std::max(lmax, 0.0)), 0.0, 1.0);
    SKNR_API_END
}

// ---- spectrum_report (spectral.cpp:195-228): top_modes at the anchor, Hessian eigenvalue pairs
// (1 -+ rho)/eps, optional right vectors v = R~^T u / rho in potential coordinates.
int sknr_spectrum_report(sknr_problem h, const double* f, const double* g, int64_t k, int include_vectors,
                         double tol, int64_t max_power_iters, double* rhos, double* hess_low, double* hess_high,
                         double* vectors_f, double* vectors_g) {
    SKNR_API_BEGIN
    Problem& P = get(h);
    const int64_t n = P.n_global, m = P.m;
    if (k < 1 || k > std::min(n, m) - 1) throw InvalidArgument("spectrum_report: need 1 <= k <= min(n,m)-1");
    if (!rhos || !hess_low || !hess_high) throw InvalidArgument("spectrum_report: null pointer");
    std::vector<double> vec(static_cast<size_t>(n) * k), vsym(static_cast<size_t>(n) * k);
    int64_t sweeps = 0;
    int rc = sknr_top_modes(h, f, g, k, tol, max_power_iters, vec.data(), vsym.data(), rhos, &sweeps);
    if (rc != SKNR_OK) return rc;
    for (int64_t a = 0; a < k; ++a) {
        hess_low[a] = (1.0 - rhos[a]) / P.eps;
        hess_high[a] = (1.0 + rhos[a]) / P.eps;
    }
    if (include_vectors) {
        if (!vectors_f || !vectors_g) throw InvalidArgument("spectrum_report: null pointer");
        std::memcpy(vectors_f, vec.data(), sizeof(double) * n * k);
        std::vector<double> vs(static_cast<size_t>(m) * k);
        rc = sknr_apply_sym_t_block(h, f, g, vsym.data(), k, vs.data());
        if (rc != SKNR_OK) return rc;
        for (int64_t a = 0; a < k; ++a)
            for (int64_t j = 0; j < m; ++j)
                vectors_g[j + a * m] = rhos[a] > 1e-12 ? (vs[j + a * m] / rhos[a]) / std::sqrt(P.h_beta[j]) : 0.0;
    }
    SKNR_API_END
}


int sknr_top_modes(sknr_problem h, const double* f, const double* g, int64_t ell, double tol,
                   int64_t max_power_iters, double* vectors, double* vectors_sym, double* rhos,
                   int64_t* sweeps) {
    return sknr_top_modes_ex(h, f, g, ell, tol, max_power_iters, 0, 1, vectors, vectors_sym, rhos, sweeps);
}

int sknr_top_modes_ex(sknr_problem h, const double* f, const double* g, int64_t ell, double tol,
                      int64_t max_power_iters, int method, int degree, double* vectors, double* vectors_sym,
                      double* rhos, int64_t* sweeps) {
    SKNR_API_BEGIN
    Problem& P = get(h);
    std::lock_guard<std::mutex> lk(P.mu);
    check_finite_vec(f, P.n_global, "SinkhornOperator(f)");
    check_finite_vec(g, P.m, "SinkhornOperator(g)");
    DBuf df, dg;
    df.ensure(P.n);
    dg.ensure(P.m);
    upload_rows(P, df.p, f);
    upload(dg.p, g, P.m, P.stream);
    if (method < 0 || method > 2)
        throw InvalidArgument("top_modes: method must be 0 (subspace), 1 (chebyshev) or 2 (lanczos)");
    Basis b = top_modes_device(P, df.p, dg.p, ell, tol, max_power_iters, method, degree);
    std::memcpy(vectors, b.vectors.data(), sizeof(double) * P.n_global * ell);
    std::memcpy(vectors_sym, b.vectors_sym.data(), sizeof(double) * P.n_global * ell);
    std::memcpy(rhos, b.rhos.data(), sizeof(double) * ell);
    if (sweeps) *sweeps = b.sweeps;
    SKNR_API_END
}

static void validate_config(const sknr_config* cfg, const double* basis, int64_t basis_ell, int64_t n) {
    if (!(cfg->tol_omega > 0.0)) throw InvalidArgument("solve: tol_omega must be positive");
    if (cfg->max_iter < 1) throw InvalidArgument("solve: max_iter must be >= 1");
    const bool use_newton = cfg->newton_enabled && cfg->ell > 0;
    if (use_newton) {
        if (basis == nullptr) throw InvalidArgument("solve: ell > 0 requires a basis");
        if (basis_ell != cfg->ell) throw InvalidArgument("solve: basis has wrong column count");
    }
    if (cfg->accept_test != 0 && cfg->accept_test != 1)
        throw InvalidArgument("solve: accept_test must be 0 (literal) or 1 (stable)");
    (void)n;
}

int sknr_solve(sknr_problem h, const sknr_config* cfg, const double* basis, int64_t basis_ell,
               const double* init_f, const double* init_g, double* f_out, double* g_out,
               int64_t* iterations, int* converged, sknr_record* trace, int64_t trace_cap,
               int64_t* trace_len) {
    SKNR_API_BEGIN
    Problem& P = get(h);
    std::lock_guard<std::mutex> lk(P.mu);
    validate_config(cfg, basis, basis_ell, P.n);
    if ((init_f == nullptr) != (init_g == nullptr))
        throw InvalidArgument("solve: init potential sizes mismatch");
    const bool use_newton = cfg->newton_enabled && cfg->ell > 0;
    const int64_t ell = use_newton ? cfg->ell : 0;
    SolveOut o = run_solve(P, cfg->tol_omega, cfg->max_iter, ell, basis, init_f, cfg->trace_enabled != 0,
                           std::max<int64_t>(trace_cap, cfg->trace_enabled ? cfg->max_iter : 1),
                           cfg->exact_marginals != 0, cfg->accept_test);
    std::memcpy(f_out, o.f.data(), sizeof(double) * P.n_global);
    std::memcpy(g_out, o.g.data(), sizeof(double) * P.m);
    if (iterations) *iterations = o.iterations;
    if (converged) *converged = o.converged ? 1 : 0;
    const int64_t len = static_cast<int64_t>(o.trace.size());
    if (trace_len) *trace_len = len;
    if (trace)
        for (int64_t t = 0; t < len && t < trace_cap; ++t) trace[t] = o.trace[t];
    P.last_trace = std::move(o.trace);
    SKNR_API_END
}

int sknr_solve_batch(const sknr_problem* problems, int64_t count, const sknr_config* cfg,
                     const double* const* bases, int64_t basis_ell, const double* const* init_f,
                     const double* const* init_g, double* const* f_out, double* const* g_out, int64_t* iterations,
                     int* converged) {
    SKNR_API_BEGIN
    if (count < 1 || !problems || !cfg || !f_out || !g_out) throw InvalidArgument("solve_batch: empty batch");
    if ((init_f == nullptr) != (init_g == nullptr)) throw InvalidArgument("solve: init potential sizes mismatch");
    std::vector<BatchItem> items(static_cast<size_t>(count));
    std::vector<std::unique_lock<std::mutex>> locks;
    for (int64_t b = 0; b < count; ++b) {
        Problem& P = get(problems[b]);
        for (int64_t c = 0; c < b; ++c)
            if (problems[c] == problems[b]) throw InvalidArgument("solve_batch: duplicate problem handle");
        if (P.shard) throw InvalidArgument("solve_batch: row-sharded problems are not supported");
        validate_config(cfg, bases ? bases[b] : nullptr, basis_ell, P.n);
        if (init_f && ((init_f[b] == nullptr) != (init_g[b] == nullptr)))
            throw InvalidArgument("solve: init potential sizes mismatch");
        if (!f_out[b] || !g_out[b]) throw InvalidArgument("solve_batch: null output");
        items[b].P = &P;
        items[b].basis = bases ? bases[b] : nullptr;
        items[b].init_f = init_f ? init_f[b] : nullptr;
        locks.emplace_back(P.mu);
    }
    const bool use_newton = cfg->newton_enabled && cfg->ell > 0;
    std::vector<SolveOut> o = run_solve_batch(items, cfg->tol_omega, cfg->max_iter, use_newton ? cfg->ell : 0,
                                              cfg->exact_marginals != 0, cfg->accept_test);
    for (int64_t b = 0; b < count; ++b) {
        std::memcpy(f_out[b], o[b].f.data(), sizeof(double) * items[b].P->n_global);
        std::memcpy(g_out[b], o[b].g.data(), sizeof(double) * items[b].P->m);
        if (iterations) iterations[b] = o[b].iterations;
        if (converged) converged[b] = o[b].converged ? 1 : 0;
    }
    SKNR_API_END
}

// Small-problem batch: every problem solved by plain SK (ell = 0) from f = 0 inside one
// kernel launch (launch_sk_small) by a group of G CTAs (G = 1 when the batch fills the
// GPU; a lone C1 problem gets 32 CTAs); point clouds of one dimension d <= 4 with
// n, m <= small_max_count(d) (8192 at d <= 2). Problems may differ in n, m, epsilon
// and cost scale.
int sknr_solve_small_batch(int64_t count, int64_t d, const int64_t* n, const int64_t* m, const double* const* x,
                           const double* const* y, const double* const* a, const double* const* b,
                           const double* eps, const double* cost_scale, double tol, int64_t max_iter,
                           double* const* f_out, double* const* g_out, int64_t* iterations, int* converged) {
    SKNR_API_BEGIN
    check_device();
    if (count < 1) throw InvalidArgument("solve_small_batch: empty batch");
    if (d < 1 || d > 4) throw InvalidArgument("solve_small_batch: 1 <= d <= 4 required");
    if (!(tol > 0.0)) throw InvalidArgument("solve: tol_omega must be positive");
    if (max_iter < 1) throw InvalidArgument("solve: max_iter must be >= 1");
    if (!n || !m || !x || !y || !a || !b || !eps || !f_out || !g_out)
        throw InvalidArgument("solve_small_batch: null pointer");
    // one device arena: per problem x (n d), y (m d), a (n), b (m), f (n), g (m), h (m)
    std::vector<size_t> off(static_cast<size_t>(count) + 1, 0);
    int64_t max_nm = 1;
    for (int64_t q = 0; q < count; ++q) {
        if (n[q] < 1 || m[q] < 1 || n[q] > small_max_count(static_cast<int>(d)) ||
            m[q] > small_max_count(static_cast<int>(d)))
            throw InvalidArgument("solve_small_batch: 1 <= n, m <= " +
                                  std::to_string(small_max_count(static_cast<int>(d))) + " required at d = " +
                                  std::to_string(d));
        max_nm = std::max<int64_t>(max_nm, std::max(n[q], m[q]));
        if (!(eps[q] > 0.0)) throw InvalidArgument("EotProblem: epsilon must be positive");
        validate_measure(a[q], n[q]);
        validate_measure(b[q], m[q]);
        off[q + 1] = off[q] + static_cast<size_t>((n[q] + m[q]) * d + 2 * n[q] + 3 * m[q]);
    }
    DBuf arena, dprobs;
    arena.ensure(off[count]);
    std::vector<SmallProbDev> hp(static_cast<size_t>(count));
    std::vector<double> host(off[count], 0.0);
    for (int64_t q = 0; q < count; ++q) {
        double* base = host.data() + off[q];
        const int64_t nq = n[q], mq = m[q];
        std::memcpy(base, x[q], sizeof(double) * nq * d);
        std::memcpy(base + nq * d, y[q], sizeof(double) * mq * d);
        std::memcpy(base + (nq + mq) * d, a[q], sizeof(double) * nq);
        std::memcpy(base + (nq + mq) * d + nq, b[q], sizeof(double) * mq);
        double* dev = arena.p + off[q];
        SmallProbDev& s = hp[q];
        s.x = dev;
        s.y = dev + nq * d;
        s.a = dev + (nq + mq) * d;
        s.b = s.a + nq;
        s.f = const_cast<double*>(s.b) + mq;  // zero-filled: SK from f = 0
        s.g = s.f + nq;
        s.h = s.g + mq;
        s.n = static_cast<int>(nq);
        s.m = static_cast<int>(mq);
        s.eps = eps[q];
        s.kappa = cost_scale ? cost_scale[q] : 1.0;
    }
    const size_t words = (sizeof(SmallProbDev) * static_cast<size_t>(count) + sizeof(double) - 1) / sizeof(double);
    dprobs.ensure(words);
    cudaStream_t s = nullptr;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    CK(cudaMemcpyAsync(arena.p, host.data(), sizeof(double) * off[count], cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(dprobs.p, hp.data(), sizeof(SmallProbDev) * count, cudaMemcpyHostToDevice, s));
    const int G = small_group_size(static_cast<int>(d), static_cast<int>(count), static_cast<int>(max_nm));
    DBuf gpart, gbar;
    if (G > 1) {
        gpart.ensure(static_cast<size_t>(count) * G * 4);
        gbar.ensure(static_cast<size_t>(count));  // 2 unsigned per problem
        CK(cudaMemsetAsync(gbar.p, 0, sizeof(double) * count, s));
    }
    launch_sk_small(static_cast<int>(d), reinterpret_cast<SmallProbDev*>(dprobs.p), static_cast<int>(count),
                    static_cast<int>(max_nm), tol, max_iter, 0, G, gpart.p, reinterpret_cast<unsigned*>(gbar.p), s);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(host.data(), arena.p, sizeof(double) * off[count], cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(hp.data(), dprobs.p, sizeof(SmallProbDev) * count, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    cudaStreamDestroy(s);
    for (int64_t q = 0; q < count; ++q) {
        const double* base = host.data() + off[q];
        const int64_t nq = n[q], mq = m[q];
        const double* fq = base + (nq + mq) * d + nq + mq;
        std::memcpy(f_out[q], fq, sizeof(double) * nq);
        std::memcpy(g_out[q], fq + nq, sizeof(double) * mq);
        if (iterations) iterations[q] = hp[q].iters;
        if (converged) converged[q] = hp[q].conv;
    }
    SKNR_API_END
}

int sknr_anneal(sknr_problem h, const double* epsilons, int64_t stages, int warm_mode, int refresh_basis,
                const sknr_config* cfg, double* f_out, double* g_out, int64_t* iterations, int* converged,
                sknr_record* trace, int64_t trace_cap, int64_t* trace_offsets, int64_t* trace_len) {
    SKNR_API_BEGIN
    Problem& P = get(h);
    std::lock_guard<std::mutex> lk(P.mu);
    if (stages < 1) throw InvalidArgument("anneal: empty schedule");
    for (int64_t s = 1; s < stages; ++s)
        if (!(epsilons[s] < epsilons[s - 1]))
            throw InvalidArgument("anneal: epsilons must be strictly decreasing");
    if (!(cfg->tol_omega > 0.0)) throw InvalidArgument("solve: tol_omega must be positive");
    if (cfg->max_iter < 1) throw InvalidArgument("solve: max_iter must be >= 1");
    const double eps0 = P.eps;
    const int64_t n = P.n_global, m = P.m;
    int64_t tl = 0;
    P.last_trace.clear();
    Basis basis;
    bool have_basis = false;
    std::vector<double> prev_f, prev_g;
    auto set_eps = [&](double e) {
        P.eps = e;
        count_launch();
        k_invalidate_refs<<<1, 32, 0, P.stream>>>(P.st);
    };
    try {
        for (int64_t s = 0; s < stages; ++s) {
            int64_t ell = 0;
            const double* bptr = nullptr;
            if (s > 0 && warm_mode == 2 && cfg->ell > 0) {
                if (!have_basis || refresh_basis) {
                    set_eps(epsilons[s - 1]);
                    DBuf df, dg;
                    df.ensure(n);
                    dg.ensure(m);
                    upload_rows(P, df.p, prev_f.data());
                    upload(dg.p, prev_g.data(), m, P.stream);
                    try {
                        basis = top_modes_device(P, df.p, dg.p, cfg->ell, 1e-8, -1);
                    } catch (const EigenFailure& e) {
                        throw EigenFailure("anneal stage " + std::to_string(s) + ": " + e.what(), e.best);
                    }
                    have_basis = true;
                }
                ell = cfg->newton_enabled ? cfg->ell : 0;
                bptr = basis.vectors.data();
            }
            set_eps(epsilons[s]);
            const double* init = (s > 0 && warm_mode != 0) ? prev_f.data() : nullptr;
            SolveOut o;
            try {
                o = run_solve(P, cfg->tol_omega, cfg->max_iter, ell, bptr, init, cfg->trace_enabled != 0,
                              cfg->max_iter, cfg->exact_marginals != 0, cfg->accept_test);
            } catch (const InvalidArgument& e) {
                throw RuntimeFailure("anneal stage " + std::to_string(s) + ": " + e.what());
            }
            std::memcpy(f_out + s * n, o.f.data(), sizeof(double) * n);
            std::memcpy(g_out + s * m, o.g.data(), sizeof(double) * m);
            iterations[s] = o.iterations;
            converged[s] = o.converged ? 1 : 0;
            trace_offsets[s] = tl;
            for (size_t t = 0; t < o.trace.size(); ++t, ++tl)
                if (trace && tl < trace_cap) trace[tl] = o.trace[t];
            P.last_trace.insert(P.last_trace.end(), o.trace.begin(), o.trace.end());
            prev_f = std::move(o.f);
            prev_g = std::move(o.g);
        }
    } catch (...) {
        set_eps(eps0);
        throw;
    }
    if (trace_len) *trace_len = tl;
    set_eps(eps0);
    CK(cudaStreamSynchronize(P.stream));
    SKNR_API_END
}

int sknr_comm_stats(int64_t* calls, int64_t* bytes, int reset) {
    SKNR_API_BEGIN
    if (calls) *calls = g_coll_calls.load();
    if (bytes) *bytes = g_coll_bytes.load();
    if (reset) {
        g_coll_calls.store(0);
        g_coll_bytes.store(0);
    }
    SKNR_API_END
}

int sknr_last_trace(sknr_problem h, sknr_record* trace, int64_t cap, int64_t* len) {
    SKNR_API_BEGIN
    Problem& P = get(h);
    std::lock_guard<std::mutex> lk(P.mu);
    const int64_t L = static_cast<int64_t>(P.last_trace.size());
    if (len) *len = L;
    if (trace)
        for (int64_t t = 0; t < L && t < cap; ++t) trace[t] = P.last_trace[t];
    SKNR_API_END
}

int sknr_bench_pass(sknr_problem h, int which, int64_t ell, int passes, double* ms_per_pass,
                    double* kernel_ms_per_pass) {
    SKNR_API_BEGIN
    Problem& P = get(h);
    std::lock_guard<std::mutex> lk(P.mu);
    const int64_t n = P.n, m = P.m;
    cudaStream_t s = P.stream;
    DBuf f, g, V, Wv, Sm, rr;
    f.ensure(n);
    g.ensure(m);
    count_launch();
    k_fill<<<grid_for(n), AUX_NT, 0, s>>>(f.p, n, 0.0);
    count_launch();
    k_state_init<<<1, 32, 0, s>>>(P.st, 1, 1.0);
    plan_for(P, 0, MODE_SUM, 0);
    plan_for(P, 1, MODE_SUM, 0);
    plan_for(P, 0, MODE_MAX, 0);
    plan_for(P, 1, MODE_MAX, 0);
    lse(P, 0, f.p, g.p, G_NONE);  // realistic g; seeds the reference state
    lse(P, 1, g.p, f.p, G_NONE);
    const int l = static_cast<int>(std::max<int64_t>(ell, 1));
    const int kt = block_kt_for(l);
    if (which >= 3) {
        V.ensure(n * l);
        Wv.ensure(std::max(n, m) * kt);
        Sm.ensure(std::max(n, m) * l);
        count_launch();
        k_fill<<<grid_for(n * l), AUX_NT, 0, s>>>(V.p, n * l, 1.0 / std::sqrt(static_cast<double>(n)));
        count_launch();
        k_pack_w<<<grid_for(n * kt), AUX_NT, 0, s>>>(V.p, n, n, l, kt, nullptr, Wv.p);
        plan_for(P, 0, which == 4 ? MODE_BLOCK_RS : MODE_BLOCK, kt, 8);
        if (which == 4) rr.ensure(n);  // 4: the fused S / r = P~ beta pass of the Newton step
    }
    CK(cudaStreamSynchronize(s));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    // the plain (unculled) sum kernel of this handle's precision
    const int smode = P.precision == 32 ? MODE_SUM_F32 : MODE_SUM;
    TilePlan tsum = plan_for(P, 0, smode, 0);
    auto one = [&]() {
        switch (which) {
            case 0: lse(P, 0, f.p, g.p, G_NONE); break;
            case 1: lse(P, 1, g.p, f.p, G_NONE); break;
            case 2: launch_tiles(tsum, tile_args(P, 0, tsum, G_NONE), s); break;
            default: {
                PassSpec sp;
                sp.dir = 0;
                sp.in_v = f.p;
                sp.in_lw = P.src.lw.p;
                sp.out_v = g.p;
                sp.W = Wv.p;
                sp.k = l;
                sp.kt = kt;
                sp.out = Sm.p;
                if (which == 4) sp.rsum_out = rr.p;
                plan_pass(P, sp);
            }
        }
    };
    one();
    CK(cudaStreamSynchronize(s));
    CK(cudaEventRecord(e0, s));
    for (int t = 0; t < passes; ++t) one();
    CK(cudaEventRecord(e1, s));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    *ms_per_pass = ms / passes;
    if (kernel_ms_per_pass) {
        // the dominant tile kernel alone, on the same stream
        TilePlan tp = which == 1 ? plan_for(P, 1, smode, 0)
                                 : (which >= 3 ? plan_for(P, 0, which == 4 ? MODE_BLOCK_RS : MODE_BLOCK, kt, 8) : tsum);
        TileArgs ta = tile_args(P, which == 1 ? 1 : 0, tp, G_NONE);
        if (which >= 3) ta.W = Wv.p;
        if (which == 4) {
            ta.out_w = P.tgt.w.p;
            ta.rsum = P.rsum.p;
        }
        if (tp.i8) {  // digit tiles of Wv, built by the plan_pass calls above
            ta.vsl = reinterpret_cast<const uint8_t*>(P.vsl.p);
            ta.vexp = reinterpret_cast<const unsigned*>(P.vexp.p);
            ta.kt = kt;
        }
        CK(cudaEventRecord(e0, s));
        for (int t = 0; t < passes; ++t) launch_tiles(tp, ta, s);
        CK(cudaEventRecord(e1, s));
        CK(cudaEventSynchronize(e1));
        CK(cudaEventElapsedTime(&ms, e0, e1));
        *kernel_ms_per_pass = ms / passes;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    CK(cudaGetLastError());
    SKNR_API_END
}

int sknr_bench_iterations(sknr_problem h, const sknr_config* cfg, const double* basis, int64_t basis_ell,
                          int64_t warmup, int64_t iters, int flush_l2, double* ms_per_iter,
                          int64_t* kernels_per_iter) {
    SKNR_API_BEGIN
    Problem& P = get(h);
    std::lock_guard<std::mutex> lk(P.mu);
    const bool use_newton = cfg->newton_enabled && cfg->ell > 0;
    if (use_newton && (basis == nullptr || basis_ell != cfg->ell))
        throw InvalidArgument("solve: ell > 0 requires a basis");
    const int64_t ell = use_newton ? cfg->ell : 0;
    if (P.emu) throw InvalidArgument("sknr_bench_iterations: not available on emulated shards");
    SolveState S;
    prepare_solve(P, S, ell, basis, nullptr, warmup + iters + 1000000, 1e-300, 1, cfg->accept_test);
    cudaStream_t s = P.stream;
    DBuf flush;
    if (flush_l2) flush.ensure((256ull << 20) / sizeof(double));  // 256 MiB > 126 MB L2
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    const int64_t l0 = launch_count();
    enqueue_iteration(P, S, ell, false, 1, false, 0, cfg->accept_test);
    if (kernels_per_iter) *kernels_per_iter = launch_count() - l0;
    CK(cudaStreamEndCapture(s, &graph));
    make_programmatic(graph);
    CK(cudaGraphInstantiate(&exec, graph, 0));
    for (int64_t t = 0; t < std::max<int64_t>(warmup, 1); ++t) CK(cudaGraphLaunch(exec, s));
    CK(cudaStreamSynchronize(s));
    std::vector<cudaEvent_t> ev(2 * iters);
    for (auto& e : ev) CK(cudaEventCreate(&e));
    for (int64_t t = 0; t < iters; ++t) {
        if (flush_l2) CK(cudaMemsetAsync(flush.p, t & 0xFF, flush.n * sizeof(double), s));
        CK(cudaEventRecord(ev[2 * t], s));
        CK(cudaGraphLaunch(exec, s));
        CK(cudaEventRecord(ev[2 * t + 1], s));
    }
    CK(cudaStreamSynchronize(s));
    double total = 0.0;
    for (int64_t t = 0; t < iters; ++t) {
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, ev[2 * t], ev[2 * t + 1]));
        total += ms;
    }
    for (auto& e : ev) cudaEventDestroy(e);
    *ms_per_iter = total / static_cast<double>(std::max<int64_t>(iters, 1));
    cudaGraphExecDestroy(exec);
    cudaGraphDestroy(graph);
    SKNR_API_END
}

// FP64 pipe ceiling on this device: 8 independent DFMA chains per thread, a
// full grid of 148 x 8 CTAs of 256 threads, timed with CUDA events.
__global__ void k_fp64_peak(double* out, int iters, double a0, double b0) {
    SKNR_PDL_ENTRY();
    // per-thread register operands (3 distinct register pairs per DFMA)
    const double a = a0 + threadIdx.x * 1e-12, b = b0 * (1.0 + threadIdx.x * 1e-9);
    double x0 = threadIdx.x * 1e-9, x1 = x0 + 1e-10, x2 = x0 + 2e-10, x3 = x0 + 3e-10;
    double x4 = x0 + 4e-10, x5 = x0 + 5e-10, x6 = x0 + 6e-10, x7 = x0 + 7e-10;
    double y0 = a * 1.5, y1 = a * 1.25, y2 = a * 1.125, y3 = a, y4 = a * 0.5, y5 = a * 0.75, y6 = a * 0.875, y7 = a;
    for (int i = 0; i < iters; ++i) {
        x0 = fma(x0, y0, b); x1 = fma(x1, y1, b); x2 = fma(x2, y2, b); x3 = fma(x3, y3, b);
        x4 = fma(x4, y4, b); x5 = fma(x5, y5, b); x6 = fma(x6, y6, b); x7 = fma(x7, y7, b);
    }
    const double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
    if (s == 12345.678) out[0] = s;
}

// MUFU ex2 ceiling (the fp32 sum pass's bound): 8 independent ex2.approx chains per
// thread over the same full grid.
__global__ void k_mufu_peak(float* out, int iters, float a0) {
    SKNR_PDL_ENTRY();
    float x[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = -1.0f - (threadIdx.x + c) * 1e-6f;
    const float a = a0 + threadIdx.x * 1e-9f;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            float r;
            asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x[c]));
            x[c] = r - a;  // stays in (-1.0, 0): one FADD per ex2 keeps the chain live
        }
    }
    float s = 0.0f;
#pragma unroll
    for (int c = 0; c < 8; ++c) s += x[c];
    if (s == 12345.678f) out[0] = s;
}

int sknr_set_tensor_block_pass(int on) {
    SKNR_API_BEGIN
    set_i8_block_enabled(on != 0);
    SKNR_API_END
}

int sknr_get_tensor_block_pass(void) { return i8_block_enabled() ? 1 : 0; }

int sknr_bench_mufu_peak(double* gex2_per_s, double* ms) {
    SKNR_API_BEGIN
    check_device();
    int sms = 0, dev = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    DBuf out;
    out.ensure(1);
    float* o = reinterpret_cast<float*>(out.p);
    const int iters = 8000, grid = sms * 8, block = 256;
    k_mufu_peak<<<grid, block>>>(o, 100, 1.5f);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0));
    count_launch();
    k_mufu_peak<<<grid, block>>>(o, iters, 1.5f);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float t = 0;
    CK(cudaEventElapsedTime(&t, e0, e1));
    *gex2_per_s = 8.0 * iters * static_cast<double>(grid) * block / (t * 1e-3) / 1e9;
    if (ms) *ms = t;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    SKNR_API_END
}

// Time launch-configuration variant v of the d=2 column-LSE sum kernel on this
// problem's current packed state (tuning aid; see tools/tune_lse.py).
int sknr_tune_variant(sknr_problem h, int variant, int passes, double* kernel_ms) {
    SKNR_API_BEGIN
    Problem& P = get(h);
    std::lock_guard<std::mutex> lk(P.mu);
    const bool anchor = variant >= 400 && variant < 500;  // 4-column anchor pass (stable accept test)
    const bool block = (variant >= 200 && variant < 300) || anchor;
    if ((variant < 100 || variant >= 300) && P.dim != 2) throw InvalidArgument("sknr_tune_variant: needs a d=2 point problem");
    if (variant >= 100 && variant < 200 && P.dim != 0)
        throw InvalidArgument("sknr_tune_variant: needs a stored-cost problem");
    if (block && P.dim != 2) throw InvalidArgument("sknr_tune_variant: needs a d=2 point problem");
    const int64_t n = P.n, m = P.m;
    cudaStream_t s = P.stream;
    DBuf f, g, V, Wv;
    f.ensure(n);
    g.ensure(m);
    count_launch();
    k_fill<<<grid_for(n), AUX_NT, 0, s>>>(f.p, n, 0.0);
    count_launch();
    k_state_init<<<1, 32, 0, s>>>(P.st, 1, 1.0);
    plan_for(P, 0, MODE_SUM, 0);
    plan_for(P, 0, MODE_MAX, 0);
    lse(P, 0, f.p, g.p, G_NONE);
    lse(P, 0, f.p, g.p, G_NONE);  // leaves the bound-shift pack in place
    const int kt = anchor ? 4 : 32;
    TilePlan tp = plan_tiles(P.dim, block ? MODE_BLOCK : MODE_SUM, block ? kt : 0, m, n, block && !anchor ? 8 : 0, variant);
    if (!tp.fn) throw InvalidArgument("sknr_tune_variant: unknown variant");
    P.partial.ensure(static_cast<size_t>(tp.n_in_blocks) * m * (block ? kt : 1));
    TileArgs ta = tile_args(P, 0, tp, G_NONE);
    if (block) {
        V.ensure(n * kt);
        Wv.ensure(n * kt);
        count_launch();
        k_fill<<<grid_for(n * kt), AUX_NT, 0, s>>>(Wv.p, n * kt, 1.0 / std::sqrt(static_cast<double>(n)));
        ta.W = Wv.p;
        P.rsum.ensure(static_cast<size_t>(tp.n_out_tiles) * n);  // for the fused-r variants
        ta.out_w = P.tgt.w.p;
        ta.rsum = P.rsum.p;
    }
    launch_tiles(tp, ta, s);
    CK(cudaStreamSynchronize(s));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0, s));
    for (int t = 0; t < passes; ++t) launch_tiles(tp, ta, s);
    CK(cudaEventRecord(e1, s));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    *kernel_ms = ms / passes;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    CK(cudaGetLastError());
    SKNR_API_END
}

// Diagnostics: the first 16 entries of the handle's reduction scratch (sums of the last
// stopping test / acceptance test / gauge).
int sknr_debug_sums(sknr_problem h, double* out) {
    SKNR_API_BEGIN
    Problem& P = get(h);
    CK(cudaMemcpyAsync(out, P.sums.p, sizeof(double) * 16, cudaMemcpyDeviceToHost, P.stream));
    CK(cudaStreamSynchronize(P.stream));
    SKNR_API_END
}

// Diagnostics: [exact col, exact row, retry col, retry row] counters since creation.
int sknr_debug_counters(sknr_problem h, int64_t* out) {
    SKNR_API_BEGIN
    Problem& P = get(h);
    CK(cudaMemcpyAsync(P.st_host, P.st, sizeof(DevState), cudaMemcpyDeviceToHost, P.stream));
    CK(cudaStreamSynchronize(P.stream));
    out[0] = static_cast<int64_t>(P.st_host->n_exact[0]);
    out[1] = static_cast<int64_t>(P.st_host->n_exact[1]);
    out[2] = static_cast<int64_t>(P.st_host->n_retry[0]);
    out[3] = static_cast<int64_t>(P.st_host->n_retry[1]);
    out[4] = static_cast<int64_t>(P.st_host->n_cull_tested);
    out[5] = static_cast<int64_t>(P.st_host->n_cull_kept);
    SKNR_API_END
}

int sknr_bench_fp64_peak(double* tflops, double* ms) {
    SKNR_API_BEGIN
    check_device();
    int sms = 0, dev = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    DBuf out;
    out.ensure(1);
    const int iters = 16000, grid = sms * 8, block = 256;
    k_fp64_peak<<<grid, block>>>(out.p, 100, 0.5, 1e-7);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0));
    count_launch();
    k_fp64_peak<<<grid, block>>>(out.p, iters, 0.5, 1e-7);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float t = 0;
    CK(cudaEventElapsedTime(&t, e0, e1));
    const double flops = 2.0 * 8.0 * iters * static_cast<double>(grid) * block;
    *tflops = flops / (t * 1e-3) / 1e12;
    if (ms) *ms = t;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    SKNR_API_END
}

// ---------------------------------------------------------------- multi-GPU (row sharding)
int sknr_comm_unique_id(unsigned char id[128]) {
    SKNR_API_BEGIN
    g_nccl.load();
    ncclUniqueId uid;
    NK(g_nccl.GetUniqueId(&uid));
    std::memcpy(id, uid.internal, NCCL_UNIQUE_ID_BYTES);
    SKNR_API_END
}

int sknr_comm_init(int rank, int world, const unsigned char id[128], int device) {
    SKNR_API_BEGIN
    if (world < 1 || rank < 0 || rank >= world) throw InvalidArgument("sknr_comm_init: bad rank/world");
    check_device();
    if (device >= 0) CK(cudaSetDevice(device));
    g_nccl.load();
    if (g_comm.comm) {
        g_nccl.CommDestroy(g_comm.comm);
        g_comm.comm = nullptr;
    }
    ncclUniqueId uid;
    std::memcpy(uid.internal, id, NCCL_UNIQUE_ID_BYTES);
    NK(g_nccl.CommInitRank(&g_comm.comm, world, uid, rank));
    g_comm.rank = rank;
    g_comm.world = world;
    SKNR_API_END
}

// Testing: an in-process group of `world` emulated ranks on the current GPU (see
// EmuGroup). Shards created afterwards route their collectives through it; each
// rank's calls must come from its own host thread.
int sknr_comm_init_emulated(int world) {
    SKNR_API_BEGIN
    if (world < 1 || world > kEmuMax) throw InvalidArgument("sknr_comm_init_emulated: 1 <= world <= 16 required");
    check_device();
    g_emu.init(world);
    SKNR_API_END
}

int sknr_comm_destroy(void) {
    SKNR_API_BEGIN
    g_emu.destroy();
    if (g_comm.comm) {
        g_nccl.CommDestroy(g_comm.comm);
        g_comm.comm = nullptr;
    }
    g_comm.world = 1;
    g_comm.rank = 0;
    SKNR_API_END
}

// Keep only this rank's source rows; column partials, the gauge scalar, the
// marginal residuals and the Newton inner products are merged with NCCL.
int sknr_problem_shard(sknr_problem h, int64_t row_begin, int64_t row_end) {
    SKNR_API_BEGIN
    Problem& P = get(h);
    std::lock_guard<std::mutex> lk(P.mu);
    const bool emu = g_emu.world > 0;
    if (!g_comm.comm && !emu) throw RuntimeFailure("sknr_problem_shard: call sknr_comm_init first");
    if (P.shard) throw InvalidArgument("sknr_problem_shard: problem already sharded");
    const int world = emu ? g_emu.world : g_comm.world;
    int rank = emu ? -1 : g_comm.rank;
    if (emu)  // the emulated rank is the one whose standard block this is
        for (int r = 0; r < world; ++r) {
            int64_t rb, re;
            row_partition(P.n_global, world, r, rb, re);
            if (rb == row_begin && re == row_end) rank = r;
        }
    int64_t b = 0, e = 0;
    if (rank >= 0) row_partition(P.n_global, world, rank, b, e);
    if (rank < 0 || row_begin != b || row_end != e)
        throw InvalidArgument("sknr_problem_shard: rows must follow the standard partition [n*r/R, n*(r+1)/R)");
    const int64_t nl = e - b, n = P.n_global, m = P.m;
    if (nl < 1) throw InvalidArgument("sknr_problem_shard: empty row block");
    cudaStream_t s = P.stream;
    auto slice = [&](DBuf& buf, int64_t cols) {
        if (!buf.p) return;
        DBuf tmp;
        tmp.ensure(nl * cols);
        for (int64_t c = 0; c < cols; ++c)
            CK(cudaMemcpyAsync(tmp.p + c * nl, buf.p + c * n + b, sizeof(double) * nl, cudaMemcpyDeviceToDevice, s));
        CK(cudaStreamSynchronize(s));
        std::swap(buf.p, tmp.p);
        std::swap(buf.n, tmp.n);
    };
    slice(P.src.w, 1);
    slice(P.src.lw, 1);
    slice(P.src.sw, 1);
    slice(P.src.lsw, 1);
    slice(P.src.sq, 1);
    slice(P.src.coords, P.d);
    if (P.C.p) {
        DBuf c2, ct2;
        c2.ensure(nl * m);
        ct2.ensure(nl * m);
        CK(cudaMemcpy2DAsync(c2.p, sizeof(double) * nl, P.C.p + b, sizeof(double) * n, sizeof(double) * nl, m,
                             cudaMemcpyDeviceToDevice, s));
        CK(cudaMemcpyAsync(ct2.p, P.CT.p + b * m, sizeof(double) * nl * m, cudaMemcpyDeviceToDevice, s));
        CK(cudaStreamSynchronize(s));
        std::swap(P.C.p, c2.p);
        std::swap(P.C.n, c2.n);
        std::swap(P.CT.p, ct2.p);
        std::swap(P.CT.n, ct2.n);
    }
    P.src.count = nl;
    P.n = nl;
    P.row_begin = b;
    P.shard = true;
    P.emu = emu;
    P.rank = rank;
    P.world = world;
    P.plans.clear();
    if (P.cull_ready) {  // re-derive the Morton order and group boxes for the local rows
        P.cull_ready = false;
        prepare_culling(P);
    }
    count_launch();
    k_invalidate_refs<<<1, 32, 0, s>>>(P.st);
    CK(cudaStreamSynchronize(s));
    SKNR_API_END
}

}  // extern "C"

