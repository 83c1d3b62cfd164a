// sknr_b200.hpp -- header-only C++ facade over the C ABI (sknr_gpu.h) that keeps
// the reference's namespace-sknr API (proj/include/sknr/{types,core,objective,
// spectral,solver}.hpp): same type names, same function names and argument
// meaning, same exceptions (std::invalid_argument with the reference's
// messages, sknr::EigensolverError carrying best_residual, std::runtime_error).
//
// Differences a caller sees, all forced by this image or by the GPU design:
//  * Vector / Matrix are small Eigen-free column-major containers (Eigen3 is
//    absent here). With Eigen available, pass .data() of VectorXd / MatrixXd
//    (both column-major) -- the layout is identical.
//  * EotProblem owns a device-resident handle; with_epsilon() re-uploads the
//    cost like the reference copies it (types.hpp:60-62); set_epsilon() is the
//    copy-free variant.
//  * SolveResult::coupling is materialised only on request (coupling_from);
//    the reference always builds the n x m plan at the end of solve.
#pragma once

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "sknr_gpu.h"

namespace sknr {

using Index = std::int64_t;

struct Vector {
    std::vector<double> v;
    Vector() = default;
    explicit Vector(Index n, double fill = 0.0) : v(static_cast<size_t>(n), fill) {}
    Vector(std::initializer_list<double> l) : v(l) {}
    Index size() const { return static_cast<Index>(v.size()); }
    double* data() { return v.data(); }
    const double* data() const { return v.data(); }
    double& operator[](Index i) { return v[static_cast<size_t>(i)]; }
    double operator[](Index i) const { return v[static_cast<size_t>(i)]; }
};

struct Matrix {  // column-major like Eigen::MatrixXd
    Index r = 0, c = 0;
    std::vector<double> v;
    Matrix() = default;
    Matrix(Index rows, Index cols, double fill = 0.0)
        : r(rows), c(cols), v(static_cast<size_t>(rows * cols), fill) {}
    Index rows() const { return r; }
    Index cols() const { return c; }
    double* data() { return v.data(); }
    const double* data() const { return v.data(); }
    double& operator()(Index i, Index j) { return v[static_cast<size_t>(i + j * r)]; }
    double operator()(Index i, Index j) const { return v[static_cast<size_t>(i + j * r)]; }
};

class EigensolverError : public std::runtime_error {
public:
    EigensolverError(const std::string& msg, double best_residual)
        : std::runtime_error(msg), best_residual_(best_residual) {}
    double best_residual() const { return best_residual_; }

private:
    double best_residual_;
};

namespace detail {
inline void check(int rc) {
    if (rc == SKNR_OK) return;
    const std::string msg = sknr_last_error();
    if (rc == SKNR_EINVAL) throw std::invalid_argument(msg);
    if (rc == SKNR_EEIGEN) throw EigensolverError(msg, sknr_last_best_residual());
    throw std::runtime_error(msg);
}
struct HandleDeleter {
    void operator()(sknr_problem_s* p) const { sknr_problem_destroy(p); }
};
}  // namespace detail

class DiscreteMeasure {
public:
    explicit DiscreteMeasure(Vector weights) : w_(std::move(weights)) {}
    Index size() const { return w_.size(); }
    const Vector& weights() const { return w_; }

private:
    Vector w_;
};

class CostMatrix {
public:
    explicit CostMatrix(Matrix entries) : c_(std::move(entries)) {}
    Index rows() const { return c_.rows(); }
    Index cols() const { return c_.cols(); }
    const Matrix& entries() const { return c_; }

private:
    Matrix c_;
};

// EotProblem (types.hpp:47-69) backed by a device handle.
class EotProblem {
public:
    EotProblem(CostMatrix cost, DiscreteMeasure alpha, DiscreteMeasure beta, double epsilon)
        : cost_(std::move(cost)), alpha_(std::move(alpha)), beta_(std::move(beta)), eps_(epsilon) {
        if (alpha_.size() != cost_.rows() || beta_.size() != cost_.cols())
            throw std::invalid_argument("EotProblem: measure sizes must match cost shape");
        sknr_problem h = nullptr;
        detail::check(sknr_problem_create_dense(cost_.entries().data(), cost_.rows(), cost_.cols(),
                                                alpha_.weights().data(), beta_.weights().data(), eps_,
                                                &h));
        h_ = std::shared_ptr<sknr_problem_s>(h, detail::HandleDeleter());
    }
    Index n() const { return cost_.rows(); }
    Index m() const { return cost_.cols(); }
    const Matrix& cost() const { return cost_.entries(); }
    const DiscreteMeasure& alpha() const { return alpha_; }
    const DiscreteMeasure& beta() const { return beta_; }
    double epsilon() const { return eps_; }
    EotProblem with_epsilon(double epsilon) const { return EotProblem(cost_, alpha_, beta_, epsilon); }
    void set_epsilon(double epsilon) {
        detail::check(sknr_problem_set_epsilon(h_.get(), epsilon));
        eps_ = epsilon;
    }
    sknr_problem handle() const { return h_.get(); }

private:
    CostMatrix cost_;
    DiscreteMeasure alpha_, beta_;
    double eps_;
    std::shared_ptr<sknr_problem_s> h_;
};

struct Potentials {
    Vector f, g;
};
struct Coupling {
    Matrix plan;
};

struct SpectralBasis {
    Matrix vectors, vectors_sym;
    Vector rhos;
    double epsilon_built_at = 0.0;
    Index ell() const { return vectors.cols(); }
    Index dim() const { return vectors.rows(); }
};

struct SolverConfig {
    double tol_omega = 1e-9;
    Index max_iter = 100000;
    Index ell = 0;
    bool newton_enabled = true;
    bool trace_enabled = true;
};

struct IterationRecord {
    Index index = 0;
    double marginal_error = 0.0, marginal_error_inf = 0.0, semi_dual_value = 0.0;
    bool newton_attempted = false, newton_accepted = false;
    double wall_time_ms = 0.0;
};

struct SolveResult {
    Potentials potentials;
    bool converged = false;
    Index iterations = 0;
    std::vector<IterationRecord> trace;
};

enum class WarmMode { none, potentials, spectral };
struct AnnealSchedule {
    std::vector<double> epsilons;
    WarmMode warm_mode = WarmMode::none;
    bool refresh_basis = false;
};

// ---- core.hpp
inline Vector ctransform_of_f(const EotProblem& p, const Vector& f) {
    if (f.size() != p.n()) throw std::invalid_argument("ctransform_of_f: length mismatch");
    Vector g(p.m());
    detail::check(sknr_ctransform_of_f(p.handle(), f.data(), g.data()));
    return g;
}
inline Vector ctransform_of_g(const EotProblem& p, const Vector& g) {
    if (g.size() != p.m()) throw std::invalid_argument("ctransform_of_g: length mismatch");
    Vector f(p.n());
    detail::check(sknr_ctransform_of_g(p.handle(), g.data(), f.data()));
    return f;
}
inline Coupling coupling_from(const EotProblem& p, const Potentials& pots) {
    Coupling c{Matrix(p.n(), p.m())};
    detail::check(sknr_coupling(p.handle(), pots.f.data(), pots.g.data(), c.plan.data()));
    return c;
}
struct PlanMarginals {
    Vector row, col;
};
struct MarginalGap {
    double l2, inf;
};
inline PlanMarginals plan_marginals(const EotProblem& p, const Potentials& pots) {
    PlanMarginals out{Vector(p.n()), Vector(p.m())};
    double l2 = 0, inf = 0;
    detail::check(sknr_plan_marginals(p.handle(), pots.f.data(), pots.g.data(), out.row.data(),
                                      out.col.data(), &l2, &inf));
    return out;
}

// ---- objective.hpp
inline double semi_dual_value(const EotProblem& p, const Vector& f) {
    double v = 0;
    detail::check(sknr_semi_dual_value(p.handle(), f.data(), &v));
    return v;
}
struct RestrictedDerivatives {
    Vector grad;
    Matrix hess;
};
inline RestrictedDerivatives restricted_derivatives_with_transform(const EotProblem& p, const Vector& f,
                                                                   const Vector& g,
                                                                   const SpectralBasis& basis) {
    if (basis.dim() != p.n())
        throw std::invalid_argument("restricted_derivatives: basis dimension mismatch");
    if (basis.ell() < 1) throw std::invalid_argument("restricted_derivatives: empty basis");
    RestrictedDerivatives d{Vector(basis.ell()), Matrix(basis.ell(), basis.ell())};
    detail::check(sknr_restricted_derivatives(p.handle(), f.data(), g.data(), basis.vectors.data(),
                                              basis.ell(), d.grad.data(), d.hess.data()));
    return d;
}
inline RestrictedDerivatives restricted_derivatives(const EotProblem& p, const Vector& f,
                                                    const SpectralBasis& basis) {
    return restricted_derivatives_with_transform(p, f, ctransform_of_f(p, f), basis);
}

// ---- spectral.hpp
inline SpectralBasis top_modes(const EotProblem& p, const Potentials& anchor, Index ell,
                               double tol = 1e-8, Index max_power_iters = -1) {
    SpectralBasis b{Matrix(p.n(), ell), Matrix(p.n(), ell), Vector(ell), p.epsilon()};
    detail::check(sknr_top_modes(p.handle(), anchor.f.data(), anchor.g.data(), ell, tol, max_power_iters,
                                 b.vectors.data(), b.vectors_sym.data(), b.rhos.data(), nullptr));
    return b;
}

// ---- solver.hpp
inline SolveResult solve(const EotProblem& p, const SolverConfig& config,
                         const SpectralBasis* basis = nullptr, const Potentials* init = nullptr) {
    sknr_config c;
    sknr_config_default(&c);
    c.tol_omega = config.tol_omega;
    c.max_iter = config.max_iter;
    c.ell = config.ell;
    c.newton_enabled = config.newton_enabled ? 1 : 0;
    c.trace_enabled = config.trace_enabled ? 1 : 0;
    if (config.newton_enabled && config.ell > 0 && basis && basis->dim() != p.n())
        throw std::invalid_argument("solve: basis dimension mismatch");
    if (init && (init->f.size() != p.n() || init->g.size() != p.m()))
        throw std::invalid_argument("solve: init potential sizes mismatch");
    SolveResult r;
    r.potentials.f = Vector(p.n());
    r.potentials.g = Vector(p.m());
    const Index cap = config.trace_enabled ? config.max_iter : 0;
    std::vector<sknr_record> recs(static_cast<size_t>(cap > 0 ? cap : 1));
    int64_t iters = 0, tlen = 0;
    int conv = 0;
    detail::check(sknr_solve(p.handle(), &c, basis ? basis->vectors.data() : nullptr,
                             basis ? basis->ell() : 0, init ? init->f.data() : nullptr,
                             init ? init->g.data() : nullptr, r.potentials.f.data(), r.potentials.g.data(),
                             &iters, &conv, recs.data(), cap, &tlen));
    r.iterations = iters;
    r.converged = conv != 0;
    for (int64_t t = 0; t < tlen && t < cap; ++t) {
        const sknr_record& s = recs[static_cast<size_t>(t)];
        r.trace.push_back(IterationRecord{s.index, s.marginal_error, s.marginal_error_inf, s.semi_dual_value,
                                          s.newton_attempted != 0, s.newton_accepted != 0, s.wall_time_ms});
    }
    return r;
}

inline std::vector<SolveResult> anneal(const EotProblem& p, const AnnealSchedule& schedule,
                                       const SolverConfig& config) {
    const Index S = static_cast<Index>(schedule.epsilons.size());
    sknr_config c;
    sknr_config_default(&c);
    c.tol_omega = config.tol_omega;
    c.max_iter = config.max_iter;
    c.ell = config.ell;
    c.newton_enabled = config.newton_enabled ? 1 : 0;
    c.trace_enabled = config.trace_enabled ? 1 : 0;
    std::vector<double> F(static_cast<size_t>(S * p.n())), G(static_cast<size_t>(S * p.m()));
    std::vector<int64_t> iters(static_cast<size_t>(S)), offs(static_cast<size_t>(S));
    std::vector<int> conv(static_cast<size_t>(S));
    const Index cap = config.trace_enabled ? config.max_iter * S : 0;
    std::vector<sknr_record> recs(static_cast<size_t>(cap > 0 ? cap : 1));
    int64_t tlen = 0;
    const int warm = schedule.warm_mode == WarmMode::none ? 0 : schedule.warm_mode == WarmMode::potentials ? 1 : 2;
    detail::check(sknr_anneal(p.handle(), schedule.epsilons.data(), S, warm, schedule.refresh_basis ? 1 : 0, &c,
                              F.data(), G.data(), iters.data(), conv.data(), recs.data(), cap, offs.data(),
                              &tlen));
    std::vector<SolveResult> out(static_cast<size_t>(S));
    for (Index s = 0; s < S; ++s) {
        SolveResult& r = out[static_cast<size_t>(s)];
        r.potentials.f.v.assign(F.begin() + s * p.n(), F.begin() + (s + 1) * p.n());
        r.potentials.g.v.assign(G.begin() + s * p.m(), G.begin() + (s + 1) * p.m());
        r.iterations = iters[static_cast<size_t>(s)];
        r.converged = conv[static_cast<size_t>(s)] != 0;
        const int64_t hi = s + 1 < S ? offs[static_cast<size_t>(s + 1)] : tlen;
        for (int64_t t = offs[static_cast<size_t>(s)]; t < hi && t < cap; ++t) {
            const sknr_record& q = recs[static_cast<size_t>(t)];
            r.trace.push_back(IterationRecord{q.index, q.marginal_error, q.marginal_error_inf, q.semi_dual_value,
                                              q.newton_attempted != 0, q.newton_accepted != 0, q.wall_time_ms});
        }
    }
    return out;
}

}  // namespace sknr
