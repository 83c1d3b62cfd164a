// Compiles against the C++ facade exactly like a reference caller of
// namespace sknr would (solve / top_modes / anneal), linking libsknr_b200.so.
#include <cmath>
#include <cstdio>

#include "sknr_b200.hpp"

int main() {
    using namespace sknr;
    const Index n = 64, m = 48;
    Matrix cost(n, m);
    for (Index j = 0; j < m; ++j)
        for (Index i = 0; i < n; ++i) cost(i, j) = std::pow((i / double(n)) - (j / double(m)), 2.0);
    Vector a(n, 1.0 / n), b(m, 1.0 / m);
    try {
        EotProblem problem(CostMatrix(cost), DiscreteMeasure(a), DiscreteMeasure(b), 0.05);
        SolverConfig cfg;
        SolveResult warm = solve(problem.with_epsilon(0.1), cfg);
        SpectralBasis basis = top_modes(problem.with_epsilon(0.1), warm.potentials, 4);
        cfg.ell = 4;
        SolveResult r = solve(problem, cfg, &basis, &warm.potentials);
        std::printf("converged=%d iters=%lld marginal_error=%.3e\n", int(r.converged),
                    static_cast<long long>(r.iterations), r.trace.empty() ? 0.0 : r.trace.back().marginal_error);
        // the rest of the reference surface: operator, spectrum, objective, Newton step
        const SinkhornOperator op = build_operator(problem, r.potentials);
        const auto k = op.apply_K(Vector(n, 1.0), Vector(m, 1.0));
        const SpectrumReport rep = spectrum_report(problem, r.potentials, 3, true);
        const double dist = projector_distance(basis, top_modes(op, 4));
        const NewtonOutcome step = newton_step(problem, sk_sweep(problem, r.potentials).f, basis);
        const double gap = dual_value(problem, r.potentials) - semi_dual_value(problem, r.potentials.f);
        std::printf("R1[0]=%.6f Rt1[0]=%.6f rho1=%.6f dist=%.3e newton_accepted=%d dual_gap=%.2e osc=%.4f\n",
                    k.first[0], k.second[0], rep.rhos[0], dist, int(step.accepted), gap,
                    osc_norm(r.potentials.f));
        return r.converged ? 0 : 2;
    } catch (const std::exception& e) {
        std::printf("error: %s\n", e.what());
        return 1;
    }
}
