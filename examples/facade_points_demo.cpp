// SK-NR(ell) on two point clouds through the C++ facade, the way a reference caller
// builds a problem from harness::PointCloud's (proj/tools/main.cpp:57-112) -- but with
// the cost evaluated on the fly on the device instead of the dense n x m matrix of
// main.cpp:86 (BASELINE C4: 65536^2 doubles would be 32 GiB).
//
//   facade_points_demo DIR [stable|literal] [cull]
//
// DIR holds x.bin (n x d), y.bin (m x d), a.bin (n), b.bin (m) as raw column-major
// doubles and meta.txt = "n m d eps eps_warm ell". The solve follows the north-star
// protocol: SK to 1e-9 at eps_warm, top_modes (block Lanczos, 12 blocks per cycle)
// at that anchor, then SK-NR(ell) at eps from the warm potentials. Writes f.bin,
// g.bin and prints one line per stage.
#include <chrono>
#include <cstdio>
#include <fstream>
#include <string>

#include "sknr_b200.hpp"

static sknr::Matrix read_matrix(const std::string& path, sknr::Index rows, sknr::Index cols) {
    sknr::Matrix out(rows, cols);
    std::ifstream in(path, std::ios::binary);
    if (!in.read(reinterpret_cast<char*>(out.data()), static_cast<std::streamsize>(sizeof(double) * rows * cols)))
        throw std::runtime_error("cannot read " + path);
    return out;
}

static sknr::Vector read_vector(const std::string& path, sknr::Index n) {
    sknr::Matrix m = read_matrix(path, n, 1);
    sknr::Vector v(n);
    for (sknr::Index i = 0; i < n; ++i) v[i] = m(i, 0);
    return v;
}

static void write_vector(const std::string& path, const sknr::Vector& v) {
    std::ofstream out(path, std::ios::binary);
    out.write(reinterpret_cast<const char*>(v.data()), static_cast<std::streamsize>(sizeof(double) * v.size()));
}

int main(int argc, char** argv) {
    using namespace sknr;
    using Clock = std::chrono::steady_clock;
    if (argc < 2) {
        std::fprintf(stderr, "usage: %s DIR [stable|literal] [cull]\n", argv[0]);
        return 1;
    }
    const std::string dir = argv[1];
    const bool stable = argc > 2 && std::string(argv[2]) == "stable";
    const bool cull = argc > 3 && std::string(argv[3]) == "cull";
    try {
        Index n = 0, m = 0, d = 0, ell = 0;
        double eps = 0, eps_warm = 0;
        {
            std::ifstream meta(dir + "/meta.txt");
            if (!(meta >> n >> m >> d >> eps >> eps_warm >> ell)) throw std::runtime_error("bad meta.txt");
        }
        harness::PointCloud src{read_matrix(dir + "/x.bin", n, d), DiscreteMeasure(read_vector(dir + "/a.bin", n))};
        harness::PointCloud tgt{read_matrix(dir + "/y.bin", m, d), DiscreteMeasure(read_vector(dir + "/b.bin", m))};
        EotProblem warm_problem(src, tgt, eps_warm);
        if (cull) warm_problem.set_culling(60.0);
        SolverConfig cfg;
        cfg.trace_enabled = false;
        auto t0 = Clock::now();
        const SolveResult warm = solve(warm_problem, cfg);
        auto t1 = Clock::now();
        std::printf("warm: eps=%g converged=%d iterations=%lld (%.3f s)\n", eps_warm, int(warm.converged),
                    static_cast<long long>(warm.iterations), std::chrono::duration<double>(t1 - t0).count());
        const SpectralBasis basis =
            top_modes(warm_problem, warm.potentials, ell, 1e-8, -1, TopModesMethod::lanczos, 12);
        auto t2 = Clock::now();
        std::printf("basis: ell=%lld rho1=%.12f (%.3f s)\n", static_cast<long long>(ell), basis.rhos[0],
                    std::chrono::duration<double>(t2 - t1).count());
        EotProblem problem = warm_problem.with_epsilon(eps);
        cfg.ell = ell;
        cfg.trace_enabled = true;
        cfg.accept_test = stable ? AcceptTest::stable : AcceptTest::literal;
        const SolveResult r = solve(problem, cfg, &basis, &warm.potentials);
        auto t3 = Clock::now();
        int accepts = 0;
        for (const IterationRecord& rec : r.trace) accepts += rec.newton_accepted ? 1 : 0;
        std::printf("main: eps=%g converged=%d iterations=%lld accepts=%d marginal_error=%.6e (%.3f s)\n", eps,
                    int(r.converged), static_cast<long long>(r.iterations), accepts,
                    r.trace.empty() ? 0.0 : r.trace.back().marginal_error,
                    std::chrono::duration<double>(t3 - t2).count());
        write_vector(dir + "/f.bin", r.potentials.f);
        write_vector(dir + "/g.bin", r.potentials.g);
        return r.converged ? 0 : 2;
    } catch (const std::exception& e) {
        std::printf("error: %s\n", e.what());
        return 1;
    }
}
