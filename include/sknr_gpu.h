/*
 * sknr_gpu.h -- C ABI of the B200-native SK-NR(ell) core (libsknr_b200.so).
 *
 * Drop-in boundary for the reference's C++ solver API in namespace sknr
 * (/root/reference/proj/include/sknr/{types,core,objective,spectral,solver}.hpp).
 * Plain pointers and sizes only; all matrices are COLUMN-MAJOR doubles exactly
 * like the reference's Eigen::MatrixXd (types.hpp:10-12), so an Eigen caller
 * passes .data() zero-copy. Host buffers are owned by the caller; device
 * memory is owned by the problem handle. A handle owns one CUDA stream and is
 * not thread-safe; concurrent solves use separate handles (the reference's
 * "concurrent solves on a shared read-only problem", maps to
 * one handle per thread).
 *
 * Every entry point returns an sknr_status. On failure sknr_last_error()
 * returns the message (thread-local). Invalid-argument messages repeat the
 * reference's std::invalid_argument texts verbatim so the C++ facade
 * (include/sknr_b200.hpp) can rethrow the same exception with the same what().
 * There is no CPU fallback: without a usable sm_100 device every compute call
 * fails with SKNR_ECUDA.
 */
#ifndef SKNR_GPU_H
#define SKNR_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    SKNR_OK = 0,
    SKNR_EINVAL = 1,   /* std::invalid_argument in the reference            */
    SKNR_EEIGEN = 2,   /* EigensolverError (spectral.hpp:60-68)              */
    SKNR_ECUDA = 3,    /* CUDA failure / no device / extension unusable      */
    SKNR_ENCCL = 4,    /* NCCL failure (multi-GPU row sharding)              */
    SKNR_ERUNTIME = 5, /* std::runtime_error (e.g. anneal stage wrapping)    */
    SKNR_EINTERNAL = 9
} sknr_status;

typedef struct sknr_problem_s* sknr_problem;

/* Last error message of the calling thread ("" if none). */
const char* sknr_last_error(void);
/* best_residual carried by the last SKNR_EEIGEN (EigensolverError::best_residual). */
double sknr_last_best_residual(void);
/* Library / device description, e.g. "sknr_b200 0.1.0 sm_100a (NVIDIA B200, 148 SMs)". */
int sknr_version(char* buf, int cap);
/* Number of kernel launches this process issued (evidence for bench "gpu_launches"). */
int64_t sknr_kernel_launch_count(void);

/* ---------------------------------------------------------------- problems
 * sknr_problem_create_dense replaces EotProblem(CostMatrix, DiscreteMeasure,
 * DiscreteMeasure, eps) (types.hpp:47-69, types.cpp:7-43): validates weights
 * (w>0 finite, |sum-1|<=1e-12), cost finiteness and eps>0 with the same
 * messages, and uploads cost (n x m col-major) once.
 *
 * sknr_problem_create_points is the on-the-fly variant the north star asks
 * for: C_ij = cost_scale * ||x_i - y_j||^2 (sq_euclidean_cost,
 * generators.cpp:94-103) is never stored; x is n x d, y is m x d (col-major,
 * like harness::PointCloud::points, generators.hpp:12-19). cost_scale=1/maxC
 * reproduces BASELINE C2's max-normalised cost.
 *
 * Row sharding (north star): with a communicator attached
 * (sknr_problem_attach_comm) the handle holds only rows [row_begin, row_end)
 * of the source side; the C ABI still takes and returns FULL-length host
 * vectors (every rank passes identical inputs and receives identical outputs).
 */
int sknr_problem_create_dense(const double* cost, int64_t n, int64_t m, const double* alpha,
                              const double* beta, double epsilon, sknr_problem* out);
int sknr_problem_create_points(const double* x, const double* y, int64_t n, int64_t m,
                               int64_t d, double cost_scale, const double* alpha,
                               const double* beta, double epsilon, sknr_problem* out);
/* cost_mode: 0 auto (d <= 4: cost evaluated in registers; d > 4: stored on
 * device if 2 n m doubles fit, else on the fly), 1 stored, 2 on the fly (d > 4:
 * the x.y contraction runs on FP64 tensor cores, mma.sync m8n8k4). */
int sknr_problem_create_points_ex(const double* x, const double* y, int64_t n, int64_t m,
                                  int64_t d, double cost_scale, const double* alpha,
                                  const double* beta, double epsilon, int cost_mode,
                                  sknr_problem* out);
/* EotProblem::with_epsilon (types.hpp:60-62) without the dense-cost copy. */
int sknr_problem_set_epsilon(sknr_problem p, double epsilon);
int sknr_problem_info(sknr_problem p, int64_t* n, int64_t* m, int64_t* d, double* epsilon,
                      int* kind /* 0 stored cost, 1 on the fly (registers), 2 on the fly (DMMA) */);
int sknr_problem_destroy(sknr_problem p);
/* Opt-in culling of negligible terms in the column/row LSE passes (not in the
 * reference): both clouds are visited in Morton order and a (64-input group,
 * 256-output group) pair is skipped when a rigorous bound puts every one of its
 * terms below e^-threshold of the output's total (threshold >= 40, typically 60;
 * 0 turns culling off). Point clouds with d <= 4 (sharded handles cull their own
 * rows). The sums change by less than n e^-threshold relative (< 1e-21 at 60). */
int sknr_problem_set_culling(sknr_problem p, double threshold);
/* Opt-in reduced precision of the column/row LSE sum passes (not in the reference,
 * which is fp64 throughout; BASELINE north star "1e-5 if an fp32 variant is
 * offered"): bits = 32 evaluates each cell's exponent in fp32 and its exp2 on the
 * MUFU unit (accumulation, shifts, potentials and every other pass stay fp64);
 * bits = 64 (default) restores the fp64 path bit for bit. Point clouds with
 * d <= 4; combines with culling (the kept groups in fp32). The cell exponent is
 * re-expanded around the squared distance with the potential terms on a 2^-8 grid
 * (exact fp32 sums), so the fp32 rounding is a fixed perturbation of the kernel
 * (<= 2e-5 per term): the solver still converges to tol in its own marginals and the
 * potentials stay within ~1e-6 relative of the fp64 path. */
int sknr_problem_set_precision(sknr_problem p, int bits);

/* ---------------------------------------------------------------- core.hpp
 * core.hpp:16-43 / core.cpp:35-150 on host buffers (upload, device kernels,
 * download). */
int sknr_ctransform_of_f(sknr_problem p, const double* f, double* g);
int sknr_ctransform_of_g(sknr_problem p, const double* g, double* f);
int sknr_plan_marginals(sknr_problem p, const double* f, const double* g, double* row,
                        double* col, double* gap_l2, double* gap_inf);
/* coupling_from (core.cpp:84-103): n x m col-major into a host buffer. On a row-sharded
 * handle: this rank's rows only (n_local x m), f full length. */
int sknr_coupling(sknr_problem p, const double* f, const double* g, double* plan);
/* Rows [row_begin, row_end) of the same plan, col-major with leading dimension
 * row_end - row_begin: lets a caller stream an n x m coupling (e.g. the CLI's
 * coupling.csv, main.cpp:149-154) without holding it whole. Row-sharded handle: global row
 * indices inside this rank's block [row_begin, row_begin + n_local) (sknr_problem_shard). */
int sknr_coupling_rows(sknr_problem p, const double* f, const double* g, int64_t row_begin, int64_t row_end,
                       double* plan_rows);

/* ---------------------------------------------------------------- objective.hpp */
int sknr_semi_dual_value(sknr_problem p, const double* f, double* value);
/* restricted_derivatives_with_transform (objective.cpp:110-142); g = f^{C,eps}. */
int sknr_restricted_derivatives(sknr_problem p, const double* f, const double* g,
                                const double* vectors /* n x ell */, int64_t ell,
                                double* grad /* ell */, double* hess /* ell x ell */);
/* dual_value (objective.cpp:10-40): a.f + b.g - eps*expm1(log sum_ij a_i b_j e^{(f_i+g_j-C_ij)/eps}). */
int sknr_dual_value(sknr_problem p, const double* f, const double* g, double* value);
/* full_semi_dual_hessian (objective.cpp:150-171): the dense n x n semi-dual Hessian
 * -(1/eps)(diag(r) - P~ diag(b) P~^T), symmetrised, at g = f^{C,eps}; SKNR_EINVAL when
 * n > dense_limit (the reference's guard). The plan and the n^2 m product run on the device. */
int sknr_full_semi_dual_hessian(sknr_problem p, const double* f, int64_t dense_limit, double* hess);
/* semi_dual_hessian_quadform (objective.cpp:53-77): u^T H(f) u. */
int sknr_semi_dual_hessian_quadform(sknr_problem p, const double* f, const double* u, double* value);

/* ---------------------------------------------------------------- spectral.hpp
 * SinkhornOperator::apply_sym_block / apply_sym_t_block (spectral.cpp:68-102)
 * and top_modes (spectral.cpp:125-193). Returns SKNR_EEIGEN with
 * sknr_last_best_residual() when the residual target is not met. */
/* SinkhornOperator::apply_R / apply_Rt (spectral.cpp:29-62):
 * (R g1)_i = sum_j e^{(f_i+g_j-C_ij)/eps} b_j g1_j ; (R^T f1)_j = sum_i e^{..} a_i f1_i.
 * apply_K(f1, g1) = (apply_R(g1), apply_Rt(f1)) (spectral.cpp:64-66). */
int sknr_apply_R(sknr_problem p, const double* f, const double* g, const double* g1, double* out /* n */);
int sknr_apply_Rt(sknr_problem p, const double* f, const double* g, const double* f1, double* out /* m */);
int sknr_apply_sym_block(sknr_problem p, const double* f, const double* g,
                         const double* v /* m x k */, int64_t k, double* out /* n x k */);
int sknr_apply_sym_t_block(sknr_problem p, const double* f, const double* g,
                           const double* u /* n x k */, int64_t k, double* out /* m x k */);
int sknr_top_modes(sknr_problem p, const double* f, const double* g, int64_t ell, double tol,
                   int64_t max_power_iters /* -1: 500*ell */, double* vectors /* n x ell */,
                   double* vectors_sym /* n x ell */, double* rhos /* ell */,
                   int64_t* sweeps /* may be NULL */);

/* spectrum_report (spectral.cpp:195-228): rhos, (1-rho)/eps, (1+rho)/eps; with
 * include_vectors, vectors_f (n x k) and vectors_g (m x k). Needs 1 <= k <= min(n,m)-1. */
int sknr_spectrum_report(sknr_problem p, const double* f, const double* g, int64_t k, int include_vectors,
                         double tol, int64_t max_power_iters, double* rhos, double* hess_low,
                         double* hess_high, double* vectors_f, double* vectors_g);
/* projector_distance (spectral.cpp:230-242) between two n x k symmetrized bases. */
int sknr_projector_distance(int64_t n, int64_t k, const double* a_sym, const double* b_sym, double* out);

/* Opt-in accelerated variants (not in the reference): method 1 = Chebyshev-
 * filtered subspace iteration of polynomial degree `degree`; method 2 = restarted
 * block Lanczos with `degree` blocks per cycle (full reorthogonalisation). Same
 * residual test and returned basis semantics as method 0 (= top_modes). `sweeps`
 * counts operator applications R~R~^T. */
int sknr_top_modes_ex(sknr_problem p, const double* f, const double* g, int64_t ell, double tol,
                      int64_t max_power_iters, int method, int degree, double* vectors,
                      double* vectors_sym, double* rhos, int64_t* sweeps);

/* ---------------------------------------------------------------- solver.hpp */
typedef struct {
    double tol_omega;      /* 1e-9   (SolverConfig, solver.hpp:13-19) */
    int64_t max_iter;      /* 100000 */
    int64_t ell;           /* 0 = vanilla SK */
    int32_t newton_enabled;/* 1 */
    int32_t trace_enabled; /* 1 */
    int32_t exact_marginals; /* 0: column marginal from the fused transform
                                (beta_j expm1((g_j-h_j)/eps)); 1: explicit
                                plan-sum passes as core.cpp:120-143 */
    int32_t accept_test;   /* Newton accept test of try_newton (solver.cpp:46-47).
                              0 (default, the reference): Q(f') > Q(f) with both values
                              evaluated in full -- once the step's gain falls below
                              ulp(Q) the decision is rounding noise on any platform.
                              1 (stable): the same predicate as dQ = Q(f') - Q(f) > 0,
                              dQ = a.d + b.(h' - h), d = f' - f, h'_j - h_j =
                              -eps log1p(sum_i P~_ij expm1(d_i/eps) / sum_i P~_ij) at the
                              anchor h = f^{C,eps}: rounding scales with the step, so
                              decisions are reproducible (steps with max|d| > 600 eps
                              use the literal test). */
} sknr_config;

void sknr_config_default(sknr_config* c);

typedef struct {
    int64_t index;
    double marginal_error;      /* L2-sum rule, core.cpp:145-150 */
    double marginal_error_inf;
    double semi_dual_value;
    int32_t newton_attempted;
    int32_t newton_accepted;
    double wall_time_ms;        /* device globaltimer per iteration */
} sknr_record;

/* solve (solver.cpp:71-156). basis: n x ell potential-coordinate vectors
 * (SpectralBasis::vectors) or NULL; init_f/init_g both NULL or both set.
 * trace may be NULL (trace_cap 0); trace_len returns the full length. */
int sknr_solve(sknr_problem p, const sknr_config* cfg, const double* basis, int64_t basis_ell,
               const double* init_f, const double* init_g, double* f_out, double* g_out,
               int64_t* iterations, int* converged, sknr_record* trace, int64_t trace_cap,
               int64_t* trace_len);

/* The full trace of the last sknr_solve / sknr_anneal on this handle (concatenated over
 * anneal stages): lets a caller size its record array from the trace_len the solve
 * returned instead of from max_iter (the reference push_back()s the iterations run). */
int sknr_last_trace(sknr_problem p, sknr_record* trace, int64_t cap, int64_t* len);

/* Batched solve (not in the reference): `count` independent
 * problems (any sizes / cost kinds, distinct unsharded handles) solved with the
 * same config in one device loop -- one CUDA graph per iteration with one
 * concurrent branch per problem. Per-problem arrays: bases[b] (n_b x ell, or
 * bases NULL when ell = 0), init_f[b]/init_g[b] (both arrays NULL or both set),
 * f_out[b], g_out[b]; iterations[count], converged[count]. Results equal the
 * one-by-one sknr_solve bit for bit. No trace. */
int sknr_solve_batch(const sknr_problem* problems, int64_t count, const sknr_config* cfg,
                     const double* const* bases, int64_t basis_ell, const double* const* init_f,
                     const double* const* init_g, double* const* f_out, double* const* g_out,
                     int64_t* iterations, int* converged);

/* Small-problem batch (not in the reference): `count` point-cloud problems of one
 * dimension d <= 4 with n, m <= 8192 (d <= 2), 6224 (d = 3), 4979 (d = 4), each
 * solved by plain SK (ell = 0) from f = 0 to tol inside a single kernel launch (no
 * launch per iteration): one CTA per problem when the batch fills the GPU, a
 * cooperative group of CTAs per problem when it does not (count = 1 is the
 * low-latency single solve). Per
 * problem q: n[q], m[q], x[q] (n x d), y[q] (m x d), a[q], b[q], eps[q],
 * cost_scale[q] (NULL: 1); outputs f_out[q], g_out[q], iterations[q], converged[q].
 * Same iteration and stopping test as sknr_solve; sums in a different order. */
int sknr_solve_small_batch(int64_t count, int64_t d, const int64_t* n, const int64_t* m,
                           const double* const* x, const double* const* y, const double* const* a,
                           const double* const* b, const double* eps, const double* cost_scale,
                           double tol, int64_t max_iter, double* const* f_out, double* const* g_out,
                           int64_t* iterations, int* converged);

/* newton_step (solver.cpp:59-69, try_newton :30-56): one restricted Newton step
 * from f with basis vectors (n x ell). f_out = accepted ? f + V delta : f. */
int sknr_newton_step(sknr_problem p, const double* f, const double* vectors, int64_t ell, double* f_out,
                     int* accepted, int* factorization_failed);
/* Same with the accept test selected as in sknr_config.accept_test (0 literal, 1 stable). */
int sknr_newton_step_ex(sknr_problem p, const double* f, const double* vectors, int64_t ell, int accept_test,
                        double* f_out, int* accepted, int* factorization_failed);

/* anneal (solver.cpp:158-222). warm_mode 0 none, 1 potentials, 2 spectral.
 * Per stage s: f_out[s*n ..], g_out[s*m ..], iterations[s], converged[s];
 * trace records are concatenated, stage s starting at trace_offsets[s]. */
int sknr_anneal(sknr_problem p, const double* epsilons, int64_t stages, int warm_mode,
                int refresh_basis, const sknr_config* cfg, double* f_out, double* g_out,
                int64_t* iterations, int* converged, sknr_record* trace, int64_t trace_cap,
                int64_t* trace_offsets, int64_t* trace_len);

/* ---------------------------------------------------------------- measurement
 * Runs `passes` back-to-back transforms on device-resident data (no host
 * copies) and reports the mean device time per pass (CUDA events on the
 * handle's stream). which: 0 column LSE (ctransform_of_f), 1 row LSE
 * (ctransform_of_g), 2 fixed-shift column sum pass (the steady-state kernel),
 * 3 Newton restricted-derivative pass, 4 top_modes block pass. */
int sknr_bench_pass(sknr_problem p, int which, int64_t ell, int passes, double* ms_per_pass,
                    double* kernel_ms_per_pass);
/* Runs `warmup` untimed then `iters` timed SK-NR iterations (stopping test
 * disabled) on device-resident state, one CUDA graph per iteration; each timed
 * iteration is bracketed by CUDA events on the handle's stream and, with
 * flush_l2, preceded (untimed) by a 256 MiB memset that evicts the 126 MB L2.
 * Returns mean device ms per iteration and the kernel count of one iteration's
 * graph; bench.py's "value" leg. */
int sknr_bench_iterations(sknr_problem p, const sknr_config* cfg, const double* basis,
                          int64_t basis_ell, int64_t warmup, int64_t iters, int flush_l2,
                          double* ms_per_iter, int64_t* kernels_per_iter);

/* Measured FP64 FMA ceiling of the current device (TFLOP/s, FMA = 2 flops):
 * the denominator of the on-the-fly roofline (MEASURED_PEAKS.json has no FP64 entry). */
int sknr_bench_fp64_peak(double* tflops, double* ms);
/* Measured MUFU ex2.approx.f32 ceiling (G ex2/s): the denominator of the fp32 roofline. */
int sknr_bench_mufu_peak(double* gex2_per_s, double* ms);
/* Tuning aid: device ms of launch variant `variant` of the d=2 column-LSE sum
 * kernel on this problem (tools/tune_lse.py). */
int sknr_tune_variant(sknr_problem p, int variant, int passes, double* kernel_ms);
/* Newton block pass S = V^T P~, r = P~ beta (objective.cpp:127-131) on the tensor cores:
 * tcgen05 int8 GEMMs over exact byte slices of P~ and V (i8_kernels.cu), on by default
 * for point clouds (d <= 4), ell <= 32 and n*m >= 2^22; 0 selects the FP64 DMMA pass.
 * Process-wide; applies to plans made afterwards (each setting keeps its own plans). */
int sknr_set_tensor_block_pass(int on);
int sknr_get_tensor_block_pass(void);
/* Testing aid: D[128][n] = A[128][k] (uint8, row-major) x B (int8, given as Bt[n][k]) with
 * one tcgen05.mma.kind::i8 per 32 inputs, in the block pass's operand layouts (A MN-major,
 * B K-major); 32 <= n <= 256 and 32 <= k <= 256, multiples of 32. Returns 0 on success. */
int sknr_probe_i8_mma(const uint8_t* A, const int8_t* Bt, int n, int k, int32_t* D);
/* Diagnostics: out[0..3] = exact-shift passes (column, row), bound-shift
 * validation failures that triggered the exact retry (column, row); out[4..5] =
 * culling group tests and kept groups (sknr_problem_set_culling). */
int sknr_debug_counters(sknr_problem p, int64_t* out /* 6 */);

/* ---------------------------------------------------------------- multi-GPU
 * One process per GPU. Rank 0 calls sknr_comm_unique_id, the id travels over
 * any side channel (torch.distributed in bench.py), every rank calls
 * sknr_comm_init with the same id. Problems created afterwards with
 * sknr_problem_shard() keep only their row block; column (max,sum) partials,
 * Krylov inner products and the gauge scalar are merged with NCCL over
 * NVLink. NCCL is loaded with dlopen at sknr_comm_init (RTLD_NOLOAD first, so
 * the copy torch already mapped is reused). */
int sknr_comm_unique_id(unsigned char id[128]);
int sknr_comm_init(int rank, int world, const unsigned char id[128], int device);
/* Testing aid: an in-process group of `world` emulated ranks on the current GPU.
 * Shards created after this call exchange their collectives in-process (one host
 * thread per rank, eager launches ordered by stream events); sknr_comm_destroy
 * ends it. Used to check the sharded path at R > 1 on a single GPU. */
int sknr_comm_init_emulated(int world);
int sknr_comm_destroy(void);
/* Collectives this process issued for sharded handles since the last reset: calls and
 * payload bytes (allreduce counts once per call with its buffer size; a row gather
 * counts the full gathered vector). reset != 0 zeroes the counters after reading. */
int sknr_comm_stats(int64_t* calls, int64_t* bytes, int reset);
/* Restrict a freshly created problem to rows [row_begin,row_end) of this rank
 * under the attached communicator. */
int sknr_problem_shard(sknr_problem p, int64_t row_begin, int64_t row_end);

#ifdef __cplusplus
}
#endif

#endif /* SKNR_GPU_H */
