// sknr_device.cuh -- device-side building blocks shared by every sm_100a kernel.
//
// Scaled log domain. Every O(nm) kernel evaluates a cell exponent
//   E_ij = la_i + (f_i - C_ij)/eps - s_j        (core.cpp:47-50, natural log)
// in units of 1/256 of a binary order of magnitude: u = LS * E, LS = 256 log2(e).
// The host-side prep folds all per-row / per-column terms into two vectors A
// (inputs) and B (outputs) and, for point clouds, scales the coordinates by
// sigma = sqrt(2 LS kappa / eps) so that
//   u = A_in + B_out + <X_in, Y_out>           (on-the-fly cost: 1 DADD + d DFMA)
//   u = A_in + B_out - (LS/eps) * C[out,in]     (stored cost: 1 DADD + 1 DFMA)
// and exp(E) = 2^(u/256) is evaluated by pexp() below in 8 FP64 issue slots:
// Cody-Waite rounding against the biased magic constant 1.5*2^52 + 1023*256
// (3 DADD), a degree-4 polynomial for 2^(r/256), |r| <= 1/2 (4 DFMA,
// truncation < 4e-17), and a 256-entry table of 2^(e/256) whose biased
// exponent field (k>>8)+1023 is OR-ed in with integer ops (no FP64 slot).
// The table is stored with the exponent field cleared (and the hi word pre-biased
// by -(e << (20 - kTB)), see pexp_parts) and replicated 16x in shared memory, so the 16 lanes of each half-warp hit 16 distinct 8-byte bank
// pairs: a warp's table read is always the minimum 2 wavefronts.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace sknr {

// Programmatic dependent launch: the solver's graphs join consecutive kernel nodes with
// programmatic edges (make_programmatic in engine.cu), so a kernel can be scheduled while
// its predecessor drains. Every kernel therefore first waits for its prerequisite grids
// to complete (their writes visible), then lets its own dependents begin launching.
// Both instructions are no-ops for a kernel launched without a programmatic dependency.
#define SKNR_PDL_ENTRY() asm volatile("griddepcontrol.wait;\n\tgriddepcontrol.launch_dependents;" ::: "memory")


// Table resolution: SKNR_TB = 8 -> 256 entries x 16 replicas (32 KiB), degree-4
// polynomial (11 FP64 slots per cell); SKNR_TB = 10 -> 1024 entries x 8 replicas
// (64 KiB), degree-3 minimax polynomial (10 slots per cell).
#ifndef SKNR_TB
#define SKNR_TB 8
#endif
constexpr int kTB = SKNR_TB;
#if SKNR_TB == 10
constexpr double kLS = 1477.3197218702985;       // 1024 * log2(e)
constexpr double kInvLS = 1.0 / 1477.3197218702985;
constexpr double kMagicB = 6755399442103296.0;   // 1.5 * 2^52 + 1023 * 1024
constexpr int kKcMax = 2046 * 1024 + 1023;
constexpr int kTabRep = 8;
// minimax-adjusted coefficients of 2^(r/1024), |r| <= 1/2 (max rel. error 1.4e-16)
constexpr double kP1 = 0.0006769015435155716;
constexpr double kP2 = 2.29097851993791e-07;
constexpr double kP3 = 5.1692229383458926e-11;
constexpr double kP4 = 0.0;
#else
constexpr double kLS = 369.3299304675746;       // 256 * log2(e)
constexpr double kInvLS = 1.0 / 369.3299304675746;
constexpr double kMagicB = 6755399441317632.0;  // 1.5 * 2^52 + 1023 * 256
constexpr int kKcMax = 2046 * 256 + 255;        // largest biased k before the exponent field overflows
constexpr int kTabRep = 16;
// (ln2/256)^k / k!
constexpr double kP1 = 0.0027076061740622863;
constexpr double kP2 = 3.6655655969101062e-06;
constexpr double kP3 = 3.3083026805413713e-09;
constexpr double kP4 = 2.239395190875157e-12;
#endif
constexpr int kMagicHi = 0x43380000;            // hi word of 1.5 * 2^52
constexpr int kTabEntries = 1 << kTB;
constexpr int kTabWords = kTabEntries * kTabRep;
constexpr int kRepShift = (kTabRep == 16) ? 7 : 6;  // log2(kTabRep * 8 bytes)

// Device flags / scalars of one problem handle. Kernels consult them through
// a guard word so a whole iteration can live in one CUDA graph: work that is
// not needed this time exits at its first instruction.
struct DevState {
    int done;          // solve finished: every guarded kernel is a no-op
    int iter_active;   // this iteration started before `done` was set
    int conv;          // converged flag of the current solve
    int newton_ok;     // Newton step alive (attempted and factorisation ok)
    int accept;        // Newton candidate accepted
    int attempted;     // Newton attempted this iteration
    int need_exact[2]; // LSE direction needs the exact max pass (0 col, 1 row)
    int retry[2];      // bound-shift validation failed -> redo exact
    int ref_valid[2];  // a previous LSE of this direction can seed the shift
    long long iter;        // current iteration index (1-based)
    long long max_iter;
    unsigned long long t_iter0;  // globaltimer at iteration start
    double tol;
    double c_gauge;
    double gap_l2, gap_inf;
    double q0, q1;
    double dmax[2], dmin[2];     // max/min of (in - ref_in) per direction
    double scratch[16];
    unsigned int counters[32];   // last-block tickets of fused reductions
    unsigned long long n_exact[2];  // diagnostics: exact-shift passes per direction
    unsigned long long n_retry[2];  // diagnostics: bound-shift validation failures
    unsigned long long n_cull_tested, n_cull_kept;  // diagnostics: culling group tests / kept groups
    // stable accept test (sknr_config.accept_test = 1): dQ = a.d + b.(h' - h), see engine_solver.cuh
    int lit;            // this step falls back to the literal Q1 > Q0 test (max|d| > lit_dmax)
    double lit_dmax;    // largest max|f' - f| the stable evaluation takes (600 eps)
    double adq;         // a.(f' - f) of the current step
    long long trace_base;  // iteration index of the device trace buffer's first slot (chunked trace)
};

enum Guard : unsigned {
    G_NONE = 0,
    G_DONE = 1u,        // skip when st->done
    G_NEWTON = 2u,      // skip unless st->newton_ok
    G_EXACT0 = 4u,      // skip unless st->need_exact[0]
    G_EXACT1 = 8u,      // skip unless st->need_exact[1]
    G_RETRY0 = 16u,     // skip unless st->retry[0]
    G_RETRY1 = 32u,     // skip unless st->retry[1]
    G_ACTIVE = 64u,     // skip unless st->iter_active
    G_ACCEPT = 128u,    // skip unless st->accept
    G_LIT = 256u,       // skip unless st->lit (stable accept test fell back to literal)
    G_NOLIT = 512u,     // skip if st->lit
};

__device__ __forceinline__ bool guard_skip(const DevState* st, unsigned g) {
    if (g == 0u) return false;
    if ((g & G_DONE) && st->done) return true;
    if ((g & G_NEWTON) && !st->newton_ok) return true;
    if ((g & G_EXACT0) && !st->need_exact[0]) return true;
    if ((g & G_EXACT1) && !st->need_exact[1]) return true;
    if ((g & G_RETRY0) && !st->retry[0]) return true;
    if ((g & G_RETRY1) && !st->retry[1]) return true;
    if ((g & G_ACTIVE) && !st->iter_active) return true;
    if ((g & G_ACCEPT) && !st->accept) return true;
    if ((g & G_LIT) && !st->lit) return true;
    if ((g & G_NOLIT) && st->lit) return true;
    return false;
}

// Polynomial coefficients and the magic constant as constant-bank operands:
// DFMA/DADD read c[bank][offset] directly, so the loop carries no UMOV
// re-materialisations of uniform registers. Defined in tile_kernels.cu.
static __constant__ double c_pexp_k[6] = {kMagicB, kP1, kP2, kP3, kP4, 0.0};

// Split evaluation 2^(u/256) = T' * p. `tab` = shared replicated table,
// `laneoff` = (lane & 15) * 8 bytes, `c3` = kP3 held in a register by the caller
// (the first Horner step has two constant operands and would otherwise
// rematerialise one per cell). Terms below 2^-1022 come out as 0 / subnormal;
// HI_CLAMP caps terms at 2^1023 for passes whose exponents are not bounded
// above by construction.
// FASTCLAMP: clamp the biased exponent with one IMNMX instead of ISETP+SEL;
// valid only while |u| < 2^31 (callers guarantee it from the exponent range).
template <bool HI_CLAMP, bool FASTCLAMP = false>
__device__ __forceinline__ void pexp_parts(double u, const unsigned long long* __restrict__ tab,
                                           unsigned laneoff, double c3, double& Tp, double& p) {
    const double t = u + c_pexp_k[0];
    const double kf = t - c_pexp_k[0];
    const double r = u - kf;
#if SKNR_TB == 10
    p = fma(r, c_pexp_k[3], c3);  // c3 holds kP2 in a register
    p = fma(p, r, c_pexp_k[1]);
    p = fma(p, r, 1.0);
#else
    p = fma(r, c_pexp_k[4], c3);
    p = fma(p, r, c_pexp_k[2]);
    p = fma(p, r, c_pexp_k[1]);
    p = fma(p, r, 1.0);
#endif
    int kc = FASTCLAMP ? max(__double2loint(t), 0)
                       : ((__double2hiint(t) >= kMagicHi) ? __double2loint(t) : 0);
    if (HI_CLAMP) kc = min(kc, kKcMax);
    const unsigned off = ((static_cast<unsigned>(kc) << kRepShift) & (((1u << kTB) - 1u) << kRepShift)) | laneoff;
    const uint2 T = *reinterpret_cast<const uint2*>(reinterpret_cast<const char*>(tab) + off);
    // hi word = biased exponent (kc >> kTB) << 20 | mantissa bits of 2^(e/2^kTB), e = kc mod 2^kTB.
    // The table's hi words are stored minus e << (20 - kTB) (load_exp2_table), so one IMAD
    // kc * 2^(20 - kTB) + T.y assembles it (the e part cancels; arithmetic mod 2^32).
    Tp = __hiloint2double(static_cast<int>(static_cast<unsigned>(kc) * (1u << (20 - kTB)) + T.y),
                          static_cast<int>(T.x));
}

// register-resident first Horner constant for pexp_parts
__device__ __forceinline__ double pexp_c3() {
#if SKNR_TB == 10
    double v = kP2;
#else
    double v = kP3;
#endif
    asm volatile("" : "+d"(v));
    return v;
}

template <bool HI_CLAMP>
__device__ __forceinline__ double pexp(double u, const unsigned long long* __restrict__ tab,
                                       unsigned laneoff, double c3) {
    double Tp, p;
    pexp_parts<HI_CLAMP>(u, tab, laneoff, c3, Tp, p);
    return Tp * p;
}

template <bool HI_CLAMP, bool FASTCLAMP = false>
__device__ __forceinline__ double pexp_acc(double u, const unsigned long long* __restrict__ tab,
                                           unsigned laneoff, double c3, double acc) {
    double Tp, p;
    pexp_parts<HI_CLAMP, FASTCLAMP>(u, tab, laneoff, c3, Tp, p);
    return fma(Tp, p, acc);
}

// Keeps a constant in a register (opaque to constant propagation).
__device__ __forceinline__ double reg_const(double v) {
    asm volatile("" : "+d"(v));
    return v;
}

// Atomic max/min on doubles (exact and order independent, hence deterministic).
__device__ __forceinline__ void atomic_max_double(double* addr, double v) {
    unsigned long long* a = reinterpret_cast<unsigned long long*>(addr);
    unsigned long long old = *a;
    while (__longlong_as_double(static_cast<long long>(old)) < v) {
        const unsigned long long prev =
            atomicCAS(a, old, static_cast<unsigned long long>(__double_as_longlong(v)));
        if (prev == old) break;
        old = prev;
    }
}

__device__ __forceinline__ void atomic_min_double(double* addr, double v) {
    unsigned long long* a = reinterpret_cast<unsigned long long*>(addr);
    unsigned long long old = *a;
    while (__longlong_as_double(static_cast<long long>(old)) > v) {
        const unsigned long long prev =
            atomicCAS(a, old, static_cast<unsigned long long>(__double_as_longlong(v)));
        if (prev == old) break;
        old = prev;
    }
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

}  // namespace sknr
