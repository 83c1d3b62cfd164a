// sknr_device.cuh -- device-side building blocks shared by every sm_100a kernel.
//
// Scaled log domain. Every O(nm) kernel evaluates a cell exponent
//   E_ij = la_i + (f_i - C_ij)/eps - s_j        (core.cpp:47-50, natural log)
// in units of 1/64 of a binary order of magnitude: u = L64 * E, L64 = 64 log2(e).
// The host-side prep folds all per-row / per-column terms into two vectors A
// (inputs) and B (outputs) and, for point clouds, scales the coordinates by
// sigma = sqrt(2 L64 kappa / eps) so that
//   u = A_in + B_out + <X_in, Y_out>           (on-the-fly cost, d FMAs)
//   u = A_in + B_out - (L64/eps) * C[out,in]    (stored cost, 1 FMA)
// and exp(E) = 2^(u/64) is evaluated by pexp() below: Cody-Waite rounding with
// the 1.5*2^52 magic constant (3 DADD), a degree-5 polynomial for 2^(r/64),
// |r| <= 1/2 (5 DFMA, truncation < 4e-17), and a 64-entry table of 2^(e/64)
// whose exponent field absorbs k>>6 with integer adds (no FP64 slot). The
// table lives in shared memory replicated 16x so the 16 lanes of each
// half-warp hit 16 distinct 8-byte bank pairs: a warp-wide table read costs the
// minimum 2 wavefronts regardless of the index pattern.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace sknr {

constexpr double kL64 = 92.33248261689366;      // 64 * log2(e)
constexpr double kInvL64 = 1.0 / 92.33248261689366;
constexpr double kMagic = 6755399441055744.0;   // 1.5 * 2^52
constexpr long long kMagicBits = 0x4338000000000000LL;
constexpr int kKmin = -64000;                   // 2^-1000: below, a term is flushed to 0
constexpr int kKmax = 64000;                    // 2^+1000: above, +inf (unshifted passes only)
constexpr int kTabRep = 16;
constexpr int kTabDoubles = 64 * kTabRep;

// (ln2/64)^k / k!
constexpr double kP1 = 0.010830424696249145;
constexpr double kP2 = 5.86490495505617e-05;
constexpr double kP3 = 2.1173137155464776e-07;
constexpr double kP4 = 5.732851688640402e-10;
constexpr double kP5 = 1.2417843701716925e-12;

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
    return false;
}

// Split evaluation: 2^(u/64) = T' * p. `tabl` = shared table + (lane & 15).
// HI_CLAMP adds the +inf branch for unshifted passes whose exponents are not
// bounded above by construction.
template <bool HI_CLAMP>
__device__ __forceinline__ void pexp_parts(double u, const double* __restrict__ tabl, double& Tp,
                                           double& p) {
    const double t = u + kMagic;
    const double kf = t - kMagic;
    const double r = u - kf;
    p = fma(r, kP5, kP4);
    p = fma(p, r, kP3);
    p = fma(p, r, kP2);
    p = fma(p, r, kP1);
    p = fma(p, r, 1.0);
    const long long tb = __double_as_longlong(t);
    const int k = static_cast<int>(tb);
    const double T = tabl[(k & 63) << 4];
    int hi = __double2hiint(T) + ((k >> 6) << 20);
    hi = (tb >= kMagicBits + kKmin) ? hi : 0;
    int lo = __double2loint(T);
    if (HI_CLAMP) {
        const bool over = tb > kMagicBits + kKmax;
        hi = over ? 0x7FF00000 : hi;
        lo = over ? 0 : lo;
    }
    Tp = __hiloint2double(hi, lo);
}

template <bool HI_CLAMP>
__device__ __forceinline__ double pexp(double u, const double* __restrict__ tabl) {
    double Tp, p;
    pexp_parts<HI_CLAMP>(u, tabl, Tp, p);
    return Tp * p;
}

template <bool HI_CLAMP>
__device__ __forceinline__ double pexp_acc(double u, const double* __restrict__ tabl, double acc) {
    double Tp, p;
    pexp_parts<HI_CLAMP>(u, tabl, Tp, p);
    return fma(Tp, p, acc);
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
