// tile_kernels.cu -- the O(nm) hot loop of SK-NR(ell) on sm_100a.
//
// One persistent-kernel family covers every pass the reference spends its
// time in:
//   MODE_SUM   partial[ib][o]      = sum_{in in block ib} 2^(u/64)
//              -> column LSE ctransform_of_f (core.cpp:35-54), row LSE
//                 ctransform_of_g (core.cpp:56-82), plan marginals
//                 (core.cpp:120-143), r = P~ beta (objective.cpp:127-128)
//   MODE_MAX   partial[ib][o]      = max_{in} u        (exact shift, core.cpp:47)
//   MODE_BLOCK partial[ib][c][o]   = sum_{in} 2^(u/256) W[in][c]
//              -> S = V^T P~ (objective.cpp:131), R~^T X / R~ Z for top_modes
//                 (spectral.cpp:68-102)
// "in" is the reduced index, "o" the output index; the column transform runs
// with o=j,in=i and the row transform with o=i,in=j over the same kernel.
//
// Work decomposition: a tile is (output tile of NT*JT consecutive outputs) x
// (input block). Each thread owns JT outputs in registers (B, Y) and streams
// the block's inputs through shared memory in chunks (broadcast reads). Tiles
// are dealt round-robin to a persistent grid sized to the resident-CTA count
// of the 148 SMs; the input blocks give deterministic split-K partials that
// the finalize kernels merge in fixed order (no floating-point atomics, so
// reruns are bitwise identical).
//
// Stored cost: the output index is the contiguous one (C for the row
// transform, C^T for the column transform), so a warp's 32 loads of one input
// are one coalesced 256 B request and every fp64 cost element is read once per
// pass: 8 B/cell, the HBM roofline of BASELINE.md section 4.
#include <atomic>
#include <cstdlib>

#include "internal.h"

namespace sknr {

__constant__ unsigned long long c_exp2_tab[kTabEntries] = {
#if SKNR_TB == 10
#include "exp2_table1024.inc"
#else
#include "exp2_table.inc"
#endif
};

#if SKNR_TB != 10
// 2^(e/1024) mantissas for the 1024-entry LSE sum kernel (pts_sum10_kernel)
__constant__ unsigned long long c_exp2_tab10[1024] = {
#include "exp2_table1024.inc"
};
#else
#define c_exp2_tab10 c_exp2_tab
#endif

// 2^(e/4096) mantissas for the 4096-entry LSE sum kernel (pts_sum12_kernel); global
// memory (32 KiB would crowd the constant bank), copied into shared memory per CTA
__device__ const unsigned long long g_exp2_tab12[4096] = {
#include "exp2_table4096.inc"
};

// Fill the replicated table: tab[e*kTabRep + r] = mantissa bits of 2^(e/2^kTB).
// The hi word is pre-biased by -(e << (20 - kTB)) (mod 2^32) so that pexp_parts assembles
// exponent and mantissa with one IMAD.
__device__ __forceinline__ void load_exp2_table(unsigned long long* tab, int tid, int nthreads) {
    for (int t = tid; t < kTabWords; t += nthreads) {
        const unsigned e = static_cast<unsigned>(t / kTabRep);
        const unsigned long long v = c_exp2_tab[e];
        const unsigned hi = static_cast<unsigned>(v >> 32) - (e << (20 - kTB));
        tab[t] = (static_cast<unsigned long long>(hi) << 32) | (v & 0xFFFFFFFFull);
    }
}

namespace {

// threads per CTA: 256 for the sum/max passes (the 32 KiB exp2 table is then
// shared by 8 warps and 4 CTAs fit per SM), 128 for the register-heavy block passes
template <int MODE>
struct NT_of {
    static constexpr int value = MODE == MODE_BLOCK ? 128 : 256;
};

template <int D>
struct PK_of {
    static constexpr int value = ((D + 2) / 2) * 2;  // A + D coords, padded to even
};

template <int MODE, int KT>
struct Chunk {
    // inputs staged per shared-memory round
    static constexpr int value = (MODE == MODE_BLOCK) ? (KT > 32 ? 32 : 64) : 256;
};

template <int MODE, int KA>
__device__ __forceinline__ void acc_init(double* acc) {
#pragma unroll
    for (int c = 0; c < KA; ++c)
        acc[c] = (MODE == MODE_MAX) ? -__longlong_as_double(0x7FF0000000000000LL) : 0.0;
}

// ------------------------------------------------------------- point clouds
template <int D, int JT, int MODE, int KT, int NTT = NT_of<MODE>::value, int UNR = 2, bool FASTCLAMP = false,
          int MINB = 1>
__global__ void __launch_bounds__(NTT, MINB) pts_tile_kernel(TileArgs a) {
    SKNR_PDL_ENTRY();
    if (guard_skip(a.st, a.guard)) return;
    constexpr int NT = NTT;
    constexpr int PK = PK_of<D>::value;
    constexpr int CH = Chunk<MODE, KT>::value;
    constexpr int KA = KT > 0 ? KT : 1;
    extern __shared__ __align__(16) double sm[];
    unsigned long long* tab = reinterpret_cast<unsigned long long*>(sm);
    double* sin = sm + kTabWords;
    double* sw = sin + CH * PK;
    const int tid = threadIdx.x;
    load_exp2_table(tab, tid, NT);
    const unsigned laneoff = (tid & (kTabRep - 1)) << 3;
    const double c3 = pexp_c3();
    const int64_t out_tile = static_cast<int64_t>(NT) * JT;

    for (int64_t tile = blockIdx.x; tile < a.n_tiles; tile += gridDim.x) {
        const int64_t ot = tile % a.n_out_tiles, ib = tile / a.n_out_tiles;
        double B[JT], Y[JT][D];
        double acc[JT][KA];
        int64_t o[JT];
#pragma unroll
        for (int jt = 0; jt < JT; ++jt) {
            o[jt] = ot * out_tile + jt * NT + tid;
            const int64_t oc = o[jt] < a.n_out ? o[jt] : a.n_out - 1;
            B[jt] = a.out_pack[oc * PK];
#pragma unroll
            for (int d = 0; d < D; ++d) Y[jt][d] = a.out_pack[oc * PK + 1 + d];
            acc_init<MODE, KA>(acc[jt]);
        }
        const int64_t i0 = ib * a.in_block;
        const int64_t i1 = (i0 + a.in_block < a.n_in) ? i0 + a.in_block : a.n_in;
        for (int64_t c0 = i0; c0 < i1; c0 += CH) {
            const int cnt = static_cast<int>((i1 - c0) < CH ? (i1 - c0) : CH);
            __syncthreads();
            {
                const double2* src = reinterpret_cast<const double2*>(a.in_pack + c0 * PK);
                double2* dst = reinterpret_cast<double2*>(sin);
                for (int t = tid; t < cnt * PK / 2; t += NT) dst[t] = src[t];
                if (MODE == MODE_BLOCK) {
                    const double2* wsrc = reinterpret_cast<const double2*>(a.W + c0 * KA);
                    double2* wdst = reinterpret_cast<double2*>(sw);
                    for (int t = tid; t < cnt * KA / 2; t += NT) wdst[t] = wsrc[t];
                }
            }
            __syncthreads();
#pragma unroll UNR
            for (int k = 0; k < cnt; ++k) {
                double x[PK];
#pragma unroll
                for (int q = 0; q < PK / 2; ++q) {
                    const double2 v = reinterpret_cast<const double2*>(sin + k * PK)[q];
                    x[2 * q] = v.x;
                    x[2 * q + 1] = v.y;
                }
#pragma unroll
                for (int jt = 0; jt < JT; ++jt) {
                    double u = x[0] + B[jt];
#pragma unroll
                    for (int d = 0; d < D; ++d) u = fma(x[1 + d], Y[jt][d], u);
                    if (MODE == MODE_SUM) {
                        acc[jt][0] = pexp_acc<false, FASTCLAMP>(u, tab, laneoff, c3, acc[jt][0]);
                    } else if (MODE == MODE_MAX) {
                        acc[jt][0] = fmax(acc[jt][0], u);
                    } else {
                        const double e = pexp<true>(u, tab, laneoff, c3);
#pragma unroll
                        for (int c = 0; c < KA; c += 2) {
                            const double2 w = reinterpret_cast<const double2*>(sw + k * KA)[c / 2];
                            acc[jt][c] = fma(e, w.x, acc[jt][c]);
                            acc[jt][c + 1] = fma(e, w.y, acc[jt][c + 1]);
                        }
                    }
                }
            }
        }
#pragma unroll
        for (int jt = 0; jt < JT; ++jt) {
            if (o[jt] >= a.n_out) continue;
            if (MODE == MODE_BLOCK) {
#pragma unroll
                for (int c = 0; c < KA; ++c) a.partial[(ib * KA + c) * a.n_out + o[jt]] = acc[jt][c];
            } else {
                a.partial[ib * a.n_out + o[jt]] = acc[jt][0];
            }
        }
    }
}

// ------------------------------------------------------------- LSE sum pass, 1024-entry table
// MODE_SUM with one FP64 slot fewer per cell than pts_tile_kernel: 2^(u/256) is evaluated
// as 2^(u'/1024), u' = 4u, from a 1024-entry table of 2^(e/1024) and a degree-3 minimax
// polynomial of 2^(r/1024), |r| <= 1/2 (max rel. error 1.4e-16; the degree-4 Taylor form
// of the 256-entry table is 4e-17):
//   per cell 1 DADD + D DFMA (u') + 3 DADD (Cody-Waite) + 3 DFMA (p) + 1 DFMA (acc) = 10 (d=2)
// u' costs nothing extra: the inputs are scaled by (4, 2, 2, ..) while they are staged into
// shared memory (A' = 4A, X' = 2X) and the outputs by the same factors when loaded into
// registers (B' = 4B, Y' = 2Y) -- powers of two, exact. The table is replicated 16x (one
// copy per lane of a half-warp: conflict-free LDS.64), which takes 128 KiB of shared
// memory: one 512-thread CTA per SM (16 warps, as two 256-thread CTAs of the 256-entry
// kernel). Partials are the same sums in the same [ib][n_out] layout.
constexpr int kTab10Rep = 16;
constexpr int kTab10Words = 1024 * kTab10Rep;
constexpr double kMagic10 = 6755399442103296.0;  // 1.5 * 2^52 + 1023 * 1024
constexpr double kQ1 = 0.0006769015435155716;   // minimax 2^(r/1024) = 1 + r(q1 + r(q2 + r q3))
constexpr double kQ2 = 2.29097851993791e-07;
constexpr double kQ3 = 5.1692229383458926e-11;
static __constant__ double c_pexp10_k[4] = {kMagic10, kQ1, kQ2, kQ3};

template <bool FASTCLAMP = false>
__device__ __forceinline__ double pexp10_acc(double u, const unsigned long long* __restrict__ tab,
                                             unsigned laneoff, double q2, double acc) {
    const double t = u + c_pexp10_k[0];
    const double kf = t - c_pexp10_k[0];
    const double r = u - kf;
    double p = fma(r, c_pexp10_k[3], q2);
    p = fma(p, r, c_pexp10_k[1]);
    p = fma(p, r, 1.0);
    // biased k = round(u') + 1023*1024 from the magic sum's low word, flushed at 0 (terms
    // below 2^-1023 underflow to zero, as in pexp_parts)
    // (FASTCLAMP: one IMNMX on the low word, valid while |u'| < 2^31 - 2^20)
    const int kc = FASTCLAMP ? max(__double2loint(t), 0)
                             : ((__double2hiint(t) >= kMagicHi) ? __double2loint(t) : 0);
    const unsigned off = ((static_cast<unsigned>(kc) << 7) & (1023u << 7)) | laneoff;
    const uint2 T = *reinterpret_cast<const uint2*>(reinterpret_cast<const char*>(tab) + off);
    // hi word = biased exponent (kc >> 10) << 20 | mantissa bits of 2^(e/1024), e = kc & 1023:
    // the table's hi words are stored minus e << 10, so kc * 1024 + T.y is that word in one
    // IMAD (the e << 10 part of kc * 1024 cancels; arithmetic mod 2^32)
    const double Tp = __hiloint2double(static_cast<int>(static_cast<unsigned>(kc) * 1024u + T.y),
                                       static_cast<int>(T.x));
    return fma(Tp, p, acc);
}

template <int D, int JT, int NTT, bool FC = false>
__global__ void __launch_bounds__(NTT, 1) pts_sum10_kernel(TileArgs a) {
    SKNR_PDL_ENTRY();
    if (guard_skip(a.st, a.guard)) return;
    constexpr int NT = NTT;
    constexpr int PK = PK_of<D>::value;
    constexpr int CH = 256;
    extern __shared__ __align__(16) double sm[];
    unsigned long long* tab = reinterpret_cast<unsigned long long*>(sm);
    double* sin = sm + kTab10Words;
    const int tid = threadIdx.x;
    for (int t = tid; t < kTab10Words; t += NT) {  // hi word pre-biased by -(e << 10), see pexp10_acc
        const unsigned e = static_cast<unsigned>(t / kTab10Rep);
        const unsigned long long v = c_exp2_tab10[e];
        const unsigned hi = static_cast<unsigned>(v >> 32) - (e << 10);
        tab[t] = (static_cast<unsigned long long>(hi) << 32) | (v & 0xFFFFFFFFull);
    }
    const unsigned laneoff = (tid & (kTab10Rep - 1)) << 3;
    double q2 = kQ2;
    asm volatile("" : "+d"(q2));
    const int64_t out_tile = static_cast<int64_t>(NT) * JT;

    for (int64_t tile = blockIdx.x; tile < a.n_tiles; tile += gridDim.x) {
        const int64_t ot = tile % a.n_out_tiles, ib = tile / a.n_out_tiles;
        double B[JT], Y[JT][D], acc[JT];
        int64_t o[JT];
#pragma unroll
        for (int jt = 0; jt < JT; ++jt) {
            o[jt] = ot * out_tile + jt * NT + tid;
            const int64_t oc = o[jt] < a.n_out ? o[jt] : a.n_out - 1;
            B[jt] = 4.0 * a.out_pack[oc * PK];
#pragma unroll
            for (int d = 0; d < D; ++d) Y[jt][d] = 2.0 * a.out_pack[oc * PK + 1 + d];
            acc[jt] = 0.0;
        }
        const int64_t i0 = ib * a.in_block;
        const int64_t i1 = (i0 + a.in_block < a.n_in) ? i0 + a.in_block : a.n_in;
        for (int64_t c0 = i0; c0 < i1; c0 += CH) {
            const int cnt = static_cast<int>((i1 - c0) < CH ? (i1 - c0) : CH);
            __syncthreads();
            for (int t = tid; t < cnt * PK; t += NT) {
                const int q = t % PK;
                sin[t] = (q == 0 ? 4.0 : 2.0) * a.in_pack[c0 * PK + t];
            }
            __syncthreads();
#pragma unroll 1
            for (int k = 0; k < cnt; ++k) {
                double x[PK];
#pragma unroll
                for (int q = 0; q < PK / 2; ++q) {
                    const double2 v = reinterpret_cast<const double2*>(sin + k * PK)[q];
                    x[2 * q] = v.x;
                    x[2 * q + 1] = v.y;
                }
#pragma unroll
                for (int jt = 0; jt < JT; ++jt) {
                    double u = x[0] + B[jt];
#pragma unroll
                    for (int d = 0; d < D; ++d) u = fma(x[1 + d], Y[jt][d], u);
                    acc[jt] = pexp10_acc<FC>(u, tab, laneoff, q2, acc[jt]);
                }
            }
        }
#pragma unroll
        for (int jt = 0; jt < JT; ++jt)
            if (o[jt] < a.n_out) a.partial[ib * a.n_out + o[jt]] = acc[jt];
    }
}

// ------------------------------------------------------------- LSE sum pass, 4096-entry table
// MODE_SUM in 10 FP64 slots per cell with the 32 KiB shared-memory footprint of the
// 256-entry kernel: 2^(u/256) = 2^(u'/4096), u' = 16u, from a 4096-entry table of
// 2^(e/4096) held ONCE per CTA (REP copies; REP = 1: lanes read random entries and pay the
// bank conflicts -- the shared-memory pipe has the slack, the FP64 pipe does not) and a
// degree-3 Taylor polynomial of 2^(r/4096), |r| <= 1/2 (truncation 2e-18):
//   per cell 1 DADD + D DFMA (u') + 3 DADD (Cody-Waite) + 3 DFMA (p) + 1 DFMA (acc) = 10 (d=2)
// u' is exact: inputs are staged as (16A, 4X), outputs loaded as (16B, 4Y) -- powers of two.
// Same partial sums in the same [ib][n_out] layout as pts_tile_kernel<SUM>.
constexpr double kMagic12 = 6755399445245952.0;  // 1.5 * 2^52 + 1023 * 4096
constexpr double kR1 = 0.0001692253858788929;    // (ln2/4096)^k / k!
constexpr double kR2 = 1.4318615612930102e-08;
constexpr double kR3 = 8.076910841165457e-13;
static __constant__ double c_pexp12_k[4] = {kMagic12, kR1, kR2, kR3};

template <int REP, bool FASTCLAMP>
__device__ __forceinline__ double pexp12_acc(double u, const unsigned long long* __restrict__ tab,
                                             unsigned laneoff, double r2, double acc) {
    const double t = u + c_pexp12_k[0];
    const double kf = t - c_pexp12_k[0];
    const double r = u - kf;
    double p = fma(r, c_pexp12_k[3], r2);
    p = fma(p, r, c_pexp12_k[1]);
    p = fma(p, r, 1.0);
    // biased k = round(u') + 1023*4096 (low word of the magic sum), flushed at 0
    const int kc = FASTCLAMP ? max(__double2loint(t), 0)
                             : ((__double2hiint(t) >= kMagicHi) ? __double2loint(t) : 0);
    constexpr int SH = REP == 1 ? 3 : (REP == 2 ? 4 : 5);
    const unsigned off = ((static_cast<unsigned>(kc) << SH) & (4095u << SH)) | laneoff;
    const uint2 T = *reinterpret_cast<const uint2*>(reinterpret_cast<const char*>(tab) + off);
    // hi word = (kc >> 12) << 20 | mantissa bits of 2^(e/4096); table hi words pre-biased
    // by -(e << 8), so kc * 256 + T.y assembles it in one IMAD (mod 2^32)
    const double Tp = __hiloint2double(static_cast<int>(static_cast<unsigned>(kc) * 256u + T.y),
                                       static_cast<int>(T.x));
    return fma(Tp, p, acc);
}

template <int D, int JT, int NTT, int REP, bool FC = false, int MINB = 1, int UNR = 1>
__global__ void __launch_bounds__(NTT, MINB) pts_sum12_kernel(TileArgs a) {
    SKNR_PDL_ENTRY();
    if (guard_skip(a.st, a.guard)) return;
    constexpr int NT = NTT;
    constexpr int PK = PK_of<D>::value;
    constexpr int CH = 256;
    constexpr int TW = 4096 * REP;
    extern __shared__ __align__(16) double sm[];
    unsigned long long* tab = reinterpret_cast<unsigned long long*>(sm);
    double* sin = sm + TW;
    const int tid = threadIdx.x;
    for (int t = tid; t < TW; t += NT) {  // hi word pre-biased by -(e << 8), see pexp12_acc
        const unsigned e = static_cast<unsigned>(t / REP);
        const unsigned long long v = g_exp2_tab12[e];
        const unsigned hi = static_cast<unsigned>(v >> 32) - (e << 8);
        tab[t] = (static_cast<unsigned long long>(hi) << 32) | (v & 0xFFFFFFFFull);
    }
    const unsigned laneoff = (tid & (REP - 1)) << 3;
    double r2 = kR2;
    asm volatile("" : "+d"(r2));
    const int64_t out_tile = static_cast<int64_t>(NT) * JT;

    for (int64_t tile = blockIdx.x; tile < a.n_tiles; tile += gridDim.x) {
        const int64_t ot = tile % a.n_out_tiles, ib = tile / a.n_out_tiles;
        double B[JT], Y[JT][D], acc[JT];
        int64_t o[JT];
#pragma unroll
        for (int jt = 0; jt < JT; ++jt) {
            o[jt] = ot * out_tile + jt * NT + tid;
            const int64_t oc = o[jt] < a.n_out ? o[jt] : a.n_out - 1;
            B[jt] = 16.0 * a.out_pack[oc * PK];
#pragma unroll
            for (int d = 0; d < D; ++d) Y[jt][d] = 4.0 * a.out_pack[oc * PK + 1 + d];
            acc[jt] = 0.0;
        }
        const int64_t i0 = ib * a.in_block;
        const int64_t i1 = (i0 + a.in_block < a.n_in) ? i0 + a.in_block : a.n_in;
        for (int64_t c0 = i0; c0 < i1; c0 += CH) {
            const int cnt = static_cast<int>((i1 - c0) < CH ? (i1 - c0) : CH);
            __syncthreads();
            for (int t = tid; t < cnt * PK; t += NT) {
                const int q = t % PK;
                sin[t] = (q == 0 ? 16.0 : 4.0) * a.in_pack[c0 * PK + t];
            }
            __syncthreads();
#pragma unroll UNR
            for (int k = 0; k < cnt; ++k) {
                double x[PK];
#pragma unroll
                for (int q = 0; q < PK / 2; ++q) {
                    const double2 v = reinterpret_cast<const double2*>(sin + k * PK)[q];
                    x[2 * q] = v.x;
                    x[2 * q + 1] = v.y;
                }
#pragma unroll
                for (int jt = 0; jt < JT; ++jt) {
                    double u = x[0] + B[jt];
#pragma unroll
                    for (int d = 0; d < D; ++d) u = fma(x[1 + d], Y[jt][d], u);
                    acc[jt] = pexp12_acc<REP, FC>(u, tab, laneoff, r2, acc[jt]);
                }
            }
        }
#pragma unroll
        for (int jt = 0; jt < JT; ++jt)
            if (o[jt] < a.n_out) a.partial[ib * a.n_out + o[jt]] = acc[jt];
    }
}

// ------------------------------------------------------------- stable-accept anchor pass
// The three column sums of the stable accept test (engine_solver.cuh, k_dh): for each
// output j, s = sum_i e, t = sum_i e w1_i, u = sum_i e w2_i, with e = P~_ij (unshifted
// pack: P~ <= 1 by construction) and W = (1, expm1(d/eps), exp(d/eps), 0) in the KT = 4
// layout of MODE_BLOCK. The exponential is pexp12's (4096-entry table), so a cell costs
// u' 3 + Cody-Waite 3 + polynomial 3 + s 1 + e 1 + t, u 2 = 13 FP64 slots (the generic
// 4-column register block pass: 16, at lower occupancy). Partials in the MODE_BLOCK
// layout [ib][c][n_out], c = 0..2 (column 3 of W is zero and is not written).
template <int D, int JT, int NTT, int REP, int UNR = 1>
__global__ void __launch_bounds__(NTT, 1) pts_anchor12_kernel(TileArgs a) {
    SKNR_PDL_ENTRY();
    if (guard_skip(a.st, a.guard)) return;
    constexpr int NT = NTT;
    constexpr int PK = PK_of<D>::value;
    constexpr int SK = PK + 2;  // staged row: 16A, 4X[D] (+ pad), w1, w2
    constexpr int CH = 256;
    constexpr int TW = 4096 * REP;
    extern __shared__ __align__(16) double sm[];
    unsigned long long* tab = reinterpret_cast<unsigned long long*>(sm);
    double* sin = sm + TW;
    const int tid = threadIdx.x;
    for (int t = tid; t < TW; t += NT) {
        const unsigned e = static_cast<unsigned>(t / REP);
        const unsigned long long v = g_exp2_tab12[e];
        const unsigned hi = static_cast<unsigned>(v >> 32) - (e << 8);
        tab[t] = (static_cast<unsigned long long>(hi) << 32) | (v & 0xFFFFFFFFull);
    }
    const unsigned laneoff = (tid & (REP - 1)) << 3;
    double r2 = kR2;
    asm volatile("" : "+d"(r2));
    const int64_t out_tile = static_cast<int64_t>(NT) * JT;

    for (int64_t tile = blockIdx.x; tile < a.n_tiles; tile += gridDim.x) {
        const int64_t ot = tile % a.n_out_tiles, ib = tile / a.n_out_tiles;
        double B[JT], Y[JT][D], as[JT], at[JT], au[JT];
        int64_t o[JT];
#pragma unroll
        for (int jt = 0; jt < JT; ++jt) {
            o[jt] = ot * out_tile + jt * NT + tid;
            const int64_t oc = o[jt] < a.n_out ? o[jt] : a.n_out - 1;
            B[jt] = 16.0 * a.out_pack[oc * PK];
#pragma unroll
            for (int d = 0; d < D; ++d) Y[jt][d] = 4.0 * a.out_pack[oc * PK + 1 + d];
            as[jt] = at[jt] = au[jt] = 0.0;
        }
        const int64_t i0 = ib * a.in_block;
        const int64_t i1 = (i0 + a.in_block < a.n_in) ? i0 + a.in_block : a.n_in;
        for (int64_t c0 = i0; c0 < i1; c0 += CH) {
            const int cnt = static_cast<int>((i1 - c0) < CH ? (i1 - c0) : CH);
            __syncthreads();
            for (int t = tid; t < cnt * SK; t += NT) {
                const int k = t / SK, q = t % SK;
                sin[t] = q < PK ? (q == 0 ? 16.0 : 4.0) * a.in_pack[(c0 + k) * PK + q]
                                : a.W[(c0 + k) * 4 + (q - PK + 1)];
            }
            __syncthreads();
#pragma unroll UNR
            for (int k = 0; k < cnt; ++k) {
                double x[SK];
#pragma unroll
                for (int q = 0; q < SK / 2; ++q) {
                    const double2 v = reinterpret_cast<const double2*>(sin + k * SK)[q];
                    x[2 * q] = v.x;
                    x[2 * q + 1] = v.y;
                }
#pragma unroll
                for (int jt = 0; jt < JT; ++jt) {
                    double u = x[0] + B[jt];
#pragma unroll
                    for (int d = 0; d < D; ++d) u = fma(x[1 + d], Y[jt][d], u);
                    const double t = u + c_pexp12_k[0];
                    const double kf = t - c_pexp12_k[0];
                    const double r = u - kf;
                    double p = fma(r, c_pexp12_k[3], r2);
                    p = fma(p, r, c_pexp12_k[1]);
                    p = fma(p, r, 1.0);
                    const int kc = (__double2hiint(t) >= kMagicHi) ? __double2loint(t) : 0;
                    constexpr int SH = REP == 1 ? 3 : (REP == 2 ? 4 : 5);
                    const unsigned off = ((static_cast<unsigned>(kc) << SH) & (4095u << SH)) | laneoff;
                    const uint2 T = *reinterpret_cast<const uint2*>(reinterpret_cast<const char*>(tab) + off);
                    const double Tp = __hiloint2double(static_cast<int>(static_cast<unsigned>(kc) * 256u + T.y),
                                                       static_cast<int>(T.x));
                    as[jt] = fma(Tp, p, as[jt]);
                    const double e = Tp * p;
                    at[jt] = fma(e, x[PK], at[jt]);
                    au[jt] = fma(e, x[PK + 1], au[jt]);
                }
            }
        }
#pragma unroll
        for (int jt = 0; jt < JT; ++jt) {
            if (o[jt] >= a.n_out) continue;
            a.partial[(ib * 4 + 0) * a.n_out + o[jt]] = as[jt];
            a.partial[(ib * 4 + 1) * a.n_out + o[jt]] = at[jt];
            a.partial[(ib * 4 + 2) * a.n_out + o[jt]] = au[jt];
        }
    }
}

// ------------------------------------------------------------- fp32 sum pass (opt-in)
// MODE_SUM_F32 (sknr_problem_set_precision(p, 32)): the sum pass of pts_tile_kernel with
// the cell exponent in fp32 and 2^v on the MUFU unit (ex2.approx.ftz.f32). The fp64 pack
// (u = A + B + <X, Y>) is re-expanded around the squared distance, in log2 units:
//   v = u/256 = A'/256 + B'/256 - |Xs - Ys|^2,  A' = A + |X|^2/2, B' = B + |Y|^2/2,
//   Xs = X / sqrt(512)
// and the potential-carrying terms are split on a 2^-8 grid:
//   A'/256 = Ah + Al, Ah = rint(A')/256, |Al| <= 2^-9   (B' likewise)
// so that, per cell, s = Ah + Bh is exact in fp32 (|Ah|, |Bh| < 2^15), the squared
// distance q = |Xs - Ys|^2 depends on the coordinates alone, and v = s - q is one
// rounding at the ulp of v (< 3e-8 for the terms that carry the sum). 2^Al enters as
// an fp32 weight per input (FFMA into the partial), 2^Bl as an fp64 factor per output.
// The coordinate rounding (|Xs| < 2^5: 1e-6 absolute) is a FIXED perturbation of the
// kernel (<= 2e-5 per term, ~1e-6 per column sum at C4), so the solver converges in its own marginals and
// the potentials stay within ~1e-6 relative of the fp64 path. Per cell: 7 FP32 ops +
// 1 MUFU; the MUFU pipe (16 ex2 / clk / SM on sm_100: 4.65 TCells/s at 1.965 GHz) and
// the issue slot (8 per cell) bound it together. Partials accumulate in fp32 over 32
// inputs, then in fp64, in the fp64 [ib][n_out] layout: the finalize kernels are shared
// (with the fp32 validity window FinalizeArgs::lo_ok).
__device__ __forceinline__ float ex2_mufu(float v) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
    return r;
}

// 2^t for |t| <= 2^-9 to fp64 accuracy (truncation below 1e-13)
__device__ __forceinline__ double exp2_small(double t) {
    const double z = t * 0.6931471805599453;
    return 1.0 + z * (1.0 + z * (0.5 + z * (1.0 / 6.0)));
}

constexpr double kInvSqrt512 = 0.04419417382415922;  // 1/sqrt(512)

template <int D>
struct PKF_of {  // fp32 input pack: Ah, 2^Al, D coords, padded to a float4 multiple
    static constexpr int value = ((D + 2 + 3) / 4) * 4;
};

// 2^(B'/256 - Bh) of an output: the fp64 factor that completes its fp32 sums
template <int D, int PK>
__device__ __forceinline__ double f32_out_split(const double* pk, float& Bh, float* Y) {
    double bv = pk[0];
#pragma unroll
    for (int d = 0; d < D; ++d) {
        const double yd = pk[1 + d];
        bv = fma(0.5 * yd, yd, bv);
        if (Y) Y[d] = static_cast<float>(yd * kInvSqrt512);
    }
    const double bh = rint(bv);
    Bh = static_cast<float>(bh * (1.0 / 256.0));
    return exp2_small((bv - bh) * (1.0 / 256.0));
}

template <int D, int JT, int NTT, int MINB = 1>
__global__ void __launch_bounds__(NTT, MINB) pts_f32_kernel(TileArgs a) {
    SKNR_PDL_ENTRY();
    if (guard_skip(a.st, a.guard)) return;
    constexpr int PK = PK_of<D>::value;
    constexpr int PKF = PKF_of<D>::value;
    constexpr int CH = 256;
    constexpr int SUB = 32;  // inputs per fp32 partial sum
    extern __shared__ __align__(16) float smf[];
    const int tid = threadIdx.x;
    const int64_t out_tile = static_cast<int64_t>(NTT) * JT;

    for (int64_t tile = blockIdx.x; tile < a.n_tiles; tile += gridDim.x) {
        const int64_t ot = tile % a.n_out_tiles, ib = tile / a.n_out_tiles;
        float B[JT], Y[JT][D];
        double acc[JT];
#pragma unroll
        for (int jt = 0; jt < JT; ++jt) {
            const int64_t o = ot * out_tile + jt * NTT + tid;
            const int64_t oc = o < a.n_out ? o : a.n_out - 1;
            f32_out_split<D, PK>(a.out_pack + oc * PK, B[jt], Y[jt]);
            acc[jt] = 0.0;
        }
        const int64_t i0 = ib * a.in_block;
        const int64_t i1 = (i0 + a.in_block < a.n_in) ? i0 + a.in_block : a.n_in;
        for (int64_t c0 = i0; c0 < i1; c0 += CH) {
            const int cnt = static_cast<int>((i1 - c0) < CH ? (i1 - c0) : CH);
            const int cnt32 = (cnt + SUB - 1) / SUB * SUB;
            __syncthreads();
            for (int t = tid; t < cnt32 * PKF; t += NTT) {
                const int k = t / PKF, q = t % PKF;
                float v = 0.0f;
                if (k >= cnt) {
                    v = q == 0 ? -1e30f : 0.0f;  // padding inputs: 2^v = 0 and weight 0
                } else if (q < 2) {
                    const double* ip = a.in_pack + (c0 + k) * PK;
                    double av = ip[0];
#pragma unroll
                    for (int d = 0; d < D; ++d) av = fma(0.5 * ip[1 + d], ip[1 + d], av);
                    const double ah = rint(av);
                    v = q == 0 ? static_cast<float>(ah * (1.0 / 256.0))
                               : static_cast<float>(exp2_small((av - ah) * (1.0 / 256.0)));
                } else if (q < 2 + D) {
                    v = static_cast<float>(a.in_pack[(c0 + k) * PK + q - 1] * kInvSqrt512);
                }
                smf[t] = v;
            }
            __syncthreads();
            for (int k0 = 0; k0 < cnt32; k0 += SUB) {
                float part[JT];
#pragma unroll
                for (int jt = 0; jt < JT; ++jt) part[jt] = 0.0f;
#pragma unroll 8
                for (int k = k0; k < k0 + SUB; ++k) {
                    float x[PKF];
#pragma unroll
                    for (int q = 0; q < PKF / 4; ++q) {
                        const float4 v = reinterpret_cast<const float4*>(smf + k * PKF)[q];
                        x[4 * q] = v.x;
                        x[4 * q + 1] = v.y;
                        x[4 * q + 2] = v.z;
                        x[4 * q + 3] = v.w;
                    }
#pragma unroll
                    for (int jt = 0; jt < JT; ++jt) {
                        const float d0 = x[2] - Y[jt][0];
                        float q = d0 * d0;
#pragma unroll
                        for (int d = 1; d < D; ++d) {
                            const float dd = x[2 + d] - Y[jt][d];
                            q = fmaf(dd, dd, q);
                        }
                        const float v = (x[0] + B[jt]) - q;
                        part[jt] = fmaf(x[1], ex2_mufu(v), part[jt]);
                    }
                }
#pragma unroll
                for (int jt = 0; jt < JT; ++jt) acc[jt] += static_cast<double>(part[jt]);
            }
        }
#pragma unroll
        for (int jt = 0; jt < JT; ++jt) {
            const int64_t o = ot * out_tile + jt * NTT + tid;
            if (o < a.n_out) {
                float bh;  // the output's split again (not held in registers across the loop)
                const double scale = f32_out_split<D, PK>(a.out_pack + o * PK, bh, nullptr);
                a.partial[ib * a.n_out + o] = acc[jt] * scale;
            }
        }
    }
}

// ------------------------------------------------------------- culled sum pass (opt-in)
// Both point clouds are visited in Morton order (perm_in / perm_out), so a warp's
// 256 outputs and a 64-input group each cover a small box. For every term
//   u_io = F_i + S_o - LS kc |x_i - y_o|^2 <= max_I F + max_O S - LS kc dist2(box_I, box_O) =: U,
// and the output's LSE satisfies L_o >= s_o - slack (slack = 0 after an exact max
// pass, (max df - min df)/eps for the bound shift). A group pair with
// U < -LS (T + slack) therefore only holds terms below e^-T of the output's total
// (n e^-60 < 1e-21 relative for T = 60): it is skipped. Each warp tests 32 groups
// at once (one per lane, ballot), stages only the kept groups and accumulates
// their terms exactly as in pts_tile_kernel.
template <int D>
__device__ __forceinline__ double box_dist2(const double* __restrict__ a, const double* __restrict__ b) {
    double s = 0.0;
#pragma unroll
    for (int d = 0; d < D; ++d) {
        const double g = fmax(fmax(a[d] - b[D + d], b[d] - a[D + d]), 0.0);
        s = fma(g, g, s);
    }
    return s;
}

// F32: the kept groups' terms in the fp32 arithmetic of pts_f32_kernel (opt-in precision).
template <int D, int JT, int NTT, bool F32 = false>
__global__ void __launch_bounds__(NTT, 2) pts_cull_kernel(TileArgs a) {
    SKNR_PDL_ENTRY();
    if (guard_skip(a.st, a.guard)) return;
    constexpr int PK = PK_of<D>::value;
    static_assert(32 * JT == CULL_GO, "one warp owns one output group");
    extern __shared__ __align__(16) double sm[];
    unsigned long long* tab = reinterpret_cast<unsigned long long*>(sm);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double* sin = sm + kTabWords + warp * CULL_GI * PK;  // warp-private input staging
    load_exp2_table(tab, tid, NTT);
    __syncthreads();
    const unsigned laneoff = (tid & (kTabRep - 1)) << 3;
    const double c3 = pexp_c3();
    const bool exact = a.retry_phase || a.st->need_exact[a.dir];
    const double slack = exact ? 0.0 : (a.st->dmax[a.dir] - a.st->dmin[a.dir]) * a.inv_eps;
    const double thr = -kLS * (a.cull_t + slack);

    // Work unit = (256-output group, input block), taken from a global queue by each
    // warp independently: culled units cost only their bound tests, and no warp
    // waits on another (the CTA only shares the exp2 table).
    while (true) {
        unsigned unit = 0;
        if (lane == 0) unit = atomicAdd(a.sched, 1u);
        unit = __shfl_sync(0xffffffffu, unit, 0);
        if (unit >= a.n_tiles) break;
        const int64_t og = unit % a.n_out_tiles, ib = unit / a.n_out_tiles;
        const int64_t wpos = og * CULL_GO;
        double B[JT], Y[JT][D], acc[JT];
        float Bf[JT], Yf[JT][D];
#pragma unroll
        for (int jt = 0; jt < JT; ++jt) {
            const int64_t pos = wpos + jt * 32 + lane;
            const int64_t oc = a.perm_out[pos < a.n_out ? pos : a.n_out - 1];
            if (F32) {
                f32_out_split<D, PK>(a.out_pack + oc * PK, Bf[jt], Yf[jt]);
            } else {
                B[jt] = a.out_pack[oc * PK];
#pragma unroll
                for (int d = 0; d < D; ++d) Y[jt][d] = a.out_pack[oc * PK + 1 + d];
            }
            acc[jt] = 0.0;
        }
        double wbox[2 * D];
#pragma unroll
        for (int q = 0; q < 2 * D; ++q) wbox[q] = a.box_go[og * 2 * D + q];
        const double s_w = a.s_go[og];
        const int64_t i0 = ib * a.in_block;
        const int64_t i1 = (i0 + a.in_block < a.n_in) ? i0 + a.in_block : a.n_in;
        unsigned tested = 0, kept = 0;
#pragma unroll 1
        for (int64_t r0 = i0; r0 < i1; r0 += 32 * CULL_GI) {
            const int64_t gl = r0 / CULL_GI + lane;
            bool keep = false;
            if (gl * CULL_GI < i1)
                keep = !(a.f_gi[gl] + s_w - a.lskc * box_dist2<D>(a.box_gi + gl * 2 * D, wbox) < thr);
            unsigned mask = __ballot_sync(0xffffffffu, keep);
            {
                const int64_t ng = (i1 - r0 + CULL_GI - 1) / CULL_GI;
                tested += static_cast<unsigned>(ng < 32 ? ng : 32);
            }
            kept += __popc(mask);
#pragma unroll 1
        while (mask) {
            const int bit = __ffs(mask) - 1;
            mask &= mask - 1;
            const int64_t g0 = r0 + static_cast<int64_t>(bit) * CULL_GI;
            const int cnt = static_cast<int>((i1 - g0) < CULL_GI ? (i1 - g0) : CULL_GI);
            __syncwarp();
            if constexpr (F32) {  // fp32 pack (Ah, 2^Al, Xs...) of the group, one input per lane
                constexpr int PKF = PKF_of<D>::value;
                static_assert(PKF <= 2 * PK, "fp32 pack fits the fp64 staging row");
                float* sf = reinterpret_cast<float*>(sin);
                for (int t = lane; t < cnt; t += 32) {
                    const double* ip = a.in_pack + static_cast<int64_t>(a.perm_in[g0 + t]) * PK;
                    double av = ip[0];
#pragma unroll
                    for (int d = 0; d < D; ++d) av = fma(0.5 * ip[1 + d], ip[1 + d], av);
                    const double ah = rint(av);
                    sf[t * PKF] = static_cast<float>(ah * (1.0 / 256.0));
                    sf[t * PKF + 1] = static_cast<float>(exp2_small((av - ah) * (1.0 / 256.0)));
#pragma unroll
                    for (int d = 0; d < D; ++d) sf[t * PKF + 2 + d] = static_cast<float>(ip[1 + d] * kInvSqrt512);
#pragma unroll
                    for (int q = D + 2; q < PKF; ++q) sf[t * PKF + q] = 0.0f;
                }
                __syncwarp();
                float part[JT];
#pragma unroll
                for (int jt = 0; jt < JT; ++jt) part[jt] = 0.0f;
#pragma unroll 8
                for (int k = 0; k < cnt; ++k) {
                    float x[PKF];
#pragma unroll
                    for (int q = 0; q < PKF / 4; ++q) {
                        const float4 v = reinterpret_cast<const float4*>(sf + k * PKF)[q];
                        x[4 * q] = v.x;
                        x[4 * q + 1] = v.y;
                        x[4 * q + 2] = v.z;
                        x[4 * q + 3] = v.w;
                    }
#pragma unroll
                    for (int jt = 0; jt < JT; ++jt) {
                        const float d0 = x[2] - Yf[jt][0];
                        float q2 = d0 * d0;
#pragma unroll
                        for (int d = 1; d < D; ++d) {
                            const float dd = x[2 + d] - Yf[jt][d];
                            q2 = fmaf(dd, dd, q2);
                        }
                        part[jt] = fmaf(x[1], ex2_mufu((x[0] + Bf[jt]) - q2), part[jt]);
                    }
                }
#pragma unroll
                for (int jt = 0; jt < JT; ++jt) acc[jt] += static_cast<double>(part[jt]);
            } else {
            for (int t = lane; t < cnt; t += 32) {
                const double2* src = reinterpret_cast<const double2*>(a.in_pack +
                                                                      static_cast<int64_t>(a.perm_in[g0 + t]) * PK);
                double2* dst = reinterpret_cast<double2*>(sin + t * PK);
#pragma unroll
                for (int q = 0; q < PK / 2; ++q) dst[q] = src[q];
            }
            __syncwarp();
#pragma unroll 4
            for (int k = 0; k < cnt; ++k) {
                double x[PK];
#pragma unroll
                for (int q = 0; q < PK / 2; ++q) {
                    const double2 v = reinterpret_cast<const double2*>(sin + k * PK)[q];
                    x[2 * q] = v.x;
                    x[2 * q + 1] = v.y;
                }
#pragma unroll
                for (int jt = 0; jt < JT; ++jt) {
                    double u = x[0] + B[jt];
#pragma unroll
                    for (int d = 0; d < D; ++d) u = fma(x[1 + d], Y[jt][d], u);
                    acc[jt] = pexp_acc<false, false>(u, tab, laneoff, c3, acc[jt]);
                }
            }
            }
        }
        }
#pragma unroll
        for (int jt = 0; jt < JT; ++jt) {
            const int64_t pos = wpos + jt * 32 + lane;
            if (pos < a.n_out) {
                const int64_t o = a.perm_out[pos];
                double scale = 1.0;
                if (F32) {
                    float bh;
                    scale = f32_out_split<D, PK>(a.out_pack + o * PK, bh, nullptr);
                }
                a.partial[ib * a.n_out + o] = acc[jt] * scale;
            }
        }
        if (lane == 0) {
            DevState* st = const_cast<DevState*>(a.st);
            atomicAdd(&st->n_cull_tested, static_cast<unsigned long long>(tested));
            atomicAdd(&st->n_cull_kept, static_cast<unsigned long long>(kept));
        }
    }
}

// ------------------------------------------------------------- small-problem batched SK
// A group of G CTAs = one problem, the whole solve loop inside the kernel (no launches
// per iteration): the inputs of each log-sum-exp are staged in every CTA's shared
// memory, one warp per output (warps of the group take outputs round-robin), lanes over
// the inputs, exact max shift then sum (core.cpp:35-82), warp-shuffle and fixed-order
// block and group reductions (deterministic for a given G). Same iteration as the
// device loop: row LSE -> gauge (solver.cpp:108-112) -> column LSE -> marginal gap ->
// stop test. G = 1 (many problems) needs only __syncthreads; G > 1 (few problems,
// one problem spread over many SMs) adds two group barriers per iteration, launched
// cooperatively so every CTA of a group is resident.
template <int D>
__device__ __forceinline__ double small_lse(const double* __restrict__ sp, int cnt, const double* yo, double ke,
                                            const unsigned long long* __restrict__ tab, unsigned laneoff,
                                            double c3, int lane) {
    constexpr int P = D + 1;
    double mx = -1e300;
    for (int k = lane; k < cnt; k += 32) {
        double d2 = 0.0;
#pragma unroll
        for (int d = 0; d < D; ++d) {
            const double t = sp[k * P + 1 + d] - yo[d];
            d2 = fma(t, t, d2);
        }
        mx = fmax(mx, sp[k * P] - ke * d2);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    double s = 0.0;
    for (int k = lane; k < cnt; k += 32) {
        double d2 = 0.0;
#pragma unroll
        for (int d = 0; d < D; ++d) {
            const double t = sp[k * P + 1 + d] - yo[d];
            d2 = fma(t, t, d2);
        }
        s = pexp_acc<true>(kLS * (sp[k * P] - ke * d2 - mx), tab, laneoff, c3, s);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    return mx + log(s);
}

__device__ __forceinline__ double small_block_sum(double v, double* red, int tid, int nthreads) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if ((tid & 31) == 0) red[tid >> 5] = v;
    __syncthreads();
    double t = 0.0;
    for (int w = 0; w < nthreads / 32; ++w) t += red[w];  // same order in every thread
    return t;
}

// Generation barrier of the G CTAs of one group (bar[0] arrivals, bar[1] generation).
__device__ __forceinline__ void group_barrier(unsigned* bar, int G) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned* vgen = bar + 1;
        const unsigned gen = *vgen;
        __threadfence();
        if (atomicAdd(bar, 1u) == static_cast<unsigned>(G - 1)) {
            atomicExch(bar, 0u);
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            while (*vgen == gen) __nanosleep(32);
        }
        __threadfence();
    }
    __syncthreads();
}

// Sum over the group of the block totals of v0 (and v1): block totals in fixed order,
// then the G CTA totals in CTA order (identical in every CTA of the group).
template <int NV>
__device__ __forceinline__ void group_sums(double* v, double* red, int tid, int nthreads, int G, int r,
                                           double* part, int slot, unsigned* bar) {
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] = small_block_sum(v[k], red, tid, nthreads);
    if (G == 1) return;
    if (tid == 0)
#pragma unroll
        for (int k = 0; k < NV; ++k) part[r * 4 + slot + k] = v[k];
    group_barrier(bar, G);
#pragma unroll
    for (int k = 0; k < NV; ++k) {
        double t = __ldcg(part + slot + k);
        for (int c = 1; c < G; ++c) t += __ldcg(part + c * 4 + slot + k);
        v[k] = t;
    }
}

template <int D>
__global__ void __launch_bounds__(512, 1)
    k_sk_small(SmallProbDev* probs, double tol, long long max_iter, int warm_g, int G, double* gpart,
               unsigned* gbar) {
    SKNR_PDL_ENTRY();
    constexpr int P = D + 1;
    constexpr int NT = 512;
    constexpr int WPB = NT / 32;
    extern __shared__ __align__(16) double sm[];
    unsigned long long* tab = reinterpret_cast<unsigned long long*>(sm);
    double* red = sm + kTabWords;
    double* sp = red + 64;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int q = blockIdx.x / G, r = blockIdx.x % G;
    const int W = G * WPB, gw = r * WPB + warp;  // warps of the group, this warp's rank in it
    double* part = gpart ? gpart + static_cast<int64_t>(q) * G * 4 : nullptr;
    unsigned* bar = gbar ? gbar + 2 * q : nullptr;
    load_exp2_table(tab, tid, NT);
    const unsigned laneoff = (tid & (kTabRep - 1)) << 3;
    const double c3 = pexp_c3();
    SmallProbDev& pr = probs[q];
    const int n = pr.n, m = pr.m;
    const double eps = pr.eps, ie = 1.0 / eps, ke = pr.kappa * ie;
    double* f = pr.f;
    double* g = pr.g;
    double* h = pr.h;
    // Cross-CTA data (f, g, h, partials) is read with ld.global.cg: L1 is not coherent.
    // column LSE at f - c into h (ctransform_of_f): inputs i (la_i + (f_i - c)/eps, x_i),
    // outputs j owned by warp j mod W, whose lane 0 also stores the gauged g_j = gsrc_j + c;
    // then the CTA's threads form the column residuals b_j expm1((g_j - h_j)/eps) of the
    // CTA's own columns (j = 16 r + w + k W, w < 16) in parallel.
    auto col_lse = [&](double c, const double* gsrc, double& csq) {
        __syncthreads();
        for (int i = tid; i < n; i += NT) {
            sp[i * P] = log(pr.a[i]) + (__ldcg(f + i) - c) * ie;
#pragma unroll
            for (int d = 0; d < D; ++d) sp[i * P + 1 + d] = pr.x[i + d * n];
        }
        __syncthreads();
        for (int j = gw; j < m; j += W) {
            double yo[D];
#pragma unroll
            for (int d = 0; d < D; ++d) yo[d] = pr.y[j + d * m];
            const double gprev = gsrc ? __ldcg(gsrc + j) : 0.0;  // loaded ahead of the LSE
            const double L = small_lse<D>(sp, n, yo, ke, tab, laneoff, c3, lane);
            if (lane == 0) {
                h[j] = -eps * L;
                if (gsrc) g[j] = gprev + c;
            }
        }
        if (!gsrc) return;
        __syncthreads();
        for (int t = tid;; t += NT) {
            const int k = t >> 4;
            if (static_cast<int64_t>(k) * W >= m) break;
            const int j = r * WPB + (t & 15) + k * W;
            if (j >= m) continue;
            const double cr = pr.b[j] * expm1((g[j] - h[j]) * ie);
            csq = fma(cr, cr, csq);
        }
    };
    double dummy = 0.0;
    if (!warm_g) {  // first sweep's g = f0^{C,eps}
        col_lse(0.0, nullptr, dummy);
        if (G > 1) group_barrier(bar, G);
    }
    const double* gsrc = warm_g ? g : h;  // g of the coming sweep (previous h, gauged below)
    long long it = 0;
    int conv = 0;
    while (it < max_iter) {
        ++it;
        // row LSE at gsrc (ctransform_of_g): f_i = -eps L_i; row residual a_i expm1(f_i/eps + L_i)
        __syncthreads();
        for (int j = tid; j < m; j += NT) {
            sp[j * P] = log(pr.b[j]) + __ldcg(gsrc + j) * ie;
#pragma unroll
            for (int d = 0; d < D; ++d) sp[j * P + 1 + d] = pr.y[j + d * m];
        }
        __syncthreads();
        double rs[2] = {0.0, 0.0};  // a.f, |row - a|^2
        for (int i = gw; i < n; i += W) {
            double xo[D];
#pragma unroll
            for (int d = 0; d < D; ++d) xo[d] = pr.x[i + d * n];
            const double ai = pr.a[i];
            const double L = small_lse<D>(sp, m, xo, ke, tab, laneoff, c3, lane);
            if (lane == 0) {
                const double fi = -eps * L;
                const double rr = ai * expm1(fi * ie + L);
                f[i] = fi;
                rs[1] = fma(rr, rr, rs[1]);
                rs[0] = fma(ai, fi, rs[0]);
            }
        }
        // gauge (solver.cpp:108-112): c = a.f over the whole group
        group_sums<2>(rs, red, tid, NT, G, r, part, 0, bar);
        const double c = rs[0], row2 = rs[1];
        // column LSE at the gauged f: next h, column residual, gauged g
        double cs[1] = {0.0};
        col_lse(c, gsrc, cs[0]);
        group_sums<1>(cs, red, tid, NT, G, r, part, 2, bar);
        // f -= c on the rows this warp owns (lanes split them; the warp writes them again
        // in the next sweep, after a __syncthreads)
        for (int i = gw + lane * W; i < n; i += 32 * W) f[i] = f[i] - c;
        if (sqrt(row2) + sqrt(cs[0]) < tol) {
            conv = 1;
            break;
        }
        gsrc = h;
    }
    if (tid == 0 && r == 0) {
        pr.iters = it;
        pr.conv = conv;
    }
}

// ------------------------------------------------------------- block pass on FP64 tensor cores
// out[o][c] += sum_in e(o,in) W[in][c] as a GEMM: A = e (generated in registers,
// one cell per lane: row o = lane>>2, col in = lane&3), B = W (smem), C in
// registers, via mma.sync.m8n8k4.f64 (DMMA). DMMA shares the FP64 pipe with
// DFMA on sm_100 (tools/dmma_probe.cu) but replaces KT DFMAs + KT/2 shared-memory
// broadcasts per cell with KT/8 tensor instructions per 32 cells, which turns
// the issue-bound DFMA formulation into a pipe-bound one. Each warp owns MB
// 8-output blocks so B fragments are reused MB times.
__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

template <int KT>
struct WStride {  // smem row stride of W, == 4 (mod 16) doubles: the 16 lanes of a half-warp
                  // (rows lane>>2, k = lane&3) hit 16 distinct bank pairs for a B-fragment load
    static constexpr int value = KT + ((4 - KT % 16) + 16) % 16;
};

constexpr int MMA_NT = 128;  // 4 warps
constexpr int MMA_CH = 64;   // inputs per shared-memory round

// RS: also emit rsum[out_tile][in] = sum_o e(o, in) out_w[o] (the transposed,
// output-weighted sums, e.g. r = P~ beta of restricted_derivatives). Each lane's
// per-step partial over its MB outputs goes to the warp's staging rows in shared
// memory; at the end of a chunk each warp sums its 8 rows (warp-synchronous), and
// the 4 warp sums are combined after the next chunk's existing barrier. All sums
// run in a fixed order, so the result is deterministic, and every (out_tile, in)
// slot is written exactly once.
// MCH: inputs staged per shared-memory round (32 with RS keeps 4 CTAs per SM).
template <int D, int KT, int MB, bool RS = false, int MCH = MMA_CH>
__global__ void __launch_bounds__(MMA_NT) pts_mma_kernel(TileArgs a) {
    SKNR_PDL_ENTRY();
    constexpr int RS_LD = MCH + 4;  // staging row stride (conflict-free half-warp stores)
    if (guard_skip(a.st, a.guard)) return;
    constexpr int PK = PK_of<D>::value;
    constexpr int NCB = KT / 8;
    constexpr int WS = WStride<KT>::value;
    constexpr int OUT_WARP = 8 * MB;
    constexpr int OUT_CTA = OUT_WARP * (MMA_NT / 32);
    extern __shared__ __align__(16) double sm[];
    unsigned long long* tab = reinterpret_cast<unsigned long long*>(sm);
    double* sin = sm + kTabWords;
    double* sw = sin + MCH * PK;
    double* srs = sw + MCH * WS;                    // RS: staging [warp*8 + row][RS_LD]
    double* srw = srs + (MMA_NT / 32) * 8 * RS_LD;  // RS: warp sums [warp][MCH]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    load_exp2_table(tab, tid, MMA_NT);
    const unsigned laneoff = (lane & (kTabRep - 1)) << 3;
    const double c3 = pexp_c3();
    const int row = lane >> 2, kq = lane & 3;

    for (int64_t tile = blockIdx.x; tile < a.n_tiles; tile += gridDim.x) {
        const int64_t ot = tile % a.n_out_tiles, ib = tile / a.n_out_tiles;
        const int64_t obase = ot * OUT_CTA + warp * OUT_WARP;
        double Bo[MB], Yo[MB][D], Bw[MB];
#pragma unroll
        for (int mb = 0; mb < MB; ++mb) {
            int64_t o = obase + mb * 8 + row;
            if (RS) Bw[mb] = o < a.n_out ? a.out_w[o] : 0.0;
            o = o < a.n_out ? o : a.n_out - 1;
            Bo[mb] = a.out_pack[o * PK];
#pragma unroll
            for (int d = 0; d < D; ++d) Yo[mb][d] = a.out_pack[o * PK + 1 + d];
        }
        double acc[MB][NCB][2];
#pragma unroll
        for (int mb = 0; mb < MB; ++mb)
#pragma unroll
            for (int cb = 0; cb < NCB; ++cb) acc[mb][cb][0] = acc[mb][cb][1] = 0.0;

        const int64_t i0 = ib * a.in_block;
        const int64_t i1 = (i0 + a.in_block < a.n_in) ? i0 + a.in_block : a.n_in;
        int pend = 0;       // RS: inputs of the previous chunk whose warp sums await combining
        int64_t pbase = 0;  // RS: first input of that chunk
        auto rs_combine = [&]() {
            for (int k = tid; k < pend; k += MMA_NT)
                a.rsum[ot * a.n_in + pbase + k] = (srw[k] + srw[MCH + k]) + (srw[2 * MCH + k] + srw[3 * MCH + k]);
        };
        for (int64_t c0 = i0; c0 < i1; c0 += MCH) {
            const int cnt = static_cast<int>((i1 - c0) < MCH ? (i1 - c0) : MCH);
            const int cnt4 = (cnt + 3) & ~3;
            __syncthreads();
            if (RS) rs_combine();
            for (int t = tid; t < cnt4 * PK; t += MMA_NT) {
                const int k = t / PK, q = t % PK;
                sin[t] = k < cnt ? a.in_pack[(c0 + k) * PK + q] : (q == 0 ? -1e300 : 0.0);
            }
            for (int t = tid; t < cnt4 * KT; t += MMA_NT) {
                const int k = t / KT, c = t % KT;
                sw[k * WS + c] = k < cnt ? a.W[(c0 + k) * KT + c] : 0.0;
            }
            __syncthreads();
            for (int k4 = 0; k4 < cnt4; k4 += 4) {
                const double* xin = sin + (k4 + kq) * PK;
                double x[PK];
#pragma unroll
                for (int q = 0; q < PK / 2; ++q) {
                    const double2 v = reinterpret_cast<const double2*>(xin)[q];
                    x[2 * q] = v.x;
                    x[2 * q + 1] = v.y;
                }
                double bf[NCB];
#pragma unroll
                for (int cb = 0; cb < NCB; ++cb) bf[cb] = sw[(k4 + kq) * WS + cb * 8 + row];
                double rt = 0.0;
#pragma unroll
                for (int mb = 0; mb < MB; ++mb) {
                    double u = x[0] + Bo[mb];
#pragma unroll
                    for (int d = 0; d < D; ++d) u = fma(x[1 + d], Yo[mb][d], u);
                    const double e = pexp<true>(u, tab, laneoff, c3);
#pragma unroll
                    for (int cb = 0; cb < NCB; ++cb) dmma_8x8x4(acc[mb][cb][0], acc[mb][cb][1], e, bf[cb]);
                    if (RS) rt = mb == 0 ? e * Bw[0] : fma(e, Bw[mb], rt);
                }
                if (RS) srs[(warp * 8 + row) * RS_LD + k4 + kq] = rt;
            }
            if (RS) {
                __syncwarp();
                const double* st8 = srs + warp * 8 * RS_LD;
#pragma unroll
                for (int h = 0; h < MCH / 32; ++h) {
                    const int k = lane + 32 * h;
                    const double s01 = st8[k] + st8[RS_LD + k], s23 = st8[2 * RS_LD + k] + st8[3 * RS_LD + k];
                    const double s45 = st8[4 * RS_LD + k] + st8[5 * RS_LD + k];
                    const double s67 = st8[6 * RS_LD + k] + st8[7 * RS_LD + k];
                    srw[warp * MCH + k] = (s01 + s23) + (s45 + s67);
                }
                __syncwarp();
                pend = cnt;
                pbase = c0;
            }
        }
        if (RS) {
            __syncthreads();
            rs_combine();
        }
#pragma unroll
        for (int mb = 0; mb < MB; ++mb) {
            const int64_t o = obase + mb * 8 + row;
            if (o >= a.n_out) continue;
#pragma unroll
            for (int cb = 0; cb < NCB; ++cb) {
                const int c = cb * 8 + kq * 2;
                a.partial[(ib * KT + c) * a.n_out + o] = acc[mb][cb][0];
                a.partial[(ib * KT + c + 1) * a.n_out + o] = acc[mb][cb][1];
            }
        }
    }
}

// ------------------------------------------------------------- block pass v2 (double-buffered)
// Same arithmetic as pts_mma_kernel (DMMA m8n8k4 over the cell values e(o, in) generated in
// registers, optional fused RS row sums), restructured for the FP64 pipe:
//  * the input chunks (pack rows and W rows) are staged with cp.async into a double
//    buffer, so chunk c+1 streams in from L2 while chunk c is multiplied (one barrier per
//    chunk; the staging latency no longer stalls the CTA's warps);
//  * the work stream runs across tiles (the next tile's first chunk is prefetched during
//    the current tile's last chunk);
//  * NW warps per CTA share each staged chunk (NW = 8: 256-output tiles, half the
//    r-partial rows of the 128-output v1 tiles);
//  * RS warp sums are double-buffered by chunk parity, so the cross-warp combine of chunk
//    c (after the next barrier) never races the warps writing chunk c+1.
// Tail chunks are zero-filled (cp.async src-size 0): padded inputs have W = 0 and add 0
// to S; their RS slots are never written.
__device__ __forceinline__ void cp_async16_zfill(double* smem_dst, const double* gmem_src, int src_bytes) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem_src), "r"(src_bytes)
                 : "memory");
}

template <int D, int KT, int MB, bool RS, int MCH, int NW>
struct Mma2Layout {
    static constexpr int PK = PK_of<D>::value;
    static constexpr int WS = WStride<KT>::value;
    static constexpr int BUF = MCH * PK + MCH * WS;  // doubles per stage
    static constexpr int RS_LD = MCH + 4;
    static constexpr int words = kTabWords + 2 * BUF + (RS ? NW * 8 * RS_LD + 2 * NW * MCH : 0);
};

template <int D, int KT, int MB, bool RS, int MCH, int NW>
__global__ void __launch_bounds__(NW * 32) pts_mma2_kernel(TileArgs a) {
    SKNR_PDL_ENTRY();
    if (guard_skip(a.st, a.guard)) return;
    using L = Mma2Layout<D, KT, MB, RS, MCH, NW>;
    constexpr int NT = NW * 32;
    constexpr int PK = L::PK;
    constexpr int WS = L::WS;
    constexpr int NCB = KT / 8;
    constexpr int OUT_WARP = 8 * MB;
    constexpr int OUT_CTA = OUT_WARP * NW;
    constexpr int RS_LD = L::RS_LD;
    extern __shared__ __align__(16) double sm[];
    unsigned long long* tab = reinterpret_cast<unsigned long long*>(sm);
    double* stage = sm + kTabWords;
    double* srs = stage + 2 * L::BUF;     // RS: [NW*8][RS_LD] per-lane partials of one chunk
    double* srw = srs + NW * 8 * RS_LD;   // RS: [2][NW][MCH] warp sums, by chunk parity
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int row = lane >> 2, kq = lane & 3;
    if (static_cast<int64_t>(blockIdx.x) >= a.n_tiles) return;
    load_exp2_table(tab, tid, NT);
    const unsigned laneoff = (lane & (kTabRep - 1)) << 3;
    const double c3 = pexp_c3();

    auto blk_begin = [&](int64_t t) { return (t / a.n_out_tiles) * a.in_block; };
    auto blk_end = [&](int64_t t) {
        const int64_t e = blk_begin(t) + a.in_block;
        return e < a.n_in ? e : a.n_in;
    };
    auto issue = [&](int64_t t, int64_t c0, int b) {
        const int64_t c1 = blk_end(t);
        const int cnt = static_cast<int>((c1 - c0) < MCH ? (c1 - c0) : MCH);
        double* sin = stage + b * L::BUF;
        double* sw = sin + MCH * PK;
        for (int g = tid; g < MCH * PK / 2; g += NT) {
            const int k = g / (PK / 2);
            const bool ok = k < cnt;
            cp_async16_zfill(sin + 2 * g, a.in_pack + (c0 + (ok ? k : 0)) * PK + 2 * (g % (PK / 2)), ok ? 16 : 0);
        }
        for (int g = tid; g < MCH * KT / 2; g += NT) {
            const int k = g / (KT / 2), c2 = g % (KT / 2);
            const bool ok = k < cnt;
            cp_async16_zfill(sw + k * WS + 2 * c2, a.W + (c0 + (ok ? k : 0)) * KT + 2 * c2, ok ? 16 : 0);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };

    int64_t tile = blockIdx.x, c0 = blk_begin(tile);
    issue(tile, c0, 0);
    int buf = 0;
    double Bo[MB], Yo[MB][D], Bw[MB];
    double acc[MB][NCB][2];
    auto begin_tile = [&](int64_t t) {
        const int64_t obase = (t % a.n_out_tiles) * OUT_CTA + warp * OUT_WARP;
#pragma unroll
        for (int mb = 0; mb < MB; ++mb) {
            int64_t o = obase + mb * 8 + row;
            if (RS) Bw[mb] = o < a.n_out ? a.out_w[o] : 0.0;
            o = o < a.n_out ? o : a.n_out - 1;
            Bo[mb] = a.out_pack[o * PK];
#pragma unroll
            for (int d = 0; d < D; ++d) Yo[mb][d] = a.out_pack[o * PK + 1 + d];
#pragma unroll
            for (int cb = 0; cb < NCB; ++cb) acc[mb][cb][0] = acc[mb][cb][1] = 0.0;
        }
    };
    begin_tile(tile);
    // RS: the chunk whose warp sums (srw[parity]) await the cross-warp combine
    int pend = 0, pbuf = 0;
    int64_t pbase = 0, pot = 0;
    auto rs_combine = [&]() {
        const double* w = srw + pbuf * NW * MCH;
        for (int k = tid; k < pend; k += NT) {
            double v = w[k];
#pragma unroll
            for (int q = 1; q < NW; ++q) v += w[q * MCH + k];
            a.rsum[pot * a.n_in + pbase + k] = v;
        }
        pend = 0;
    };

    while (true) {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncthreads();  // chunk `buf` landed for every thread; all reads of buf^1 are done
        if (RS && pend) rs_combine();
        // next work item: the following chunk of this tile, else the first chunk of the next tile
        const int64_t c1 = blk_end(tile);
        int64_t ntile = tile, nc0 = c0 + MCH;
        if (nc0 >= c1) {
            ntile = tile + gridDim.x;
            nc0 = ntile < a.n_tiles ? blk_begin(ntile) : 0;
        }
        if (ntile < a.n_tiles) issue(ntile, nc0, buf ^ 1);
        const int cnt = static_cast<int>((c1 - c0) < MCH ? (c1 - c0) : MCH);
        const int cnt4 = (cnt + 3) & ~3;
        const double* sin = stage + buf * L::BUF;
        const double* sw = sin + MCH * PK;
        double* srs_w = srs + warp * 8 * RS_LD;
        for (int k4 = 0; k4 < cnt4; k4 += 4) {
            const double* xin = sin + (k4 + kq) * PK;
            double x[PK];
#pragma unroll
            for (int q = 0; q < PK / 2; ++q) {
                const double2 v = reinterpret_cast<const double2*>(xin)[q];
                x[2 * q] = v.x;
                x[2 * q + 1] = v.y;
            }
            double bf[NCB];
#pragma unroll
            for (int cb = 0; cb < NCB; ++cb) bf[cb] = sw[(k4 + kq) * WS + cb * 8 + row];
            double rt = 0.0;
#pragma unroll
            for (int mb = 0; mb < MB; ++mb) {
                double u = x[0] + Bo[mb];
#pragma unroll
                for (int d = 0; d < D; ++d) u = fma(x[1 + d], Yo[mb][d], u);
                const double e = pexp<true>(u, tab, laneoff, c3);
#pragma unroll
                for (int cb = 0; cb < NCB; ++cb) dmma_8x8x4(acc[mb][cb][0], acc[mb][cb][1], e, bf[cb]);
                if (RS) rt = mb == 0 ? e * Bw[0] : fma(e, Bw[mb], rt);
            }
            if (RS) srs_w[row * RS_LD + k4 + kq] = rt;
        }
        if (RS) {
            __syncwarp();
            double* w = srw + buf * NW * MCH + warp * MCH;
#pragma unroll
            for (int h = 0; h < MCH / 32; ++h) {
                const int k = lane + 32 * h;
                const double s01 = srs_w[k] + srs_w[RS_LD + k], s23 = srs_w[2 * RS_LD + k] + srs_w[3 * RS_LD + k];
                const double s45 = srs_w[4 * RS_LD + k] + srs_w[5 * RS_LD + k];
                const double s67 = srs_w[6 * RS_LD + k] + srs_w[7 * RS_LD + k];
                w[k] = (s01 + s23) + (s45 + s67);
            }
            __syncwarp();
            pend = cnt;
            pbuf = buf;
            pbase = c0;
            pot = tile % a.n_out_tiles;
        }
        if (ntile != tile) {  // tile done: its split-K partial of S
            const int64_t ib = tile / a.n_out_tiles;
            const int64_t obase = (tile % a.n_out_tiles) * OUT_CTA + warp * OUT_WARP;
#pragma unroll
            for (int mb = 0; mb < MB; ++mb) {
                const int64_t o = obase + mb * 8 + row;
                if (o >= a.n_out) continue;
#pragma unroll
                for (int cb = 0; cb < NCB; ++cb) {
                    const int c = cb * 8 + kq * 2;
                    a.partial[(ib * KT + c) * a.n_out + o] = acc[mb][cb][0];
                    a.partial[(ib * KT + c + 1) * a.n_out + o] = acc[mb][cb][1];
                }
            }
            if (ntile >= a.n_tiles) break;
            begin_tile(ntile);
        }
        tile = ntile;
        c0 = nc0;
        buf ^= 1;
    }
    if (RS) {
        __syncthreads();
        rs_combine();
    }
}

// Culled block pass (opt-in, see pts_cull_kernel): work unit = (32 Morton-ordered
// outputs, input block), taken from a queue by each warp; inputs are tested in
// groups of 32 against the unit's box with the output-normalised bound
// S'_o = S_o - LS log(total_o) supplied by the caller (0 when every output's terms
// sum to 1, e.g. P~ at h = f^{C,eps}); kept groups are staged warp-privately
// (inputs and their W rows gathered through perm_in) and multiplied on DMMA as
// in pts_mma_kernel.
constexpr int CULL_GB = 32;  // block-pass input group size
constexpr int CULL_GBO = 16;  // block-pass output group (one warp, MB = 2)

__device__ __forceinline__ void cp_async16(double* smem_dst, const double* gmem_src) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}

template <int D, int KT, int MB>
__global__ void __launch_bounds__(MMA_NT, 3) pts_mma_cull_kernel(TileArgs a) {
    SKNR_PDL_ENTRY();
    if (guard_skip(a.st, a.guard)) return;
    constexpr int PK = PK_of<D>::value;
    constexpr int NCB = KT / 8;
    constexpr int WS = WStride<KT>::value;
    static_assert(8 * MB == CULL_GBO, "one warp owns one output group");
    extern __shared__ __align__(16) double sm[];
    unsigned long long* tab = reinterpret_cast<unsigned long long*>(sm);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double* sin = sm + kTabWords + warp * (CULL_GB * PK + CULL_GB * WS);
    double* sw = sin + CULL_GB * PK;
    load_exp2_table(tab, tid, MMA_NT);
    __syncthreads();
    const unsigned laneoff = (lane & (kTabRep - 1)) << 3;
    const double c3 = pexp_c3();
    const int row = lane >> 2, kq = lane & 3;
    const double thr = -kLS * a.cull_t;

    while (true) {
        unsigned unit = 0;
        if (lane == 0) unit = atomicAdd(a.sched, 1u);
        unit = __shfl_sync(0xffffffffu, unit, 0);
        if (unit >= a.n_tiles) break;
        const int64_t og = unit % a.n_out_tiles, ib = unit / a.n_out_tiles;
        const int64_t obase = og * CULL_GBO;
        double Bo[MB], Yo[MB][D];
#pragma unroll
        for (int mb = 0; mb < MB; ++mb) {
            const int64_t pos = obase + mb * 8 + row;
            const int64_t oc = a.perm_out[pos < a.n_out ? pos : a.n_out - 1];
            Bo[mb] = a.out_pack[oc * PK];
#pragma unroll
            for (int d = 0; d < D; ++d) Yo[mb][d] = a.out_pack[oc * PK + 1 + d];
        }
        double acc[MB][NCB][2];
#pragma unroll
        for (int mb = 0; mb < MB; ++mb)
#pragma unroll
            for (int cb = 0; cb < NCB; ++cb) acc[mb][cb][0] = acc[mb][cb][1] = 0.0;
        double wbox[2 * D];
#pragma unroll
        for (int q = 0; q < 2 * D; ++q) wbox[q] = a.box_go[og * 2 * D + q];
        const double s_w = a.s_go[og];
        const int64_t i0 = ib * a.in_block;
        const int64_t i1 = (i0 + a.in_block < a.n_in) ? i0 + a.in_block : a.n_in;
        unsigned tested = 0, kept = 0;
        // the group tests of 32 consecutive groups run in parallel (one per lane);
        // the kept ones are then processed in order
#pragma unroll 1
        for (int64_t r0 = i0; r0 < i1; r0 += 32 * CULL_GB) {
            const int64_t gl = r0 / CULL_GB + lane;
            bool keep = false;
            if (gl * CULL_GB < i1)
                keep = !(a.f_gi[gl] + s_w - a.lskc * box_dist2<D>(a.box_gi + gl * 2 * D, wbox) < thr);
            unsigned mask = __ballot_sync(0xffffffffu, keep);
            {
                const int64_t ng = (i1 - r0 + CULL_GB - 1) / CULL_GB;
                tested += static_cast<unsigned>(ng < 32 ? ng : 32);
            }
            kept += __popc(mask);
#pragma unroll 1
        while (mask) {
            const int bit = __ffs(mask) - 1;
            mask &= mask - 1;
            const int64_t g0 = r0 + static_cast<int64_t>(bit) * CULL_GB;
            const int cnt = static_cast<int>((i1 - g0) < CULL_GB ? (i1 - g0) : CULL_GB);
            const int cnt4 = (cnt + 3) & ~3;
            __syncwarp();
            {
                // asynchronous gather (cp.async, 16 B per request, all in flight at once):
                // the group's inputs and their W rows; padded inputs get A = -inf, W = 0
                const int ii = lane < cnt ? a.perm_in[g0 + lane] : 0;
                if (lane < cnt) {
#pragma unroll
                    for (int q = 0; q < PK / 2; ++q)
                        cp_async16(sin + lane * PK + 2 * q, a.in_pack + static_cast<int64_t>(ii) * PK + 2 * q);
                } else {
#pragma unroll
                    for (int q = 0; q < PK; ++q) sin[lane * PK + q] = q == 0 ? -1e300 : 0.0;
                }
                constexpr int HC = KT / 2;  // 16-byte chunks per W row
#pragma unroll 4
                for (int c = lane; c < CULL_GB * HC; c += 32) {
                    const int k = c / HC, q = c - k * HC;
                    const int ik = __shfl_sync(0xffffffffu, ii, k);
                    if (k < cnt)
                        cp_async16(sw + k * WS + 2 * q, a.W + static_cast<int64_t>(ik) * KT + 2 * q);
                    else
                        *reinterpret_cast<double2*>(sw + k * WS + 2 * q) = make_double2(0.0, 0.0);
                }
                cp_async_wait_all();
            }
            __syncwarp();
#pragma unroll 1
            for (int k4 = 0; k4 < cnt4; k4 += 4) {
                const double* xin = sin + (k4 + kq) * PK;
                double x[PK];
#pragma unroll
                for (int q = 0; q < PK / 2; ++q) {
                    const double2 v = reinterpret_cast<const double2*>(xin)[q];
                    x[2 * q] = v.x;
                    x[2 * q + 1] = v.y;
                }
                double bf[NCB];
#pragma unroll
                for (int cb = 0; cb < NCB; ++cb) bf[cb] = sw[(k4 + kq) * WS + cb * 8 + row];
#pragma unroll
                for (int mb = 0; mb < MB; ++mb) {
                    double u = x[0] + Bo[mb];
#pragma unroll
                    for (int d = 0; d < D; ++d) u = fma(x[1 + d], Yo[mb][d], u);
                    const double e = pexp<true>(u, tab, laneoff, c3);
#pragma unroll
                    for (int cb = 0; cb < NCB; ++cb) dmma_8x8x4(acc[mb][cb][0], acc[mb][cb][1], e, bf[cb]);
                }
            }
        }
        }
#pragma unroll
        for (int mb = 0; mb < MB; ++mb) {
            const int64_t pos = obase + mb * 8 + row;
            if (pos >= a.n_out) continue;
            const int64_t o = a.perm_out[pos];
#pragma unroll
            for (int cb = 0; cb < NCB; ++cb) {
                const int c = cb * 8 + kq * 2;
                a.partial[(ib * KT + c) * a.n_out + o] = acc[mb][cb][0];
                a.partial[(ib * KT + c + 1) * a.n_out + o] = acc[mb][cb][1];
            }
        }
        if (lane == 0) {
            DevState* st = const_cast<DevState*>(a.st);
            atomicAdd(&st->n_cull_tested, static_cast<unsigned long long>(tested));
            atomicAdd(&st->n_cull_kept, static_cast<unsigned long long>(kept));
        }
    }
}

// Stored-cost block pass on DMMA: like pts_mma_kernel, with the A fragment's cell
// e(o, in) computed from C[o + in*ldc] (one global load per lane per 4 inputs,
// 8 consecutive outputs per 64 B segment), the next step's loads issued before
// the current step's math.
template <int KT, int MB>
__global__ void __launch_bounds__(MMA_NT) dense_mma_kernel(TileArgs a) {
    SKNR_PDL_ENTRY();
    if (guard_skip(a.st, a.guard)) return;
    constexpr int NCB = KT / 8;
    constexpr int WS = WStride<KT>::value;
    constexpr int OUT_WARP = 8 * MB;
    constexpr int OUT_CTA = OUT_WARP * (MMA_NT / 32);
    extern __shared__ __align__(16) double sm[];
    unsigned long long* tab = reinterpret_cast<unsigned long long*>(sm);
    double* sin = sm + kTabWords;
    double* sw = sin + MMA_CH;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    load_exp2_table(tab, tid, MMA_NT);
    const unsigned laneoff = (lane & (kTabRep - 1)) << 3;
    const double c3 = pexp_c3();
    const int row = lane >> 2, kq = lane & 3;
    const double nk = -a.kappa;

    for (int64_t tile = blockIdx.x; tile < a.n_tiles; tile += gridDim.x) {
        const int64_t ot = tile % a.n_out_tiles, ib = tile / a.n_out_tiles;
        const int64_t obase = ot * OUT_CTA + warp * OUT_WARP;
        double Bo[MB];
        int64_t oc[MB];
#pragma unroll
        for (int mb = 0; mb < MB; ++mb) {
            const int64_t o = obase + mb * 8 + row;
            oc[mb] = o < a.n_out ? o : a.n_out - 1;
            Bo[mb] = a.out_pack[oc[mb]];
        }
        double acc[MB][NCB][2];
#pragma unroll
        for (int mb = 0; mb < MB; ++mb)
#pragma unroll
            for (int cb = 0; cb < NCB; ++cb) acc[mb][cb][0] = acc[mb][cb][1] = 0.0;
        const int64_t i0 = ib * a.in_block;
        const int64_t i1 = (i0 + a.in_block < a.n_in) ? i0 + a.in_block : a.n_in;
        for (int64_t c0 = i0; c0 < i1; c0 += MMA_CH) {
            const int cnt = static_cast<int>((i1 - c0) < MMA_CH ? (i1 - c0) : MMA_CH);
            const int cnt4 = (cnt + 3) & ~3;
            __syncthreads();
            for (int t = tid; t < cnt4; t += MMA_NT) sin[t] = t < cnt ? a.in_pack[c0 + t] : -1e300;
            for (int t = tid; t < cnt4 * KT; t += MMA_NT) {
                const int k = t / KT, c = t % KT;
                sw[k * WS + c] = k < cnt ? a.W[(c0 + k) * KT + c] : 0.0;
            }
            __syncthreads();
            double cv[MB];
            {
                const int64_t in = c0 + (kq < cnt ? kq : cnt - 1);
#pragma unroll
                for (int mb = 0; mb < MB; ++mb) cv[mb] = __ldcs(a.C + in * a.ldc + oc[mb]);
            }
            for (int k4 = 0; k4 < cnt4; k4 += 4) {
                double nv[MB];
                const int kn = k4 + 4 + kq;
                const int64_t inn = c0 + (kn < cnt ? kn : cnt - 1);
#pragma unroll
                for (int mb = 0; mb < MB; ++mb) nv[mb] = __ldcs(a.C + inn * a.ldc + oc[mb]);
                const double ak = sin[k4 + kq];
                double bf[NCB];
#pragma unroll
                for (int cb = 0; cb < NCB; ++cb) bf[cb] = sw[(k4 + kq) * WS + cb * 8 + row];
#pragma unroll
                for (int mb = 0; mb < MB; ++mb) {
                    const double u = fma(nk, cv[mb], ak + Bo[mb]);
                    const double e = pexp<true>(u, tab, laneoff, c3);
#pragma unroll
                    for (int cb = 0; cb < NCB; ++cb) dmma_8x8x4(acc[mb][cb][0], acc[mb][cb][1], e, bf[cb]);
                    cv[mb] = nv[mb];
                }
            }
        }
#pragma unroll
        for (int mb = 0; mb < MB; ++mb) {
            const int64_t o = obase + mb * 8 + row;
            if (o >= a.n_out) continue;
#pragma unroll
            for (int cb = 0; cb < NCB; ++cb) {
                const int c = cb * 8 + kq * 2;
                a.partial[(ib * KT + c) * a.n_out + o] = acc[mb][cb][0];
                a.partial[(ib * KT + c + 1) * a.n_out + o] = acc[mb][cb][1];
            }
        }
    }
}

// ------------------------------------------------------------- on-the-fly, large d
// u = A_in + B_out + <X_in, Y_out> with the d-contraction on FP64 tensor cores:
// each warp forms 8x8 (output x input) blocks of u with DK/4 DMMAs (A = Y_out
// fragment, registers; B = X_in fragment, shared memory), then evaluates the
// exponentials from the accumulator fragment (2 cells per lane). MODE_BLOCK
// re-shuffles the exponentials into A fragments of a second DMMA chain against
// W (the ell-wide pass). Pack rows: (A, x_0 .. x_{d-1}, 0-padding), stride DK+2.
template <int DK>
struct XStride {  // smem stride of staged X rows: == 4 or 12 (mod 16) -> conflict-free B fragments
    static constexpr int value = DK + 4;
};

constexpr int CT_NT = 128;
constexpr int CT_CH = 64;

template <int DK, int MODE, int KT, int MB>
__global__ void __launch_bounds__(CT_NT) pts_contract_kernel(TileArgs a) {
    SKNR_PDL_ENTRY();
    if (guard_skip(a.st, a.guard)) return;
    constexpr int PK = DK + 2;
    constexpr int NK = DK / 4;
    constexpr int XS = XStride<DK>::value;
    constexpr int KA = KT > 0 ? KT : 8;
    constexpr int NCB = KA / 8;
    constexpr int WS = WStride<KA>::value;
    constexpr int OUT_WARP = 8 * MB;
    constexpr int OUT_CTA = OUT_WARP * (CT_NT / 32);
    extern __shared__ __align__(16) double sm[];
    unsigned long long* tab = reinterpret_cast<unsigned long long*>(sm);
    double* sX = sm + kTabWords;
    double* sA = sX + CT_CH * XS;
    double* sw = sA + CT_CH;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    load_exp2_table(tab, tid, CT_NT);
    const unsigned laneoff = (lane & (kTabRep - 1)) << 3;
    const double c3 = pexp_c3();
    const int row = lane >> 2, kq = lane & 3;
    const double ninf = -__longlong_as_double(0x7FF0000000000000LL);

    for (int64_t tile = blockIdx.x; tile < a.n_tiles; tile += gridDim.x) {
        const int64_t ot = tile % a.n_out_tiles, ib = tile / a.n_out_tiles;
        const int64_t obase = ot * OUT_CTA + warp * OUT_WARP;
        double yf[MB][NK], Bo[MB];
        double acc[MB];
        double bacc[MB][NCB][2];
#pragma unroll
        for (int mb = 0; mb < MB; ++mb) {
            int64_t o = obase + mb * 8 + row;
            o = o < a.n_out ? o : a.n_out - 1;
            const double* yo = a.out_pack + o * PK;
            Bo[mb] = yo[0];
#pragma unroll
            for (int kk = 0; kk < NK; ++kk) yf[mb][kk] = yo[1 + kk * 4 + kq];
            acc[mb] = (MODE == MODE_MAX) ? ninf : 0.0;
#pragma unroll
            for (int cb = 0; cb < NCB; ++cb) bacc[mb][cb][0] = bacc[mb][cb][1] = 0.0;
        }
        const int64_t i0 = ib * a.in_block;
        const int64_t i1 = (i0 + a.in_block < a.n_in) ? i0 + a.in_block : a.n_in;
        for (int64_t c0 = i0; c0 < i1; c0 += CT_CH) {
            const int cnt = static_cast<int>((i1 - c0) < CT_CH ? (i1 - c0) : CT_CH);
            const int cnt8 = (cnt + 7) & ~7;
            __syncthreads();
            for (int t = tid; t < cnt8 * DK; t += CT_NT) {
                const int k = t / DK, q = t % DK;
                sX[k * XS + q] = k < cnt ? a.in_pack[(c0 + k) * PK + 1 + q] : 0.0;
            }
            for (int t = tid; t < cnt8; t += CT_NT) sA[t] = t < cnt ? a.in_pack[(c0 + t) * PK] : -1e300;
            if (MODE == MODE_BLOCK)
                for (int t = tid; t < cnt8 * KA; t += CT_NT) {
                    const int k = t / KA, c = t % KA;
                    sw[k * WS + c] = k < cnt ? a.W[(c0 + k) * KA + c] : 0.0;
                }
            __syncthreads();
            for (int j8 = 0; j8 < cnt8; j8 += 8) {
                double xf[NK];
#pragma unroll
                for (int kk = 0; kk < NK; ++kk) xf[kk] = sX[(j8 + row) * XS + kk * 4 + kq];
                const double a0 = sA[j8 + 2 * kq], a1 = sA[j8 + 2 * kq + 1];
                double wf[2][NCB];
                if (MODE == MODE_BLOCK) {
#pragma unroll
                    for (int h = 0; h < 2; ++h)
#pragma unroll
                        for (int cb = 0; cb < NCB; ++cb) wf[h][cb] = sw[(j8 + 4 * h + kq) * WS + cb * 8 + row];
                }
#pragma unroll
                for (int mb = 0; mb < MB; ++mb) {
                    double u0 = 0.0, u1 = 0.0;
#pragma unroll
                    for (int kk = 0; kk < NK; ++kk) dmma_8x8x4(u0, u1, yf[mb][kk], xf[kk]);
                    u0 += a0 + Bo[mb];
                    u1 += a1 + Bo[mb];
                    if (MODE == MODE_SUM) {
                        acc[mb] = pexp_acc<false>(u0, tab, laneoff, c3, acc[mb]);
                        acc[mb] = pexp_acc<false>(u1, tab, laneoff, c3, acc[mb]);
                    } else if (MODE == MODE_MAX) {
                        acc[mb] = fmax(acc[mb], fmax(u0, u1));
                    } else {
                        const double e0 = pexp<true>(u0, tab, laneoff, c3);
                        const double e1 = pexp<true>(u1, tab, laneoff, c3);
                        // A fragment of chunk h needs e(row, 4h + kq), held by lane
                        // row*4 + 2h + kq/2 as element kq&1
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int src = (lane & ~3) + 2 * h + (kq >> 1);
                            const double s0 = __shfl_sync(0xffffffffu, e0, src);
                            const double s1 = __shfl_sync(0xffffffffu, e1, src);
                            const double af = (kq & 1) ? s1 : s0;
#pragma unroll
                            for (int cb = 0; cb < NCB; ++cb)
                                dmma_8x8x4(bacc[mb][cb][0], bacc[mb][cb][1], af, wf[h][cb]);
                        }
                    }
                }
            }
        }
#pragma unroll
        for (int mb = 0; mb < MB; ++mb) {
            const int64_t o = obase + mb * 8 + row;
            if (MODE == MODE_BLOCK) {
                if (o >= a.n_out) continue;
#pragma unroll
                for (int cb = 0; cb < NCB; ++cb) {
                    const int c = cb * 8 + kq * 2;
                    a.partial[(ib * KA + c) * a.n_out + o] = bacc[mb][cb][0];
                    a.partial[(ib * KA + c + 1) * a.n_out + o] = bacc[mb][cb][1];
                }
            } else {
                double v = acc[mb];
                const double w1 = __shfl_xor_sync(0xffffffffu, v, 1);
                v = (MODE == MODE_MAX) ? fmax(v, w1) : v + w1;
                const double w2 = __shfl_xor_sync(0xffffffffu, v, 2);
                v = (MODE == MODE_MAX) ? fmax(v, w2) : v + w2;
                if (kq == 0 && o < a.n_out) a.partial[ib * a.n_out + o] = v;
            }
        }
    }
}

// ------------------------------------------------------------- stored cost
template <int JT, int MODE, int KT>
__global__ void __launch_bounds__(NT_of<MODE>::value) dense_tile_kernel(TileArgs a) {
    SKNR_PDL_ENTRY();
    if (guard_skip(a.st, a.guard)) return;
    constexpr int NT = NT_of<MODE>::value;
    constexpr int CH = Chunk<MODE, KT>::value;
    constexpr int KA = KT > 0 ? KT : 1;
    constexpr int U = 4;  // inputs per unrolled step: U*JT independent loads in flight
    extern __shared__ __align__(16) double sm[];
    unsigned long long* tab = reinterpret_cast<unsigned long long*>(sm);
    double* sin = sm + kTabWords;
    double* sw = sin + CH;
    const int tid = threadIdx.x;
    load_exp2_table(tab, tid, NT);
    const unsigned laneoff = (tid & (kTabRep - 1)) << 3;
    const double c3 = pexp_c3();
    const int64_t out_tile = static_cast<int64_t>(NT) * JT;
    const double nk = -a.kappa;

    for (int64_t tile = blockIdx.x; tile < a.n_tiles; tile += gridDim.x) {
        const int64_t ot = tile % a.n_out_tiles, ib = tile / a.n_out_tiles;
        double B[JT];
        double acc[JT][KA];
        int64_t o[JT], oc[JT];
#pragma unroll
        for (int jt = 0; jt < JT; ++jt) {
            o[jt] = ot * out_tile + jt * NT + tid;
            oc[jt] = o[jt] < a.n_out ? o[jt] : a.n_out - 1;
            B[jt] = a.out_pack[oc[jt]];
            acc_init<MODE, KA>(acc[jt]);
        }
        const int64_t i0 = ib * a.in_block;
        const int64_t i1 = (i0 + a.in_block < a.n_in) ? i0 + a.in_block : a.n_in;
        for (int64_t c0 = i0; c0 < i1; c0 += CH) {
            const int cnt = static_cast<int>((i1 - c0) < CH ? (i1 - c0) : CH);
            __syncthreads();
            for (int t = tid; t < cnt; t += NT) sin[t] = a.in_pack[c0 + t];
            if (MODE == MODE_BLOCK) {
                const double2* wsrc = reinterpret_cast<const double2*>(a.W + c0 * KA);
                double2* wdst = reinterpret_cast<double2*>(sw);
                for (int t = tid; t < cnt * KA / 2; t += NT) wdst[t] = wsrc[t];
            }
            __syncthreads();
            const double* Cb = a.C + c0 * a.ldc;
            int k = 0;
            for (; k + U <= cnt; k += U) {
                double cv[U][JT];
#pragma unroll
                for (int q = 0; q < U; ++q)
#pragma unroll
                    for (int jt = 0; jt < JT; ++jt)
                        cv[q][jt] = __ldcs(Cb + (k + q) * a.ldc + oc[jt]);
#pragma unroll
                for (int q = 0; q < U; ++q) {
                    const double ak = sin[k + q];
#pragma unroll
                    for (int jt = 0; jt < JT; ++jt) {
                        const double u = fma(nk, cv[q][jt], ak + B[jt]);
                        if (MODE == MODE_SUM) {
                            acc[jt][0] = pexp_acc<false>(u, tab, laneoff, c3, acc[jt][0]);
                        } else if (MODE == MODE_MAX) {
                            acc[jt][0] = fmax(acc[jt][0], u);
                        } else {
                            const double e = pexp<true>(u, tab, laneoff, c3);
#pragma unroll
                            for (int c = 0; c < KA; c += 2) {
                                const double2 w =
                                    reinterpret_cast<const double2*>(sw + (k + q) * KA)[c / 2];
                                acc[jt][c] = fma(e, w.x, acc[jt][c]);
                                acc[jt][c + 1] = fma(e, w.y, acc[jt][c + 1]);
                            }
                        }
                    }
                }
            }
            for (; k < cnt; ++k) {
                const double ak = sin[k];
#pragma unroll
                for (int jt = 0; jt < JT; ++jt) {
                    const double u = fma(nk, __ldcs(Cb + k * a.ldc + oc[jt]), ak + B[jt]);
                    if (MODE == MODE_SUM) {
                        acc[jt][0] = pexp_acc<false>(u, tab, laneoff, c3, acc[jt][0]);
                    } else if (MODE == MODE_MAX) {
                        acc[jt][0] = fmax(acc[jt][0], u);
                    } else {
                        const double e = pexp<true>(u, tab, laneoff, c3);
#pragma unroll
                        for (int c = 0; c < KA; c += 2) {
                            const double2 w = reinterpret_cast<const double2*>(sw + k * KA)[c / 2];
                            acc[jt][c] = fma(e, w.x, acc[jt][c]);
                            acc[jt][c + 1] = fma(e, w.y, acc[jt][c + 1]);
                        }
                    }
                }
            }
        }
#pragma unroll
        for (int jt = 0; jt < JT; ++jt) {
            if (o[jt] >= a.n_out) continue;
            if (MODE == MODE_BLOCK) {
#pragma unroll
                for (int c = 0; c < KA; ++c) a.partial[(ib * KA + c) * a.n_out + o[jt]] = acc[jt][c];
            } else {
                a.partial[ib * a.n_out + o[jt]] = acc[jt][0];
            }
        }
    }
}

// Stored cost, 128-bit loads: each thread owns JT2 pairs of adjacent outputs and
// streams them with one double2 load per input (requires even ldc and n_out).
template <int JT2, int U, int NTT, int MODE>
__global__ void __launch_bounds__(NTT) dense_v2_kernel(TileArgs a) {
    SKNR_PDL_ENTRY();
    if (guard_skip(a.st, a.guard)) return;
    constexpr int NT = NTT;
    constexpr int CH = 256;
    extern __shared__ __align__(16) double sm[];
    unsigned long long* tab = reinterpret_cast<unsigned long long*>(sm);
    double* sin = sm + kTabWords;
    const int tid = threadIdx.x;
    load_exp2_table(tab, tid, NT);
    const unsigned laneoff = (tid & (kTabRep - 1)) << 3;
    const double c3 = pexp_c3();
    const int64_t out_tile = static_cast<int64_t>(NT) * 2 * JT2;
    const double nk = -a.kappa;
    for (int64_t tile = blockIdx.x; tile < a.n_tiles; tile += gridDim.x) {
        const int64_t ot = tile % a.n_out_tiles, ib = tile / a.n_out_tiles;
        double B0[JT2], B1[JT2], acc0[JT2], acc1[JT2];
        int64_t o[JT2], oc[JT2];
#pragma unroll
        for (int jt = 0; jt < JT2; ++jt) {
            o[jt] = ot * out_tile + 2 * (jt * NT + tid);
            oc[jt] = o[jt] < a.n_out ? o[jt] : a.n_out - 2;
            B0[jt] = a.out_pack[oc[jt]];
            B1[jt] = a.out_pack[oc[jt] + 1];
            acc0[jt] = acc1[jt] = (MODE == MODE_MAX) ? -__longlong_as_double(0x7FF0000000000000LL) : 0.0;
        }
        const int64_t i0 = ib * a.in_block;
        const int64_t i1 = (i0 + a.in_block < a.n_in) ? i0 + a.in_block : a.n_in;
        for (int64_t c0 = i0; c0 < i1; c0 += CH) {
            const int cnt = static_cast<int>((i1 - c0) < CH ? (i1 - c0) : CH);
            __syncthreads();
            for (int t = tid; t < cnt; t += NT) sin[t] = a.in_pack[c0 + t];
            __syncthreads();
            const double* Cb = a.C + c0 * a.ldc;
            int k = 0;
            for (; k < cnt; k += U) {
                double2 cv[U][JT2];
#pragma unroll
                for (int q = 0; q < U; ++q)
#pragma unroll
                    for (int jt = 0; jt < JT2; ++jt)
                        cv[q][jt] = (k + q < cnt)
                                        ? __ldcs(reinterpret_cast<const double2*>(Cb + (k + q) * a.ldc + oc[jt]))
                                        : make_double2(0.0, 0.0);
#pragma unroll
                for (int q = 0; q < U; ++q) {
                    if (k + q >= cnt) break;
                    const double ak = sin[k + q];
#pragma unroll
                    for (int jt = 0; jt < JT2; ++jt) {
                        const double u0 = fma(nk, cv[q][jt].x, ak + B0[jt]);
                        const double u1 = fma(nk, cv[q][jt].y, ak + B1[jt]);
                        if (MODE == MODE_SUM) {
                            acc0[jt] = pexp_acc<false>(u0, tab, laneoff, c3, acc0[jt]);
                            acc1[jt] = pexp_acc<false>(u1, tab, laneoff, c3, acc1[jt]);
                        } else {
                            acc0[jt] = fmax(acc0[jt], u0);
                            acc1[jt] = fmax(acc1[jt], u1);
                        }
                    }
                }
            }
        }
#pragma unroll
        for (int jt = 0; jt < JT2; ++jt) {
            if (o[jt] >= a.n_out) continue;
            a.partial[ib * a.n_out + o[jt]] = acc0[jt];
            a.partial[ib * a.n_out + o[jt] + 1] = acc1[jt];
        }
    }
}

// ------------------------------------------------------------- dispatch
struct KernelInfo {
    const void* fn = nullptr;
    int jt = 1;
    int nt = 128;
    int out_tile = 0;  // outputs per CTA tile (0: nt * jt)
    int smem = 0;
    int occ = 0;
};

template <int D, int JT, int MODE, int KT, int NTT = NT_of<MODE>::value, int UNR = 2, bool FC = false,
          int MINB = 1>
KernelInfo make_pts() {
    KernelInfo k;
    k.fn = reinterpret_cast<const void*>(&pts_tile_kernel<D, JT, MODE, KT, NTT, UNR, FC, MINB>);
    k.jt = JT;
    k.nt = NTT;
    constexpr int CH = Chunk<MODE, KT>::value;
    k.smem = static_cast<int>(sizeof(double)) *
             (kTabWords + CH * PK_of<D>::value + (MODE == MODE_BLOCK ? CH * KT : 0));
    return k;
}

template <int D, int JT, int NTT, bool FC = false>
KernelInfo make_sum10() {
    KernelInfo k;
    k.fn = reinterpret_cast<const void*>(&pts_sum10_kernel<D, JT, NTT, FC>);
    k.jt = JT;
    k.nt = NTT;
    k.smem = static_cast<int>(sizeof(double)) * (kTab10Words + 256 * PK_of<D>::value);
    return k;
}

template <int D, int JT, int NTT, int REP, bool FC = false, int MINB = 1, int UNR = 1>
KernelInfo make_sum12() {
    KernelInfo k;
    k.fn = reinterpret_cast<const void*>(&pts_sum12_kernel<D, JT, NTT, REP, FC, MINB, UNR>);
    k.jt = JT;
    k.nt = NTT;
    k.smem = static_cast<int>(sizeof(double)) * (4096 * REP + 256 * PK_of<D>::value);
    return k;
}

template <int D, int JT, int NTT, int REP, int UNR = 1>
KernelInfo make_anchor12() {
    KernelInfo k;
    k.fn = reinterpret_cast<const void*>(&pts_anchor12_kernel<D, JT, NTT, REP, UNR>);
    k.jt = JT;
    k.nt = NTT;
    k.smem = static_cast<int>(sizeof(double)) * (4096 * REP + 256 * (PK_of<D>::value + 2));
    return k;
}

template <int D, int JT, int NTT, int MINB = 1>
KernelInfo make_f32() {
    KernelInfo k;
    k.fn = reinterpret_cast<const void*>(&pts_f32_kernel<D, JT, NTT, MINB>);
    k.jt = JT;
    k.nt = NTT;
    k.smem = static_cast<int>(sizeof(float)) * 256 * PKF_of<D>::value;
    return k;
}

template <int D, bool F32 = false>
KernelInfo make_cull() {
    KernelInfo k;
    k.fn = reinterpret_cast<const void*>(&pts_cull_kernel<D, 4, 256, F32>);
    k.jt = 4;
    k.nt = 256;
    k.out_tile = CULL_GO;  // work units are per warp
    k.smem = static_cast<int>(sizeof(double)) * (kTabWords + 8 * CULL_GI * PK_of<D>::value);
    return k;
}

template <int JT, int MODE, int KT>
KernelInfo make_dense() {
    KernelInfo k;
    k.fn = reinterpret_cast<const void*>(&dense_tile_kernel<JT, MODE, KT>);
    k.jt = JT;
    k.nt = NT_of<MODE>::value;
    constexpr int CH = Chunk<MODE, KT>::value;
    k.smem = static_cast<int>(sizeof(double)) * (kTabWords + CH + (MODE == MODE_BLOCK ? CH * KT : 0));
    return k;
}

template <int D, int KT, int MB, bool RS = false, int MCH = MMA_CH>
KernelInfo make_mma() {
    static_assert(MCH % 32 == 0 && MCH <= MMA_CH, "chunk must be a multiple of 32");
    KernelInfo k;
    k.fn = reinterpret_cast<const void*>(&pts_mma_kernel<D, KT, MB, RS, MCH>);
    k.jt = 1;
    k.nt = MMA_NT;
    k.out_tile = 8 * MB * (MMA_NT / 32);
    k.smem = static_cast<int>(sizeof(double)) * (kTabWords + MCH * PK_of<D>::value + MCH * WStride<KT>::value +
                                                 (RS ? (MMA_NT / 32) * (8 * (MCH + 4) + MCH) : 0));
    return k;
}

template <int D, int KT, int MB, bool RS, int MCH, int NW>
KernelInfo make_mma2() {
    KernelInfo k;
    k.fn = reinterpret_cast<const void*>(&pts_mma2_kernel<D, KT, MB, RS, MCH, NW>);
    k.jt = 1;
    k.nt = NW * 32;
    k.out_tile = 8 * MB * NW;
    k.smem = static_cast<int>(sizeof(double)) * Mma2Layout<D, KT, MB, RS, MCH, NW>::words;
    return k;
}

template <int D, int KT>
KernelInfo make_mma_cull() {
    KernelInfo k;
    k.fn = reinterpret_cast<const void*>(&pts_mma_cull_kernel<D, KT, 2>);
    k.jt = 1;
    k.nt = MMA_NT;
    k.out_tile = CULL_GBO;
    k.smem = static_cast<int>(sizeof(double)) *
             (kTabWords + (MMA_NT / 32) * (CULL_GB * PK_of<D>::value + CULL_GB * WStride<KT>::value));
    return k;
}

template <int DK, int MODE, int KT, int MB>
KernelInfo make_contract() {
    KernelInfo k;
    k.fn = reinterpret_cast<const void*>(&pts_contract_kernel<DK, MODE, KT, MB>);
    k.jt = 1;
    k.nt = CT_NT;
    k.out_tile = 8 * MB * (CT_NT / 32);
    constexpr int KA = KT > 0 ? KT : 8;
    k.smem = static_cast<int>(sizeof(double)) *
             (kTabWords + CT_CH * XStride<DK>::value + CT_CH + (MODE == MODE_BLOCK ? CT_CH * WStride<KA>::value : 0));
    return k;
}

template <int DK>
KernelInfo pick_contract(int mode, int kt) {
    if (mode == MODE_BLOCK_RS || mode == MODE_SUM_CULL || mode == MODE_BLOCK_CULL || mode == MODE_SUM_F32 ||
        mode == MODE_SUM_CULL_F32)
        return KernelInfo{};
    if (mode == MODE_SUM) return make_contract<DK, MODE_SUM, 0, 2>();
    if (mode == MODE_MAX) return make_contract<DK, MODE_MAX, 0, 2>();
    switch (kt) {
        case 8: return make_contract<DK, MODE_BLOCK, 8, 1>();
        case 16: return make_contract<DK, MODE_BLOCK, 16, 1>();
        case 24: return make_contract<DK, MODE_BLOCK, 24, 1>();
        case 32: return make_contract<DK, MODE_BLOCK, 32, 1>();
        case 40: return make_contract<DK, MODE_BLOCK, 40, 1>();
        case 48: return make_contract<DK, MODE_BLOCK, 48, 1>();
        case 64: return make_contract<DK, MODE_BLOCK, 64, 1>();
        default: return KernelInfo{};
    }
}

KernelInfo tune_variant(int v);

template <int D>
KernelInfo pick_pts(int mode, int kt) {
    // SKNR_SUM_VARIANT=v (d = 2): run the sum passes with tune variant v (numerics checks of
    // the variants, tools/tune_lse.py)
    static const int sum_variant = std::getenv("SKNR_SUM_VARIANT") ? std::atoi(std::getenv("SKNR_SUM_VARIANT")) : -1;
    if (mode == MODE_SUM && D == 2 && sum_variant >= 0 && sum_variant < 100) return tune_variant(sum_variant);
    // 4096-entry table (10 FP64 slots per cell), JT=8, 512 threads, 4 table copies, inner
    // loop unrolled 2x: best of the launch sweep (tools/tune_lse.py, variants 4-69: C4
    // column LSE 3.08 ms vs 3.57 ms for the 256-entry pts_tile_kernel)
    if (mode == MODE_SUM) return D == 4 ? make_sum12<4, 6, 512, 4, false, 1, 2>()  // 8 outputs spill at d = 4
                                        : make_sum12<D, 8, 512, 4, false, 1, 2>();
    if (mode == MODE_MAX) return make_pts<D, 4, MODE_MAX, 0>();
    if (mode == MODE_SUM_CULL) return make_cull<D>();
    if (mode == MODE_SUM_CULL_F32) return make_cull<D, true>();
    if (mode == MODE_SUM_F32) return make_f32<D, 8, 512, 2>();  // best of tools/fp32_probe.py variants 300-311
    if (mode == MODE_BLOCK_CULL) {
        switch (kt) {
            case 8: return make_mma_cull<D, 8>();
            case 16: return make_mma_cull<D, 16>();
            case 24: return make_mma_cull<D, 24>();
            case 32: return make_mma_cull<D, 32>();
            case 40: return make_mma_cull<D, 40>();
            case 48: return make_mma_cull<D, 48>();
            case 64: return make_mma_cull<D, 64>();
            default: return KernelInfo{};
        }
    }
    if (mode == MODE_BLOCK && kt == 4)  // the stable accept test's anchor pass (s, t, u)
        return D == 4 ? make_anchor12<4, 4, 512, 4, 1>() : make_anchor12<D, 4, 512, 4, 2>();  // tune 400-405
    // FP64 tensor-core (DMMA) block passes. Default: the double-buffered v2 kernel (8 warps,
    // 256-output tiles, 32-input chunks); SKNR_BLOCK_V1=1 selects the round-1 kernel.
    static const bool v1 = std::getenv("SKNR_BLOCK_V1") != nullptr;
    if (mode == MODE_BLOCK_RS) {
        if (v1) {  // 32-input rounds: 4 CTAs/SM fit (C4 ell=32: 13.9 ms vs 14.1 ms at 64)
            switch (kt) {
                case 8: return make_mma<D, 8, 4, true, 32>();
                case 16: return make_mma<D, 16, 4, true, 32>();
                case 24: return make_mma<D, 24, 4, true, 32>();
                case 32: return make_mma<D, 32, 4, true, 32>();
                case 40: return make_mma<D, 40, 4, true, 32>();
                case 48: return make_mma<D, 48, 2, true, 32>();
                case 64: return make_mma<D, 64, 2, true, 32>();
                default: return KernelInfo{};
            }
        }
        switch (kt) {
            case 8: return make_mma2<D, 8, 4, true, 32, 8>();
            case 16: return make_mma2<D, 16, 4, true, 32, 8>();
            case 24: return make_mma2<D, 24, 4, true, 32, 8>();
            case 32: return make_mma2<D, 32, 4, true, 32, 8>();
            case 40: return make_mma2<D, 40, 4, true, 32, 8>();
            case 48: return make_mma2<D, 48, 2, true, 32, 8>();
            case 64: return make_mma2<D, 64, 2, true, 32, 8>();
            default: return KernelInfo{};
        }
    }
    if (v1) {
        switch (kt) {  // 4 x 8-output blocks per warp
            case 8: return make_mma<D, 8, 4>();
            case 16: return make_mma<D, 16, 4>();
            case 24: return make_mma<D, 24, 4>();
            case 32: return make_mma<D, 32, 4>();
            case 40: return make_mma<D, 40, 4>();
            case 48: return make_mma<D, 48, 2>();
            case 64: return make_mma<D, 64, 2>();
            default: return KernelInfo{};
        }
    }
    switch (kt) {
        case 8: return make_mma2<D, 8, 4, false, 32, 8>();
        case 16: return make_mma2<D, 16, 4, false, 32, 8>();
        case 24: return make_mma2<D, 24, 4, false, 32, 8>();
        case 32: return make_mma2<D, 32, 4, false, 32, 8>();
        case 40: return make_mma2<D, 40, 4, false, 32, 8>();
        case 48: return make_mma2<D, 48, 2, false, 32, 8>();
        case 64: return make_mma2<D, 64, 2, false, 32, 8>();
        default: return KernelInfo{};
    }
}

template <int JT2, int U, int NTT, int MODE>
KernelInfo make_dense_v2() {
    KernelInfo k;
    k.fn = reinterpret_cast<const void*>(&dense_v2_kernel<JT2, U, NTT, MODE>);
    k.jt = 2 * JT2;
    k.nt = NTT;
    k.smem = static_cast<int>(sizeof(double)) * (kTabWords + 256);
    return k;
}

template <int KT, int MB>
KernelInfo make_dense_mma() {
    KernelInfo k;
    k.fn = reinterpret_cast<const void*>(&dense_mma_kernel<KT, MB>);
    k.jt = 1;
    k.nt = MMA_NT;
    k.out_tile = 8 * MB * (MMA_NT / 32);
    k.smem = static_cast<int>(sizeof(double)) * (kTabWords + MMA_CH + MMA_CH * WStride<KT>::value);
    return k;
}

KernelInfo pick_dense(int mode, int kt) {
    if (mode == MODE_BLOCK_RS || mode == MODE_SUM_CULL || mode == MODE_BLOCK_CULL || mode == MODE_SUM_F32 ||
        mode == MODE_SUM_CULL_F32)
        return KernelInfo{};
    if (mode == MODE_SUM) return make_dense<2, MODE_SUM, 0>();
    if (mode == MODE_MAX) return make_dense<2, MODE_MAX, 0>();
    switch (kt) {  // FP64 tensor-core (DMMA) block pass
        case 8: return make_dense_mma<8, 4>();
        case 16: return make_dense_mma<16, 4>();
        case 24: return make_dense_mma<24, 4>();
        case 32: return make_dense_mma<32, 4>();
        case 40: return make_dense_mma<40, 4>();
        case 48: return make_dense_mma<48, 2>();
        case 64: return make_dense_mma<64, 2>();
        default: return KernelInfo{};
    }
}

// Launch-configuration variants of the d=2 column-LSE sum kernel, timed by
// sknr_tune_variant (tools/tune_lse.py) to choose the default above.
KernelInfo tune_variant(int v) {
    switch (v) {
        case 0: return make_pts<2, 4, MODE_SUM, 0, 256, 2, false>();
        case 1: return make_pts<2, 4, MODE_SUM, 0, 256, 1, false>();
        case 2: return make_pts<2, 4, MODE_SUM, 0, 256, 4, false>();
        case 3: return make_pts<2, 2, MODE_SUM, 0, 256, 2, false>();
        case 4: return make_pts<2, 8, MODE_SUM, 0, 256, 1, false>();
        case 5: return make_pts<2, 8, MODE_SUM, 0, 256, 2, false>();
        case 6: return make_pts<2, 4, MODE_SUM, 0, 128, 2, false>();
        case 7: return make_pts<2, 4, MODE_SUM, 0, 512, 2, false>();
        case 8: return make_pts<2, 4, MODE_SUM, 0, 256, 2, true>();
        case 9: return make_pts<2, 8, MODE_SUM, 0, 256, 1, true>();
        case 10: return make_pts<2, 2, MODE_SUM, 0, 512, 4, false>();
        case 11: return make_pts<2, 4, MODE_SUM, 0, 512, 2, true>();
        case 12: return make_pts<2, 8, MODE_SUM, 0, 128, 1, false>();
        case 13: return make_pts<2, 8, MODE_SUM, 0, 512, 1, false>();
        case 14: return make_pts<2, 16, MODE_SUM, 0, 128, 1, false>();
        case 15: return make_pts<2, 16, MODE_SUM, 0, 256, 1, false>();
        case 16: return make_pts<2, 6, MODE_SUM, 0, 256, 1, false>();
        case 17: return make_pts<2, 12, MODE_SUM, 0, 256, 1, false>();
        case 18: return make_pts<2, 12, MODE_SUM, 0, 128, 1, false>();
        case 19: return make_pts<2, 8, MODE_SUM, 0, 256, 1, true>();
        case 20: return make_pts<2, 8, MODE_SUM, 0, 256, 1, false, 3>();
        case 21: return make_pts<2, 8, MODE_SUM, 0, 128, 1, false, 6>();
        case 22: return make_pts<2, 6, MODE_SUM, 0, 256, 1, false, 3>();
        case 23: return make_pts<2, 4, MODE_SUM, 0, 256, 2, false, 4>();
        case 24: return make_pts<2, 8, MODE_SUM, 0, 256, 1, false, 2>();
        case 25: return make_pts<2, 8, MODE_SUM, 0, 128, 1, false, 4>();
        case 26: return make_pts<2, 6, MODE_SUM, 0, 256, 1, false, 2>();
        // 1024-entry table, 10 FP64 slots per cell (pts_sum10_kernel <D, JT, threads>)
        case 40: return make_sum10<2, 8, 512>();
        case 41: return make_sum10<2, 4, 512>();
        case 42: return make_sum10<2, 8, 256>();
        case 43: return make_sum10<2, 6, 512>();
        case 44: return make_sum10<2, 12, 256>();
        case 45: return make_sum10<2, 8, 384>();
        case 46: return make_sum10<2, 8, 512, true>();
        case 47: return make_sum10<2, 6, 512, true>();
        // 4096-entry table, 10 FP64 slots per cell (pts_sum12_kernel <D, JT, threads, REP, FC>)
        case 50: return make_sum12<2, 8, 256, 1, false, 2>();
        case 51: return make_sum12<2, 8, 256, 2, false, 2>();
        case 52: return make_sum12<2, 8, 256, 1, true, 2>();
        case 53: return make_sum12<2, 8, 256, 2, true, 2>();
        case 54: return make_sum12<2, 8, 512, 4>();
        case 55: return make_sum12<2, 6, 256, 1, false, 2>();
        case 56: return make_sum12<2, 4, 256, 1, false, 3>();
        case 57: return make_sum12<2, 8, 128, 1, false, 4>();
        case 58: return make_sum12<2, 8, 256, 1, false, 1>();
        case 59: return make_sum12<2, 8, 256, 1, false, 2, 2>();
        case 60: return make_sum12<2, 8, 256, 1, true, 2, 2>();
        case 61: return make_sum12<2, 8, 256, 2, false, 2, 2>();
        case 62: return make_sum12<2, 8, 512, 4, false, 1, 2>();
        case 63: return make_sum12<2, 8, 512, 1, false, 1, 2>();
        case 64: return make_sum12<2, 8, 512, 1, false, 1>();
        case 65: return make_sum12<2, 8, 512, 2, false, 1, 2>();
        case 66: return make_sum12<2, 8, 512, 4, false, 1, 4>();
        case 67: return make_sum12<2, 8, 512, 4, true, 1, 2>();
        case 68: return make_sum12<2, 6, 512, 4, false, 1, 2>();
        case 69: return make_sum12<2, 8, 384, 4, false, 1, 2>();
        // stable-accept anchor pass, d=2 (timed with W = 1/sqrt(n) in every column)
        case 400: return make_pts<2, 4, MODE_BLOCK, 4, 256, 1>();
        case 401: return make_anchor12<2, 6, 512, 4, 1>();
        case 402: return make_anchor12<2, 4, 512, 4, 1>();
        case 403: return make_anchor12<2, 6, 512, 4, 2>();
        case 404: return make_anchor12<2, 8, 512, 4, 1>();
        case 405: return make_anchor12<2, 4, 512, 4, 2>();
        // stored cost (dim 0)
        case 100: return make_dense<2, MODE_SUM, 0>();
        case 101: return make_dense_v2<1, 4, 256, MODE_SUM>();
        case 102: return make_dense_v2<2, 4, 256, MODE_SUM>();
        case 103: return make_dense_v2<1, 8, 256, MODE_SUM>();
        case 104: return make_dense_v2<2, 2, 256, MODE_SUM>();
        case 105: return make_dense_v2<1, 4, 512, MODE_SUM>();
        case 106: return make_dense_v2<4, 2, 256, MODE_SUM>();
        case 107: return make_dense_v2<2, 4, 128, MODE_SUM>();
        // DMMA block pass, d=2, KT=32 (MB = 8-output blocks per warp)
        case 200: return make_mma<2, 32, 2>();
        case 201: return make_mma<2, 32, 4>();
        case 202: return make_mma<2, 32, 8>();
        case 203: return make_mma<2, 32, 6>();
        case 204: return make_mma<2, 32, 4, true>();
        case 205: return make_mma<2, 32, 2, true>();
        case 206: return make_mma<2, 32, 4, true, 32>();
        case 207: return make_mma<2, 32, 4, false, 32>();
        // double-buffered v2 (pts_mma2_kernel): <D, KT, MB, RS, MCH, NW>
        case 210: return make_mma2<2, 32, 4, true, 32, 8>();
        case 211: return make_mma2<2, 32, 4, true, 32, 4>();
        case 212: return make_mma2<2, 32, 2, true, 32, 8>();
        case 213: return make_mma2<2, 32, 4, false, 32, 8>();
        case 214: return make_mma2<2, 32, 4, true, 64, 4>();
        case 215: return make_mma2<2, 32, 2, true, 64, 8>();
        case 216: return make_mma2<2, 32, 4, false, 64, 4>();
        // fp32 sum pass (MUFU ex2), d=2
        case 300: return make_f32<2, 8, 256>();
        case 301: return make_f32<2, 4, 256>();
        case 302: return make_f32<2, 16, 256>();
        case 303: return make_f32<2, 8, 128>();
        case 304: return make_f32<2, 16, 128>();
        case 305: return make_f32<2, 8, 512>();
        case 306: return make_f32<2, 8, 256, 3>();
        case 307: return make_f32<2, 4, 256, 4>();
        case 308: return make_f32<2, 8, 128, 6>();
        case 309: return make_f32<2, 16, 128, 3>();
        case 310: return make_f32<2, 6, 256, 3>();
        case 311: return make_f32<2, 8, 512, 2>();
        default: return KernelInfo{};
    }
}

KernelInfo pick(int dim, int mode, int kt, bool vec_ok) {
    if (dim < 0) {  // -DK: tensor-core contraction, coordinates padded to DK (multiple of 8)
        switch (-dim) {
            case 8: return pick_contract<8>(mode, kt);
            case 16: return pick_contract<16>(mode, kt);
            case 32: return pick_contract<32>(mode, kt);
            case 64: return pick_contract<64>(mode, kt);
            case 128: return pick_contract<128>(mode, kt);
            default: return KernelInfo{};
        }
    }
    switch (dim) {
        case 0:
            // 128-bit loads (4 outputs per thread): 806 GCells/s = 98 % of HBM on C5 (tools/tune_dense.py)
            if (vec_ok && mode == MODE_SUM) return make_dense_v2<2, 4, 256, MODE_SUM>();
            if (vec_ok && mode == MODE_MAX) return make_dense_v2<2, 4, 256, MODE_MAX>();
            return pick_dense(mode, kt);
        case 1: return pick_pts<1>(mode, kt);
        case 2: return pick_pts<2>(mode, kt);
        case 3: return pick_pts<3>(mode, kt);
        case 4: return pick_pts<4>(mode, kt);
        default: return KernelInfo{};
    }
}

}  // namespace

int block_kt_for(int k) {
    static const int kts[] = {8, 16, 24, 32, 40, 48, 64};
    for (int kt : kts)
        if (k <= kt) return kt;
    return 0;
}

int chunk_inputs(int mode, int kt) {
    if (mode != MODE_BLOCK) return 256;
    return kt > 32 ? 32 : 64;
}

// Tensor-core Newton block pass (i8_kernels.cu): on unless SKNR_BLOCK_I8=0.
static std::atomic<int> g_i8_on{-1};
bool i8_block_enabled() {
    int v = g_i8_on.load();
    if (v < 0) {
        const char* e = std::getenv("SKNR_BLOCK_I8");
        v = (e && e[0] == '0') ? 0 : 1;
        g_i8_on.store(v);
    }
    return v != 0;
}
void set_i8_block_enabled(bool on) { g_i8_on.store(on ? 1 : 0); }

static int sm_count_cached() {
    static thread_local int sm_count = 0;
    if (sm_count == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sm_count, cudaDevAttrMultiProcessorCount, dev);
        if (sm_count <= 0) sm_count = 148;
    }
    return sm_count;
}

// 128-output tiles x input blocks of <= 8192 inputs (int32 level bound), multiples of 32;
// one CTA per SM (persistent).
// pts_i8w_kernel: a CTA takes a work unit of og output tiles x ig input blocks. S is summed
// over the unit's input blocks in registers (one partial row per ig-group instead of one per
// input block) and r over its output tiles (one row per og-group instead of one per output
// tile), so the split-K partials shrink from (NI S-rows, NO r-rows) to (ceil(NI/ig),
// ceil(NO/og)). The shape is the one with the smallest makespan (cells on the busiest CTA)
// over the input-block counts NI and ig; ties go to fewer partial bytes.
static TilePlan plan_i8(int dim, int64_t n_out, int64_t n_in, int64_t max_in_blocks) {
    TilePlan p;
    p.fn = i8_block_kernel(dim);
    if (!p.fn) return p;
    p.i8 = true;
    p.smem = i8_block_smem();
    p.nt = i8_block_threads();
    cudaFuncSetAttribute(p.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, p.smem);
    p.occ = 1;
    const int64_t resident = sm_count_cached();
    p.out_tile = i8_block_out_tile();
    const int64_t NO = (n_out + p.out_tile - 1) / p.out_tile;
    const int64_t ni_min = (n_in + i8_max_in_block() - 1) / i8_max_in_block();
    double best_span = 0.0, best_bytes = 0.0;
    bool have = false;
    for (int64_t want = ni_min; want <= ni_min + 24; ++want) {
        int64_t in_block = (n_in + want - 1) / want;
        in_block = ((in_block + 31) / 32) * 32;
        if (in_block > i8_max_in_block()) continue;
        const int64_t NI = (n_in + in_block - 1) / in_block;
        for (int64_t ig = 1; ig <= NI; ++ig) {
            const int64_t n_ig = (NI + ig - 1) / ig;
            if (max_in_blocks > 0 && n_ig > max_in_blocks) continue;
            // og so that the units fit the resident CTAs in one or two waves, or og = 1
            // (many small units, round-robin: the fallback when NO does not split well)
            for (int waves = 0; waves <= 2; ++waves) {
                const int64_t per_ig = waves == 0 ? NO : (resident * waves) / n_ig;  // og-groups per ig-group
                if (per_ig < 1) continue;
                const int64_t og = (NO + per_ig - 1) / per_ig;
                const int64_t n_og = (NO + og - 1) / og;
                const int64_t units = n_og * n_ig;
                const int64_t rounds = (units + resident - 1) / resident;
                const double span = static_cast<double>(rounds) * og * ig * in_block;
                const double bytes = static_cast<double>(n_ig) * n_out * 32 + static_cast<double>(n_og) * n_in;
                if (!have || span < best_span * 0.99 || (span <= best_span * 1.01 && bytes < best_bytes)) {
                    have = true;
                    best_span = span;
                    best_bytes = bytes;
                    p.in_block = in_block;
                    p.i8_in_blocks = NI;
                    p.i8_ig = ig;
                    p.i8_og = og;
                    p.n_in_blocks = n_ig;
                    p.n_out_tiles = n_og;
                }
            }
        }
    }
    p.i8_out_tiles = NO;
    p.n_tiles = p.n_out_tiles * p.n_in_blocks;  // work units
    p.grid = static_cast<int>(p.n_tiles < resident ? p.n_tiles : resident);
    return p;
}

TilePlan plan_tiles(int dim, int mode, int kt, int64_t n_out, int64_t n_in, int64_t max_in_blocks,
                    int variant) {
    TilePlan p;
    if (variant < 0 && mode == MODE_BLOCK_RS && dim >= 1 && dim <= 4 && kt <= 32 && i8_block_enabled() &&
        n_out * n_in >= (int64_t(1) << 22))
        return plan_i8(dim, n_out, n_in, max_in_blocks);
    // the stored cost's leading dimension equals n_out in both directions
    KernelInfo ki = variant >= 0 ? tune_variant(variant) : pick(dim, mode, kt, n_out % 2 == 0);
    if (!ki.fn) return p;
    // Small problems (e.g. C1 512^2, C2 4096^2): the 2048-output tiles of the
    // register kernels leave most SMs idle; use 128-output tiles instead.
    const bool blk = mode == MODE_BLOCK || mode == MODE_BLOCK_RS || mode == MODE_BLOCK_CULL;
    const bool culled = mode == MODE_SUM_CULL || mode == MODE_BLOCK_CULL || mode == MODE_SUM_CULL_F32;
    if (variant < 0 && dim > 0 && mode == MODE_SUM_F32 && n_out * n_in <= (int64_t(1) << 26)) {
        switch (dim) {
            case 1: ki = make_f32<1, 1, 128>(); break;
            case 2: ki = make_f32<2, 1, 128>(); break;
            case 3: ki = make_f32<3, 1, 128>(); break;
            default: ki = make_f32<4, 1, 128>(); break;
        }
    } else if (variant < 0 && dim > 0 && !blk && !culled && n_out * n_in <= (int64_t(1) << 26)) {
        switch (dim) {
            case 1: ki = mode == MODE_SUM ? make_pts<1, 1, MODE_SUM, 0, 128, 2>() : make_pts<1, 1, MODE_MAX, 0, 128, 2>(); break;
            case 2: ki = mode == MODE_SUM ? make_pts<2, 1, MODE_SUM, 0, 128, 2>() : make_pts<2, 1, MODE_MAX, 0, 128, 2>(); break;
            case 3: ki = mode == MODE_SUM ? make_pts<3, 1, MODE_SUM, 0, 128, 2>() : make_pts<3, 1, MODE_MAX, 0, 128, 2>(); break;
            default: ki = mode == MODE_SUM ? make_pts<4, 1, MODE_SUM, 0, 128, 2>() : make_pts<4, 1, MODE_MAX, 0, 128, 2>(); break;
        }
    }
    static thread_local int sm_count = 0;
    if (sm_count == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sm_count, cudaDevAttrMultiProcessorCount, dev);
        if (sm_count <= 0) sm_count = 148;
    }
    cudaFuncSetAttribute(ki.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, ki.smem);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, ki.fn, ki.nt, ki.smem);
    if (occ < 1) occ = 1;
    const int64_t resident = static_cast<int64_t>(sm_count) * occ;
    p.out_tile = ki.out_tile > 0 ? ki.out_tile : ki.nt * ki.jt;
    p.nt = ki.nt;
    p.n_out_tiles = (n_out + p.out_tile - 1) / p.out_tile;
    // input-block granularity (the kernels stage up to their chunk size per round)
    const int ch = mode == MODE_BLOCK_CULL ? CULL_GB
                                          : (blk ? chunk_inputs(MODE_BLOCK, kt) : (mode == MODE_SUM_CULL || mode == MODE_SUM_CULL_F32 ? CULL_GI : 32));
    const int64_t max_blocks_by_chunk = (n_in + ch - 1) / ch;
    // Aim for >= 8 tiles per resident CTA so the last wave's imbalance stays small
    // (culled pass: >= 8 work units per resident warp, taken from a queue).
    const int64_t units = culled ? 8 * resident * (ki.nt / 32) : 8 * resident;
    int64_t want = (units + p.n_out_tiles - 1) / p.n_out_tiles;
    if (want < 1) want = 1;
    if (want > max_blocks_by_chunk) want = max_blocks_by_chunk;
    if (max_in_blocks > 0 && want > max_in_blocks) want = max_in_blocks;
    int64_t in_block = (n_in + want - 1) / want;
    in_block = ((in_block + ch - 1) / ch) * ch;
    p.in_block = in_block;
    p.n_in_blocks = (n_in + in_block - 1) / in_block;
    p.n_tiles = p.n_out_tiles * p.n_in_blocks;
    p.grid = static_cast<int>(p.n_tiles < resident ? p.n_tiles : resident);
    p.smem = ki.smem;
    p.fn = ki.fn;
    p.occ = occ;
    return p;
}

static const void* small_kernel(int d) {
    switch (d) {
        case 1: return reinterpret_cast<const void*>(&k_sk_small<1>);
        case 2: return reinterpret_cast<const void*>(&k_sk_small<2>);
        case 3: return reinterpret_cast<const void*>(&k_sk_small<3>);
        case 4: return reinterpret_cast<const void*>(&k_sk_small<4>);
        default: return nullptr;
    }
}

static int small_smem(int d, int max_nm) {
    return static_cast<int>(sizeof(double)) * (kTabWords + 64 + max_nm * (d + 1));
}

// CTAs per problem: spread few problems over the SMs (all CTAs must be co-resident for
// the group barriers), at most one warp per output of the larger side.
int small_group_size(int d, int count, int max_nm) {
    const void* fn = small_kernel(d);
    if (!fn || count < 1) return 1;
    const int smem = small_smem(d, max_nm);
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int dev = 0, sms = 0, occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, 512, smem);
    const int capacity = sms * (occ > 0 ? occ : 1);
    int G = capacity / count;
    const int useful = (max_nm + 15) / 16;
    if (G > useful) G = useful;
    return G < 1 ? 1 : G;
}

void launch_sk_small(int d, SmallProbDev* probs, int count, int max_nm, double tol, long long max_iter,
                     int warm_g, int G, double* gpart, unsigned* gbar, cudaStream_t s) {
    const void* fn = small_kernel(d);
    if (!fn) return;
    const int smem = small_smem(d, max_nm);
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    void* args[] = {&probs, &tol, &max_iter, &warm_g, &G, &gpart, &gbar};
    count_launch();
    if (G > 1)  // group barriers: every CTA must be resident
        cudaLaunchCooperativeKernel(fn, dim3(count * G), dim3(512), args, smem, s);
    else
        cudaLaunchKernel(fn, dim3(count), dim3(512), args, smem, s);
}

void launch_tiles(const TilePlan& p, TileArgs a, cudaStream_t s) {
    a.n_out_tiles = p.n_out_tiles;
    a.n_in_blocks = p.n_in_blocks;
    a.n_tiles = p.n_tiles;
    a.in_block = p.in_block;
    a.i8_og = p.i8_og;
    a.i8_ig = p.i8_ig;
    a.i8_out_tiles = p.i8_out_tiles;
    a.i8_in_blocks = p.i8_in_blocks;
    void* args[] = {&a};
    count_launch();
    cudaLaunchKernel(p.fn, dim3(p.grid), dim3(p.nt), args, p.smem, s);
}

}  // namespace sknr
