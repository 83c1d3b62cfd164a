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
#include "internal.h"

namespace sknr {

__constant__ unsigned long long c_exp2_tab[kTabEntries] = {
#include "exp2_table.inc"
};

// Fill the replicated table: tab[e*16 + r] = mantissa bits of 2^(e/256).
__device__ __forceinline__ void load_exp2_table(unsigned long long* tab, int tid, int nthreads) {
    for (int t = tid; t < kTabWords; t += nthreads) tab[t] = c_exp2_tab[t >> 4];
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
template <int D, int JT, int MODE, int KT>
__global__ void __launch_bounds__(NT_of<MODE>::value) pts_tile_kernel(TileArgs a) {
    if (guard_skip(a.st, a.guard)) return;
    constexpr int NT = NT_of<MODE>::value;
    constexpr int PK = PK_of<D>::value;
    constexpr int CH = Chunk<MODE, KT>::value;
    constexpr int KA = KT > 0 ? KT : 1;
    extern __shared__ __align__(16) double sm[];
    unsigned long long* tab = reinterpret_cast<unsigned long long*>(sm);
    double* sin = sm + kTabWords;
    double* sw = sin + CH * PK;
    const int tid = threadIdx.x;
    load_exp2_table(tab, tid, NT);
    const unsigned laneoff = (tid & 15) << 3;
    const double c3 = reg_const(kP3);
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
#pragma unroll 2
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

// ------------------------------------------------------------- stored cost
template <int JT, int MODE, int KT>
__global__ void __launch_bounds__(NT_of<MODE>::value) dense_tile_kernel(TileArgs a) {
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
    const unsigned laneoff = (tid & 15) << 3;
    const double c3 = reg_const(kP3);
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

// ------------------------------------------------------------- dispatch
struct KernelInfo {
    const void* fn = nullptr;
    int jt = 1;
    int nt = 128;
    int smem = 0;
    int occ = 0;
};

template <int D, int JT, int MODE, int KT>
KernelInfo make_pts() {
    KernelInfo k;
    k.fn = reinterpret_cast<const void*>(&pts_tile_kernel<D, JT, MODE, KT>);
    k.jt = JT;
    k.nt = NT_of<MODE>::value;
    constexpr int CH = Chunk<MODE, KT>::value;
    k.smem = static_cast<int>(sizeof(double)) *
             (kTabWords + CH * PK_of<D>::value + (MODE == MODE_BLOCK ? CH * KT : 0));
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

template <int D>
KernelInfo pick_pts(int mode, int kt) {
    if (mode == MODE_SUM) return make_pts<D, 4, MODE_SUM, 0>();
    if (mode == MODE_MAX) return make_pts<D, 4, MODE_MAX, 0>();
    switch (kt) {
        case 8: return make_pts<D, 2, MODE_BLOCK, 8>();
        case 16: return make_pts<D, 2, MODE_BLOCK, 16>();
        case 24: return make_pts<D, 1, MODE_BLOCK, 24>();
        case 32: return make_pts<D, 1, MODE_BLOCK, 32>();
        case 40: return make_pts<D, 1, MODE_BLOCK, 40>();
        case 48: return make_pts<D, 1, MODE_BLOCK, 48>();
        case 64: return make_pts<D, 1, MODE_BLOCK, 64>();
        default: return KernelInfo{};
    }
}

KernelInfo pick_dense(int mode, int kt) {
    if (mode == MODE_SUM) return make_dense<2, MODE_SUM, 0>();
    if (mode == MODE_MAX) return make_dense<2, MODE_MAX, 0>();
    switch (kt) {
        case 8: return make_dense<2, MODE_BLOCK, 8>();
        case 16: return make_dense<1, MODE_BLOCK, 16>();
        case 24: return make_dense<1, MODE_BLOCK, 24>();
        case 32: return make_dense<1, MODE_BLOCK, 32>();
        case 40: return make_dense<1, MODE_BLOCK, 40>();
        case 48: return make_dense<1, MODE_BLOCK, 48>();
        case 64: return make_dense<1, MODE_BLOCK, 64>();
        default: return KernelInfo{};
    }
}

KernelInfo pick(int dim, int mode, int kt) {
    switch (dim) {
        case 0: return pick_dense(mode, kt);
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

TilePlan plan_tiles(int dim, int mode, int kt, int64_t n_out, int64_t n_in, int64_t max_in_blocks) {
    TilePlan p;
    KernelInfo ki = pick(dim, mode, kt);
    if (!ki.fn) return p;
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
    p.out_tile = ki.nt * ki.jt;
    p.nt = ki.nt;
    p.n_out_tiles = (n_out + p.out_tile - 1) / p.out_tile;
    const int ch = chunk_inputs(mode, kt);
    const int64_t max_blocks_by_chunk = (n_in + ch - 1) / ch;
    // Aim for >= 8 tiles per resident CTA so the last wave's imbalance stays small.
    int64_t want = (8 * resident + p.n_out_tiles - 1) / p.n_out_tiles;
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

void launch_tiles(const TilePlan& p, TileArgs a, cudaStream_t s) {
    a.n_out_tiles = p.n_out_tiles;
    a.n_in_blocks = p.n_in_blocks;
    a.n_tiles = p.n_tiles;
    a.in_block = p.in_block;
    void* args[] = {&a};
    count_launch();
    cudaLaunchKernel(p.fn, dim3(p.grid), dim3(p.nt), args, p.smem, s);
}

}  // namespace sknr
