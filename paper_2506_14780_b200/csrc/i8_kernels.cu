// i8_kernels.cu -- the Newton block pass S = V^T P~ (and r = P~ beta) with the l-wide
// contraction on the 5th-generation tensor cores (tcgen05, kind::i8), exactly.
//
// The FP64 block pass (pts_mma2_kernel<..., RS>) spends 32 of its ~44 FP64-pipe slot
// equivalents per cell on the contraction S_jc += P~_ij V_ic (DMMA shares the FP64 pipe on
// sm_100). Here the contraction runs as an integer GEMM on the tensor cores, split into
// byte slices (Ozaki-style) so that every product and every sum is exact:
//
//   P~_ij in [0, 1]: t = P~ + 2 has the 52-bit fixed-point value of P~ (2^-51 units) in its
//     mantissa; bytes k = 0..6 of t are unsigned digits p_k (byte 6 holds 4 bits).
//     Slice a = byte 6 - a:  P~ = sum_a p_a 2^(-3 - 8a) + e_lo, |e_lo| <= 2^-52; the
//     rounding residual e_lo = P~ - (t - 2) (exact) is kept as one signed slice
//     q = rint(e_lo 2^59) in [-128, 127] times V's leading digit (level 7), so P~ is
//     represented to 2^-60 absolute -- below the FP64 rounding of the terms that matter.
//   V_ic: N_ic = rint(V_ic 2^S_c) with |N| < 2^54 (S_c from the column's largest exponent),
//     written as 7 balanced base-256 digits d_b in [-128, 127]:  N = sum_b d_b 256^(6 - b).
//   level w = a + b:  L_w[j][c] = sum_i sum_{a+b=w} p_a(i,j) d_b(i,c)      (int32, exact)
//   S_jc = 2^-S_c sum_{w<=7} 2^(45 - 8w) L_w[j][c]
// Levels w >= 8 are dropped: each dropped term is below 2^-58 of the column's largest |V|
// (below the rounding of an FP64 product), and P~'s own representation error is 2^-52.
// One int32 level accumulates at most 7 * 8192 * 255 * 128 < 2^31 per tile (in_block <= 8192).
//
// Tile: 128 outputs j (MMA M) x an input block; per 32-input chunk (MMA K) the producer
// warps generate the 128 x 32 cells of P~ with the FP64 exponential of pts_sum12_kernel
// (4096-entry table, u' = 16u exact), accumulate r_i += P~_ij beta_j in FP64, and store the
// byte slices as MN-major (j contiguous) int8 tiles into a 4-stage shared-memory ring; one
// elected thread then issues 8 tcgen05.mma (A = slice a, B = the chunk's V digit tile
// [7 x 32 columns, K-major, fetched by a bulk copy], D = TMEM columns 32a.. so that product
// (a, b) lands on level a + b) and commits them to the stage's mbarrier. A tile's 8 levels
// x 32 columns of int32 live in TMEM (256 columns); after every input block they are read
// back (tcgen05.ld) and combined in FP64 into the split-K partial. See pts_i8w_kernel for
// the warp roles and the work units.
//
// Precondition: P~_ij <= 1 (+ rounding), i.e. the pass is taken at the anchor h = f^{C,eps}
// whose columns of P~ sum to 1 (objective.cpp:127-131); engine.cu only routes the Newton S
// pass here.
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "internal.h"

namespace sknr {

// 2^(e/4096) mantissas (the pexp12 table of tile_kernels.cu; a TU-local copy, no -rdc)
__device__ const unsigned long long g_exp2_tab12_i8[4096] = {
#include "exp2_table4096.inc"
};

namespace i8 {
constexpr int MT = 128;              // outputs per tile (MMA M)
constexpr int KC = 32;               // inputs per chunk (MMA K for kind::i8)
constexpr int NSL = 7;               // byte slices of P~ and digits of V
constexpr int NLEV = 8;              // levels kept
constexpr int A_SLICE = MT * KC;     // 4096 bytes per slice tile
constexpr int A_BYTES = (NSL + 1) * A_SLICE;  // + the signed low slice (slot 7)
constexpr int B_BYTES = NSL * 32 * KC;  // 7 digits x 32 columns x 32 inputs = 7168
constexpr int STAGES = 4;
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int TMEM_COLS = 256;
constexpr int MAX_IN_BLOCK = 8192;
// instruction descriptor: D s32 (bits 4-5 = 2), A u8 (7-9 = 0), B s8 (10-12 = 1),
// A MN-major (bit 15), B K-major, M = 128 (bits 24-28 = 128 >> 4); N (bits 17-22) per MMA
constexpr uint32_t IDESC = (2u << 4) | (0u << 7) | (1u << 10) | (1u << 15) | ((128u >> 4) << 24);
// the low slice: A s8 (bits 7-9 = 1), N = 32 (V's leading digit only)
constexpr uint32_t IDESC_LO = (2u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | ((32u >> 3) << 17) | ((128u >> 4) << 24);
}  // namespace i8

// ------------------------------------------------------------- tcgen05 / mbarrier helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// shared-memory matrix descriptor, no swizzle: start, leading / stride byte offsets
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
    d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
    d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
    d |= static_cast<uint64_t>(1) << 46;  // descriptor version (sm_100)
    return d;                             // base offset 0, layout type 0 (SWIZZLE_NONE)
}

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
}

__device__ __forceinline__ void mma_commit(uint32_t mbar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mbar)
                 : "memory");
}

__device__ __forceinline__ void mbar_init(uint32_t mbar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mbar), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra DONE_%=;\n\t"
        "bra WAIT_%=;\n"
        "DONE_%=:\n\t}\n" ::"r"(mbar),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t mbar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(bytes) : "memory");
}

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t mbar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(mbar)
                 : "memory");
}

__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_before_sync() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_after_sync() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// ld + wait in one statement, so no use of v[] can be scheduled before the wait
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n\t"
        "tcgen05.wait::ld.sync.aligned;"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr)
        : "memory");
}

__device__ __forceinline__ void tmem_zero32(uint32_t taddr) {
    const uint32_t z = 0;
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,"
        "%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(taddr),
        "r"(z)
        : "memory");
}

__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void tmem_alloc(uint32_t slot_saddr) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(slot_saddr),
                 "n"(i8::TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(i8::TMEM_COLS)
                 : "memory");
}

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
    uint32_t r;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
    return r;
}

// 4 x 4 byte transpose: out[k] = byte k of w0 | byte k of w1 << 8 | ... (k = 0..NK-1)
template <int NK>
__device__ __forceinline__ void byte_transpose(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3, uint32_t* out) {
    const uint32_t l01 = prmt(w0, w1, 0x5140), l23 = prmt(w2, w3, 0x5140);
    out[0] = prmt(l01, l23, 0x5410);
    out[1] = prmt(l01, l23, 0x7632);
    const uint32_t h01 = prmt(w0, w1, 0x7362), h23 = prmt(w2, w3, 0x7362);
    out[2] = prmt(h01, h23, 0x5410);
    if (NK > 3) out[3] = prmt(h01, h23, 0x7632);
}

// ------------------------------------------------------------- probe: one tcgen05 int8 GEMM
// D[128][N] = A[128][K] (u8, row-major) x B[K][N] (s8, given as Bt[N][K]); K % 32 == 0,
// N % 32 == 0, N <= 256. Same descriptors and layouts as the fused kernel (A MN-major,
// B K-major, SWIZZLE_NONE); used by the tests to pin the encoding.
__global__ void __launch_bounds__(128, 1) k_i8_probe(const uint8_t* __restrict__ A, const int8_t* __restrict__ Bt,
                                                     int N, int K, int32_t* __restrict__ D) {
    extern __shared__ __align__(1024) uint8_t smp[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nch = K / 32;
    uint8_t* sa = smp;                   // nch x 4096
    uint8_t* sb = smp + nch * 4096;      // nch x (N/8) x 256
    uint64_t* bar = reinterpret_cast<uint64_t*>(sb + nch * (N / 8) * 256);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
    for (int idx = tid; idx < 128 * K; idx += 128) {
        const int m = idx / K, k = idx % K, ch = k / 32, kk = k % 32;
        sa[ch * 4096 + (m / 16) * 512 + (kk / 8) * 128 + (kk % 8) * 16 + (m % 16)] = A[idx];
    }
    for (int idx = tid; idx < N * K; idx += 128) {
        const int n = idx / K, k = idx % K, ch = k / 32, kk = k % 32;
        sb[ch * (N / 8) * 256 + (n / 8) * 256 + (kk / 16) * 128 + (n % 8) * 16 + (kk % 16)] =
            static_cast<uint8_t>(Bt[idx]);
    }
    if (tid == 0) {
        mbar_init(smem_u32(bar), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) tmem_alloc(smem_u32(slot));
    fence_proxy_async();
    tc_before_sync();
    __syncthreads();
    tc_after_sync();
    const uint32_t tbase = *slot;
    if (tid == 0) {
        const uint32_t idesc = i8::IDESC | (static_cast<uint32_t>(N >> 3) << 17);
        for (int ch = 0; ch < nch; ++ch) {
            const uint64_t ad = umma_desc(smem_u32(sa + ch * 4096), 128, 512);
            const uint64_t bd = umma_desc(smem_u32(sb + ch * (N / 8) * 256), 128, 256);
            mma_i8(tbase, ad, bd, idesc, ch > 0 ? 1u : 0u);
        }
        mma_commit(smem_u32(bar));
    }
    mbar_wait(smem_u32(bar), 0);
    tc_after_sync();
    const int m = warp * 32 + lane;
    for (int c0 = 0; c0 < N; c0 += 32) {
        uint32_t v[32];
        tmem_ld32(tbase + (static_cast<uint32_t>(warp * 32) << 16) + c0, v);
#pragma unroll
        for (int q = 0; q < 32; ++q) D[m * N + c0 + q] = static_cast<int32_t>(v[q]);
    }
    tc_before_sync();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tbase);
}

// ------------------------------------------------------------- V digit tiles
// vexp[c] = 2048 + max_i ilogb|W[i][c]| (0 when the column is zero); one block per column,
// a fixed-order max (deterministic, no zero-initialised buffer needed).
__global__ void __launch_bounds__(256) k_i8_vexp(const double* __restrict__ W, int kt, int64_t n_in,
                                                 unsigned* __restrict__ vexp, const DevState* st, unsigned guard) {
    SKNR_PDL_ENTRY();
    if (guard_skip(st, guard)) return;
    __shared__ unsigned red[8];
    const int c = blockIdx.x;
    unsigned mx = 0;
    for (int64_t i = threadIdx.x; i < n_in; i += blockDim.x) {
        const double v = W[i * kt + c];
        if (v != 0.0) mx = max(mx, static_cast<unsigned>(2048 + ilogb(v)));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < 8; ++w) mx = max(mx, red[w]);
        vexp[c] = mx;
    }
}

// Digit tiles in the B-operand layout of one 32-input chunk: byte (n = b*32 + c, k) at
// (n/8)*256 + (k/16)*128 + (n%8)*16 + k%16, chunk base ch*7168; columns c >= kt and
// inputs i >= n_in are zero. One thread per (input, column 0..31).
__global__ void k_i8_vslices(const double* __restrict__ W, int kt, int64_t n_in, int64_t n_pad,
                             const unsigned* __restrict__ vexp, uint8_t* __restrict__ vsl, const DevState* st,
                             unsigned guard) {
    SKNR_PDL_ENTRY();
    if (guard_skip(st, guard)) return;
    const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= n_pad * 32) return;
    const int64_t i = idx >> 5;
    const int c = static_cast<int>(idx & 31);
    long long N = 0;
    if (i < n_in && c < kt && vexp[c] != 0u) {
        const int S = 53 - (static_cast<int>(vexp[c]) - 2048);
        N = llrint(scalbn(W[i * kt + c], S));  // |N| < 2^54
    }
    uint8_t* base = vsl + (i >> 5) * i8::B_BYTES;
    const int k = static_cast<int>(i & 31);
#pragma unroll
    for (int q = 0; q < i8::NSL; ++q) {  // least significant digit first: b = 6 - q
        const long long d = ((N + 128) & 255) - 128;
        N = (N - d) >> 8;
        const int n = (6 - q) * 32 + c;
        base[(n >> 3) * 256 + (k >> 4) * 128 + (n & 7) * 16 + (k & 15)] = static_cast<uint8_t>(static_cast<int8_t>(d));
    }
}

// ------------------------------------------------------------- fused block pass
constexpr double kI8Magic = 6755399445245952.0;  // 1.5 * 2^52 + 1023 * 4096 (as pexp12)
constexpr double kI8R1 = 0.0001692253858788929;  // (ln2/4096)^k / k!
constexpr double kI8R2 = 1.4318615612930102e-08;
constexpr double kI8R3 = 8.076910841165457e-13;
constexpr int kI8MagicHi = 0x43380000;
constexpr double kI8MagicLo = 6755399441055744.0;  // 1.5 * 2^52: low word = rint(x), |x| < 2^31

// ------------------------------------------------------------- fused block pass, warp-specialised
// No CTA-wide barrier sits in the chunk loop (the first version -- 8 warps of 16 outputs, one
// __syncthreads per chunk, r sums and MMA issue on the compute warps -- left the FP64 pipe
// idle two thirds of the time, profiles/ncu_block_i8_v1_r02.json):
//   16 producer warps (warp w: 16 outputs x 16 inputs of the chunk, a lane pair per input, 8
//     outputs per lane) generate P~, the byte slices (one 8-byte store per slice: half a
//     16-output core-matrix row, a warp's stores contiguous) and the r terms, then arrive
//     on the stage's `full` mbarrier (one arrival per warp);
//   4 service warps: one waits for `full` and the V tile and issues the chunk's 8
//     tcgen05.mma, committed to the stage's `free` mbarrier; two add the 16 r terms of each
//     input in a fixed order (even / odd chunks) and arrive on `free` as well; one fetches
//     the V digit tiles. (With the r sums on the MMA warp its serial latency, ~2000 cycles
//     per chunk, set the pace of the whole CTA.)
// Producers only wait for `free` of the stage they are about to refill, so they run up to
// STAGES chunks ahead of the tensor cores and of each other. At the end of a tile all 16
// producer warps read the levels back (lane group w % 4, columns 8 (w / 4)..+7), and the
// MMA warp waits for their `drained` arrivals before the next tile's first MMA.
namespace i8w {
constexpr int NPW = 16;                       // producer warps
constexpr int NT = (NPW + 4) * 32;            // + the MMA warp's warpgroup (setmaxnreg is per warpgroup)
constexpr int OW = i8::MT / NPW;              // outputs per producer warp = 8
constexpr int OFF_TAB = i8::STAGES * i8::STAGE_BYTES;
constexpr int OFF_RS = OFF_TAB + 4096 * 8;
constexpr int OFF_BAR = OFF_RS + i8::STAGES * NPW * 32 * 8;
constexpr int SMEM = OFF_BAR + 256;
// barriers: [0..3] free, [4..7] V tile landed, [8..11] full, [12] accumulators ready, [13] drained
constexpr int B_FREE = 0, B_VT = i8::STAGES, B_FULL = 2 * i8::STAGES, B_ACC = 3 * i8::STAGES, B_DRAIN = B_ACC + 1;
}  // namespace i8w

__device__ __forceinline__ void mbar_arrive(uint32_t mbar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(mbar) : "memory");
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&v)[8]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n\t"
        "tcgen05.wait::ld.sync.aligned;"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
        : "r"(taddr)
        : "memory");
}

__device__ __forceinline__ void tmem_zero8(uint32_t taddr) {
    const uint32_t z = 0;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(taddr), "r"(z)
                 : "memory");
}

template <int D>
__global__ void __launch_bounds__(i8w::NT, 1) pts_i8w_kernel(TileArgs a) {
    SKNR_PDL_ENTRY();
    if (guard_skip(a.st, a.guard)) return;
    constexpr int PK = ((D + 2) / 2) * 2;
    constexpr int OW = i8w::OW;
    extern __shared__ __align__(1024) uint8_t sm8[];
    uint8_t* stages = sm8;
    unsigned long long* tab = reinterpret_cast<unsigned long long*>(sm8 + i8w::OFF_TAB);
    double* rs = reinterpret_cast<double*>(sm8 + i8w::OFF_RS);
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm8 + i8w::OFF_BAR);
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + i8w::B_DRAIN + 1);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    for (int t = tid; t < 4096; t += i8w::NT) {  // 2^(e/4096), hi word pre-biased by -(e << 8)
        const unsigned e = static_cast<unsigned>(t);
        const unsigned long long v = g_exp2_tab12_i8[e];
        const unsigned hi = static_cast<unsigned>(v >> 32) - (e << 8);
        tab[t] = (static_cast<unsigned long long>(hi) << 32) | (v & 0xFFFFFFFFull);
    }
    if (tid == 0) {
        for (int q = 0; q < i8::STAGES; ++q) {
            mbar_init(smem_u32(bars + i8w::B_FREE + q), 2);  // MMAs completed + r terms read
            mbar_init(smem_u32(bars + i8w::B_VT + q), 1);
            mbar_init(smem_u32(bars + i8w::B_FULL + q), i8w::NPW);
        }
        mbar_init(smem_u32(bars + i8w::B_ACC), 1);
        mbar_init(smem_u32(bars + i8w::B_DRAIN), i8w::NPW);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) tmem_alloc(smem_u32(tslot));
    tc_before_sync();
    __syncthreads();
    tc_after_sync();
    const uint32_t tbase = *tslot;
    // this producer warp's part of the accumulators: lanes 32 (w % 4).., columns 8 (w / 4)..+7 per level
    const uint32_t tmine = tbase + (static_cast<uint32_t>((warp & 3) * 32) << 16) + static_cast<uint32_t>((warp >> 2) * 8);
    if (warp < i8w::NPW) {  // TMEM starts undefined
#pragma unroll
        for (int w = 0; w < i8::NLEV; ++w) tmem_zero8(tmine + w * 32);
        tmem_wait_st();
    }
    tc_before_sync();
    __syncthreads();
    tc_after_sync();

    uint32_t g = 0;      // chunks seen by this CTA
    uint32_t ntile = 0;  // (output tile, input block) pairs finished by this CTA
    // work units: i8_og output tiles x i8_ig input blocks; n_out_tiles / n_in_blocks count the
    // unit rows (= rows of rsum / partial), i8_out_tiles / i8_in_blocks the tiles themselves
    const int64_t n_units = a.n_out_tiles * a.n_in_blocks;
    if (warp >= i8w::NPW) {
        // ------------------------------------------------------------------ service warps
        // (their warpgroup gives registers back to the producers: 640 x 96 at launch ->
        // 512 x 112 + 128 x 32). Each walks the CTA's chunk sequence on its own:
        //   warp 16    tcgen05.mma issue (one elected lane)
        //   warp 17/18 r terms of the even / odd chunks
        //   warp 19    V digit tiles (bulk copies) one ring round ahead
        // A stage is free again when its MMAs have completed AND its r terms have been
        // read (`free` counts two arrivals).
        asm volatile("setmaxnreg.dec.sync.aligned.u32 32;");
        const int role = warp - i8w::NPW;
        for (int64_t unit = blockIdx.x; unit < n_units; unit += gridDim.x) {
            const int64_t ogi = unit % a.n_out_tiles, igi = unit / a.n_out_tiles;
            const int64_t ot0 = ogi * a.i8_og, ot1 = (ot0 + a.i8_og < a.i8_out_tiles) ? ot0 + a.i8_og : a.i8_out_tiles;
            const int64_t ib0 = igi * a.i8_ig, ib1 = (ib0 + a.i8_ig < a.i8_in_blocks) ? ib0 + a.i8_ig : a.i8_in_blocks;
            double* rrow = a.rsum + ogi * a.n_in;  // this unit's r terms: row ogi, inputs of blocks ib0..ib1-1
            for (int64_t ot = ot0; ot < ot1; ++ot)
            for (int64_t ib = ib0; ib < ib1; ++ib, ++ntile) {
            const int64_t i0 = ib * a.in_block;
            const int64_t i1 = (i0 + a.in_block < a.n_in) ? i0 + a.in_block : a.n_in;
            if (role == 0 && ntile > 0) {  // the previous tile's levels have been read and zeroed
                mbar_wait(smem_u32(bars + i8w::B_DRAIN), (ntile - 1) & 1u);
                tc_after_sync();
            }
            for (int64_t c0 = i0; c0 < i1; c0 += i8::KC, ++g) {
                const uint32_t s = g % i8::STAGES, use = g / i8::STAGES;
                uint8_t* sA = stages + s * i8::STAGE_BYTES;
                uint8_t* sB = sA + i8::A_BYTES;
                if (role == 0) {
                    if (lane == 0) {
                        mbar_wait(smem_u32(bars + i8w::B_FULL + s), use & 1u);
                        mbar_wait(smem_u32(bars + i8w::B_VT + s), use & 1u);
                        tc_after_sync();
                        const uint64_t bd = umma_desc(smem_u32(sB), 128, 256);
#pragma unroll
                        for (int sa = 0; sa < i8::NSL; ++sa) {  // P~ slice sa = byte 6 - sa
                            const int nb = (i8::NLEV - sa) < i8::NSL ? (i8::NLEV - sa) : i8::NSL;
                            const uint64_t ad = umma_desc(smem_u32(sA + (6 - sa) * i8::A_SLICE), 128, 512);
                            mma_i8(tbase + sa * 32, ad, bd, i8::IDESC | (static_cast<uint32_t>(nb * 32 >> 3) << 17), 1u);
                        }
                        mma_i8(tbase + 7 * 32, umma_desc(smem_u32(sA + 7 * i8::A_SLICE), 128, 512), bd, i8::IDESC_LO,
                               1u);
                        mma_commit(smem_u32(bars + i8w::B_FREE + s));
                        if (c0 + i8::KC >= i1) mma_commit(smem_u32(bars + i8w::B_ACC));
                    }
                    __syncwarp();
                } else if (role == 3) {
                    if (lane == 0) {
                        if (use > 0) mbar_wait(smem_u32(bars + i8w::B_FREE + s), (use - 1) & 1u);
                        mbar_expect_tx(smem_u32(bars + i8w::B_VT + s), i8::B_BYTES);
                        bulk_g2s(smem_u32(sB), a.vsl + (c0 >> 5) * i8::B_BYTES, i8::B_BYTES,
                                 smem_u32(bars + i8w::B_VT + s));
                    }
                    __syncwarp();
                } else if (static_cast<int>(g & 1u) == role - 1) {
                    // r accumulates over the unit's output tiles in this row (L2-resident
                    // read-modify-write; the load overlaps the wait below)
                    const bool rok = c0 + lane < i1;
                    double rold = 0.0;
                    if (rok && ot > ot0) rold = rrow[c0 + lane];
                    mbar_wait(smem_u32(bars + i8w::B_FULL + s), use & 1u);
                    // r of input `lane` over the tile's 128 outputs: the 16 producer terms
                    // (output group 0..7, half 0..1) as a fixed pairwise tree; producer warp
                    // 2 og + (lane >> 4) holds them in lanes 2 (lane & 15) + half
                    const double* rr = rs + s * (i8w::NPW * 32) + (lane >> 4) * 32 + 2 * (lane & 15);
                    double q[i8w::NPW / 2];
#pragma unroll
                    for (int og = 0; og < i8w::NPW / 2; ++og) {
                        const double2 pr = *reinterpret_cast<const double2*>(rr + og * 64);
                        q[og] = pr.x + pr.y;
                    }
                    const double v = ((q[0] + q[1]) + (q[2] + q[3])) + ((q[4] + q[5]) + (q[6] + q[7]));
                    if (rok) rrow[c0 + lane] = rold + v;
                    __syncwarp();
                    if (lane == 0) mbar_arrive(smem_u32(bars + i8w::B_FREE + s));
                }
            }
            }
        }
    } else {
        // ------------------------------------------------------------------ producer warps
        asm volatile("setmaxnreg.inc.sync.aligned.u32 112;");
        const double r2 = reg_const(kI8R2);
        const double c59 = reg_const(0x1p59), cm59 = reg_const(-0x1p59);
        // 2^60 + 1.5 * 2^52: -(tf - 2) 2^59 + this is exact (a multiple of 2^8 below 2^60)
        const double c60m = reg_const(0x1p60 + kI8MagicLo);
        // warp w: output group w >> 1 (16 outputs) x input half w & 1 (16 inputs); lane:
        // input lane >> 1 of that half, outputs 8 (lane & 1)..+7 of the group. A lane pair
        // then writes one 16-byte core-matrix row and a warp 256 contiguous bytes per slice
        // (conflict-free 8-byte stores; a lane = input mapping strides them by 16 bytes).
        const int og16 = warp >> 1;
        const int kin = (warp & 1) * 16 + (lane >> 1);   // input within the chunk
        const int oh = lane & 1;
        for (int64_t unit = blockIdx.x; unit < n_units; unit += gridDim.x) {
            const int64_t ogi = unit % a.n_out_tiles, igi = unit / a.n_out_tiles;
            const int64_t ot0 = ogi * a.i8_og, ot1 = (ot0 + a.i8_og < a.i8_out_tiles) ? ot0 + a.i8_og : a.i8_out_tiles;
            const int64_t ib0 = igi * a.i8_ig, ib1 = (ib0 + a.i8_ig < a.i8_in_blocks) ? ib0 + a.i8_ig : a.i8_in_blocks;
            for (int64_t ot = ot0; ot < ot1; ++ot) {
            // Operands stay unscaled in registers: u = A_i + B_j + x.y, and the exact factor 16
            // of u' = 16 u (table step 2^(1/4096)) rides on the Cody-Waite FMAs below -- the
            // same values as staging (16A, 4X), (16B, 4Y), without a multiply on the loaded
            // inputs (which made every chunk wait for its own prefetch).
            double Bj[OW], Yj[OW][D], Wj[OW];
#pragma unroll
            for (int q = 0; q < OW; ++q) {
                int64_t o = ot * i8::MT + og16 * 16 + oh * 8 + q;
                Wj[q] = o < a.n_out ? a.out_w[o] : 0.0;
                o = o < a.n_out ? o : a.n_out - 1;
                Bj[q] = a.out_pack[o * PK];
#pragma unroll
                for (int d = 0; d < D; ++d) Yj[q][d] = a.out_pack[o * PK + 1 + d];
            }
            for (int64_t ib = ib0; ib < ib1; ++ib, ++ntile) {
            const int64_t i0 = ib * a.in_block;
            const int64_t i1 = (i0 + a.in_block < a.n_in) ? i0 + a.in_block : a.n_in;
            double xn0, Xn[D];
            {
                const int64_t ic = (i0 + kin < i1) ? i0 + kin : i1 - 1;
                xn0 = a.in_pack[ic * PK];
#pragma unroll
                for (int d = 0; d < D; ++d) Xn[d] = a.in_pack[ic * PK + 1 + d];
            }
            for (int64_t c0 = i0; c0 < i1; c0 += i8::KC, ++g) {
                const uint32_t s = g % i8::STAGES, use = g / i8::STAGES;
                uint8_t* sA = stages + s * i8::STAGE_BYTES;
                const int64_t i = c0 + kin;
                double x0 = xn0, X[D];
#pragma unroll
                for (int d = 0; d < D; ++d) X[d] = Xn[d];
                if (i >= i1) x0 = -1.0e300;  // e = 0: every byte slice 0, no contribution
                if (c0 + i8::KC < i1) {  // prefetch the next chunk's inputs (used one chunk later)
                    const int64_t inx = (i + i8::KC < i1) ? i + i8::KC : i1 - 1;
                    xn0 = a.in_pack[inx * PK];
#pragma unroll
                    for (int d = 0; d < D; ++d) Xn[d] = a.in_pack[inx * PK + 1 + d];
                }
                if (use > 0) mbar_wait(smem_u32(bars + i8w::B_FREE + s), (use - 1) & 1u);
                double rt = 0.0;
                uint32_t wl[2][4], wh[2][3], wq[2];  // [group of 4 outputs][byte], low slice
#pragma unroll
                for (int q4 = 0; q4 < 2; ++q4) {
                    uint32_t lo[4], hi[4], ql[4];
#pragma unroll
                    for (int qq = 0; qq < 4; ++qq) {
                        const int q = q4 * 4 + qq;
                        double u = x0 + Bj[q];
#pragma unroll
                        for (int d = 0; d < D; ++d) u = fma(X[d], Yj[q][d], u);
                        const double t = fma(u, 16.0, kI8Magic);  // u' + magic, u' = 16 u exact
                        const double kf = t - kI8Magic;
                        const double r = fma(u, 16.0, -kf);
                        double p = fma(r, kI8R3, r2);
                        p = fma(p, r, kI8R1);
                        p = fma(p, r, 1.0);
                        const int kc = (__double2hiint(t) >= kI8MagicHi) ? __double2loint(t) : 0;
                        const unsigned off = (static_cast<unsigned>(kc) << 3) & (4095u << 3);
                        const uint2 T = *reinterpret_cast<const uint2*>(reinterpret_cast<const char*>(tab) + off);
                        const double Tp = __hiloint2double(static_cast<int>(static_cast<unsigned>(kc) * 256u + T.y),
                                                           static_cast<int>(T.x));
                        const double e = Tp * p;
                        rt = fma(e, Wj[q], rt);
                        const double tf = e + 2.0;  // mantissa = P~ in 2^-51 units
                        lo[qq] = static_cast<uint32_t>(__double2loint(tf));
                        hi[qq] = static_cast<uint32_t>(__double2hiint(tf));
                        // residual e - (tf - 2), exact, as rint(. 2^59) in the low word of tq
                        const double nh = fma(tf, cm59, c60m);  // -(tf - 2) 2^59 + 1.5 2^52, exact
                        const double tq = fma(e, c59, nh);
                        ql[qq] = static_cast<uint32_t>(min(__double2loint(tq), 127));
                    }
                    byte_transpose<4>(lo[0], lo[1], lo[2], lo[3], wl[q4]);
                    byte_transpose<3>(hi[0], hi[1], hi[2], hi[3], wh[q4]);
                    wq[q4] = prmt(prmt(ql[0], ql[1], 0x40), prmt(ql[2], ql[3], 0x40), 0x5410);
                }
                // core matrix (og16, kin >> 3): 16 bytes (outputs) per input row kin & 7
                uint8_t* dst = sA + og16 * 512 + kin * 16 + oh * 8;
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    *reinterpret_cast<uint2*>(dst + k * i8::A_SLICE) = make_uint2(wl[0][k], wl[1][k]);
#pragma unroll
                for (int k = 0; k < 3; ++k)
                    *reinterpret_cast<uint2*>(dst + (4 + k) * i8::A_SLICE) = make_uint2(wh[0][k], wh[1][k]);
                *reinterpret_cast<uint2*>(dst + 7 * i8::A_SLICE) = make_uint2(wq[0], wq[1]);
                rs[s * (i8w::NPW * 32) + warp * 32 + lane] = rt;
                fence_proxy_async();
                __syncwarp();
                if (lane == 0) mbar_arrive(smem_u32(bars + i8w::B_FULL + s));
            }
            // input block done: levels -> FP64; warp w: rows 32 (w % 4) + lane, columns 8 (w / 4)..+7
            mbar_wait(smem_u32(bars + i8w::B_ACC), ntile & 1u);
            tc_after_sync();
            double acc[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) acc[c] = 0.0;
#pragma unroll
            for (int w = i8::NLEV - 1; w >= 0; --w) {  // smallest level first
                uint32_t v[8];
                tmem_ld8(tmine + w * 32, v);
                const double sc = __hiloint2double((1023 + 45 - 8 * w) << 20, 0);
#pragma unroll
                for (int c = 0; c < 8; ++c) acc[c] = fma(static_cast<double>(static_cast<int32_t>(v[c])), sc, acc[c]);
                tmem_zero8(tmine + w * 32);
            }
            tmem_wait_st();
            tc_before_sync();
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(bars + i8w::B_DRAIN));
            // the unit's split-K partial of this output tile (row igi of [n_ig][kt][n_out]) sums
            // its input blocks in order: read-modify-write by the owning thread (L2-resident;
            // the scale is a power of two, so scaling each block's term is exact)
            const int64_t o = ot * i8::MT + (warp & 3) * 32 + lane;
            if (o < a.n_out) {
#pragma unroll
                for (int cc = 0; cc < 8; ++cc) {
                    const int c = (warp >> 2) * 8 + cc;
                    if (c < a.kt) {
                        const unsigned ve = a.vexp[c];
                        const double sc = ve ? scalbn(1.0, -(53 - (static_cast<int>(ve) - 2048))) : 0.0;
                        double* pp = a.partial + (igi * a.kt + c) * a.n_out + o;
                        double v = acc[cc] * sc;
                        if (ib > ib0) v += *pp;
                        *pp = v;
                    }
                }
            }
            }
            }
        }
    }
    tc_before_sync();
    __syncthreads();
    tc_after_sync();
    if (warp == 0) tmem_dealloc(tbase);
}

const void* i8_block_kernel(int d) {
    switch (d) {
        case 1: return reinterpret_cast<const void*>(&pts_i8w_kernel<1>);
        case 2: return reinterpret_cast<const void*>(&pts_i8w_kernel<2>);
        case 3: return reinterpret_cast<const void*>(&pts_i8w_kernel<3>);
        case 4: return reinterpret_cast<const void*>(&pts_i8w_kernel<4>);
        default: return nullptr;
    }
}
int i8_block_smem() { return i8w::SMEM; }
int i8_block_threads() { return i8w::NT; }
int i8_block_out_tile() { return i8::MT; }
int i8_max_in_block() { return i8::MAX_IN_BLOCK; }
int64_t i8_vslice_bytes(int64_t n_in) { return ((n_in + 31) / 32) * i8::B_BYTES; }

void launch_i8_vprep(const double* W, int kt, int64_t n_in, uint8_t* vsl, unsigned* vexp, const DevState* st,
                     unsigned guard, cudaStream_t s) {
    count_launch();
    k_i8_vexp<<<kt, 256, 0, s>>>(W, kt, n_in, vexp, st, guard);
    const int64_t n_pad = ((n_in + 31) / 32) * 32;
    count_launch();
    k_i8_vslices<<<static_cast<int>((n_pad * 32 + 255) / 256), 256, 0, s>>>(W, kt, n_in, n_pad, vexp, vsl, st,
                                                                          guard);
}

}  // namespace sknr

// Probe of the tcgen05 int8 encoding (tests): host arrays in, host array out.
extern "C" int sknr_probe_i8_mma(const uint8_t* A, const int8_t* Bt, int n, int k, int32_t* D) {
    using namespace sknr;
    if (n < 32 || n > 256 || n % 32 || k < 32 || k % 32 || k > 256) return 1;
    uint8_t *dA = nullptr, *dB = nullptr;
    int32_t* dD = nullptr;
    cudaError_t e = cudaMalloc(&dA, 128 * k);
    if (e == cudaSuccess) e = cudaMalloc(&dB, n * k);
    if (e == cudaSuccess) e = cudaMalloc(&dD, 128 * n * sizeof(int32_t));
    if (e == cudaSuccess) e = cudaMemcpy(dA, A, 128 * k, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(dB, Bt, n * k, cudaMemcpyHostToDevice);
    const int smem = (k / 32) * 4096 + (k / 32) * (n / 8) * 256 + 64;
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_i8_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess) {
        k_i8_probe<<<1, 128, smem>>>(dA, reinterpret_cast<const int8_t*>(dB), n, k, dD);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e == cudaSuccess) e = cudaMemcpy(D, dD, 128 * n * sizeof(int32_t), cudaMemcpyDeviceToHost);
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dD);
    if (e != cudaSuccess) {
        std::fprintf(stderr, "sknr_probe_i8_mma: %s\n", cudaGetErrorString(e));
        return 2;
    }
    return 0;
}
