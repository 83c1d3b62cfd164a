// engine.cu -- host orchestration of SK-NR(ell) on one B200 (C++ host code +
// the small kernels it sequences). The C ABI at the bottom is the drop-in
// boundary declared in include/sknr_gpu.h.
//
// Device-resident solve loop (solver.cpp:104-151): one CUDA graph
// per iteration, every kernel guarded by device flags (DevState) so that
// convergence, Newton rejection and the exact-shift fallback never need a host
// round trip; the host only polls the done flag between graph batches.
//
// Pass accounting per iteration (n*m cells each):
//   SK     : row LSE (f) + column LSE (h = next g)                    = 2 passes
//   SK-NR  : + row LSE at (f,h) for r + block pass S = V^T P~ (ell wide)
//            + column LSE at the candidate                           = 4 + 1 block
// The reference spends 3-6 passes (4 with its default trace); the column
// marginal is taken from the fused transform: col_j - beta_j =
// beta_j expm1((g_j - h_j)/eps) (SURVEY 3.2 "bitwise-safe reuse").
#include <dlfcn.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <map>
#include <set>
#include <tuple>
#include <unordered_map>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include <nccl.h>  // types only; entry points are resolved with dlopen/dlsym

#include "../../include/sknr_gpu.h"
#include "aux_kernels.cuh"

namespace sknr {

// ============================================================ errors
struct InvalidArgument : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct CudaFailure : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct EigenFailure : std::runtime_error {
    double best;
    EigenFailure(const std::string& m, double b) : std::runtime_error(m), best(b) {}
};
struct RuntimeFailure : std::runtime_error {
    using std::runtime_error::runtime_error;
};

#define CK(x)                                                                                 \
    do {                                                                                      \
        cudaError_t e_ = (x);                                                                 \
        if (e_ != cudaSuccess)                                                                \
            throw CudaFailure(std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " + \
                              __FILE__ + ":" + std::to_string(__LINE__));                     \
    } while (0)

struct NcclFailure : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// ============================================================ NCCL (row sharding)
// Loaded lazily with dlopen so the library never pins a second libnccl next to
// the one torch already mapped (RTLD_NOLOAD first).
struct NcclApi {
    void* lib = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*ReduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                  cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;

    void load() {
        if (lib) return;
        lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!lib) lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!lib) throw NcclFailure(std::string("sknr: cannot load libnccl.so.2: ") + dlerror());
        auto sym = [&](const char* name) {
            void* p = dlsym(lib, name);
            if (!p) throw NcclFailure(std::string("sknr: NCCL symbol missing: ") + name);
            return p;
        };
        GetUniqueId = reinterpret_cast<decltype(GetUniqueId)>(sym("ncclGetUniqueId"));
        CommInitRank = reinterpret_cast<decltype(CommInitRank)>(sym("ncclCommInitRank"));
        AllReduce = reinterpret_cast<decltype(AllReduce)>(sym("ncclAllReduce"));
        Broadcast = reinterpret_cast<decltype(Broadcast)>(sym("ncclBroadcast"));
        AllGather = reinterpret_cast<decltype(AllGather)>(sym("ncclAllGather"));
        ReduceScatter = reinterpret_cast<decltype(ReduceScatter)>(sym("ncclReduceScatter"));
        GroupStart = reinterpret_cast<decltype(GroupStart)>(sym("ncclGroupStart"));
        GroupEnd = reinterpret_cast<decltype(GroupEnd)>(sym("ncclGroupEnd"));
        CommDestroy = reinterpret_cast<decltype(CommDestroy)>(sym("ncclCommDestroy"));
        GetErrorString = reinterpret_cast<decltype(GetErrorString)>(sym("ncclGetErrorString"));
    }
};

static NcclApi g_nccl;

struct Comm {
    int rank = 0, world = 1;
    ncclComm_t comm = nullptr;
};
static Comm g_comm;

#define NK(x)                                                                                      \
    do {                                                                                           \
        ncclResult_t r_ = (x);                                                                     \
        if (r_ != ncclSuccess)                                                                     \
            throw NcclFailure(std::string("NCCL error: ") + g_nccl.GetErrorString(r_) + " at " + \
                              __FILE__ + ":" + std::to_string(__LINE__));                         \
    } while (0)

// Standard contiguous row partition of n rows over `world` ranks.
static void row_partition(int64_t n, int world, int rank, int64_t& begin, int64_t& end) {
    begin = n * rank / world;
    end = n * (rank + 1) / world;
}

static std::atomic<int64_t> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
int64_t launch_count() { return g_launches.load(); }

template <typename... KArgs, typename... Args>
static void launch(void (*kern)(KArgs...), int grid, int block, cudaStream_t s, Args... args) {
    count_launch();
    kern<<<grid, block, 0, s>>>(args...);
}

// Rewrites the plain kernel->kernel edges of a captured graph into programmatic edges
// (see SKNR_PDL_ENTRY): the successor may launch as soon as every CTA of the predecessor
// has started, and waits in griddepcontrol.wait for its completion. Only edges into this
// library's kernels are rewritten (foreign kernels, e.g. NCCL's, do not wait).
// SKNR_NO_PDL=1 keeps plain edges.
static bool own_kernel(cudaGraphNode_t node) {
    static std::mutex mu;
    static std::unordered_map<const void*, bool> cache;
    cudaKernelNodeParams kp = {};
    if (cudaGraphKernelNodeGetParams(node, &kp) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(kp.func);
    if (it != cache.end()) return it->second;
    const char* name = nullptr;
    bool ours = cudaFuncGetName(&name, kp.func) == cudaSuccess && name && std::strstr(name, "4sknr") != nullptr;
    cudaGetLastError();
    cache.emplace(kp.func, ours);
    return ours;
}

static void make_programmatic(cudaGraph_t g) {
    static const bool off = std::getenv("SKNR_NO_PDL") != nullptr;
    if (off || !g) return;
    size_t ne = 0;
    CK(cudaGraphGetEdges_v2(g, nullptr, nullptr, nullptr, &ne));
    if (ne == 0) return;
    std::vector<cudaGraphNode_t> from(ne), to(ne);
    std::vector<cudaGraphEdgeData> ed(ne);
    CK(cudaGraphGetEdges_v2(g, from.data(), to.data(), ed.data(), &ne));
    for (size_t e = 0; e < ne; ++e) {
        if (ed[e].type != cudaGraphDependencyTypeDefault || ed[e].from_port != cudaGraphKernelNodePortDefault)
            continue;
        cudaGraphNodeType tf, tt;
        CK(cudaGraphNodeGetType(from[e], &tf));
        CK(cudaGraphNodeGetType(to[e], &tt));
        if (tf != cudaGraphNodeTypeKernel || tt != cudaGraphNodeTypeKernel || !own_kernel(to[e])) continue;
        CK(cudaGraphRemoveDependencies_v2(g, &from[e], &to[e], &ed[e], 1));
        cudaGraphEdgeData pe = {};
        pe.from_port = cudaGraphKernelNodePortProgrammatic;
        pe.type = cudaGraphDependencyTypeProgrammatic;
        CK(cudaGraphAddDependencies_v2(g, &from[e], &to[e], &pe, 1));
    }
}

static int grid_for(int64_t count, int threads = AUX_NT) {
    int64_t g = (count + threads - 1) / threads;
    if (g < 1) g = 1;
    if (g > 148 * 8) g = 148 * 8;
    return static_cast<int>(g);
}

// ============================================================ device buffers
// Device allocations come from the device's stream-ordered memory pool (release
// threshold raised once, so memory freed by a destroyed problem is reused by the next
// one without going back to the driver) on a dedicated allocation stream.
static cudaStream_t alloc_stream() {
    static std::mutex mu;
    static int dev_init = -1;
    static cudaStream_t s = nullptr;
    std::lock_guard<std::mutex> lk(mu);
    int dev = 0;
    CK(cudaGetDevice(&dev));
    if (dev_init != dev) {
        cudaMemPool_t pool;
        CK(cudaDeviceGetDefaultMemPool(&pool, dev));
        uint64_t thr = UINT64_MAX;
        CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
        if (!s) CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        dev_init = dev;
    }
    return s;
}

// Frees are stream-ordered on the stream of the problem that used the buffer (no
// device-wide barrier): every API entry point makes its problem's stream this thread's
// owner stream (own_stream), and a buffer allocated under it is returned to the pool
// after the work already queued there. Streams are registered while alive, so a buffer
// never frees on a destroyed stream (unowned buffers -- host-synchronised temporaries --
// free on the allocation stream).
static std::mutex g_live_mu;
static std::set<cudaStream_t> g_live_streams;
static thread_local cudaStream_t tl_owner = nullptr;
static void own_stream(cudaStream_t s) { tl_owner = s; }
static cudaStream_t live_owner() {
    if (!tl_owner) return nullptr;
    std::lock_guard<std::mutex> lk(g_live_mu);
    return g_live_streams.count(tl_owner) ? tl_owner : nullptr;
}

struct DBuf {
    double* p = nullptr;
    size_t n = 0;
    cudaStream_t owner = nullptr;
    DBuf() = default;
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    ~DBuf() { release(); }
    // Returns the memory to the pool after the work queued on the owner stream.
    void release() {
        if (!p) return;
        cudaStream_t o = owner;
        if (o) {
            std::lock_guard<std::mutex> lk(g_live_mu);
            if (!g_live_streams.count(o)) o = nullptr;  // its problem is gone (and was synchronised)
        }
        cudaFreeAsync(p, o ? o : alloc_stream());
        p = nullptr;
        n = 0;
        owner = nullptr;
    }
    // Grows (never inside stream capture). The zero fill is complete before
    // returning: the problem streams are non-blocking, so the allocation stream's
    // work must be finished before they touch the buffer.
    void ensure(size_t count) {
        if (count <= n) return;
        release();
        const size_t bytes = std::max<size_t>(count, 1) * sizeof(double);
        cudaStream_t s = alloc_stream();
        CK(cudaMallocAsync(reinterpret_cast<void**>(&p), bytes, s));
        CK(cudaMemsetAsync(p, 0, bytes, s));
        CK(cudaStreamSynchronize(s));
        n = count;
        owner = live_owner();
    }
};

struct IBuf {  // int32 device buffer (permutations)
    int* p = nullptr;
    size_t n = 0;
    IBuf() = default;
    IBuf(const IBuf&) = delete;
    IBuf& operator=(const IBuf&) = delete;
    ~IBuf() {
        if (p) cudaFree(p);
    }
    void assign(const std::vector<int>& h) {
        if (p) CK(cudaFree(p));
        p = nullptr;
        n = 0;
        CK(cudaMalloc(&p, std::max<size_t>(h.size(), 1) * sizeof(int)));
        CK(cudaMemcpy(p, h.data(), h.size() * sizeof(int), cudaMemcpyHostToDevice));
        n = h.size();
    }
};

#include "engine_kernels.cuh"

// ============================================================ problem
struct Side {
    int64_t count = 0;
    DBuf w, lw, sw, lsw, coords, sq;
    // culling (opt-in): Morton order and bounding boxes of groups of 64 / 256 / 2048
    // consecutive permuted points, [group][2d] = lo..., hi...
    IBuf perm;
    DBuf box16, box32, box64, box128;
};

struct SolveState;

struct StreamReaper {
    cudaStream_t s = nullptr;
    ~StreamReaper() {
        if (s) cudaStreamDestroy(s);
    }
};

struct Problem {
    StreamReaper reaper;  // first member: destroyed after every DBuf member
    int kind = 0;  // 0 dense, 1 points
    int64_t n = 0, m = 0, d = 0;
    double eps = 1.0, kappa = 1.0;
    int dim = 0;  // tile-kernel dimension: 0 stored cost, 1..4 points
    Side src, tgt;
    DBuf C, CT;
    DevState* st = nullptr;
    DevState* st_host = nullptr;  // pinned mirror for polling
    cudaStream_t stream = nullptr;

    // per-direction LSE state
    DBuf L[2], ref[2], shift[2], pack_in[2], pack_out[2], stats;
    DBuf partial, rsum;
    DBuf vsl, vexp;  // tensor-core block pass: V digit tiles, column exponents (i8_kernels.cu)
    const double* vsl_src = nullptr;  // the static W whose digit tiles vsl holds (a solve's basis), or nullptr
    std::shared_ptr<SolveState> solve_cache;  // per-solve device buffers, reused across solves
    // culling (sknr_problem_set_culling): threshold T (0 = off) and per-direction group bounds
    double cull_t = 0.0;
    // sknr_problem_set_precision: 64 (default) or 32 (LSE sum passes in fp32 on MUFU, points d <= 4)
    int precision = 64;
    bool cull_ready = false;
    DBuf f_gi[2], s_go[2], f_g32[2], s_g16[2];
    DBuf gram_part, sums, misc;
    std::mutex mu;

    ~Problem() {
        if (stream) {
            cudaStreamSynchronize(stream);
            std::lock_guard<std::mutex> lk(g_live_mu);
            g_live_streams.erase(stream);
        }
        if (tl_owner == stream) tl_owner = nullptr;
        // the member buffers free after this body (the stream is idle and unregistered, so
        // on the allocation stream); the stream itself goes last (StreamReaper)
        if (st) cudaFree(st);
        if (st_host) cudaFreeHost(st_host);
    }

    std::map<std::tuple<int, int, int, int64_t, bool>, TilePlan> plans;

    // row sharding: this handle holds source rows [row_begin, row_begin + n)
    bool shard = false;
    bool emu = false;           // collectives through the in-process emulated group (testing)
    int rank = 0, world = 1;
    int64_t n_global = 0, row_begin = 0;
    DBuf red_tmp, gather_buf;
    // sharded column LSE: rank-local LSE of the last pass (bound-shift reference), the
    // exchange row [shift | S] (2m) and the gathered rows of every rank [R][2m]
    DBuf L_loc, xrow, xall;
    std::vector<double> h_alpha, h_beta;  // full host copies (validation, host-side dots)
    std::vector<sknr_record> last_trace;  // trace of the last solve / anneal (sknr_last_trace)

    bool otf() const { return dim != 0; }  // on-the-fly cost (dim > 0: registers, dim < 0: DMMA contraction)
    double inv_eps() const { return 1.0 / eps; }
    double kc() const { return otf() ? kappa / eps : 0.0; }
    double sigma() const { return otf() ? std::sqrt(2.0 * kLS * kappa / eps) : 0.0; }
    int pk() const { return dim > 0 ? (dim + 2) / 2 * 2 : (dim < 0 ? -dim + 2 : 1); }
    Side& in_side(int dir) { return dir == 0 ? src : tgt; }
    Side& out_side(int dir) { return dir == 0 ? tgt : src; }
    const double* cost_for(int dir) const { return dir == 0 ? CT.p : C.p; }
    int64_t ldc_for(int dir) const { return dir == 0 ? m : n; }
};

static void upload(double* dst, const double* src, size_t count, cudaStream_t s) {
    CK(cudaMemcpyAsync(dst, src, count * sizeof(double), cudaMemcpyHostToDevice, s));
}
static void download(double* dst, const double* src, size_t count, cudaStream_t s) {
    CK(cudaMemcpyAsync(dst, src, count * sizeof(double), cudaMemcpyDeviceToHost, s));
}

static void check_device() {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count < 1)
        throw CudaFailure("sknr_b200: no CUDA device available (this library has no CPU fallback)");
}

// DiscreteMeasure validation (types.cpp:7-18) with the reference's messages.
static void validate_measure(const double* w, int64_t len) {
    if (len == 0) throw InvalidArgument("DiscreteMeasure: empty weight vector");
    double total = 0.0;
    for (int64_t i = 0; i < len; ++i) {
        if (!std::isfinite(w[i]) || w[i] <= 0.0)
            throw InvalidArgument("DiscreteMeasure: weights must be strictly positive and finite");
        total += w[i];
    }
    if (std::abs(total - 1.0) > 1e-12) throw InvalidArgument("DiscreteMeasure: weights must sum to 1");
}

static void setup_side(Side& s, const double* w, int64_t count, cudaStream_t stream) {
    s.count = count;
    std::vector<double> lw(count), sw(count), lsw(count);
    for (int64_t i = 0; i < count; ++i) {
        lw[i] = std::log(w[i]);  // scalar std::log like types.cpp:19-23
        sw[i] = std::sqrt(w[i]);
        lsw[i] = std::log(sw[i]);
    }
    s.w.ensure(count);
    s.lw.ensure(count);
    s.sw.ensure(count);
    s.lsw.ensure(count);
    upload(s.w.p, w, count, stream);
    upload(s.lw.p, lw.data(), count, stream);
    upload(s.sw.p, sw.data(), count, stream);
    upload(s.lsw.p, lsw.data(), count, stream);
    CK(cudaStreamSynchronize(stream));
}

static Problem* new_problem(int64_t n, int64_t m, const double* alpha, const double* beta, double eps) {
    if (n < 1 || m < 1) throw InvalidArgument("CostMatrix: need at least a 1x1 matrix");
    validate_measure(alpha, n);
    validate_measure(beta, m);
    if (!(eps > 0.0) || !std::isfinite(eps)) throw InvalidArgument("EotProblem: epsilon must be positive");
    check_device();
    std::unique_ptr<Problem> p(new Problem());
    p->n = n;
    p->n_global = n;
    p->m = m;
    p->eps = eps;
    CK(cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking));
    p->reaper.s = p->stream;
    {
        std::lock_guard<std::mutex> lk(g_live_mu);
        g_live_streams.insert(p->stream);
    }
    own_stream(p->stream);
    CK(cudaMalloc(&p->st, sizeof(DevState)));
    CK(cudaMemsetAsync(p->st, 0, sizeof(DevState), p->stream));
    CK(cudaMallocHost(&p->st_host, sizeof(DevState)));
    setup_side(p->src, alpha, n, p->stream);
    setup_side(p->tgt, beta, m, p->stream);
    for (int dir = 0; dir < 2; ++dir) {
        const int64_t nin = dir == 0 ? n : m, nout = dir == 0 ? m : n;
        p->L[dir].ensure(nout);
        p->ref[dir].ensure(nin);
        p->shift[dir].ensure(nout);
    }
    p->stats.ensure(2 * 148 * 8);
    p->red_tmp.ensure(std::max(n, m));
    p->h_alpha.assign(alpha, alpha + n);
    p->h_beta.assign(beta, beta + m);
    p->gram_part.ensure(296 * 64 * 64 + 64);
    p->sums.ensure(64);
    return p.release();
}

static void finish_points(Problem* p, const double* x, const double* y, int64_t d, double cost_scale,
                          int cost_mode = 0) {
    const int64_t n = p->n, m = p->m;
    p->kind = 1;
    p->d = d;
    p->kappa = cost_scale;
    // Centre on the midpoint of the joint bounding box: ||x-y||^2 is translation
    // invariant, and smaller norms keep the expanded form's rounding small.
    std::vector<double> xc(x, x + n * d), yc(y, y + m * d), sx(n, 0.0), sy(m, 0.0);
    for (int64_t q = 0; q < d; ++q) {
        double lo = x[q * n], hi = x[q * n];
        for (int64_t i = 0; i < n; ++i) {
            lo = std::min(lo, x[i + q * n]);
            hi = std::max(hi, x[i + q * n]);
        }
        for (int64_t j = 0; j < m; ++j) {
            lo = std::min(lo, y[j + q * m]);
            hi = std::max(hi, y[j + q * m]);
        }
        const double mid = 0.5 * (lo + hi);
        for (int64_t i = 0; i < n; ++i) {
            xc[i + q * n] -= mid;
            sx[i] += xc[i + q * n] * xc[i + q * n];
        }
        for (int64_t j = 0; j < m; ++j) {
            yc[j + q * m] -= mid;
            sy[j] += yc[j + q * m] * yc[j + q * m];
        }
    }
    p->src.coords.ensure(n * d);
    p->tgt.coords.ensure(m * d);
    p->src.sq.ensure(n);
    p->tgt.sq.ensure(m);
    upload(p->src.coords.p, xc.data(), n * d, p->stream);
    upload(p->tgt.coords.p, yc.data(), m * d, p->stream);
    upload(p->src.sq.p, sx.data(), n, p->stream);
    upload(p->tgt.sq.p, sy.data(), m, p->stream);
    // cost_mode 0 auto: d <= 4 register kernels, larger d stored (fits: 2 n m 8 B < 1/2 free HBM)
    // else DMMA contraction; 1 stored; 2 on the fly.
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    const bool fits = 2.0 * static_cast<double>(n) * m * 8.0 < 0.5 * static_cast<double>(free_b);
    int dk = 8;
    while (dk < d) dk *= 2;
    const bool contract_ok = d > 4 && dk <= 128;
    if (cost_mode != 1 && d >= 1 && d <= 4) {
        p->dim = static_cast<int>(d);
    } else if (contract_ok && (cost_mode == 2 || (cost_mode == 0 && !fits))) {
        p->dim = -dk;  // coordinates zero-padded to dk in the packs
    } else {
        // No register-resident on-the-fly kernel for this dimension yet: the
        // cost is materialised once on device (both layouts) and streamed.
        p->dim = 0;
        p->C.ensure(n * m);
        p->CT.ensure(n * m);
        count_launch();
        k_build_cost<<<grid_for(n * m), AUX_NT, 0, p->stream>>>(p->src.coords.p, p->tgt.coords.p, n,
                                                               m, static_cast<int>(d), cost_scale,
                                                               p->C.p, p->CT.p);
        CK(cudaGetLastError());
    }
    for (int dir = 0; dir < 2; ++dir) {
        const int64_t nin = dir == 0 ? n : m, nout = dir == 0 ? m : n;
        p->pack_in[dir].ensure(nin * p->pk());
        p->pack_out[dir].ensure(nout * p->pk());
    }
    CK(cudaStreamSynchronize(p->stream));
}

static void finish_dense(Problem* p, const double* cost) {
    const int64_t n = p->n, m = p->m;
    for (int64_t e = 0; e < n * m; ++e)
        if (!std::isfinite(cost[e])) throw InvalidArgument("CostMatrix: entries must be finite");
    p->kind = 0;
    p->dim = 0;
    p->d = 0;
    p->C.ensure(n * m);
    p->CT.ensure(n * m);
    upload(p->C.p, cost, n * m, p->stream);
    count_launch();
    k_transpose<<<dim3(std::min<int64_t>((n + 31) / 32, 256), std::min<int64_t>((m + 31) / 32, 256)),
                  dim3(32, 8), 0, p->stream>>>(p->C.p, n, m, p->CT.p);
    CK(cudaGetLastError());
    for (int dir = 0; dir < 2; ++dir) {
        const int64_t nin = dir == 0 ? n : m, nout = dir == 0 ? m : n;
        p->pack_in[dir].ensure(nin);
        p->pack_out[dir].ensure(nout);
    }
    CK(cudaStreamSynchronize(p->stream));
}

// ============================================================ collectives
// In-process emulation of the row-sharded collectives (sknr_comm_init_emulated): R
// shard handles on one GPU, driven by R host threads, meet at every collective; the
// last thread to arrive enqueues one reduction kernel over all R buffers on a shared
// stream after waiting (cudaStreamWaitEvent) for every rank's arrival event, and each
// rank's stream then waits for its completion event. Ordering is by stream/event
// dependencies only -- no kernel ever waits on another -- and the solve loop runs
// eagerly (no graph capture) in this mode. The rank order of the merge is fixed.
constexpr int kEmuMax = 16;

struct EmuPtrs {
    double* buf[kEmuMax];
};

__global__ void k_emu_allreduce(EmuPtrs p, int world, int64_t count, int op) {
    SKNR_PDL_ENTRY();
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < count;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        double acc = p.buf[0][e];
        for (int r = 1; r < world; ++r) {
            const double v = p.buf[r][e];
            acc = op == 0 ? acc + v : fmax(acc, v);
        }
        for (int r = 0; r < world; ++r) p.buf[r][e] = acc;
    }
}

// recv[q][e] = sum_r send[r][q * count + e], ranks in order (reduce-scatter)
__global__ void k_emu_reduce_scatter(EmuPtrs send, EmuPtrs recv, int world, int64_t count) {
    SKNR_PDL_ENTRY();
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < count * world;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int q = static_cast<int>(t / count);
        double acc = send.buf[0][t];
        for (int r = 1; r < world; ++r) acc += send.buf[r][t];
        recv.buf[q][t - q * count] = acc;
    }
}

struct EmuGroup {
    int world = 0;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    int64_t generation = 0;
    EmuPtrs bufs{};
    const double* locals[kEmuMax] = {};
    int64_t counts[kEmuMax] = {};
    cudaEvent_t ev_arrive[kEmuMax] = {};
    cudaEvent_t ev_done = nullptr;
    cudaStream_t red = nullptr;

    void init(int w) {
        destroy();
        world = w;
        for (int r = 0; r < w; ++r) CK(cudaEventCreateWithFlags(&ev_arrive[r], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&ev_done, cudaEventDisableTiming));
        CK(cudaStreamCreateWithFlags(&red, cudaStreamNonBlocking));
    }
    void destroy() {
        for (auto& e : ev_arrive)
            if (e) cudaEventDestroy(e), e = nullptr;
        if (ev_done) cudaEventDestroy(ev_done), ev_done = nullptr;
        if (red) cudaStreamDestroy(red), red = nullptr;
        world = 0;
    }
    // Rendezvous of rank r; `leader` runs once with every rank's arguments in place.
    template <typename F>
    void meet(int r, cudaStream_t s, F&& leader) {
        static const bool dbg_sync = std::getenv("SKNR_EMU_SYNC") != nullptr;
        if (dbg_sync) CK(cudaStreamSynchronize(s));
        CK(cudaEventRecord(ev_arrive[r], s));
        {
            std::unique_lock<std::mutex> lk(mu);
            const int64_t gen = generation;
            if (++arrived == world) {
                for (int q = 0; q < world; ++q) CK(cudaStreamWaitEvent(red, ev_arrive[q], 0));
                leader();
                CK(cudaEventRecord(ev_done, red));
                if (dbg_sync) CK(cudaStreamSynchronize(red));
                arrived = 0;
                ++generation;
                cv.notify_all();
            } else {
                cv.wait(lk, [&] { return generation != gen; });
            }
        }
        CK(cudaStreamWaitEvent(s, ev_done, 0));
    }
};
static EmuGroup g_emu;

static int nccl_op_code(ncclRedOp_t op) { return op == ncclMax ? 1 : 0; }

// Collective accounting (sknr_comm_stats): calls and payload bytes issued by this process.
static std::atomic<int64_t> g_coll_calls{0}, g_coll_bytes{0};
static void count_collective(size_t bytes) {
    g_coll_calls.fetch_add(1, std::memory_order_relaxed);
    g_coll_bytes.fetch_add(static_cast<int64_t>(bytes), std::memory_order_relaxed);
}

// In-place allreduce on the problem's stream; a no-op unless the handle is row-sharded.
static void allreduce(Problem& P, double* buf, size_t count, ncclRedOp_t op) {
    if (!P.shard || count == 0) return;
    count_collective(count * sizeof(double));
    if (P.emu) {
        std::unique_lock<std::mutex> lk(g_emu.mu);
        g_emu.bufs.buf[P.rank] = buf;
        lk.unlock();
        const int code = nccl_op_code(op);
        g_emu.meet(P.rank, P.stream, [&] {
            count_launch();
            k_emu_allreduce<<<static_cast<int>(std::min<int64_t>((count + 255) / 256, 1184)), 256, 0, g_emu.red>>>(
                g_emu.bufs, g_emu.world, static_cast<int64_t>(count), code);
            CK(cudaGetLastError());
        });
        return;
    }
    NK(g_nccl.AllReduce(buf, buf, count, ncclDouble, op, g_comm.comm, P.stream));
}

// All-gather `count` doubles per rank into recv[R][count] (rank order), on the problem's stream.
static void allgather(Problem& P, const double* send, double* recv, size_t count) {
    count_collective(count * sizeof(double) * static_cast<size_t>(P.world));
    if (P.emu) {
        {
            std::lock_guard<std::mutex> lk(g_emu.mu);
            g_emu.locals[P.rank] = send;
            g_emu.bufs.buf[P.rank] = recv;
        }
        g_emu.meet(P.rank, P.stream, [&] {
            for (int q = 0; q < g_emu.world; ++q)
                for (int r = 0; r < g_emu.world; ++r)
                    CK(cudaMemcpyAsync(g_emu.bufs.buf[r] + q * count, g_emu.locals[q], sizeof(double) * count,
                                       cudaMemcpyDeviceToDevice, g_emu.red));
        });
        return;
    }
    NK(g_nccl.AllGather(send, recv, count, ncclDouble, g_comm.comm, P.stream));
}

// Reduce-scatter (sum): send holds R blocks of `count` doubles, rank q receives the sum of
// block q over all ranks (NCCL's layout), on the problem's stream.
static void reduce_scatter(Problem& P, const double* send, double* recv, size_t count) {
    count_collective(count * sizeof(double) * static_cast<size_t>(P.world));
    if (P.emu) {
        {
            std::lock_guard<std::mutex> lk(g_emu.mu);
            g_emu.locals[P.rank] = send;
            g_emu.bufs.buf[P.rank] = recv;
        }
        g_emu.meet(P.rank, P.stream, [&] {
            EmuPtrs sp{};
            for (int r = 0; r < g_emu.world; ++r) sp.buf[r] = const_cast<double*>(g_emu.locals[r]);
            const int64_t tot = static_cast<int64_t>(count) * g_emu.world;
            count_launch();
            k_emu_reduce_scatter<<<static_cast<int>(std::min<int64_t>((tot + 255) / 256, 1184)), 256, 0, g_emu.red>>>(
                sp, g_emu.bufs, g_emu.world, static_cast<int64_t>(count));
            CK(cudaGetLastError());
        });
        return;
    }
    NK(g_nccl.ReduceScatter(send, recv, count, ncclDouble, ncclSum, g_comm.comm, P.stream));
}

// All-gather of an n_local x k column-major row block (ld = n_local) into the full
// n_global x k block (ld = n_global) on every rank: one NCCL broadcast per rank (ragged
// row blocks) into a staging buffer, then a strided copy into place.
static void gather_row_block(Problem& P, const double* X, int k, double* full) {
    const size_t pitch = sizeof(double) * static_cast<size_t>(P.n_global);
    if (P.emu) {
        {
            std::lock_guard<std::mutex> lk(g_emu.mu);
            g_emu.locals[P.rank] = X;
            g_emu.bufs.buf[P.rank] = full;
        }
        g_emu.meet(P.rank, P.stream, [&] {
            for (int q = 0; q < g_emu.world; ++q) {
                int64_t b, e;
                row_partition(P.n_global, g_emu.world, q, b, e);
                if (e == b) continue;
                for (int r = 0; r < g_emu.world; ++r)
                    CK(cudaMemcpy2DAsync(g_emu.bufs.buf[r] + b, pitch, g_emu.locals[q], sizeof(double) * (e - b),
                                         sizeof(double) * (e - b), k, cudaMemcpyDeviceToDevice, g_emu.red));
            }
        });
        return;
    }
    P.gather_buf.ensure(static_cast<size_t>(P.n_global) * k);
    count_collective(static_cast<size_t>(P.n_global) * k * sizeof(double));
    NK(g_nccl.GroupStart());
    for (int r = 0; r < g_comm.world; ++r) {
        int64_t b, e;
        row_partition(P.n_global, g_comm.world, r, b, e);
        NK(g_nccl.Broadcast(X, P.gather_buf.p + b * k, (e - b) * k, ncclDouble, r, g_comm.comm, P.stream));
    }
    NK(g_nccl.GroupEnd());
    for (int r = 0; r < g_comm.world; ++r) {
        int64_t b, e;
        row_partition(P.n_global, g_comm.world, r, b, e);
        if (e == b) continue;
        CK(cudaMemcpy2DAsync(full + b, pitch, P.gather_buf.p + b * k, sizeof(double) * (e - b), sizeof(double) * (e - b),
                             k, cudaMemcpyDeviceToDevice, P.stream));
    }
}

// Column blocks of the m-side for the reduce-scattered S = V^T P~: rank q
// owns target rows [q * mb, min(m, (q + 1) * mb)), mb = ceil(m / R) (NCCL needs equal blocks).
static int64_t scatter_rows(const Problem& P) { return (P.m + P.world - 1) / P.world; }

// Upload the local row block of a full-length, `cols`-column column-major host array.
static void upload_rows(Problem& P, double* dev, const double* host_full, int64_t cols = 1) {
    for (int64_t c = 0; c < cols; ++c)
        upload(dev + c * P.n, host_full + c * P.n_global + P.row_begin, P.n, P.stream);
}

// All-gather the local row block of a device vector into a full host vector.
static void gather_rows(Problem& P, const double* dev_local, double* host_full) {
    if (!P.shard) {
        download(host_full, dev_local, P.n, P.stream);
        CK(cudaStreamSynchronize(P.stream));
        return;
    }
    P.gather_buf.ensure(P.n_global);
    if (P.emu) {
        {
            std::lock_guard<std::mutex> lk(g_emu.mu);
            g_emu.locals[P.rank] = dev_local;
            g_emu.bufs.buf[P.rank] = P.gather_buf.p;
        }
        g_emu.meet(P.rank, P.stream, [&] {
            for (int q = 0; q < g_emu.world; ++q) {
                int64_t b, e;
                row_partition(P.n_global, g_emu.world, q, b, e);
                for (int r = 0; r < g_emu.world; ++r)
                    CK(cudaMemcpyAsync(g_emu.bufs.buf[r] + b, g_emu.locals[q], sizeof(double) * (e - b),
                                       cudaMemcpyDeviceToDevice, g_emu.red));
            }
        });
        download(host_full, P.gather_buf.p, P.n_global, P.stream);
        CK(cudaStreamSynchronize(P.stream));
        return;
    }
    count_collective(static_cast<size_t>(P.n_global) * sizeof(double));
    NK(g_nccl.GroupStart());
    for (int r = 0; r < g_comm.world; ++r) {
        int64_t b, e;
        row_partition(P.n_global, g_comm.world, r, b, e);
        NK(g_nccl.Broadcast(dev_local, P.gather_buf.p + b, e - b, ncclDouble, r, g_comm.comm, P.stream));
    }
    NK(g_nccl.GroupEnd());
    download(host_full, P.gather_buf.p, P.n_global, P.stream);
    CK(cudaStreamSynchronize(P.stream));
}

// ============================================================ passes
static TilePlan plan_for(Problem& P, int dir, int mode, int kt, int64_t max_in_blocks = 0) {
    const int64_t nout = dir == 0 ? P.m : P.n, nin = dir == 0 ? P.n : P.m;
    const auto key = std::make_tuple(dir, mode, kt, max_in_blocks, i8_block_enabled());
    auto it = P.plans.find(key);
    if (it != P.plans.end()) return it->second;
    TilePlan tp = plan_tiles(P.dim, mode, kt, nout, nin, max_in_blocks);
    if (!tp.fn) throw CudaFailure("sknr_b200: no tile kernel for this configuration");
    P.plans[key] = tp;
    const bool blk = mode == MODE_BLOCK || mode == MODE_BLOCK_RS || mode == MODE_BLOCK_CULL;
    const size_t need = static_cast<size_t>(tp.n_in_blocks) * nout * (blk ? kt : 1);
    P.partial.ensure(need);
    if (mode == MODE_BLOCK_RS) P.rsum.ensure(static_cast<size_t>(tp.n_out_tiles) * nin);
    if (tp.i8) {
        P.vsl.ensure(static_cast<size_t>(i8_vslice_bytes(nin) / 8));
        P.vexp.ensure(16);
    }
    return tp;
}

static TileArgs tile_args(Problem& P, int dir, const TilePlan& tp, unsigned guard) {
    TileArgs a;
    a.n_out = dir == 0 ? P.m : P.n;
    a.n_in = dir == 0 ? P.n : P.m;
    a.out_pack = P.pack_out[dir].p;
    a.in_pack = P.pack_in[dir].p;
    a.C = P.cost_for(dir);
    a.ldc = P.ldc_for(dir);
    a.kappa = kLS * P.inv_eps();
    a.partial = P.partial.p;
    a.st = P.st;
    a.guard = guard;
    (void)tp;
    return a;
}

// Culled column/row LSE (opt-in): register point kernels, unsharded, large enough
// for whole cull tiles.
static bool cull_active(const Problem& P, int dir) {
    if (!(P.cull_t > 0.0) || !P.cull_ready || P.dim < 1 || P.dim > 4) return false;
    const int64_t nin = dir == 0 ? P.n : P.m, nout = dir == 0 ? P.m : P.n;
    return nout >= 8 * CULL_GO && nin >= 4 * CULL_GI;
}

static TileArgs cull_args(Problem& P, int dir, const TilePlan& tp, unsigned guard, int retry_phase) {
    TileArgs a = tile_args(P, dir, tp, guard);
    Side& in = P.in_side(dir);
    Side& out = P.out_side(dir);
    a.perm_in = in.perm.p;
    a.perm_out = out.perm.p;
    a.box_gi = in.box32.p;
    a.box_go = out.box128.p;
    a.f_gi = P.f_gi[dir].p;
    a.s_go = P.s_go[dir].p;
    a.lskc = kLS * P.kc();
    a.cull_t = P.cull_t;
    a.inv_eps = P.inv_eps();
    a.dir = dir;
    a.retry_phase = retry_phase;
    return a;
}

// Per-group maxima (groups of gs permuted positions) of the culling bound terms.
static void cull_group_max(Problem& P, const Side& side, const double* pack, double* out, int gs, unsigned guard,
                           unsigned* zero_counter = nullptr, const double* sub = nullptr) {
    count_launch();
    k_group_max<<<static_cast<int>((side.count + AUX_NT - 1) / AUX_NT), AUX_NT, 0, P.stream>>>(
        pack, P.pk(), side.sq.p, kLS * P.kc(), side.perm.p, side.count, gs, out, P.st, guard, zero_counter, sub);
}

// Culled block pass (opt-in): same conditions as the culled LSE, sizes above one work unit.
static bool cull_block_active(const Problem& P, int dir) {
    if (!(P.cull_t > 0.0) || !P.cull_ready || P.dim < 1 || P.dim > 4) return false;
    const int64_t nin = dir == 0 ? P.n : P.m, nout = dir == 0 ? P.m : P.n;
    return nout >= 1024 && nin >= 1024;
}

static unsigned exact_bit(int dir) { return dir == 0 ? G_EXACT0 : G_EXACT1; }
static unsigned retry_bit(int dir) { return dir == 0 ? G_RETRY0 : G_RETRY1; }

// (C,eps)-transform in direction dir (0: g <- f^{C,eps}, core.cpp:35-54; 1: f <-
// g^{C,eps}, core.cpp:56-82). Writes L (natural-log LSE) into P.L[dir] and, if
// pot != nullptr, the potential -eps*L.
// Sum-pass kernel family of an LSE direction: culled and/or fp32 (both opt-in), else fp64.
static int sum_mode(const Problem& P, int dir) {
    const bool f32 = P.precision == 32;
    if (cull_active(P, dir)) return f32 ? MODE_SUM_CULL_F32 : MODE_SUM_CULL;
    return f32 ? MODE_SUM_F32 : MODE_SUM;
}

static void lse(Problem& P, int dir, const double* in_vec, double* pot, unsigned guard) {
    Side& in = P.in_side(dir);
    Side& out = P.out_side(dir);
    const int64_t nin = in.count, nout = out.count;
    cudaStream_t s = P.stream;
    const TilePlan tmax = plan_for(P, dir, MODE_MAX, 0);
    const bool cull = cull_active(P, dir);
    const bool f32 = P.precision == 32;
    const TilePlan tsum = plan_for(P, dir, sum_mode(P, dir), 0);
    // Row-sharded column transform: every rank runs the whole single-GPU
    // pipeline on its own rows -- its own bound-shift / exact-max decision, shift and
    // validity retry, all rank-local (no collective inside the guarded branches) -- and
    // ends with its (shift_j, S_j) per column. ONE all-gather of those 2m doubles per rank
    // and a fixed rank-order merge L_j = M_j + log(sum_r S_rj e^{shift_rj - M_j}),
    // M_j = max_r shift_rj, give every rank the same global transform.
    const bool split = P.shard && dir == 0;
    double* Lbuf = P.L[dir].p;
    double* shift = P.shift[dir].p;
    if (split) {
        P.L_loc.ensure(nout);
        P.xrow.ensure(2 * nout);
        P.xall.ensure(2 * nout * P.world);
        Lbuf = P.L_loc.p;
        shift = P.xrow.p;
    }

    PrepInArgs pi;
    pi.count = nin;
    pi.d = P.otf() ? static_cast<int>(P.d) : 0;
    pi.pk = P.pk();
    pi.v = in_vec;
    pi.lw = in.lw.p;
    pi.sq = P.otf() ? in.sq.p : nullptr;
    pi.coords = P.otf() ? in.coords.p : nullptr;
    pi.inv_eps = P.inv_eps();
    pi.kc = P.kc();
    pi.sigma = P.sigma();
    pi.pack = P.pack_in[dir].p;
    pi.ref = P.ref[dir].p;
    pi.dir = dir;
    pi.part = P.stats.p;
    pi.st = P.st;
    pi.guard = guard;
    // fp32 terms underflow below 2^-126: take the exact shift once the bound could sit
    // more than 40 nats (58 bits) above the true maximum
    if (f32) pi.exact_spread = 40.0;
    const int gin = std::min(grid_for(nin), 148 * 8);
    count_launch();
    k_prep_in<<<gin, AUX_NT, 0, s>>>(pi);

    PrepOutArgs po;
    po.count = nout;
    po.d = pi.d;
    po.pk = pi.pk;
    po.sq = P.otf() ? out.sq.p : nullptr;
    po.coords = P.otf() ? out.coords.p : nullptr;
    po.inv_eps = P.inv_eps();
    po.kc = P.kc();
    po.sigma = P.sigma();
    po.shift_mode = SHIFT_BOUND;
    po.Lref = Lbuf;
    po.shift = shift;
    po.pack = P.pack_out[dir].p;
    po.dir = dir;
    po.st = P.st;
    po.guard = guard;
    count_launch();
    k_prep_out<<<grid_for(nout), AUX_NT, 0, s>>>(po);
    if (cull)  // input-group maxima of F (the inputs do not change between phases)
        cull_group_max(P, in, P.pack_in[dir].p, P.f_gi[dir].p, CULL_GI, guard);

    FinalizeArgs fa;
    fa.partial = P.partial.p;
    fa.n_out = nout;
    fa.shift = shift;
    fa.pack = P.pack_out[dir].p;
    fa.pk = P.pk();
    fa.sq = P.otf() ? out.sq.p : nullptr;
    fa.kc = P.kc();
    fa.eps = P.eps;
    fa.L = Lbuf;
    fa.pot = split ? nullptr : pot;
    fa.S = split ? P.xrow.p + nout : nullptr;
    fa.dir = dir;
    fa.st = P.st;
    if (f32) fa.lo_ok = 0x1p-60;  // smallest sum whose leading fp32 terms are still normal

    for (int phase = 0; phase < 2; ++phase) {
        const unsigned gmax = guard | (phase == 0 ? exact_bit(dir) : retry_bit(dir));
        const unsigned gsum = guard | (phase == 0 ? 0u : retry_bit(dir));
        launch_tiles(tmax, tile_args(P, dir, tmax, gmax), s);
        fa.partial = P.partial.p;
        fa.nb = tmax.n_in_blocks;
        fa.guard = gmax;
        count_launch();
        k_max_finalize<<<fold_grid(nout), AUX_NT, 0, s>>>(fa);
        if (cull) {  // output-group maxima of S with this phase's shift
            unsigned* sched = &P.st->counters[10 + dir];
            cull_group_max(P, out, P.pack_out[dir].p, P.s_go[dir].p, CULL_GO, gsum, sched);
            TileArgs ca = cull_args(P, dir, tsum, gsum, phase);
            ca.sched = sched;
            launch_tiles(tsum, ca, s);
        } else {
            launch_tiles(tsum, tile_args(P, dir, tsum, gsum), s);
        }
        fa.partial = P.partial.p;
        fa.nb = tsum.n_in_blocks;
        fa.guard = gsum;
        fa.retry_phase = phase;
        count_launch();
        k_lse_finalize<<<fold_grid(nout), AUX_NT, 0, s>>>(fa);
    }
    if (split) {
        allgather(P, P.xrow.p, P.xall.p, static_cast<size_t>(2 * nout));
        count_launch();
        k_lse_merge<<<grid_for(nout), AUX_NT, 0, s>>>(P.xall.p, P.world, nout, P.eps, P.L[dir].p, pot, P.st,
                                                      guard);
    }
    count_launch();
    k_lse_commit<<<grid_for(nin), AUX_NT, 0, s>>>(in_vec, P.ref[dir].p, nin, dir, P.st, guard);
    CK(cudaGetLastError());
}

// Unshifted pass family: out_o = oscale_o * sum_in exp(ia_in + ob_o - C/eps)
// [ * W[in][c] for block mode ], with ia = lw_in + v_in/eps (log weights
// chosen by the caller) and ob likewise.
struct PassSpec {
    int dir = 0;
    const double* in_v = nullptr;
    const double* in_lw = nullptr;
    const double* out_v = nullptr;
    const double* out_lw = nullptr;
    const double* W = nullptr;  // packed [nin][kt] or nullptr (sum mode)
    int k = 0, kt = 0;
    const double* out_scale = nullptr;
    double* out = nullptr;  // sum: [nout]; block: col-major nout x k (ld = nout)
    double* rsum_out = nullptr;  // block, dir 0 only: r_i = sum_j e(j, i) b_j fused into the pass
    // block, dir 0, sharded: reduce-scatter instead of allreduce -- `out` (R * scatter_rows
    // x k, rank-blocked) is summed over the shards and this rank receives its block
    // (scatter_rows x k, ld = scatter_rows) here
    double* scatter_out = nullptr;
    bool w_static = false;             // W is the solve's packed basis: its int8 digit tiles are made once per solve
    bool cull = false;                 // block pass may skip negligible terms (culling enabled)
    const double* cull_logtot = nullptr;  // per-output log of sum_in e (nullptr: 0, i.e. sums are 1)
    unsigned guard = 0;
};

// Input-block cap of a pass's split-K partials: the ell-wide block passes keep at most 8
// (their partials are kt x n_out each); sum passes and the 4-column anchor pass are
// split like the LSE sums (enough tiles for every SM).
static int64_t anchor_in_blocks(int kt) { return kt > 4 ? 8 : 0; }

// Columns of the stable accept test's anchor pass W = (1, expm1(d/eps), exp(d/eps), 0):
// the register point kernels take 4 columns with DFMA; the DMMA kernels need a multiple of 8.
static int anchor_kt(const Problem& P) { return P.dim >= 1 && P.dim <= 4 ? 4 : 8; }

// Whether the block pass can fuse r = P~ beta (register point kernels, d <= 4).
static bool block_rs_fusable(const Problem& P) { return P.dim >= 1 && P.dim <= 4; }

static void plan_pass(Problem& P, const PassSpec& ps) {
    Side& in = P.in_side(ps.dir);
    Side& out = P.out_side(ps.dir);
    const int64_t nin = in.count, nout = out.count;
    cudaStream_t s = P.stream;
    const bool rs = ps.W && ps.rsum_out;
    if (rs && (ps.dir != 0 || !block_rs_fusable(P))) throw InvalidArgument("sknr_b200: fused row sums unsupported here");
    const bool scatter = ps.scatter_out && P.shard && ps.W && ps.dir == 0;
    const bool bcull = ps.W && !rs && ps.cull && cull_block_active(P, ps.dir);
    const int mode = ps.W ? (rs ? MODE_BLOCK_RS : (bcull ? MODE_BLOCK_CULL : MODE_BLOCK)) : MODE_SUM;
    const TilePlan tp = plan_for(P, ps.dir, mode, ps.W ? ps.kt : 0, anchor_in_blocks(ps.W ? ps.kt : 0));

    PrepInArgs pi;
    pi.count = nin;
    pi.d = P.otf() ? static_cast<int>(P.d) : 0;
    pi.pk = P.pk();
    pi.v = ps.in_v;
    pi.lw = ps.in_lw;
    pi.sq = P.otf() ? in.sq.p : nullptr;
    pi.coords = P.otf() ? in.coords.p : nullptr;
    pi.inv_eps = P.inv_eps();
    pi.kc = P.kc();
    pi.sigma = P.sigma();
    pi.pack = P.pack_in[ps.dir].p;
    pi.st = P.st;
    pi.guard = ps.guard;
    count_launch();
    k_prep_in<<<grid_for(nin), AUX_NT, 0, s>>>(pi);

    PrepOutArgs po;
    po.count = nout;
    po.d = pi.d;
    po.pk = pi.pk;
    po.v = ps.out_v;
    po.lw = ps.out_lw;
    po.sq = P.otf() ? out.sq.p : nullptr;
    po.coords = P.otf() ? out.coords.p : nullptr;
    po.inv_eps = P.inv_eps();
    po.kc = P.kc();
    po.sigma = P.sigma();
    po.shift_mode = SHIFT_NONE;
    po.pack = P.pack_out[ps.dir].p;
    po.dir = ps.dir;
    po.st = P.st;
    po.guard = ps.guard;
    count_launch();
    k_prep_out<<<grid_for(nout), AUX_NT, 0, s>>>(po);

    TileArgs ta = tile_args(P, ps.dir, tp, ps.guard);
    if (bcull) {
        unsigned* sched = &P.st->counters[12];
        cull_group_max(P, in, P.pack_in[ps.dir].p, P.f_g32[ps.dir].p, 32, ps.guard);
        cull_group_max(P, out, P.pack_out[ps.dir].p, P.s_g16[ps.dir].p, 16, ps.guard, sched,
                       ps.cull_logtot);
        ta.perm_in = in.perm.p;
        ta.perm_out = out.perm.p;
        ta.box_gi = in.box32.p;
        ta.box_go = out.box16.p;
        ta.f_gi = P.f_g32[ps.dir].p;
        ta.s_go = P.s_g16[ps.dir].p;
        ta.lskc = kLS * P.kc();
        ta.cull_t = P.cull_t;
        ta.sched = sched;
    }
    ta.W = ps.W;
    if (rs) {
        ta.out_w = out.w.p;
        ta.rsum = P.rsum.p;
    }
    if (tp.i8) {  // tensor-core pass: V as exact int8 digit tiles, O(n kt); a solve's basis keeps
                  // the tiles made by prepare_solve, any other W is converted per pass
        uint8_t* vsl = reinterpret_cast<uint8_t*>(P.vsl.p);
        unsigned* vexp = reinterpret_cast<unsigned*>(P.vexp.p);
        if (!(ps.w_static && P.vsl_src == ps.W)) {
            launch_i8_vprep(ps.W, ps.kt, nin, vsl, vexp, P.st, ps.guard, s);
            P.vsl_src = nullptr;
        }
        ta.vsl = vsl;
        ta.vexp = vexp;
        ta.kt = ps.kt;
    }
    launch_tiles(tp, ta, s);
    if (rs) {
        count_launch();
        k_rsum_finalize<<<fold_grid(nin), AUX_NT, 0, s>>>(P.rsum.p, tp.n_out_tiles, nin, ps.rsum_out, P.st,
                                                         ps.guard);
    }
    count_launch();
    if (mode == MODE_SUM)
        k_sum_finalize<<<fold_grid(nout), AUX_NT, 0, s>>>(P.partial.p, tp.n_in_blocks, nout, ps.out_scale,
                                                         ps.out, P.st, ps.guard);
    else
        k_block_finalize<<<fold_grid(nout * ps.k), AUX_NT, 0, s>>>(P.partial.p, tp.n_in_blocks, ps.kt,
                                                                  ps.k, nout, ps.out_scale, ps.out, nout,
                                                                  P.st, ps.guard, scatter ? scatter_rows(P) : 0);
    if (scatter)  // column direction, this rank's block of the sum over the sharded rows
        reduce_scatter(P, ps.out, ps.scatter_out, static_cast<size_t>(scatter_rows(P)) * ps.k);
    else if (ps.dir == 0)  // column direction reduces over the sharded rows
        allreduce(P, ps.out, static_cast<size_t>(nout) * (mode == MODE_SUM ? 1 : ps.k), ncclSum);
    CK(cudaGetLastError());
}

// Gram / dot products: out[a + b*ka] = scale * sum_t w_t U[t,a] V[t,b]
constexpr unsigned kGramSlot = 4;  // DevState ticket counter used by k_gram
static void gram(Problem& P, int64_t T, int ka, int kb, const double* U, int64_t ldu, const double* V,
                 int64_t ldv, const double* w, double* out, unsigned guard, int diag_only = 0,
                 double scale = 1.0) {
    GramArgs ga;
    ga.T = T;
    ga.ka = ka;
    ga.kb = kb;
    ga.U = U;
    ga.ldu = ldu;
    ga.V = V;
    ga.ldv = ldv;
    ga.w = w;
    ga.diag_only = diag_only;
    ga.part = P.gram_part.p;
    ga.out = out;
    ga.out_scale = scale;
    ga.counter = &P.st->counters[kGramSlot];
    ga.st = P.st;
    ga.guard = guard;
    const int G = gram_blocks(T);
    count_launch();
    k_gram<<<G, AUX_NT, 0, P.stream>>>(ga);
    if (G > 1) {
        const int64_t Q = diag_only ? ka : static_cast<int64_t>(ka) * kb;
        count_launch();
        k_fold_sum<<<fold_grid(Q), AUX_NT, 0, P.stream>>>(ga.part, G, Q, scale, out, P.st, guard);
    }
    CK(cudaGetLastError());
}


// gram() followed by the cross-rank sum when the rows are sharded.
static void gram_all(Problem& P, int64_t T, int ka, int kb, const double* U, int64_t ldu, const double* V,
                     int64_t ldv, const double* w, double* out, unsigned guard, int diag_only = 0) {
    gram(P, T, ka, kb, U, ldu, V, ldv, w, out, guard, diag_only);
    allreduce(P, out, static_cast<size_t>(diag_only ? ka : ka * kb), ncclSum);
}

#include "engine_spectral.cuh"
#include "engine_solver.cuh"

}  // namespace sknr

#include "engine_capi.cuh"
