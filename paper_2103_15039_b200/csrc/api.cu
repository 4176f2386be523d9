// C ABI of liblsgcpd.so (see include/lsgcpd.h for the contract of every entry point).
#include <dlfcn.h>
#include <stdarg.h>
#include <string.h>

#include <mutex>
#include <vector>

#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: ranges for Nsight / ncu --nvtx

#include "common.cuh"
#include "kernels.h"

#define LSG_EXPORT extern "C" __attribute__((visibility("default")))

namespace lsg {

static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

int cuda_fail(cudaError_t e, const char* what) {
    set_error("CUDA error %s (%s) in %s", cudaGetErrorName(e), cudaGetErrorString(e), what);
    return LSGCPD_ECUDA;
}

static bool finite_vec(const double* v, int n) {
    for (int i = 0; i < n; ++i)
        if (!isfinite(v[i])) return false;
    return true;
}

static bool is_rotation(const double* R) {
    if (!finite_vec(R, 9)) return false;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double s = 0.0;
            for (int k = 0; k < 3; ++k) s += R[3 * k + i] * R[3 * k + j];
            if (fabs(s - (i == j ? 1.0 : 0.0)) > 1e-6) return false;
        }
    const double det = R[0] * (R[4] * R[8] - R[5] * R[7]) - R[1] * (R[3] * R[8] - R[5] * R[6]) +
                       R[2] * (R[3] * R[7] - R[4] * R[6]);
    return det > 0.0;
}

// affine group: a finite linear part with positive determinant (GA⁺(3))
static bool is_affine_linear(const double* A) {
    if (!finite_vec(A, 9)) return false;
    const double det = A[0] * (A[4] * A[8] - A[5] * A[7]) - A[1] * (A[3] * A[8] - A[5] * A[6]) +
                       A[2] * (A[3] * A[7] - A[4] * A[6]);
    return det > 0.0;
}
static bool pose_ok(const double* R, int group) { return group ? is_affine_linear(R) : is_rotation(R); }

// RAII NVTX range (SURVEY §5 tracing): one per public call and per registration phase
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

// Owns the capture stream, event, graph and executable of one EM-loop replay; released on every exit path.
struct GraphRun {
    cudaStream_t cs = nullptr;
    cudaEvent_t ev = nullptr;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    ~GraphRun() {
        if (exec) cudaGraphExecDestroy(exec);
        if (graph) cudaGraphDestroy(graph);
        if (ev) cudaEventDestroy(ev);
        if (cs) cudaStreamDestroy(cs);
    }
};

// Instantiated EM-iteration graphs of recent lsgcpd_register calls on this thread, keyed by every value the
// captured kernels receive (pointers, sizes, schedule, EM parameters).  Capture + instantiate costs ≈ 0.3 ms
// per call, a fifth of a 50-iteration registration of 1,000 points; a repeated call with the same buffers and
// parameters replays the cached graph; a call with other buffers or values but the same launch shapes (another
// problem of the same size) captures its graph and updates a cached executable in place (cudaGraphExecUpdate)
// instead of instantiating one.  The work before the loop (memsets, setup, σ²₀) runs every call.
struct GraphCache {
    struct Entry {
        std::vector<unsigned char> key, topo;   // every kernel argument; the launch shapes only
        GraphRun* run = nullptr;
        uint64_t used = 0;
    };
    std::vector<Entry> e;
    uint64_t tick = 0;
    static constexpr int kMaxDev = 64;
    cudaStream_t cap[kMaxDev] = {};   // capture stream of this thread, per device (a stream belongs to one device)
    static constexpr size_t kMax = 4;
    Entry* find(const std::vector<unsigned char>& k, bool topo) {
        for (auto& x : e)
            if ((topo ? x.topo : x.key) == k) {
                x.used = ++tick;
                return &x;
            }
        return nullptr;
    }
    void insert(std::vector<unsigned char> k, std::vector<unsigned char> t, GraphRun* r) {
        if (e.size() >= kMax) {
            size_t lru = 0;
            for (size_t i = 1; i < e.size(); ++i)
                if (e[i].used < e[lru].used) lru = i;
            delete e[lru].run;
            e.erase(e.begin() + (long)lru);
        }
        e.push_back({std::move(k), std::move(t), r, ++tick});
    }
    ~GraphCache() {
        for (auto& x : e) delete x.run;
        for (auto c : cap)
            if (c) cudaStreamDestroy(c);
    }
};
static thread_local GraphCache g_graphs;

template <typename T>
static void key_put(std::vector<unsigned char>& k, const T& v) {
    const unsigned char* b = reinterpret_cast<const unsigned char*>(&v);
    k.insert(k.end(), b, b + sizeof(T));
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
static size_t al(size_t x) { return (x + 255) & ~size_t(255); }

// ---------------------------------------------------------------------------------------------
// NCCL, loaded at run time (the library does not link it; torch's libnccl.so.2 is reused if loaded)
// ---------------------------------------------------------------------------------------------
typedef int ncclResult_t;
typedef struct ncclComm* ncclComm_t;
typedef struct {
    char internal[128];
} ncclUniqueId;
enum { kNcclFloat64 = 8, kNcclSum = 0 };

struct Nccl {
    bool loaded = false;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
static Nccl g_nccl;
static std::mutex g_nccl_mu;

static int nccl_load() {
    std::lock_guard<std::mutex> lk(g_nccl_mu);
    if (g_nccl.loaded) return 0;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    LSG_CHECK(h != nullptr, LSGCPD_ENCCL, "cannot load libnccl.so.2: %s", dlerror());
    g_nccl.GetUniqueId = (ncclResult_t(*)(ncclUniqueId*))dlsym(h, "ncclGetUniqueId");
    g_nccl.CommInitRank = (ncclResult_t(*)(ncclComm_t*, int, ncclUniqueId, int))dlsym(h, "ncclCommInitRank");
    g_nccl.AllReduce =
        (ncclResult_t(*)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t))dlsym(h, "ncclAllReduce");
    g_nccl.CommDestroy = (ncclResult_t(*)(ncclComm_t))dlsym(h, "ncclCommDestroy");
    g_nccl.GetErrorString = (const char* (*)(ncclResult_t))dlsym(h, "ncclGetErrorString");
    LSG_CHECK(g_nccl.GetUniqueId && g_nccl.CommInitRank && g_nccl.AllReduce && g_nccl.CommDestroy, LSGCPD_ENCCL,
              "libnccl.so.2 lacks required symbols");
    g_nccl.loaded = true;
    return 0;
}

static int nccl_fail(ncclResult_t r, const char* what) {
    set_error("NCCL error %d (%s) in %s", r, g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "?", what);
    return LSGCPD_ENCCL;
}

struct Comm {
    ncclComm_t nc;
    int rank, world;
};

// ---------------------------------------------------------------------------------------------
// Workspace layouts
// ---------------------------------------------------------------------------------------------
struct EstepLayout {
    size_t state, part, total;
};
static int estep_layout(int64_t M_pad, int64_t N, EstepLayout* L, Sched* sc) {
    const int rc = estep_plan(M_pad, N, sc);
    if (rc) return rc;
    size_t o = 0;
    L->state = o; o += al(sizeof(IterState));
    L->part = o; o += al(estep_partial_bytes(*sc));
    L->total = o;
    return 0;
}

struct RegLayout {
    size_t state, mom, sums, blockpart, counters, nll, sig2, iters, part, rec, total;
    size_t srt, sphi, ssort;   // the Morton-ordered source copy and its sort scratch (0: sources not reordered)
    int sorted;
};
// Sources of at least this many points are registered in Morton order (DESIGN §8 "far points"); below it the
// sort's launches cost more than the E steps gain
constexpr int64_t kSortMinN = 4096;
static int reg_layout(int64_t M_pad, int64_t N, int max_iters, RegLayout* L, Sched* sc) {
    const int rc = estep_plan(M_pad, N, sc);
    if (rc) return rc;
    size_t o = 0;
    L->state = o; o += al(sizeof(IterState));
    L->mom = o; o += al(sizeof(double) * 80);
    L->sums = o; o += al(sizeof(double) * 4);
    L->blockpart = o; o += al(sizeof(double) * kMomentBlocks * kMomentCount);
    L->counters = o; o += al(sizeof(unsigned) * 8);
    L->nll = o; o += al(sizeof(double) * (max_iters + 1));
    L->sig2 = o; o += al(sizeof(double) * (max_iters + 2));
    L->iters = o; o += al(sizeof(int) * 4);
    L->part = o; o += al(estep_partial_bytes(*sc));
    L->rec = o; o += al(sizeof(float) * LSGCPD_REC * (size_t)N);
    L->sorted = N >= kSortMinN && N < ((int64_t)1 << 31);
    if (L->sorted) {
        L->srt = o; o += al(sizeof(float) * 3 * (size_t)N);
        L->sphi = o; o += al(sizeof(float) * (size_t)N);
        L->ssort = o; o += al(source_sort_ws_bytes(N));
    } else {
        L->srt = L->sphi = L->ssort = 0;
    }
    L->total = o;
    return 0;
}
// The source the EM iterations read: a Morton-ordered copy in the workspace when the layout has one and the
// sort_source option is on (the confidences φ reordered with it), else the caller's arrays.
static int order_source(const float** src, const float** phi, int64_t N, char* ws, const RegLayout& L,
                        cudaStream_t s) {
    if (!L.sorted || options().sort_source.load() == 0) return 0;
    float* out = reinterpret_cast<float*>(ws + L.srt);
    float* phi_out = *phi ? reinterpret_cast<float*>(ws + L.sphi) : nullptr;
    const int rc = source_sort_launch(*src, *phi, N, out, phi_out, ws + L.ssort, s);
    if (rc) return rc;
    *src = out;
    if (*phi) *phi = phi_out;
    return 0;
}

static int read_header(const void* d_target, int64_t M, TargetHeader* h, cudaStream_t stream) {
    LSG_CUDA(cudaMemcpyAsync(h, d_target, sizeof(TargetHeader), cudaMemcpyDeviceToHost, stream));
    LSG_CUDA(cudaStreamSynchronize(stream));
    LSG_CHECK(h->magic == kTargetMagic, LSGCPD_EINVAL, "d_target is not a prepared target (bad magic)");
    LSG_CHECK(h->M == M, LSGCPD_EINVAL, "M=%lld does not match the prepared target (M=%lld)", (long long)M,
              (long long)h->M);
    return 0;
}

// The two halves of one EM iteration around the moment all-reduce (async).
// First half: E step → merge → the 75 moments in `mom`.  With fuse_newton (no communicator) the N ≤ 2^17 path
// also runs Newton + σ² inside em_tail_kernel and the iteration is complete.
static int enqueue_moments(const void* d_target, const float* d_src, int64_t N, char* ws, const RegLayout& L,
                           const Sched& sc, const RegParams& rp, bool fuse_newton, cudaStream_t stream) {
    IterState* st = reinterpret_cast<IterState*>(ws + L.state);
    double* mom = reinterpret_cast<double*>(ws + L.mom);
    float* rec = reinterpret_cast<float*>(ws + L.rec);
    if (N <= kTailMaxN && options().no_fuse.load() != 1) {   // one launch for merge + moments (+ Newton w/o comm)
        const int rc = estep_launch(d_target, d_src, N, st, sc, reinterpret_cast<float*>(ws + L.part), rec,
                                    rp.consistent, rp.phi, stream, 0);
        if (rc) return rc;
        em_tail_launch(reinterpret_cast<float*>(ws + L.part), d_src, N, st, sc, rp.phi,
                       reinterpret_cast<double*>(ws + L.blockpart), mom, reinterpret_cast<unsigned*>(ws + L.counters),
                       rp, reinterpret_cast<double*>(ws + L.nll), reinterpret_cast<double*>(ws + L.sig2),
                       reinterpret_cast<int*>(ws + L.iters), fuse_newton ? 1 : 0, stream);
        return 0;
    }
    const int rc = estep_launch(d_target, d_src, N, st, sc, reinterpret_cast<float*>(ws + L.part), rec, rp.consistent,
                                rp.phi, stream);
    if (rc) return rc;
    moments_launch(rec, d_src, N, st, reinterpret_cast<double*>(ws + L.blockpart), mom,
                   reinterpret_cast<unsigned*>(ws + L.counters), stream);
    return 0;
}
static bool moments_fused_newton(int64_t N) { return N <= kTailMaxN && options().no_fuse.load() != 1; }
// Second half: damped Newton + σ² from the (all-reduced) moments; writes the next IterState.
static void enqueue_newton(char* ws, const RegLayout& L, const RegParams& rp, cudaStream_t stream) {
    newton_launch(reinterpret_cast<IterState*>(ws + L.state), reinterpret_cast<double*>(ws + L.mom), rp,
                  reinterpret_cast<double*>(ws + L.nll), reinterpret_cast<double*>(ws + L.sig2),
                  reinterpret_cast<int*>(ws + L.iters), stream);
}

// One EM iteration (async): E step → moments → [all-reduce] → Newton + σ².
static int enqueue_iteration(const void* d_target, const float* d_src, int64_t N, char* ws, const RegLayout& L,
                             const Sched& sc, const RegParams& rp, Comm* comm, cudaStream_t stream) {
    const int rc = enqueue_moments(d_target, d_src, N, ws, L, sc, rp, comm == nullptr, stream);
    if (rc) return rc;
    if (!comm && moments_fused_newton(N)) return 0;
    if (comm) {
        double* mom = reinterpret_cast<double*>(ws + L.mom);
        const ncclResult_t r = g_nccl.AllReduce(mom, mom, kMomentCount, kNcclFloat64, kNcclSum, comm->nc, stream);
        if (r != 0) return nccl_fail(r, "ncclAllReduce(moments)");
    }
    enqueue_newton(ws, L, rp, stream);
    return 0;
}

// The all-reduce of lsgcpd_register_shards: out = Σ_g v_g in shard order, written back to every shard's vector
// (every "rank" receives the same sum, as from ncclAllReduce).
constexpr int kMaxShards = 16;
struct ShardPtrs {
    double* p[kMaxShards];
};
__global__ void shard_allreduce_kernel(ShardPtrs v, int G, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double s = v.p[0][i];
    for (int g = 1; g < G; ++g) s += v.p[g][i];
    for (int g = 0; g < G; ++g) v.p[g][i] = s;
}

}  // namespace lsg

using namespace lsg;

// =============================================================================================
// exported C ABI
// =============================================================================================
LSG_EXPORT int lsgcpd_version(void) { return 10400; }
LSG_EXPORT const char* lsgcpd_last_error(void) { return g_err; }

LSG_EXPORT void lsgcpd_prep_params_default(lsgcpd_prep_params* p) {
    if (!p) return;
    p->alpha_max = 50.0f;
    p->lambda = 0.5f;
    p->knn_k = 10;
    p->volume_margin = 0.1;
}

LSG_EXPORT void lsgcpd_em_params_default(lsgcpd_em_params* p) {
    if (!p) return;
    p->w = 0.1;
    p->max_iters = 50;
    p->newton_max = 10;
    p->consistent_normalizer = 1;
    p->sigma2_init = 0.0;
    p->sigma2_floor_rel = 1e-12;
    p->tol = 0.0;
    p->eta = -1.0;
    p->d_src_conf = nullptr;
    p->group = 0;
}

LSG_EXPORT size_t lsgcpd_target_bytes(int64_t M) {
    if (M < 0) return 0;
    return target_total_bytes(pad_targets(M));
}

LSG_EXPORT size_t lsgcpd_prepare_workspace_bytes(int64_t M, int knn_k) {
    (void)knn_k;
    if (M < 0) return 0;
    return prepare_ws_bytes(M);
}

LSG_EXPORT size_t lsgcpd_pack_workspace_bytes(int64_t M) {
    if (M < 0) return 0;
    return pack_ws_bytes(M);
}

LSG_EXPORT int lsgcpd_prepare_target(const float* d_xyz, int64_t M, const lsgcpd_prep_params* params, void* d_target,
                                     void* d_ws, size_t ws_bytes, lsgcpd_target_info* h_info,
                                     const lsgcpd_annotations* annotations, lsgcpd_stream_t stream) {
    lsgcpd_prep_params p;
    lsgcpd_prep_params_default(&p);
    if (params) p = *params;
    LSG_CHECK(d_xyz && d_target && d_ws, LSGCPD_EINVAL, "null pointer argument");
    LSG_CHECK(aligned16(d_target), LSGCPD_EINVAL, "d_target must be 16-byte aligned");
    LSG_CHECK(M >= 3 && M < (int64_t)1 << 30, LSGCPD_EINVAL, "M=%lld out of range [3, 2^30)", (long long)M);
    LSG_CHECK(p.knn_k >= 3 && p.knn_k <= 32 && p.knn_k <= M, LSGCPD_EINVAL, "knn_k=%d out of range [3, min(32, M)]",
              p.knn_k);
    LSG_CHECK(isfinite(p.alpha_max) && p.alpha_max >= 0.f && isfinite(p.lambda) && p.lambda > 0.f, LSGCPD_EINVAL,
              "alpha_max must be >= 0 and lambda > 0");
    LSG_CHECK(isfinite(p.volume_margin) && p.volume_margin >= 0.0, LSGCPD_EINVAL, "volume_margin must be >= 0");
    LSG_CHECK(ws_bytes >= prepare_ws_bytes(M), LSGCPD_EINVAL, "workspace too small (%zu < %zu)", ws_bytes,
              prepare_ws_bytes(M));
    NvtxRange r("lsgcpd_prepare_target");
    return prepare_target_impl(d_xyz, M, p, d_target, d_ws, h_info, annotations, (cudaStream_t)stream);
}

LSG_EXPORT size_t lsgcpd_prepare_batch_workspace_bytes(const int64_t* h_M, int B, int knn_k) {
    (void)knn_k;
    if (!h_M || B < 1) return 0;
    for (int b = 0; b < B; ++b)
        if (h_M[b] < 3 || h_M[b] >= (int64_t)1 << 30) return 0;
    return prepare_batch_ws_bytes(h_M, B);
}

LSG_EXPORT int lsgcpd_prepare_batch(const float* const* h_d_xyz, const int64_t* h_M, int B,
                                    const lsgcpd_prep_params* params, void* const* h_d_target, void* d_ws,
                                    size_t ws_bytes, lsgcpd_target_info* h_info, lsgcpd_stream_t stream) {
    lsgcpd_prep_params p;
    lsgcpd_prep_params_default(&p);
    if (params) p = *params;
    LSG_CHECK(h_d_xyz && h_M && h_d_target && d_ws && B >= 1 && B <= (1 << 20), LSGCPD_EINVAL,
              "null pointer argument or bad B=%d", B);
    for (int b = 0; b < B; ++b) {
        LSG_CHECK(h_d_xyz[b] && h_d_target[b], LSGCPD_EINVAL, "problem %d: null pointer", b);
        LSG_CHECK(aligned16(h_d_target[b]), LSGCPD_EINVAL, "problem %d: d_target must be 16-byte aligned", b);
        LSG_CHECK(h_M[b] >= 3 && h_M[b] < (int64_t)1 << 30 && p.knn_k <= h_M[b], LSGCPD_EINVAL,
                  "problem %d: M=%lld out of range [max(3, knn_k), 2^30)", b, (long long)h_M[b]);
    }
    LSG_CHECK(p.knn_k >= 3 && p.knn_k <= 32, LSGCPD_EINVAL, "knn_k=%d out of range [3, 32]", p.knn_k);
    LSG_CHECK(isfinite(p.alpha_max) && p.alpha_max >= 0.f && isfinite(p.lambda) && p.lambda > 0.f, LSGCPD_EINVAL,
              "alpha_max must be >= 0 and lambda > 0");
    LSG_CHECK(isfinite(p.volume_margin) && p.volume_margin >= 0.0, LSGCPD_EINVAL, "volume_margin must be >= 0");
    LSG_CHECK(aligned16(d_ws), LSGCPD_EINVAL, "d_ws must be 16-byte aligned");
    LSG_CHECK(ws_bytes >= prepare_batch_ws_bytes(h_M, B), LSGCPD_EINVAL, "workspace too small (%zu < %zu)", ws_bytes,
              prepare_batch_ws_bytes(h_M, B));
    NvtxRange r("lsgcpd_prepare_batch");
    return prepare_batch_impl(h_d_xyz, h_M, B, p, h_d_target, d_ws, h_info, (cudaStream_t)stream);
}

LSG_EXPORT int lsgcpd_pack_target(const float* d_xyz, const float* d_normals, const float* d_alpha, int64_t M,
                                  double volume_margin, void* d_target, void* d_ws, size_t ws_bytes,
                                  lsgcpd_target_info* h_info, lsgcpd_stream_t stream) {
    LSG_CHECK(d_xyz && d_normals && d_alpha && d_target && d_ws, LSGCPD_EINVAL, "null pointer argument");
    LSG_CHECK(aligned16(d_target), LSGCPD_EINVAL, "d_target must be 16-byte aligned");
    LSG_CHECK(M >= 1 && M < (int64_t)1 << 30, LSGCPD_EINVAL, "M=%lld out of range", (long long)M);
    LSG_CHECK(isfinite(volume_margin) && volume_margin >= 0.0, LSGCPD_EINVAL, "volume_margin must be >= 0");
    LSG_CHECK(ws_bytes >= pack_ws_bytes(M), LSGCPD_EINVAL, "workspace too small (%zu < %zu)", ws_bytes,
              pack_ws_bytes(M));
    const int rc = pack_target_impl(d_xyz, d_normals, d_alpha, M, volume_margin, d_target, d_ws, h_info,
                                    (cudaStream_t)stream);
    if (rc == LSGCPD_EDEGENERATE && h_info && !isfinite(h_info->extent)) {
        set_error("non-finite coordinate in d_xyz");
        return LSGCPD_EINVAL;
    }
    return rc;
}

LSG_EXPORT size_t lsgcpd_estep_workspace_bytes(int64_t M, int64_t N) {
    if (M < 1 || N < 1) return 0;
    EstepLayout L;
    Sched sc;
    if (estep_layout(pad_targets(M), N, &L, &sc)) return 0;
    return L.total;
}

static int estep_impl(const void* d_target, int64_t M, const float* d_src, int64_t N, const double R[9],
                      const double t[3], double sigma2, double w, double eta, const float* phi, double volume,
                      int consistent_normalizer, float* d_record, void* d_ws, size_t ws_bytes, cudaStream_t s,
                      int group = 0);

LSG_EXPORT int lsgcpd_estep(const void* d_target, int64_t M, const float* d_src, int64_t N, const double R[9],
                            const double t[3], double sigma2, double w, double volume, int consistent_normalizer,
                            float* d_record, void* d_ws, size_t ws_bytes, lsgcpd_stream_t stream) {
    return estep_impl(d_target, M, d_src, N, R, t, sigma2, w, -1.0, nullptr, volume, consistent_normalizer,
                      d_record, d_ws, ws_bytes, (cudaStream_t)stream);
}

LSG_EXPORT int lsgcpd_estep_ex(const void* d_target, int64_t M, const float* d_src, int64_t N, const double R[9],
                               const double t[3], double sigma2, const lsgcpd_em_params* params, double volume,
                               float* d_record, void* d_ws, size_t ws_bytes, lsgcpd_stream_t stream) {
    LSG_CHECK(params, LSGCPD_EINVAL, "null params");
    LSG_CHECK(!(params->eta >= 1.0) && !isnan(params->eta), LSGCPD_EINVAL, "eta must be < 1 (negative: off)");
    LSG_CHECK(params->group == 0 || params->group == 1, LSGCPD_EINVAL, "group must be 0 (SE(3)) or 1 (affine)");
    return estep_impl(d_target, M, d_src, N, R, t, sigma2, params->eta >= 0.0 ? 0.0 : params->w, params->eta,
                      params->d_src_conf, volume, params->consistent_normalizer, d_record, d_ws, ws_bytes,
                      (cudaStream_t)stream, params->group);
}

static int estep_impl(const void* d_target, int64_t M, const float* d_src, int64_t N, const double R[9],
                      const double t[3], double sigma2, double w, double eta, const float* phi, double volume,
                      int consistent_normalizer, float* d_record, void* d_ws, size_t ws_bytes, cudaStream_t s,
                      int group) {
    LSG_CHECK(d_target && d_src && d_record && d_ws && R && t, LSGCPD_EINVAL, "null pointer argument");
    LSG_CHECK(aligned16(d_target) && aligned16(d_record) && aligned16(d_ws), LSGCPD_EINVAL,
              "d_target, d_record and d_ws must be 16-byte aligned");
    LSG_CHECK(M >= 1 && N >= 1 && M < (int64_t)1 << 30 && N < (int64_t)1 << 34, LSGCPD_EINVAL,
              "M=%lld N=%lld out of range", (long long)M, (long long)N);
    LSG_CHECK(isfinite(sigma2) && sigma2 > 0.0, LSGCPD_EINVAL, "sigma2 must be finite and > 0");
    LSG_CHECK(isfinite(w) && w >= 0.0 && w < 1.0, LSGCPD_EINVAL, "w must be in [0, 1)");
    LSG_CHECK(isfinite(volume) && volume > 0.0, LSGCPD_EINVAL, "volume must be finite and > 0");
    LSG_CHECK(pose_ok(R, group), LSGCPD_EINVAL,
              group ? "A must be finite with det A > 0" : "R is not a rotation matrix (to 1e-6)");
    LSG_CHECK(finite_vec(t, 3), LSGCPD_EINVAL, "t must be finite");
    EstepLayout L;
    Sched sc;
    int rc = estep_layout(pad_targets(M), N, &L, &sc);
    if (rc) return rc;
    LSG_CHECK(ws_bytes >= L.total, LSGCPD_EINVAL, "workspace too small (%zu < %zu)", ws_bytes, L.total);
    if (!consistent_normalizer) {   // the Eq. 9-10 literal form has π(m) = 1/M (reads the header: a host sync)
        TargetHeader h;
        rc = read_header(d_target, M, &h, s);
        if (rc) return rc;
        LSG_CHECK(!h.prior, LSGCPD_EINVAL, "component priors require consistent_normalizer = 1");
    }
    NvtxRange r("lsgcpd_estep");
    char* ws = static_cast<char*>(d_ws);
    IterState* st = reinterpret_cast<IterState*>(ws + L.state);
    estep_launch_setup(st, d_target, R, t, sigma2, w, volume, M, consistent_normalizer ? 1 : 0, eta, s);
    rc = estep_launch(d_target, d_src, N, st, sc, reinterpret_cast<float*>(ws + L.part), d_record,
                      consistent_normalizer ? 1 : 0, phi, s);
    if (rc) return rc;
    LSG_CUDA(cudaGetLastError());
    return 0;
}

LSG_EXPORT int lsgcpd_comm_unique_id(void* h_out128) {
    LSG_CHECK(h_out128, LSGCPD_EINVAL, "null pointer argument");
    int rc = nccl_load();
    if (rc) return rc;
    ncclUniqueId id;
    const ncclResult_t r = g_nccl.GetUniqueId(&id);
    if (r != 0) return nccl_fail(r, "ncclGetUniqueId");
    memcpy(h_out128, &id, sizeof(id));
    return 0;
}

LSG_EXPORT int lsgcpd_comm_init(int rank, int world_size, const void* h_id128, void** comm_out) {
    LSG_CHECK(h_id128 && comm_out, LSGCPD_EINVAL, "null pointer argument");
    LSG_CHECK(world_size >= 1 && rank >= 0 && rank < world_size, LSGCPD_EINVAL, "bad rank/world_size");
    int rc = nccl_load();
    if (rc) return rc;
    ncclUniqueId id;
    memcpy(&id, h_id128, sizeof(id));
    Comm* c = new Comm();
    c->rank = rank;
    c->world = world_size;
    const ncclResult_t r = g_nccl.CommInitRank(&c->nc, world_size, id, rank);
    if (r != 0) {
        delete c;
        return nccl_fail(r, "ncclCommInitRank");
    }
    *comm_out = c;
    return 0;
}

LSG_EXPORT int lsgcpd_comm_destroy(void* comm) {
    if (!comm) return 0;
    Comm* c = static_cast<Comm*>(comm);
    ncclResult_t r = 0;
    if (g_nccl.loaded) r = g_nccl.CommDestroy(c->nc);
    delete c;
    if (r != 0) return nccl_fail(r, "ncclCommDestroy");
    return 0;
}

LSG_EXPORT size_t lsgcpd_register_workspace_bytes(int64_t M, int64_t N_local, int max_iters) {
    if (M < 1 || N_local < 1 || max_iters < 0) return 0;
    RegLayout L;
    Sched sc;
    if (reg_layout(pad_targets(M), N_local, max_iters, &L, &sc)) return 0;
    return L.total;
}

namespace lsg {
// EM parameters common to lsgcpd_register and lsgcpd_register_shards (the checks of include/lsgcpd.h)
static int check_em_params(const lsgcpd_em_params& p, const double* R, const double* t) {
    LSG_CHECK(isfinite(p.w) && p.w >= 0.0 && p.w < 1.0, LSGCPD_EINVAL, "w must be in [0, 1)");
    LSG_CHECK(p.max_iters >= 0 && p.max_iters <= 100000, LSGCPD_EINVAL, "max_iters out of range");
    LSG_CHECK(p.newton_max >= 0 && p.newton_max <= 1000, LSGCPD_EINVAL, "newton_max out of range");
    LSG_CHECK(isfinite(p.sigma2_floor_rel) && p.sigma2_floor_rel >= 0.0, LSGCPD_EINVAL, "bad sigma2_floor_rel");
    LSG_CHECK(isfinite(p.sigma2_init) && isfinite(p.tol), LSGCPD_EINVAL, "sigma2_init and tol must be finite");
    LSG_CHECK(!(p.eta >= 1.0) && !isnan(p.eta), LSGCPD_EINVAL, "eta must be < 1 (negative: off)");
    LSG_CHECK(p.group == 0 || p.group == 1, LSGCPD_EINVAL, "group must be 0 (SE(3)) or 1 (affine)");
    LSG_CHECK(pose_ok(R, p.group), LSGCPD_EINVAL,
              p.group ? "A0 must be finite with det A0 > 0" : "R0 is not a rotation matrix (to 1e-6)");
    LSG_CHECK(finite_vec(t, 3), LSGCPD_EINVAL, "t0 must be finite");
    return 0;
}
static RegParams reg_params(const lsgcpd_em_params& p, const TargetHeader& h, double V, int64_t M) {
    RegParams rp;
    memset(&rp, 0, sizeof(rp));
    rp.w = p.eta >= 0.0 ? 0.0 : p.w;
    rp.eta = p.eta >= 0.0 ? p.eta : -1.0;
    rp.spc = h.spc;
    rp.phi = p.d_src_conf;
    rp.V = V;
    rp.floor = p.sigma2_floor_rel * h.extent * h.extent;
    rp.tol = p.tol;
    rp.omega_ref_target = h.omega_ref;
    rp.M = M;
    rp.newton_max = p.newton_max;
    rp.consistent = p.consistent_normalizer ? 1 : 0;
    rp.max_iters = p.max_iters;
    rp.group = p.group;
    return rp;
}
}  // namespace lsg

LSG_EXPORT int lsgcpd_register(const void* d_target, int64_t M, double volume, const float* d_src_local,
                               int64_t N_local, const lsgcpd_em_params* params, const double R0[9], const double t0[3],
                               double R_out[9], double t_out[3], double* sigma2_out, int* iters_out,
                               double* nll_trace, double* sigma2_trace, void* comm, void* d_ws, size_t ws_bytes,
                               lsgcpd_stream_t stream) {
    lsgcpd_em_params p;
    lsgcpd_em_params_default(&p);
    if (params) p = *params;
    LSG_CHECK(d_target && d_src_local && d_ws && R_out && t_out && sigma2_out && iters_out, LSGCPD_EINVAL,
              "null pointer argument");
    LSG_CHECK(aligned16(d_target) && aligned16(d_ws), LSGCPD_EINVAL, "d_target and d_ws must be 16-byte aligned");
    LSG_CHECK(M >= 1 && N_local >= 1 && M < (int64_t)1 << 30 && N_local < (int64_t)1 << 34, LSGCPD_EINVAL,
              "M=%lld N_local=%lld out of range", (long long)M, (long long)N_local);
    double Rid[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1}, tid[3] = {0, 0, 0};
    const double* R = R0 ? R0 : Rid;
    const double* t = t0 ? t0 : tid;
    int rc0 = check_em_params(p, R, t);
    if (rc0) return rc0;
    cudaStream_t s = (cudaStream_t)stream;
    TargetHeader h;
    int rc = read_header(d_target, M, &h, s);
    if (rc) return rc;
    LSG_CHECK(p.consistent_normalizer || !h.prior, LSGCPD_EINVAL, "component priors require consistent_normalizer = 1");
    const double V = volume > 0.0 ? volume : h.volume;
    LSG_CHECK(isfinite(V) && V > 0.0, LSGCPD_EINVAL, "volume must be finite and > 0");
    RegLayout L;
    Sched sc;
    rc = reg_layout(h.M_pad, N_local, p.max_iters, &L, &sc);
    if (rc) return rc;
    LSG_CHECK(ws_bytes >= L.total, LSGCPD_EINVAL, "workspace too small (%zu < %zu)", ws_bytes, L.total);
    Comm* c = static_cast<Comm*>(comm);
    if (c) {
        rc = nccl_load();
        if (rc) return rc;
    }

    NvtxRange r("lsgcpd_register");
    char* ws = static_cast<char*>(d_ws);
    IterState* st = reinterpret_cast<IterState*>(ws + L.state);
    double* mom = reinterpret_cast<double*>(ws + L.mom);
    double* sums = reinterpret_cast<double*>(ws + L.sums);
    RegParams rp = reg_params(p, h, V, M);
    const float* d_src = d_src_local;
    rc = order_source(&d_src, &rp.phi, N_local, ws, L, s);
    if (rc) return rc;

    LSG_CUDA(cudaMemsetAsync(ws + L.counters, 0, sizeof(unsigned) * 8, s));
    LSG_CUDA(cudaMemsetAsync(ws + L.iters, 0, sizeof(int) * 4, s));
    LSG_CUDA(cudaMemsetAsync(ws + L.nll, 0, sizeof(double) * (p.max_iters + 1), s));
    LSG_CUDA(cudaMemsetAsync(ws + L.sig2, 0, sizeof(double) * (p.max_iters + 2), s));
    // initial pose, then σ²₀ (CPD closed form over all ranks' points)
    estep_launch_setup(st, d_target, R, t, 1.0, rp.w, V, M, rp.consistent, rp.eta, s);
    sigma2_sums_launch(d_src, N_local, st, d_target, reinterpret_cast<double*>(ws + L.blockpart), sums,
                       reinterpret_cast<unsigned*>(ws + L.counters), s);
    if (c) {
        const ncclResult_t r = g_nccl.AllReduce(sums, sums, 2, kNcclFloat64, kNcclSum, c->nc, s);
        if (r != 0) return nccl_fail(r, "ncclAllReduce(sigma2 sums)");
    }
    sigma2_init_launch(st, d_target, sums, rp, p.sigma2_init, reinterpret_cast<double*>(ws + L.sig2), mom + 75, s);
    LSG_CUDA(cudaGetLastError());

    // EM iterations: captured once into a CUDA graph and replayed (no host sync per iteration)
    NvtxRange rem("EM iterations");
    const Options& op = options();
    // With a communicator of more than one rank the iterations are launched directly (no stream capture of
    // ncclAllReduce): ≈ 6 launches per EM iteration against ≥ 10 ms of E step per rank on the scale config, and
    // no dependence on NCCL's graph-capture support on the multi-GPU path.
    const bool use_graph = p.max_iters > 1 && op.no_graph.load() != 1 && !(c && c->world > 1);
    if (use_graph) {
        // (not with a communicator: a destroyed and re-created comm could reuse the address)
        const bool cache = op.graph_cache.load() != 0 && c == nullptr;
        std::vector<unsigned char> key, topo;
        int dev = 0;
        LSG_CUDA(cudaGetDevice(&dev));
        const int nofuse = op.no_fuse.load() == 1 ? 1 : 0;
        key_put(topo, dev);
        key_put(topo, N_local);
        key_put(topo, sc);
        key_put(topo, rp.consistent);
        key_put(topo, nofuse);
        key = topo;
        key_put(key, d_target);
        key_put(key, d_src);
        key_put(key, ws);
        key_put(key, L);
        key_put(key, rp);
        GraphCache::Entry* hit = cache ? g_graphs.find(key, false) : nullptr;
        GraphRun* g = hit ? hit->run : nullptr;
        GraphRun local;
        if (!g) {
            // capture this call's iteration on a scratch stream of this thread
            LSG_CHECK(dev >= 0 && dev < GraphCache::kMaxDev, LSGCPD_ECUDA, "device ordinal %d out of range", dev);
            cudaStream_t& cap = g_graphs.cap[dev];
            if (!cap) LSG_CUDA(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
            LSG_CUDA(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
            cudaGraph_t graph = nullptr;
            rc = enqueue_iteration(d_target, d_src, N_local, ws, L, sc, rp, c, cap);
            cudaError_t ce = cudaStreamEndCapture(cap, &graph);
            if (rc || ce != cudaSuccess) {
                if (graph) cudaGraphDestroy(graph);
                return rc ? rc : cuda_fail(ce, "cudaStreamEndCapture");
            }
            GraphCache::Entry* same = cache ? g_graphs.find(topo, true) : nullptr;
            cudaGraphExecUpdateResultInfo info;
            if (same && cudaGraphExecUpdate(same->run->exec, graph, &info) == cudaSuccess) {
                // same launch shapes: the cached executable now carries this call's arguments
                cudaGraphDestroy(same->run->graph);
                same->run->graph = graph;
                same->key = key;
                g = same->run;
            } else {
                cudaGetLastError();   // a refused update is not an error: instantiate instead
                GraphRun* fresh = cache ? new GraphRun() : &local;
                fresh->graph = graph;
                ce = cudaStreamCreateWithFlags(&fresh->cs, cudaStreamNonBlocking);
                if (ce == cudaSuccess) ce = cudaEventCreateWithFlags(&fresh->ev, cudaEventDisableTiming);
                if (ce == cudaSuccess) ce = cudaGraphInstantiate(&fresh->exec, fresh->graph, 0);
                if (ce != cudaSuccess) {
                    if (fresh != &local) delete fresh;
                    return cuda_fail(ce, "graph instantiate");
                }
                if (cache) g_graphs.insert(key, topo, fresh);
                g = fresh;
            }
        }
        LSG_CUDA(cudaEventRecord(g->ev, s));
        LSG_CUDA(cudaStreamWaitEvent(g->cs, g->ev, 0));
        for (int k = 0; k < p.max_iters; ++k) LSG_CUDA(cudaGraphLaunch(g->exec, g->cs));
        LSG_CUDA(cudaEventRecord(g->ev, g->cs));
        LSG_CUDA(cudaStreamWaitEvent(s, g->ev, 0));
        LSG_CUDA(cudaStreamSynchronize(s));
    } else {
        for (int k = 0; k < p.max_iters; ++k) {
            rc = enqueue_iteration(d_target, d_src, N_local, ws, L, sc, rp, c, s);
            if (rc) return rc;
        }
        LSG_CUDA(cudaGetLastError());
    }

    IterState fin;
    int iters = 0;
    LSG_CUDA(cudaMemcpyAsync(&fin, st, sizeof(fin), cudaMemcpyDeviceToHost, s));
    LSG_CUDA(cudaMemcpyAsync(&iters, ws + L.iters, sizeof(int), cudaMemcpyDeviceToHost, s));
    if (nll_trace && p.max_iters > 0)
        LSG_CUDA(cudaMemcpyAsync(nll_trace, ws + L.nll, sizeof(double) * p.max_iters, cudaMemcpyDeviceToHost, s));
    if (sigma2_trace)
        LSG_CUDA(cudaMemcpyAsync(sigma2_trace, ws + L.sig2, sizeof(double) * (p.max_iters + 1), cudaMemcpyDeviceToHost,
                                 s));
    LSG_CUDA(cudaStreamSynchronize(s));
    LSG_CUDA(cudaGetLastError());
    for (int i = 0; i < 9; ++i) R_out[i] = fin.R[i];
    for (int i = 0; i < 3; ++i) t_out[i] = fin.t[i];
    *sigma2_out = fin.sigma2;
    *iters_out = iters;
    if (fin.status == LSGCPD_ENOMASS) {
        set_error("no inlier mass (sum P <= 1e-12 N) for 3 consecutive iterations");
        return LSGCPD_ENOMASS;
    }
    if (fin.status == LSGCPD_EINVAL) {
        set_error("non-finite coordinate in the source cloud");
        return LSGCPD_EINVAL;
    }
    return 0;
}

// The multi-GPU protocol of lsgcpd_register (source shards, replicated target, one 75-double all-reduce of the
// moments per EM iteration and one of the σ²₀ sums, Newton run redundantly per rank) with G shards on ONE
// device: every shard's E step, merge, moments and Newton are the kernels lsgcpd_register enqueues with a
// communicator; only the all-reduce is a fixed-order device sum (shard_allreduce_kernel).  Test support for
// SURVEY §8(c).6 step 4 on a one-GPU box; no graph capture.
LSG_EXPORT int lsgcpd_register_shards(const void* d_target, int64_t M, double volume, const float* const* h_d_src,
                                      const int64_t* h_N, int G, const lsgcpd_em_params* params, const double R0[9],
                                      const double t0[3], double* R_out, double* t_out, double* sigma2_out,
                                      int* iters_out, void* d_ws, size_t ws_stride, lsgcpd_stream_t stream) {
    lsgcpd_em_params p;
    lsgcpd_em_params_default(&p);
    if (params) p = *params;
    LSG_CHECK(d_target && h_d_src && h_N && d_ws && R_out && t_out && sigma2_out && iters_out, LSGCPD_EINVAL,
              "null pointer argument");
    LSG_CHECK(G >= 1 && G <= kMaxShards, LSGCPD_EINVAL, "G=%d out of range [1, %d]", G, kMaxShards);
    LSG_CHECK(aligned16(d_target) && aligned16(d_ws) && (ws_stride & 255) == 0, LSGCPD_EINVAL,
              "d_target and d_ws must be 16-byte aligned, ws_stride a multiple of 256");
    double Rid[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1}, tid[3] = {0, 0, 0};
    const double* R = R0 ? R0 : Rid;
    const double* t = t0 ? t0 : tid;
    int rc = check_em_params(p, R, t);
    if (rc) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    TargetHeader h;
    rc = read_header(d_target, M, &h, s);
    if (rc) return rc;
    LSG_CHECK(p.consistent_normalizer || !h.prior, LSGCPD_EINVAL, "component priors require consistent_normalizer = 1");
    LSG_CHECK(p.d_src_conf == nullptr, LSGCPD_EINVAL, "per-point confidences are not supported with shards");
    const double V = volume > 0.0 ? volume : h.volume;
    LSG_CHECK(isfinite(V) && V > 0.0, LSGCPD_EINVAL, "volume must be finite and > 0");
    const RegParams rp = reg_params(p, h, V, M);
    std::vector<RegLayout> L(G);
    std::vector<Sched> sc(G);
    std::vector<char*> ws(G);
    ShardPtrs mom{}, sums{};
    for (int g = 0; g < G; ++g) {
        LSG_CHECK(h_d_src[g] && h_N[g] >= 1 && h_N[g] < (int64_t)1 << 34, LSGCPD_EINVAL, "shard %d: bad source", g);
        rc = reg_layout(h.M_pad, h_N[g], p.max_iters, &L[g], &sc[g]);
        if (rc) return rc;
        LSG_CHECK(ws_stride >= L[g].total, LSGCPD_EINVAL, "ws_stride too small (%zu < %zu)", ws_stride, L[g].total);
        ws[g] = static_cast<char*>(d_ws) + (size_t)g * ws_stride;
        mom.p[g] = reinterpret_cast<double*>(ws[g] + L[g].mom);
        sums.p[g] = reinterpret_cast<double*>(ws[g] + L[g].sums);
    }
    NvtxRange r("lsgcpd_register_shards");
    std::vector<const float*> src(G);
    for (int g = 0; g < G; ++g) {   // each shard in Morton order, as lsgcpd_register orders its source
        src[g] = h_d_src[g];
        const float* no_phi = nullptr;
        rc = order_source(&src[g], &no_phi, h_N[g], ws[g], L[g], s);
        if (rc) return rc;
    }
    for (int g = 0; g < G; ++g) {
        char* w = ws[g];
        LSG_CUDA(cudaMemsetAsync(w + L[g].counters, 0, sizeof(unsigned) * 8, s));
        LSG_CUDA(cudaMemsetAsync(w + L[g].iters, 0, sizeof(int) * 4, s));
        LSG_CUDA(cudaMemsetAsync(w + L[g].nll, 0, sizeof(double) * (p.max_iters + 1), s));
        LSG_CUDA(cudaMemsetAsync(w + L[g].sig2, 0, sizeof(double) * (p.max_iters + 2), s));
        estep_launch_setup(reinterpret_cast<IterState*>(w + L[g].state), d_target, R, t, 1.0, rp.w, V, M,
                           rp.consistent, rp.eta, s);
        sigma2_sums_launch(src[g], h_N[g], reinterpret_cast<IterState*>(w + L[g].state), d_target,
                           reinterpret_cast<double*>(w + L[g].blockpart), sums.p[g],
                           reinterpret_cast<unsigned*>(w + L[g].counters), s);
    }
    shard_allreduce_kernel<<<1, 32, 0, s>>>(sums, G, 2);
    for (int g = 0; g < G; ++g)
        sigma2_init_launch(reinterpret_cast<IterState*>(ws[g] + L[g].state), d_target, sums.p[g], rp, p.sigma2_init,
                           reinterpret_cast<double*>(ws[g] + L[g].sig2), mom.p[g] + 75, s);
    LSG_CUDA(cudaGetLastError());
    for (int k = 0; k < p.max_iters; ++k) {
        for (int g = 0; g < G; ++g) {
            rc = enqueue_moments(d_target, src[g], h_N[g], ws[g], L[g], sc[g], rp, false, s);
            if (rc) return rc;
        }
        shard_allreduce_kernel<<<(kMomentCount + 127) / 128, 128, 0, s>>>(mom, G, kMomentCount);
        for (int g = 0; g < G; ++g) enqueue_newton(ws[g], L[g], rp, s);
    }
    LSG_CUDA(cudaGetLastError());
    std::vector<IterState> fin(G);
    for (int g = 0; g < G; ++g) {
        LSG_CUDA(cudaMemcpyAsync(&fin[g], ws[g] + L[g].state, sizeof(IterState), cudaMemcpyDeviceToHost, s));
        LSG_CUDA(cudaMemcpyAsync(iters_out + g, ws[g] + L[g].iters, sizeof(int), cudaMemcpyDeviceToHost, s));
    }
    LSG_CUDA(cudaStreamSynchronize(s));
    int status = 0;
    for (int g = 0; g < G; ++g) {
        for (int i = 0; i < 9; ++i) R_out[9 * g + i] = fin[g].R[i];
        for (int i = 0; i < 3; ++i) t_out[3 * g + i] = fin[g].t[i];
        sigma2_out[g] = fin[g].sigma2;
        if (fin[g].status) status = fin[g].status;
    }
    if (status == LSGCPD_ENOMASS) {
        set_error("no inlier mass (sum P <= 1e-12 N) for 3 consecutive iterations");
        return LSGCPD_ENOMASS;
    }
    if (status == LSGCPD_EINVAL) {
        set_error("non-finite coordinate in the source cloud");
        return LSGCPD_EINVAL;
    }
    return 0;
}

// Run-time options (diagnostics and tests); see include/lsgcpd.h.
LSG_EXPORT int lsgcpd_set_option(const char* name, double value) {
    LSG_CHECK(name && isfinite(value), LSGCPD_EINVAL, "bad option name or value");
    Options& o = options();
    const int iv = (int)value;
    if (!strcmp(name, "tc")) {
        LSG_CHECK(iv >= 0 && iv <= 2, LSGCPD_EINVAL, "tc must be 0, 1 or 2");
        o.tc.store(iv);
    } else if (!strcmp(name, "estep_variant")) {
        LSG_CHECK(iv >= -1 && iv <= 2, LSGCPD_EINVAL, "estep_variant must be -1..2");
        o.estep_variant.store(iv);
    } else if (!strcmp(name, "halves")) {
        o.halves.store(iv);
    } else if (!strcmp(name, "no_fuse")) {
        o.no_fuse.store(iv);
    } else if (!strcmp(name, "graph_cache")) {
        o.graph_cache.store(iv);
    } else if (!strcmp(name, "no_graph")) {
        o.no_graph.store(iv);
    } else if (!strcmp(name, "tile_gate")) {
        o.tile_gate.store((float)value);
    } else if (!strcmp(name, "far_rule")) {
        o.far_rule.store(iv ? 1 : 0);
    } else if (!strcmp(name, "sort_source")) {
        o.sort_source.store(iv ? 1 : 0);
    } else {
        set_error("unknown option '%s'", name);
        return LSGCPD_EINVAL;
    }
    return 0;
}

LSG_EXPORT int lsgcpd_get_option(const char* name, double* value) {
    LSG_CHECK(name && value, LSGCPD_EINVAL, "null pointer argument");
    const Options& o = options();
    if (!strcmp(name, "tc")) *value = o.tc.load();
    else if (!strcmp(name, "estep_variant")) *value = o.estep_variant.load();
    else if (!strcmp(name, "halves")) *value = o.halves.load();
    else if (!strcmp(name, "no_fuse")) *value = o.no_fuse.load();
    else if (!strcmp(name, "graph_cache")) *value = o.graph_cache.load();
    else if (!strcmp(name, "no_graph")) *value = o.no_graph.load();
    else if (!strcmp(name, "tile_gate")) *value = o.tile_gate.load();
    else if (!strcmp(name, "far_rule")) *value = o.far_rule.load();
    else if (!strcmp(name, "sort_source")) *value = o.sort_source.load();
    else {
        set_error("unknown option '%s'", name);
        return LSGCPD_EINVAL;
    }
    return 0;
}

LSG_EXPORT size_t lsgcpd_target_prior_workspace_bytes(int64_t M) {
    if (M < 1) return 0;
    return prior_ws_bytes(M);
}

LSG_EXPORT int lsgcpd_target_set_prior(void* d_target, int64_t M, const float* d_phi, void* d_ws, size_t ws_bytes,
                                       double* h_spc, lsgcpd_stream_t stream) {
    LSG_CHECK(d_target && d_phi && d_ws, LSGCPD_EINVAL, "null pointer argument");
    LSG_CHECK(aligned16(d_target), LSGCPD_EINVAL, "d_target must be 16-byte aligned");
    LSG_CHECK(M >= 1 && M < (int64_t)1 << 30, LSGCPD_EINVAL, "M=%lld out of range", (long long)M);
    LSG_CHECK(ws_bytes >= prior_ws_bytes(M), LSGCPD_EINVAL, "workspace too small (%zu < %zu)", ws_bytes,
              prior_ws_bytes(M));
    cudaStream_t s = (cudaStream_t)stream;
    TargetHeader h;
    int rc = read_header(d_target, M, &h, s);
    if (rc) return rc;
    return set_prior_impl(d_target, M, d_phi, d_ws, h_spc, s);
}

LSG_EXPORT size_t lsgcpd_select_workspace_bytes(int64_t n) {
    if (n < 1 || n >= (int64_t)1 << 31) return 0;
    return select_ws_bytes(n);
}

LSG_EXPORT int lsgcpd_select_confident(const float* d_xyz, const float* d_phi, int64_t n, float threshold,
                                       float* d_xyz_out, float* d_phi_out, int64_t* h_n_out, void* d_ws,
                                       size_t ws_bytes, lsgcpd_stream_t stream) {
    LSG_CHECK(d_xyz && d_phi && d_xyz_out && h_n_out && d_ws, LSGCPD_EINVAL, "null pointer argument");
    LSG_CHECK(n >= 1 && n < (int64_t)1 << 31, LSGCPD_EINVAL, "n=%lld out of range", (long long)n);
    LSG_CHECK(isfinite(threshold), LSGCPD_EINVAL, "threshold must be finite");
    LSG_CHECK(aligned16(d_ws), LSGCPD_EINVAL, "d_ws must be 16-byte aligned");
    LSG_CHECK(ws_bytes >= select_ws_bytes(n), LSGCPD_EINVAL, "workspace too small (%zu < %zu)", ws_bytes,
              select_ws_bytes(n));
    return select_confident_impl(d_xyz, d_phi, n, threshold, d_xyz_out, d_phi_out, h_n_out, d_ws,
                                 (cudaStream_t)stream);
}

LSG_EXPORT int lsgcpd_depth_confidence(const float* d_xyz, int64_t n, double c0, double c1, double z_min,
                                       float* d_phi, lsgcpd_stream_t stream) {
    LSG_CHECK(d_xyz && d_phi, LSGCPD_EINVAL, "null pointer argument");
    LSG_CHECK(n >= 1, LSGCPD_EINVAL, "n must be >= 1");
    LSG_CHECK(isfinite(c0) && isfinite(c1) && isfinite(z_min) && c0 >= 0.0 && c1 >= 0.0 &&
                  c0 + c1 * z_min * z_min > 0.0,
              LSGCPD_EINVAL, "error model must have c0, c1 >= 0 and e(z_min) > 0");
    depth_confidence_launch(d_xyz, n, c0, c1, z_min, d_phi, (cudaStream_t)stream);
    LSG_CUDA(cudaGetLastError());
    return 0;
}

// ---------------------------------------------------------------------------------------------
// Batched registrations
// ---------------------------------------------------------------------------------------------
namespace lsg {
struct BatchLayout {
    size_t desc, st, mom, bpart, ctr, nll, sig2, iters, err, part, rec, total;
    int64_t units, nblk_tot, pts, kmax;
    Sched sc;
};

static int batch_layout(const lsgcpd_problem* P, int B, int max_iters, BatchLayout* L, std::vector<BatchProblem>* out,
                        int group = 0) {
    LSG_CHECK(P && B >= 1 && B <= (1 << 20), LSGCPD_EINVAL, "bad problem list (B=%d)", B);
    LSG_CHECK(max_iters >= 0 && max_iters <= 100000, LSGCPD_EINVAL, "max_iters out of range");
    const int64_t kB = batch_block_points();
    std::vector<BatchProblem> bp(B);
    int64_t units = 0, pts = 0, nblk_tot = 0;
    for (int b = 0; b < B; ++b) {
        const lsgcpd_problem& p = P[b];
        LSG_CHECK(p.d_target && p.d_src, LSGCPD_EINVAL, "problem %d: null pointer", b);
        LSG_CHECK(aligned16(p.d_target), LSGCPD_EINVAL, "problem %d: d_target must be 16-byte aligned", b);
        LSG_CHECK(p.M >= 1 && p.N >= 1 && p.M < (int64_t)1 << 30 && p.N < (int64_t)1 << 30, LSGCPD_EINVAL,
                  "problem %d: M=%lld N=%lld out of range", b, (long long)p.M, (long long)p.N);
        LSG_CHECK(pose_ok(p.R0, group) && finite_vec(p.t0, 3), LSGCPD_EINVAL, "problem %d: bad initial pose", b);
        LSG_CHECK(isfinite(p.volume), LSGCPD_EINVAL, "problem %d: volume must be finite", b);
        BatchProblem& q = bp[b];
        memset(&q, 0, sizeof(q));
        const int64_t M_pad = pad_targets(p.M);
        q.target = p.d_target;
        q.body = target_body(p.d_target);
        q.tc = reinterpret_cast<const char*>(target_tc(p.d_target, M_pad));
        q.src = p.d_src;
        q.conf = p.d_src_conf;
        q.M = p.M;
        q.N = p.N;
        q.T = M_pad / kTT_host;
        q.nblk = (p.N + kB - 1) / kB;
        q.unit0 = units;
        q.pt0 = pts;
        q.volume = p.volume;
        for (int i = 0; i < 9; ++i) q.R0[i] = p.R0[i];
        for (int i = 0; i < 3; ++i) q.t0[i] = p.t0[i];
        units += q.nblk * q.T;
        pts += p.N;
        nblk_tot += q.nblk;
    }
    int dev, nsm;
    LSG_CUDA(cudaGetDevice(&dev));
    LSG_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    Sched sc;
    memset(&sc, 0, sizeof(sc));
    sc.halves = 1;
    sc.gate_g = options().tile_gate.load();
    sc.far_rule = options().far_rule.load() ? 1 : 0;
    sc.U = units;
    const int64_t slots = (int64_t)nsm;       // one CTA per SM (both batched E-step kernels)
    sc.G = units < slots ? units : slots;
    sc.B = kB;
    int64_t kmax = 1;
    for (int b = 0; b < B; ++b)
        for (int64_t j = 0; j < bp[b].nblk; ++j) {
            const int64_t k = sched_owner(sc, bp[b].unit0 + (j + 1) * bp[b].T - 1) -
                              sched_owner(sc, bp[b].unit0 + j * bp[b].T) + 1;
            if (k > kmax) kmax = k;
        }
    sc.kmax = kmax;
    int64_t part0 = 0;
    for (int b = 0; b < B; ++b) {
        bp[b].part0 = part0;
        part0 += (int64_t)batch_partial_floats(bp[b].nblk, kmax);
    }
    size_t o = 0;
    L->desc = o; o += al(sizeof(BatchProblem) * B);
    L->st = o; o += al(sizeof(IterState) * B);
    L->mom = o; o += al(sizeof(double) * kBatchMom * B);
    L->bpart = o; o += al(sizeof(double) * 80 * B);
    L->ctr = o; o += al(sizeof(unsigned) * B);
    L->nll = o; o += al(sizeof(double) * (max_iters + 1) * B);
    L->sig2 = o; o += al(sizeof(double) * (max_iters + 2) * B);
    L->iters = o; o += al(sizeof(int) * B);
    L->err = o; o += al(sizeof(int) * B);
    L->part = o; o += al(sizeof(float) * (size_t)part0);
    L->rec = o; o += al(sizeof(float) * LSGCPD_REC * (size_t)pts);
    L->total = o;
    L->units = units;
    L->nblk_tot = nblk_tot;
    L->pts = pts;
    L->kmax = kmax;
    L->sc = sc;
    if (out) out->swap(bp);
    return 0;
}
}  // namespace lsg

LSG_EXPORT size_t lsgcpd_register_batch_workspace_bytes(const lsgcpd_problem* h_problems, int B, int max_iters) {
    BatchLayout L;
    if (batch_layout(h_problems, B, max_iters, &L, nullptr)) return 0;
    return L.total;
}

LSG_EXPORT int lsgcpd_register_batch(const lsgcpd_problem* h_problems, int B, const lsgcpd_em_params* params,
                                     double* R_out, double* t_out, double* sigma2_out, int* iters_out, int* status_out,
                                     void* d_ws, size_t ws_bytes, lsgcpd_stream_t stream) {
    lsgcpd_em_params p;
    lsgcpd_em_params_default(&p);
    if (params) p = *params;
    LSG_CHECK(R_out && t_out && sigma2_out && iters_out && status_out && d_ws, LSGCPD_EINVAL, "null pointer argument");
    LSG_CHECK(aligned16(d_ws), LSGCPD_EINVAL, "d_ws must be 16-byte aligned");
    LSG_CHECK(isfinite(p.w) && p.w >= 0.0 && p.w < 1.0, LSGCPD_EINVAL, "w must be in [0, 1)");
    LSG_CHECK(!(p.eta >= 1.0) && !isnan(p.eta), LSGCPD_EINVAL, "eta must be < 1 (negative: off)");
    LSG_CHECK(p.newton_max >= 0 && p.newton_max <= 1000, LSGCPD_EINVAL, "newton_max out of range");
    LSG_CHECK(isfinite(p.sigma2_floor_rel) && p.sigma2_floor_rel >= 0.0, LSGCPD_EINVAL, "bad sigma2_floor_rel");
    LSG_CHECK(isfinite(p.sigma2_init) && isfinite(p.tol), LSGCPD_EINVAL, "sigma2_init and tol must be finite");
    LSG_CHECK(p.group == 0 || p.group == 1, LSGCPD_EINVAL, "group must be 0 (SE(3)) or 1 (affine)");
    BatchLayout L;
    std::vector<BatchProblem> bp;
    int rc = batch_layout(h_problems, B, p.max_iters, &L, &bp, p.group);
    if (rc) return rc;
    LSG_CHECK(ws_bytes >= L.total, LSGCPD_EINVAL, "workspace too small (%zu < %zu)", ws_bytes, L.total);
    cudaStream_t s = (cudaStream_t)stream;
    NvtxRange r("lsgcpd_register_batch");
    char* ws = static_cast<char*>(d_ws);
    BatchProblem* dbp = reinterpret_cast<BatchProblem*>(ws + L.desc);
    IterState* st = reinterpret_cast<IterState*>(ws + L.st);
    double* mom = reinterpret_cast<double*>(ws + L.mom);
    int* err = reinterpret_cast<int*>(ws + L.err);
    LSG_CUDA(cudaMemcpyAsync(dbp, bp.data(), sizeof(BatchProblem) * B, cudaMemcpyHostToDevice, s));
    const int consistent = p.consistent_normalizer ? 1 : 0;
    batch_fill_launch(dbp, B, consistent, err, s);
    std::vector<int> herr(B);
    LSG_CUDA(cudaMemcpyAsync(herr.data(), err, sizeof(int) * B, cudaMemcpyDeviceToHost, s));
    LSG_CUDA(cudaStreamSynchronize(s));
    for (int b = 0; b < B; ++b) {
        LSG_CHECK(herr[b] != 1, LSGCPD_EINVAL, "problem %d: d_target is not a prepared target with M=%lld", b,
                  (long long)bp[b].M);
        LSG_CHECK(herr[b] != 2, LSGCPD_EINVAL, "problem %d: component priors require consistent_normalizer = 1", b);
    }
    RegParams rp;
    memset(&rp, 0, sizeof(rp));
    rp.w = p.eta >= 0.0 ? 0.0 : p.w;
    rp.eta = p.eta >= 0.0 ? p.eta : -1.0;
    rp.floor = p.sigma2_floor_rel;   // relative: scaled by each problem's extent² on the device
    rp.tol = p.tol;
    rp.newton_max = p.newton_max;
    rp.consistent = consistent;
    rp.max_iters = p.max_iters;
    rp.group = p.group;
    LSG_CUDA(cudaMemsetAsync(ws + L.iters, 0, sizeof(int) * B, s));
    LSG_CUDA(cudaMemsetAsync(ws + L.nll, 0, sizeof(double) * (p.max_iters + 1) * B, s));
    init_batch_launch(dbp, B, st, rp, p.sigma2_init, mom, reinterpret_cast<double*>(ws + L.sig2), s);
    LSG_CUDA(cudaGetLastError());
    float* part = reinterpret_cast<float*>(ws + L.part);
    float* rec = reinterpret_cast<float*>(ws + L.rec);
    auto enqueue = [&](cudaStream_t q) {
        estep_batch_launch(dbp, B, L.sc, st, part, rec, L.pts, consistent, q);
        moments_batch_launch(dbp, B, rec, st, reinterpret_cast<double*>(ws + L.bpart), mom,
                             reinterpret_cast<unsigned*>(ws + L.ctr), q);
        newton_batch_launch(dbp, B, st, mom, rp, reinterpret_cast<double*>(ws + L.nll),
                            reinterpret_cast<double*>(ws + L.sig2), reinterpret_cast<int*>(ws + L.iters), q);
    };
    if (p.max_iters > 0) {
        GraphRun g;
        LSG_CUDA(cudaStreamCreateWithFlags(&g.cs, cudaStreamNonBlocking));
        LSG_CUDA(cudaEventCreateWithFlags(&g.ev, cudaEventDisableTiming));
        LSG_CUDA(cudaEventRecord(g.ev, s));
        LSG_CUDA(cudaStreamWaitEvent(g.cs, g.ev, 0));
        LSG_CUDA(cudaStreamBeginCapture(g.cs, cudaStreamCaptureModeThreadLocal));
        enqueue(g.cs);
        cudaError_t ce = cudaStreamEndCapture(g.cs, &g.graph);
        if (ce != cudaSuccess) return cuda_fail(ce, "cudaStreamEndCapture");
        LSG_CUDA(cudaGraphInstantiate(&g.exec, g.graph, 0));
        for (int k = 0; k < p.max_iters; ++k) LSG_CUDA(cudaGraphLaunch(g.exec, g.cs));
        LSG_CUDA(cudaEventRecord(g.ev, g.cs));
        LSG_CUDA(cudaStreamWaitEvent(s, g.ev, 0));
        LSG_CUDA(cudaStreamSynchronize(s));
    }
    std::vector<IterState> fin(B);
    LSG_CUDA(cudaMemcpyAsync(fin.data(), st, sizeof(IterState) * B, cudaMemcpyDeviceToHost, s));
    LSG_CUDA(cudaMemcpyAsync(iters_out, ws + L.iters, sizeof(int) * B, cudaMemcpyDeviceToHost, s));
    LSG_CUDA(cudaStreamSynchronize(s));
    LSG_CUDA(cudaGetLastError());
    for (int b = 0; b < B; ++b) {
        for (int i = 0; i < 9; ++i) R_out[9 * b + i] = fin[b].R[i];
        for (int i = 0; i < 3; ++i) t_out[3 * b + i] = fin[b].t[i];
        sigma2_out[b] = fin[b].sigma2;
        status_out[b] = (fin[b].status == LSGCPD_ENOMASS || fin[b].status == LSGCPD_EINVAL) ? fin[b].status : 0;
    }
    return 0;
}
