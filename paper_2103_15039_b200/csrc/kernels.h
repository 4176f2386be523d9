// Host-side launchers shared between the translation units of liblsgcpd.so.
#pragma once
#include <atomic>

#include "common.cuh"

namespace lsg {

// Run-time knobs (diagnostics and tests; the defaults are the product configuration).  Initialised once from
// the environment (LSGCPD_TC, LSGCPD_ESTEP_VARIANT, LSGCPD_HALVES, LSGCPD_NO_FUSE, LSGCPD_GRAPH_CACHE,
// LSGCPD_NO_GRAPH, LSGCPD_TILE_GATE, LSGCPD_FAR_RULE, LSGCPD_SORT_SOURCE); lsgcpd_set_option changes them.  Atomic: calls on other threads see a
// consistent value per field.
constexpr float kDefaultTileGate = 24.f;   // E_tile ≤ gate·σ → tile-centred residual
struct Options {
    std::atomic<int> tc;              // 0 CUDA cores only, 1 tensor cores forced, 2 automatic
    std::atomic<int> estep_variant;   // -1 automatic, else the CUDA-core configuration (estep.cu)
    std::atomic<int> halves;          // 0 automatic, 1 one sweep over the target
    std::atomic<int> no_fuse;         // 1: separate merge / moments kernels instead of em_tail_kernel
    std::atomic<int> graph_cache;     // 0: no cached EM-iteration graphs
    std::atomic<int> no_graph;        // 1: plain launches instead of a captured EM iteration
    std::atomic<float> tile_gate;     // gate_g of Sched (≤ 0: hi/lo residual on every tile)
    std::atomic<int> far_rule;        // far_rule of Sched (0: the tile gate alone picks the residual)
    std::atomic<int> sort_source;     // 1: lsgcpd_register runs on a Morton-ordered copy of the source
    Options();
};
Options& options();

// Registration parameters passed by value to the device-side EM state machine.
struct RegParams {
    double w, V, floor, tol, omega_ref_target;
    double eta, spc;          // outlier ratio (< 0: use w) and the target's Σ π √(1+α) (Eq. 7)
    const float* phi;         // per-source-point confidences φ(x_n) (Eq. 8) or NULL
    int64_t M;
    int newton_max, consistent, max_iters;
    int group;                // 0: SE(3) (rigid, the paper's M step); 1: affine GA⁺(3)
};

// Batched registrations (NEXT-3): one descriptor per problem, in device memory.  Units of all problems
// are concatenated: problem b owns global units [unit0, unit0 + nblk·T), points [pt0, pt0 + N) of the
// concatenated record, and partial slots from part0 (floats).
struct BatchProblem {
    const void* target;        // prepared target (header + body + tensor-core section)
    const float* body;         // pair-interleaved body (CUDA-core E step)
    const char* tc;            // tensor-core section (tensor-core E step)
    const float* src;          // [N][3]
    const float* conf;         // optional φ(x_n) [N] or NULL
    int64_t M, N, T, nblk, unit0, pt0, part0;
    double volume, extent, omega_ref, spc;
    double R0[9], t0[3];
};
constexpr int kBatchMom = 80;   // doubles per problem in the moment array (75 moments + N at [75])

// batch.cu
int batch_block_points();
size_t batch_partial_floats(int64_t nblk, int64_t kmax);
void batch_fill_launch(BatchProblem* bp, int B, int consistent, int* err, cudaStream_t stream);
void estep_batch_launch(const BatchProblem* bp, int B, const Sched& sc, const IterState* st, float* part, float* rec,
                        int64_t Ntot, int consistent, cudaStream_t stream);
// mstep.cu (batched)
void moments_batch_launch(const BatchProblem* bp, int B, const float* rec, IterState* st, double* blockpart,
                          double* mom, unsigned* counters, cudaStream_t stream);
void newton_batch_launch(const BatchProblem* bp, int B, IterState* st, const double* mom, const RegParams& rp0,
                         double* nll_trace, double* sigma2_trace, int* iters_done, cudaStream_t stream);
void init_batch_launch(const BatchProblem* bp, int B, IterState* st, const RegParams& rp0, double sigma2_user,
                       double* mom, double* sigma2_trace, cudaStream_t stream);

// estep.cu
int sm_count();   // SM count of the current device (cached per device); 0 on a CUDA error
int estep_plan(int64_t M_pad, int64_t N, Sched* sc);
size_t estep_partial_bytes(const Sched& s);
void estep_launch_setup(IterState* st, const void* d_target, const double* R, const double* t, double sigma2,
                        double w, double V, int64_t M, int consistent, double eta, cudaStream_t stream);
// phi: optional per-source-point confidence φ(x_n) (Eq. 8: w_n = 1 - (1 - w0) φ(x_n)), NULL = uniform w0
int estep_launch(const void* d_target, const float* d_src, int64_t N, const IterState* st, const Sched& sc,
                 float* part, float* rec, int consistent, const float* phi, cudaStream_t stream, int merge = 1);

// mstep.cu
constexpr int kMomentCount = 75;          // G 60, U 12, σ²ΣD, ΣP, Σ ln p
constexpr int kMomentBlocks = 256;
void moments_launch(const float* rec, const float* src, int64_t N, const IterState* st, double* blockpart,
                    double* out, unsigned int* counter, cudaStream_t stream);
void sigma2_sums_launch(const float* src, int64_t N, const IterState* st, const void* d_target, double* blockpart,
                        double* out, unsigned int* counter, cudaStream_t stream);
void sigma2_init_launch(IterState* st, const void* d_target, const double* sums, const RegParams& rp,
                        double sigma2_user, double* sigma2_trace, double* ntot_out, cudaStream_t stream);
void newton_launch(IterState* st, const double* mom, const RegParams& rp, double* nll_trace, double* sigma2_trace,
                   int* iters_done, cudaStream_t stream);
// merge + moments (+ Newton/σ² when run_newton) in one launch after the pair kernels (estep_launch, merge = 0)
void em_tail_launch(const float* part, const float* src, int64_t N, IterState* st, const Sched& sc, const float* phi,
                    double* blockpart, double* mom, unsigned* counter, const RegParams& rp, double* nll_trace,
                    double* sigma2_trace, int* iters_done, int run_newton, cudaStream_t stream);
constexpr int64_t kTailMaxN = 1 << 17;   // above this the separate merge / moments grids are used

// target.cu
size_t prepare_ws_bytes(int64_t M);
size_t source_sort_ws_bytes(int64_t N);
int source_sort_launch(const float* src, const float* phi, int64_t N, float* out, float* phi_out, void* d_ws,
                       cudaStream_t stream);
size_t pack_ws_bytes(int64_t M);
int pack_target_impl(const float* d_xyz, const float* d_nrm, const float* d_alpha, int64_t M, double margin,
                     void* d_target, void* d_ws, lsgcpd_target_info* info, cudaStream_t stream);
size_t prior_ws_bytes(int64_t M);
int set_prior_impl(void* d_target, int64_t M, const float* d_phi, void* d_ws, double* h_spc, cudaStream_t stream);
size_t select_ws_bytes(int64_t n);
int select_confident_impl(const float* d_xyz, const float* d_phi, int64_t n, float threshold, float* d_xyz_out,
                          float* d_phi_out, int64_t* h_n_out, void* d_ws, cudaStream_t stream);
void depth_confidence_launch(const float* d_xyz, int64_t n, double c0, double c1, double z_min, float* d_phi,
                             cudaStream_t stream);
size_t prepare_batch_ws_bytes(const int64_t* M, int B);
int prepare_batch_impl(const float* const* xyz, const int64_t* M, int B, const lsgcpd_prep_params& p,
                       void* const* targets, void* d_ws, lsgcpd_target_info* info, cudaStream_t stream);
int prepare_target_impl(const float* d_xyz, int64_t M, const lsgcpd_prep_params& p, void* d_target, void* d_ws,
                        lsgcpd_target_info* info, const lsgcpd_annotations* ann, cudaStream_t stream);

}  // namespace lsg
