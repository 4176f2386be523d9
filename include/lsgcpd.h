/*
 * lsgcpd.h — C ABI of the B200-native LSG-CPD library (liblsgcpd.so).
 *
 * LSG-CPD: Coherent Point Drift with Local Surface Geometry (arXiv 2103.15039).
 * Citations "P:<line>" refer to the paper's LaTeX source; see DESIGN.md.
 *
 * Conventions for every entry point
 *   - d_* pointers are DEVICE pointers owned by the caller (e.g. torch tensors); h_* / plain
 *     pointers to double arrays are HOST pointers.  The library allocates no device memory:
 *     scratch space is the caller-provided workspace sized by the matching *_bytes() query.
 *   - Point clouds are row-major float32 [count][3] (x, y, z), 4-byte aligned.
 *   - Rotations are row-major double[9]; translations double[3]; a pose g = (R, t) acts as
 *     g(x) = R x + t.
 *   - Return value: 0 on success, a negative LSGCPD_E* code otherwise; lsgcpd_last_error()
 *     returns a thread-local message describing the last failure on the calling thread.
 *   - "async" calls only enqueue work on `stream`; "sync" calls return after the stream work
 *     they issued has completed.
 *   - No entry point reads or writes memory outside the documented buffers.
 */
#ifndef LSGCPD_H_
#define LSGCPD_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* lsgcpd_stream_t; /* == cudaStream_t; NULL = legacy default stream */

#define LSGCPD_OK 0
#define LSGCPD_EINVAL (-1)      /* bad argument: null pointer, size, non-finite value, ws too small */
#define LSGCPD_EDEGENERATE (-2) /* degenerate target (fewer than 3 points, zero-volume box) */
#define LSGCPD_ECUDA (-3)       /* a CUDA runtime error (message in lsgcpd_last_error) */
#define LSGCPD_ENCCL (-4)       /* NCCL unavailable or failed */
#define LSGCPD_ENOMASS (-5)     /* Σ_mn P_mn ≤ 1e-12·N for 3 consecutive EM iterations */

/* Per-source-point E-step record: LSGCPD_REC floats per point, row-major [N][16].
 * P_mn is the posterior of Eq. 5 at the E-step pose, x̂_n = R x_n + t.          */
#define LSGCPD_REC 16
enum {
    LSGCPD_REC_P = 0,       /* Σ_m P_mn                                                      */
    LSGCPD_REC_PY = 1,      /* [1..3]  Σ_m P_mn y_m                                          */
    LSGCPD_REC_A = 4,       /* [4..9]  Σ_m P_mn α_m n_m n_mᵀ   (xx, xy, xz, yy, yz, zz)      */
    LSGCPD_REC_B = 10,      /* [10..12] Σ_m P_mn α_m (n_m·y_m) n_m                           */
    LSGCPD_REC_D = 13,      /* Σ_m P_mn d_mn, d_mn = (x̂_n-y_m)ᵀ(α_m n_m n_mᵀ+I)(x̂_n-y_m)/σ² */
    LSGCPD_REC_LNP = 14,    /* ln p(x̂_n), Eq. 1 density; NLL = -Σ_n (Eq. 4)     */
    LSGCPD_REC_POUT = 15    /* outlier posterior w p_o / p(x̂_n); Σ_m P_mn + P_out = 1       */
};

/* Target preparation parameters (defaults are readings R8-R9 in DESIGN.md). */
typedef struct {
    float alpha_max;      /* α_max of Eq. 3 (default 50)                                     */
    float lambda;         /* λ of Eq. 3 (default 0.5)                                         */
    int knn_k;            /* neighbourhood size k, self included (default 10; 3 ≤ k ≤ 32)    */
    double volume_margin; /* V = Π_a extent_a (1 + 2·margin)  (default 0.1, R5)   */
} lsgcpd_prep_params;

/* Host-side summary returned by prepare/pack. */
typedef struct {
    double volume;        /* V of the uniform outlier density p_o = 1/V          */
    double extent;        /* diagonal of the target's axis-aligned bounding box              */
    double aabb_lo[3], aabb_hi[3];
    double alpha_mean;    /* mean α_m (the ᾱ of Fig. 3(d))                        */
    int64_t n_degenerate; /* targets whose k neighbours all coincide (κ = 1/3, n = (0,0,1))  */
} lsgcpd_target_info;

/* Optional per-target annotations written by lsgcpd_prepare_target (each pointer may be NULL). */
typedef struct {
    float* d_normals;     /* [M][3] unit normal n_m (eigenvector of λ_min), sign unspecified */
    float* d_kappa;       /* [M] surface variation κ_m ∈ [1e-12, 1/3]            */
    float* d_alpha;       /* [M] α_m of Eq. 3                                                */
    int32_t* d_knn;       /* [M][k] neighbour ids, ascending distance, ties → lower id       */
} lsgcpd_annotations;

/* EM parameters (§3.5). */
typedef struct {
    double w;                  /* uniform outlier weight w ∈ [0, 1); 0 = no outlier term */
    int max_iters;             /* EM iterations (fixed count unless tol > 0)                     */
    int newton_max;            /* Newton iterations per M step (default 10, reading R13)         */
    int consistent_normalizer; /* 1: c_m ∝ sqrt(1+α_m) of Eq. 2; 0: Eq. 9-10 literal (R1)      */
    double sigma2_init;        /* ≤ 0: CPD closed form Σ_mn||x̂_n-y_m||²/(3MN) (R7)  */
    double sigma2_floor_rel;   /* σ² ≥ sigma2_floor_rel · extent² (default 1e-12, R16)           */
    double tol;                /* > 0: stop when |Δσ²|/σ² < tol and the pose step < tol          */
    /* Model extensions (§3.2-3.3).  Defaults (eta < 0, NULL) reproduce the uniform model above.   */
    double eta;                /* outlier ratio η ∈ [0,1): w0 = w_max(η) = ηVΣπc/((1-η)+ηVΣπc)     */
                               /* (Eq. 7), re-evaluated from σ² at every E step (reading    */
                               /* R22); w is then ignored.  < 0: use w.                            */
    const float* d_src_conf;   /* DEVICE [N] source confidences φ(x_n) ∈ [0,1] (Eq. 8):  */
                               /* w_n = 1 - (1 - w0) φ(x_n); NULL: w_n = w0 for every point          */
    int group;                 /* transformation group of the M step: 0 = SE(3) rigid   */
                               /* (default); 1 = affine GA⁺(3), basis e_i e_jᵀ (9) + translations   */
                               /* (3), reading R24.  With 1, "R" is the linear part A (det A > 0).   */
} lsgcpd_em_params;

/* Library identity. */
int lsgcpd_version(void);                 /* MAJOR*10000 + MINOR*100 + PATCH                */
const char* lsgcpd_last_error(void);      /* thread-local; never NULL                         */

/* ---------------------------------------------------------------------------------------
 * Target model.  The prepared target is an opaque device buffer of lsgcpd_target_bytes(M)
 * bytes (16-byte aligned, caller-owned) holding, per target m, y_m, √α_m n_m, α_m n_m n_mᵀ,
 * α_m (n_m·y_m) n_m and the log-determinant weight ½log2(1+α_m), plus a small header.  The
 * targets are stored in a spatial (Morton) order with per-tile centres (the E step's
 * precision device); every result is a sum over targets and does not depend on
 * that order.  Layout 2 (ABI 1.3): a target prepared by an older library is refused (EINVAL).
 * ------------------------------------------------------------------------------------- */
size_t lsgcpd_target_bytes(int64_t M);
size_t lsgcpd_prepare_workspace_bytes(int64_t M, int knn_k);

/* Build the target GMM from raw points: exact kNN (k, self included) → centred
 * scatter → FP64 symmetric eigen-decomposition → n_m, κ_m (clamped to [1e-12, 1/3]) →
 * α_m (Eq. 3) → pack; V and extent from the AABB.  sync.
 * Errors: EINVAL (null, M < 3, k ∉ [3, 32], k > M, non-finite coordinate, ws too small),
 * EDEGENERATE (all points identical), ECUDA. */
int lsgcpd_prepare_target(const float* d_xyz, int64_t M, const lsgcpd_prep_params* params,
                          void* d_target, void* d_ws, size_t ws_bytes,
                          lsgcpd_target_info* h_info, const lsgcpd_annotations* annotations,
                          lsgcpd_stream_t stream);

/* B targets in one call (many small registrations, §8(f) NEXT-3): byte for byte the targets of B calls of
 * lsgcpd_prepare_target (no annotations), with two host synchronisations in all instead of two per
 * target; every stage runs once per wave of up to 64 targets.  h_d_xyz[b] / h_d_target[b]: HOST arrays of
 * B DEVICE pointers (cloud b [M_b][3], target b of lsgcpd_target_bytes(M_b) bytes); h_M: HOST [B];
 * h_info: HOST [B] or NULL.  One workspace of lsgcpd_prepare_batch_workspace_bytes() bytes serves all
 * targets: about 512 MB of per-target regions for a wave plus O(B) bookkeeping (smaller for few targets).
 * sync.
 * Errors: as lsgcpd_prepare_target, the message naming the problem; EINVAL also for B < 1. */
size_t lsgcpd_prepare_batch_workspace_bytes(const int64_t* h_M, int B, int knn_k);
int lsgcpd_prepare_batch(const float* const* h_d_xyz, const int64_t* h_M, int B,
                         const lsgcpd_prep_params* params, void* const* h_d_target, void* d_ws,
                         size_t ws_bytes, lsgcpd_target_info* h_info, lsgcpd_stream_t stream);

/* Pack a target from caller-supplied normals and α (e.g. an oracle's or a sensor's), no kNN.
 * d_normals [M][3] (normalised to unit length by the pack; a zero or non-finite normal makes
 * component m isotropic, α_m := 0), d_alpha [M] (α_m ≥ 0).  sync (returns h_info).
 * Errors: EINVAL (null, M < 1, negative or non-finite α, ws too small), ECUDA. */
size_t lsgcpd_pack_workspace_bytes(int64_t M);
int lsgcpd_pack_target(const float* d_xyz, const float* d_normals, const float* d_alpha, int64_t M,
                       double volume_margin, void* d_target, void* d_ws, size_t ws_bytes,
                       lsgcpd_target_info* h_info, lsgcpd_stream_t stream);

/* ---------------------------------------------------------------------------------------
 * E step: for every source point x_n, against every target m,
 *   d_mn = ((x̂_n-y_m)ᵀ(x̂_n-y_m) + α_m (n_m·(x̂_n-y_m))²)/σ²,
 *   P_mn = (1-w)/M c_m e^{-d_mn/2} / (w/V + (1-w)/M Σ_k c_k e^{-d_kn/2}),
 * reduced to the 16-float record above.  P is never materialised.  async.
 * d_target must be a target prepared for this M: that is checked on the device (no host
 * synchronisation) and a mismatch (wrong M, not a prepared target) writes an all-NaN record.
 * Errors: EINVAL (null, N < 1, M < 1, σ² ≤ 0 or non-finite, w ∉ [0,1), V ≤ 0, R not a
 * rotation to 1e-6, ws too small), ECUDA. */
size_t lsgcpd_estep_workspace_bytes(int64_t M, int64_t N);
int lsgcpd_estep(const void* d_target, int64_t M, const float* d_src, int64_t N,
                 const double R[9], const double t[3], double sigma2, double w, double volume,
                 int consistent_normalizer, float* d_record, void* d_ws, size_t ws_bytes,
                 lsgcpd_stream_t stream);

/* E step with the §3.2-3.3 model extensions: w, eta, consistent_normalizer and d_src_conf are
 * taken from `params` (the other fields are ignored); the target's component priors π(m) are
 * whatever lsgcpd_target_set_prior last installed (uniform 1/M by default).  With per-point w_n:
 *   P_mn = (1-w_n) π(m) c_m e^{-d_mn/2} / (w_n/V + (1-w_n) Σ_k π(k) c_k e^{-d_kn/2}),
 * and a point with φ(x_n) = 0 (w_n = 1) is all outlier (P_out = 1, ln p = -ln V).  async.
 * Errors: as lsgcpd_estep, plus EINVAL for eta ≥ 1. */
int lsgcpd_estep_ex(const void* d_target, int64_t M, const float* d_src, int64_t N,
                    const double R[9], const double t[3], double sigma2, const lsgcpd_em_params* params,
                    double volume, float* d_record, void* d_ws, size_t ws_bytes, lsgcpd_stream_t stream);

/* ---------------------------------------------------------------------------------------
 * Confidence filtering.  φ(x) = e_min/e(x) is a sensor's measurement confidence.
 * ------------------------------------------------------------------------------------- */
/* Install component priors π(m) = φ(y_m)/Σ_m φ(y_m) (Eq. 8) into a prepared target, in place:
 * the per-target log weight becomes ½log2(1+α_m) + log2(M π(m)).  Idempotent (α_m is read back
 * from the packed model; a uniform φ restores π = 1/M).  d_phi: DEVICE [M], φ ≥ 0, Σφ > 0;
 * φ(y_m) = 0 removes component m.  h_spc (may be NULL) receives Σ_m π(m)√(1+α_m).  sync.
 * Non-uniform priors need consistent_normalizer = 1 in the E step / registration (the Eq. 9-10
 * literal form has π(m) = 1/M): with 0 those calls return EINVAL (and the E step then reads the
 * target header, a host sync).
 * Errors: EINVAL (null, M mismatch, negative / non-finite φ, all zero, ws too small), ECUDA. */
size_t lsgcpd_target_prior_workspace_bytes(int64_t M);
int lsgcpd_target_set_prior(void* d_target, int64_t M, const float* d_phi, void* d_ws, size_t ws_bytes,
                            double* h_spc, lsgcpd_stream_t stream);

/* Truncation of low-confidence points: copy the points with φ ≥ threshold, in their original
 * order, to d_xyz_out [n][3] (and their φ to d_phi_out [n], may be NULL); *h_n_out = count.  The
 * output buffers must hold n points.  sync.  Errors: EINVAL (null, n < 1, ws too small), ECUDA. */
size_t lsgcpd_select_workspace_bytes(int64_t n);
int lsgcpd_select_confident(const float* d_xyz, const float* d_phi, int64_t n, float threshold,
                            float* d_xyz_out, float* d_phi_out, int64_t* h_n_out, void* d_ws,
                            size_t ws_bytes, lsgcpd_stream_t stream);

/* Depth error model (reading R23): for points in their sensor's camera frame
 * (z = depth), φ = e(z_min)/e(z) with e(z) = c0 + c1 z², clipped to [0, 1].  d_phi: DEVICE [n].
 * async.  Errors: EINVAL (null, n < 1, c0 < 0, c1 < 0, c0 + c1 z_min² ≤ 0). */
int lsgcpd_depth_confidence(const float* d_xyz, int64_t n, double c0, double c1, double z_min,
                            float* d_phi, lsgcpd_stream_t stream);

/* ---------------------------------------------------------------------------------------
 * Multi-GPU communicator (one process per GPU).  Wraps an NCCL communicator loaded at run time
 * (libnccl.so.2); the 128-byte id is produced on rank 0 and broadcast by the caller (e.g. over
 * torch.distributed).  comm_init is collective over all ranks.
 * ------------------------------------------------------------------------------------- */
int lsgcpd_comm_unique_id(void* h_out128);
int lsgcpd_comm_init(int rank, int world_size, const void* h_id128, void** comm_out);
int lsgcpd_comm_destroy(void* comm);

/* ---------------------------------------------------------------------------------------
 * Registration (the EM loop): σ²₀ (CPD closed form) → for k < max_iters:
 * E step → per-point FP64 moments (75 numbers) → [all-reduce over comm] → damped SE(3)
 * Newton on the exact frozen-P objective (Eq. 11-13, readings R11-R13) → σ².
 * params->eta and params->d_src_conf (indexed like d_src_local) select the §3.2-3.3 model as in
 * lsgcpd_estep_ex; the target's priors are those installed by lsgcpd_target_set_prior.
 * Each rank passes its own contiguous source shard (N_local points) and the same prepared
 * target; all ranks return bit-identical R, t, σ².  volume ≤ 0 uses the target's V.
 * Optional host traces (may be NULL): nll_trace[max_iters] (NLL at each E step, Eq. 4),
 * sigma2_trace[max_iters+1] (σ²_0 … σ²_k).  sync.
 * Errors: EINVAL (also for a non-finite source coordinate, detected by the σ²₀ reduction), ECUDA,
 * ENCCL, ENOMASS (results still written). */
size_t lsgcpd_register_workspace_bytes(int64_t M, int64_t N_local, int max_iters);
int lsgcpd_register(const void* d_target, int64_t M, double volume, const float* d_src_local,
                    int64_t N_local, const lsgcpd_em_params* params, const double R0[9],
                    const double t0[3], double R_out[9], double t_out[3], double* sigma2_out,
                    int* iters_out, double* nll_trace, double* sigma2_trace, void* comm,
                    void* d_ws, size_t ws_bytes, lsgcpd_stream_t stream);

/* ---------------------------------------------------------------------------------------
 * Batched registrations (many small independent problems in one EM loop, SURVEY §8(f) NEXT-3;
 * the paper's workloads are 3.5k-5k-point pairs).  Every iteration is
 * ONE batched E-step launch over the units of all problems (stream-K), one merge, one moments
 * launch (a CTA per problem) and one Newton launch (a warp per problem), replayed as a CUDA graph.
 * Per problem: its own prepared target (priors as installed), source, volume and initial pose;
 * shared: params (w / eta, iterations, normaliser, floors).  Results match per-problem
 * lsgcpd_register up to FP32 summation order (the batched E step runs on CUDA cores).
 * ------------------------------------------------------------------------------------- */
typedef struct {
    const void* d_target;      /* prepared target of this problem (16-byte aligned)               */
    int64_t M;                 /* its number of targets                                          */
    const float* d_src;        /* DEVICE [N][3] source points                                    */
    int64_t N;                 /* ≥ 1                                                             */
    const float* d_src_conf;   /* DEVICE [N] φ(x_n) (Eq. 8) or NULL                               */
    double volume;             /* ≤ 0: the target's V                                            */
    double R0[9], t0[3];       /* initial pose (row-major R)                                     */
} lsgcpd_problem;

/* Workspace for B problems (depends on every problem's M and N).  0 on invalid sizes. */
size_t lsgcpd_register_batch_workspace_bytes(const lsgcpd_problem* h_problems, int B, int max_iters);
/* sync.  Outputs (HOST, B entries each): R_out [B][9], t_out [B][3], sigma2_out, iters_out,
 * status_out (0; LSGCPD_ENOMASS for a problem that lost its inlier mass; LSGCPD_EINVAL for a
 * problem whose source holds a non-finite coordinate, which is not iterated; the others are
 * unaffected either way).  params->d_src_conf is ignored (per-problem d_src_conf is used).
 * Errors: EINVAL (null, B < 1, bad sizes, bad target / priors with the literal form, bad
 * params, ws too small), ECUDA. */
int lsgcpd_register_batch(const lsgcpd_problem* h_problems, int B, const lsgcpd_em_params* params,
                          double* R_out, double* t_out, double* sigma2_out, int* iters_out,
                          int* status_out, void* d_ws, size_t ws_bytes, lsgcpd_stream_t stream);

/* ---------------------------------------------------------------------------------------
 * Test support: the multi-GPU protocol on ONE device.  G source
 * shards h_d_src[g] (HOST array of G DEVICE pointers, [h_N[g]][3]) are registered as G ranks of
 * lsgcpd_register with a communicator would: each shard runs the production E step, merge,
 * moment and Newton kernels on its own workspace; the moment all-reduce (75 doubles per EM
 * iteration) and the σ²₀ all-reduce are a fixed-order device sum over the shards.  d_ws holds G
 * workspaces at a stride of ws_stride bytes (a multiple of 256, each ≥ lsgcpd_register_
 * workspace_bytes(M, h_N[g], max_iters)).  Outputs per shard: R_out[9G], t_out[3G],
 * sigma2_out[G], iters_out[G] (identical across shards by construction).  1 ≤ G ≤ 16;
 * params->d_src_conf must be NULL.  sync.  Errors: as lsgcpd_register. */
int lsgcpd_register_shards(const void* d_target, int64_t M, double volume, const float* const* h_d_src,
                           const int64_t* h_N, int G, const lsgcpd_em_params* params, const double R0[9],
                           const double t0[3], double* R_out, double* t_out, double* sigma2_out,
                           int* iters_out, void* d_ws, size_t ws_stride, lsgcpd_stream_t stream);

/* Run-time options (diagnostics and tests; the defaults are the product configuration).  Read
 * once from the environment at first use (LSGCPD_TC, LSGCPD_ESTEP_VARIANT, LSGCPD_HALVES,
 * LSGCPD_NO_FUSE, LSGCPD_GRAPH_CACHE, LSGCPD_NO_GRAPH, LSGCPD_TILE_GATE), then only changed
 * by lsgcpd_set_option; each field is atomic.  Names and values:
 *   "tc"            2 automatic, 1 tensor-core E step forced, 0 CUDA cores only
 *   "estep_variant" -1 automatic, 0/1/2 the 768/512/64-point-block CUDA-core E step
 *   "halves"        0 automatic, 1 one sweep over large targets
 *   "no_fuse"       1: separate merge and moment kernels (N ≤ 2^17)
 *   "graph_cache"   0: no cached EM-iteration graphs
 *   "no_graph"      1: plain launches instead of a captured EM iteration
 *   "tile_gate"     G: tile-centred residual on tiles with E_tile ≤ G·σ (≤ 0: never)
 *   "far_rule"      1 (default): also for a warp whose points are all ≥ 2 R_tile from the tile centre; 0: off
 *   "sort_source"   1 (default): lsgcpd_register / _shards run on a Morton-ordered copy of sources of ≥ 4,096
 *                   points (kept in the workspace; only the FP summation order changes); 0: the given order
 * Errors: EINVAL (unknown name, value out of range). */
int lsgcpd_set_option(const char* name, double value);
int lsgcpd_get_option(const char* name, double* value);

/* Defaults for the parameter structs (the values documented above). */
void lsgcpd_prep_params_default(lsgcpd_prep_params* p);
void lsgcpd_em_params_default(lsgcpd_em_params* p);

#ifdef __cplusplus
}
#endif
#endif /* LSGCPD_H_ */
