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
} lsgcpd_em_params;

/* Library identity. */
int lsgcpd_version(void);                 /* MAJOR*10000 + MINOR*100 + PATCH                */
const char* lsgcpd_last_error(void);      /* thread-local; never NULL                         */

/* ---------------------------------------------------------------------------------------
 * Target model.  The prepared target is an opaque device buffer of lsgcpd_target_bytes(M)
 * bytes (16-byte aligned, caller-owned) holding, per target m, y_m, √α_m n_m, α_m n_m n_mᵀ,
 * α_m (n_m·y_m) n_m and the log-determinant weight ½log2(1+α_m), plus a small header.
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

/* Pack a target from caller-supplied normals and α (e.g. an oracle's or a sensor's), no kNN.
 * d_normals [M][3] (used as given), d_alpha [M] (α_m ≥ 0).  sync (returns h_info).
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
 * Errors: EINVAL (null, N < 1, M < 1, σ² ≤ 0 or non-finite, w ∉ [0,1), V ≤ 0, R not a
 * rotation to 1e-6, ws too small), ECUDA. */
size_t lsgcpd_estep_workspace_bytes(int64_t M, int64_t N);
int lsgcpd_estep(const void* d_target, int64_t M, const float* d_src, int64_t N,
                 const double R[9], const double t[3], double sigma2, double w, double volume,
                 int consistent_normalizer, float* d_record, void* d_ws, size_t ws_bytes,
                 lsgcpd_stream_t stream);

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
 * Each rank passes its own contiguous source shard (N_local points) and the same prepared
 * target; all ranks return bit-identical R, t, σ².  volume ≤ 0 uses the target's V.
 * Optional host traces (may be NULL): nll_trace[max_iters] (NLL at each E step, Eq. 4),
 * sigma2_trace[max_iters+1] (σ²_0 … σ²_k).  sync.
 * Errors: EINVAL, ECUDA, ENCCL, ENOMASS (results still written). */
size_t lsgcpd_register_workspace_bytes(int64_t M, int64_t N_local, int max_iters);
int lsgcpd_register(const void* d_target, int64_t M, double volume, const float* d_src_local,
                    int64_t N_local, const lsgcpd_em_params* params, const double R0[9],
                    const double t0[3], double R_out[9], double t_out[3], double* sigma2_out,
                    int* iters_out, double* nll_trace, double* sigma2_trace, void* comm,
                    void* d_ws, size_t ws_bytes, lsgcpd_stream_t stream);

/* Defaults for the parameter structs (the values documented above). */
void lsgcpd_prep_params_default(lsgcpd_prep_params* p);
void lsgcpd_em_params_default(lsgcpd_em_params* p);

#ifdef __cplusplus
}
#endif
#endif /* LSGCPD_H_ */
