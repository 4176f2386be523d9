// Shared definitions for the LSG-CPD sm_100a library (product path; no oracle code).
// Paper citations: P:<line> of arXiv 2103.15039's LaTeX source.
#pragma once
#include <cuda_runtime.h>
#include <type_traits>
#include <math.h>
#include <stdint.h>
#include <stdio.h>

#include "../../include/lsgcpd.h"

namespace lsg {

// ------------------------------------------------------------------------------------------
// Error reporting (thread-local message, C ABI codes)
// ------------------------------------------------------------------------------------------
void set_error(const char* fmt, ...);
int cuda_fail(cudaError_t e, const char* what);

#define LSG_CUDA(call)                                               \
    do {                                                             \
        cudaError_t _e = (call);                                     \
        if (_e != cudaSuccess) return ::lsg::cuda_fail(_e, #call);   \
    } while (0)

#define LSG_CHECK(cond, code, ...)                                   \
    do {                                                             \
        if (!(cond)) {                                               \
            ::lsg::set_error(__VA_ARGS__);                           \
            return (code);                                           \
        }                                                            \
    } while (0)

// ------------------------------------------------------------------------------------------
// Prepared target: header + per-target 16-float record (64 B), padded to a tile multiple.
// Stored pair-interleaved: targets (2i, 2i+1) form a 128-B pair block holding, for every field f,
// {f of 2i, f of 2i+1} adjacent — one float2 per field for the f32x2 (FFMA2) E-step kernel.
//   f[0..3]   y_x, y_y, y_z, ω̄_m = ½log2(1+α_m) - ω_ref   (log-determinant weight, ≤ 0)
//   f[4..7]   ñ_x, ñ_y, ñ_z (ñ = √α n), W_xx          (W = α n nᵀ)
//   f[8..11]  W_xy, W_xz, W_yy, W_yz
//   f[12..15] W_zz, b_x, b_y, b_z                      (b = α (n·y) n)
// Padding targets have ω̄ = -inf (zero weight) and zero geometry.
// ------------------------------------------------------------------------------------------
constexpr int kTgtFloats = 16;
constexpr int kTgtPadMultiple = 256;
constexpr size_t kHeaderBytes = 256;

struct TargetHeader {
    int64_t M, M_pad;
    double omega_ref;        // max_m ½log2(1+α_m)
    double volume, extent;
    double aabb_lo[3], aabb_hi[3];
    double ybar[3];          // centroid
    double syy;              // Σ_m ||y_m - ȳ||²
    double alpha_sum;
    double spc;              // Σ_m π(m) √(1+α_m): Σ_m π(m) c_m (2πσ²)^{3/2} for w_max of Eq. 7
    int64_t n_degenerate;
    uint32_t magic;
    uint32_t prior;          // 1: non-uniform component priors installed (lsgcpd_target_set_prior)
    uint32_t pad_[2];
};
static_assert(sizeof(TargetHeader) <= kHeaderBytes, "header too big");
constexpr uint32_t kTargetMagic = 0x4c534745u;  // "LSGE": layout 3 (slot order, tile-centred core, R_tile)

inline int64_t pad_targets(int64_t M) { return (M + kTgtPadMultiple - 1) / kTgtPadMultiple * kTgtPadMultiple; }
inline const float* target_body(const void* t) { return reinterpret_cast<const float*>(static_cast<const char*>(t) + kHeaderBytes); }
inline float* target_body(void* t) { return reinterpret_cast<float*>(static_cast<char*>(t) + kHeaderBytes); }

// Targets are stored in SLOT order: the pack sorts them along a Morton (Z-order) curve of the AABB, so the
// 64 targets of a tile are spatially compact (DESIGN §8 "tile-centred residual").  The record is a sum over
// targets and does not depend on their order.  A slot section maps original target index → slot.
//
// Tensor-core section (after the pair-interleaved body): per 64-target tile, 10 KB:
//   [0, 2048)     core: 32 target pairs × 64 B, field f of targets (2i, 2i+1) adjacent, f = y'0, y'1, y'2,
//                 ω̄, ñ0, ñ1, ñ2, meta.  y' = y - c_tile, exact in FP32 (c_a = 0 on an axis where it would
//                 not be); the CUDA-core part of the pair math, two targets per f32x2 instruction.
//                 meta of targets 0, 1, 2, 3, 4 = c_0, c_1, c_2, E_tile = R_tile·√(1 + max α), R_tile (rounded
//                 up) with R_tile = max ||y'|| over the tile's real targets (the E step's precision gates).
//   [2048, 10240) 8 K-steps × 1024 B: the 32×8 B operand [F_hi; F_lo] of one K step, where
//                 F[f][m] = (1, y, W, b, 0,0,0) (original coordinates), F_hi = F rounded to TF32 (nearest),
//                 F_lo = F - F_hi (exact in FP32, read as TF32 by the MMA); UMMA K-major, no swizzle:
//                 core matrix = 8 rows × 16 B (4 targets); LBO = 128 B (next 4 targets),
//                 SBO = 256 B (next 8 rows): byte(row r, j) = 1024 s + (r/8) 256 + (j/4) 128 + (r%8) 16 + (j%4) 4.
// Slot section (after the tensor-core section): int32 slot_of[M_pad], slot_of[m] = slot of original target m.
constexpr int kTT_host = 64;   // E-step target tile (targets), host-visible copy of estep_dev.cuh's kTT
constexpr int kTcTile = 64;
constexpr int kTcTileBytes = 10240;
constexpr int kTcCoreBytes = 2048;
constexpr int kTcBOff = 2048;
inline size_t tc_section_offset(int64_t M_pad) { return kHeaderBytes + (size_t)M_pad * kTgtFloats * sizeof(float); }
inline size_t slot_section_offset(int64_t M_pad) { return tc_section_offset(M_pad) + (size_t)(M_pad / kTcTile) * kTcTileBytes; }
inline size_t target_total_bytes(int64_t M_pad) { return slot_section_offset(M_pad) + (size_t)M_pad * sizeof(int32_t); }
inline const float* target_tc(const void* t, int64_t M_pad) { return reinterpret_cast<const float*>(static_cast<const char*>(t) + tc_section_offset(M_pad)); }
inline float* target_tc(void* t, int64_t M_pad) { return reinterpret_cast<float*>(static_cast<char*>(t) + tc_section_offset(M_pad)); }
inline int32_t* target_slots(void* t, int64_t M_pad) { return reinterpret_cast<int32_t*>(static_cast<char*>(t) + slot_section_offset(M_pad)); }

// ------------------------------------------------------------------------------------------
// Per-E-step constants, computed in FP64 on the device (setup kernel or the Newton kernel),
// read by the E-step kernels.  See DESIGN.md "E-step arithmetic".
//   l̄_mn = ω̄_m - k2 τ_mn,  τ = ||r||² + (ñ·r)²,  k2 = log2(e)/(2σ²)      (base-2 log weights)
//   outlier log2 weight relative to ω_ref:  Lo = log2(w/V) - C1/ln2 - ω_ref
//   C1 = ln((1-w)/M) - 1.5 ln(2πσ²);  ln p(x̂) = C1 + ln2 (ω_ref + μ + log2 Σ 2^{l̄-μ})
// fixed = 1 when Lo ≥ -50 (w > 0): then the constant max μ ≡ 0 is safe (all l̄ ≤ 0).
// ------------------------------------------------------------------------------------------
struct IterState {
    double R[9], t[3];       // E-step pose g_old
    double sigma2;
    double w, volume;
    double C1;
    double omega_ref;        // 0 in the Eq. 9-10 literal mode
    double Lo;               // -inf when w == 0
    double extent;
    float k2;
    int fixed;
    int active;              // 0: EM finished (kernels return immediately)
    int iter;                // EM iteration index of this E step
    int status;              // 0 or LSGCPD_ENOMASS
    int no_mass;             // consecutive iterations with Σ P ≈ 0
    double last_step_rot, last_step_trans;
};

// eta ≥ 0 replaces w by the outlier-ratio bound of §3.2 (Eq. 7) at this σ²:
//   w_max = η V S / ((1 - η) + η V S),  S = Σ_m π(m) c_m = (2πσ²)^{-3/2} · (Σ π √(1+α) | 1)
// (re-evaluated at every E step because c_m depends on σ², reading R22).
__host__ __device__ inline void make_state(IterState& s, const double* R, const double* t, double sigma2, double w,
                                           double V, int64_t M, double omega_ref_target, int consistent,
                                           double eta = -1.0, double spc = 1.0) {
    for (int i = 0; i < 9; ++i) s.R[i] = R[i];
    for (int i = 0; i < 3; ++i) s.t[i] = t[i];
    if (eta >= 0.0) {
        const double S = pow(2.0 * 3.14159265358979323846 * sigma2, -1.5) * (consistent ? spc : 1.0);
        const double a = eta * V * S;
        w = a / ((1.0 - eta) + a);
        if (!(w < 1.0)) w = 1.0 - 1e-16;
    }
    s.sigma2 = sigma2;
    s.w = w;
    s.volume = V;
    const double ln2 = 0.69314718055994530942;
    s.omega_ref = consistent ? omega_ref_target : 0.0;
    s.C1 = log((1.0 - w) / (double)M) - 1.5 * log(2.0 * 3.14159265358979323846 * sigma2);
    if (w > 0.0) {
        s.Lo = (log(w / V) - s.C1) / ln2 - s.omega_ref;
    } else {
        s.Lo = -INFINITY;
    }
    s.k2 = (float)(1.4426950408889634074 / (2.0 * sigma2));
    s.fixed = (w > 0.0 && s.Lo >= -50.0) ? 1 : 0;
}

// ------------------------------------------------------------------------------------------
// Device helpers
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Deterministic grid reduction: entries [0, KMAX) by max, [KMAX, K) by sum.  Each block writes a
// partial; the last block to finish (atomic ticket) combines the partials in block order and
// writes `out`, then re-arms the counter.  blockDim.x must equal NT.
// The last CTA's fold of the per-CTA partials p[0], p[stride], … p[(n-1)·stride] in CTA order (max or sum):
// loaded 16 at a time from L2 (ld.global.cg, after the writers' __threadfence and the atomic ticket), then
// combined in the same order as a plain loop — the same result, without n dependent L2 round trips.
template <bool kMax>
__device__ __forceinline__ double ordered_reduce_l2(const double* __restrict__ p, int64_t stride, unsigned n) {
    double s = __ldcg(p);
    for (unsigned b0 = 1; b0 < n; b0 += 16) {
        double v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) v[u] = (b0 + u < n) ? __ldcg(p + (int64_t)(b0 + u) * stride) : 0.0;
#pragma unroll
        for (int u = 0; u < 16; ++u)
            if (b0 + u < n) s = kMax ? fmax(s, v[u]) : s + v[u];
    }
    return s;
}

template <int K, int KMAX, int NT>
__device__ void block_reduce_store(double (&v)[K], double* blockpart, double* out, unsigned int* counter) {
    __shared__ double sm[NT / 32][K];
    __shared__ bool last;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
    for (int f = 0; f < K; ++f) {
        const double s = f < KMAX ? warp_max(v[f]) : warp_sum(v[f]);
        if (lane == 0) sm[warp][f] = s;
    }
    __syncthreads();
    for (int f = threadIdx.x; f < K; f += NT) {
        double s = sm[0][f];
        for (int w = 1; w < NT / 32; ++w) s = f < KMAX ? fmax(s, sm[w][f]) : s + sm[w][f];
        blockpart[(int64_t)blockIdx.x * K + f] = s;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = (atomicAdd(counter, 1u) == gridDim.x - 1);
    __syncthreads();
    if (last) {
        __threadfence();
        for (int f = threadIdx.x; f < K; f += NT)
            out[f] = f < KMAX ? ordered_reduce_l2<true>(blockpart + f, K, gridDim.x)
                              : ordered_reduce_l2<false>(blockpart + f, K, gridDim.x);
        if (threadIdx.x == 0) *counter = 0u;
    }
}

// Sum over one CTA (fixed order) of K values per thread → out[0..K) (thread 0 writes).
template <int K, int NT>
__device__ void block_reduce_single(double (&v)[K], double* out) {
    __shared__ double sm[NT / 32][K];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
    for (int f = 0; f < K; ++f) {
        const double s = warp_sum(v[f]);
        if (lane == 0) sm[warp][f] = s;
    }
    __syncthreads();
    for (int f = threadIdx.x; f < K; f += NT) {
        double s = sm[0][f];
        for (int w = 1; w < NT / 32; ++w) s += sm[w][f];
        out[f] = s;
    }
}

// E-step stream-K schedule: units = (source block j, target tile i), u = j*T + i.
// CTA g owns units [start(g), start(g+1)), start(g) = floor(g U / G).
struct Sched {
    int64_t U;        // total units
    int64_t T;        // tiles per source block
    int64_t G;        // CTAs
    int64_t nblk;     // source blocks
    int64_t kmax;     // max CTAs touching one source block (partial slots per block)
    int64_t B;        // source points per block
    int variant;      // E-step kernel variant (negative: tensor-core kernel + CUDA-core variant -1-variant)
    int tc_variant;   // tensor-core kernel configuration
    int halves;       // 2: the targets are swept as two halves, one launch each (T = tiles per half); else 1
    float gate_g;     // tile-centred residual when E_tile ≤ gate_g·σ, else the hi/lo residual
    int far_rule;     // 1: also the centred residual for a warp whose points are all ≥ 2 R_tile from the centre
    int64_t hstride;  // floats between the two halves' partial sets
};
__host__ __device__ inline int64_t sched_start(const Sched& s, int64_t g) { return g * s.U / s.G; }
__host__ __device__ inline int64_t sched_owner(const Sched& s, int64_t u) { return ((u + 1) * s.G - 1) / s.U; }

}  // namespace lsg
