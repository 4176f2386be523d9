// Target preparation for sm_100a: exact grid kNN (FP64 distances),
// centred scatter, FP64 Jacobi eigen-decomposition → n_m, κ_m, α_m (Eq. 3), working volume V, and
// the packed 64-B-per-target model the E step streams through TMA.
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace lsg {

constexpr int kRedThreads = 256;
constexpr int kRedBlocks = 148;
constexpr int kMaxK = 32;
#ifndef LSG_KNN_COARSE
#define LSG_KNN_COARSE 4
#endif
#ifndef LSG_KNN_RMAX
#define LSG_KNN_RMAX 4
#endif
#ifndef LSG_KNN_FINE
#define LSG_KNN_FINE 4
#endif
// Grid sizing (tools/prep_speed.py, round 1, ms on one B200 — object / rgbd / lidar / scale):
//   one grid, cell = (AABB volume / M)^{1/3}:                 0.5 / 101.9 / 38.4 / 3.6
//   + a 4× coarser fallback grid after 4 fine rings:          0.5 /   3.5 / 36.4 / 3.6
//   + fine cell a quarter of that (the default):              1.0 /   3.8 / 27.3 / 2.3
// The AABB-volume estimate is far too coarse for surface clouds with outliers (rgbd, lidar), whose
// isolated points then scanned O(r³) cells; LiDAR's remaining cost is its near-sensor density.
constexpr int kCoarse = LSG_KNN_COARSE;         // coarse cell = kCoarse³ fine cells
constexpr int kFineRings = LSG_KNN_RMAX;        // fine rings searched before the coarse grid takes over

// ---- reductions over the raw cloud -------------------------------------------------------------
// stats1: [max(-x), max(-y), max(-z), max x, max y, max z, Σx, Σy, Σz]
__device__ __forceinline__ void cloud_stats_body(const float* __restrict__ xyz, int64_t M, double* blockpart, double* out, unsigned* counter) {
    double v[12] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY, -INFINITY, -INFINITY, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    for (int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; m < M; m += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const double c = xyz[3 * m + a];
            v[a] = fmax(v[a], -c);
            v[3 + a] = fmax(v[3 + a], c);
            v[6 + a] += c;
            v[9 + a] = fma(c, c, v[9 + a]);
        }
    }
    block_reduce_store<12, 6, kRedThreads>(v, blockpart, out, counter);
}
__global__ void __launch_bounds__(kRedThreads)
    cloud_stats_kernel(const float* __restrict__ xyz, int64_t M, double* blockpart, double* out, unsigned* counter) {
    cloud_stats_body(xyz, M, blockpart, out, counter);
}

// The model of target m as packed: y, the unit normal n = n_in/|n_in| and α.  A zero or non-finite normal
// gives α = 0 (an isotropic component), so the packed W = α n nᵀ, the normaliser ½log2(1+α) and tr(W) (read
// back by lsgcpd_target_set_prior) all describe the same density.
__device__ __forceinline__ double model_of(const float* __restrict__ nrm, const float* __restrict__ alpha, int64_t m,
                                           double n[3]) {
    const double n0 = nrm[3 * m], n1 = nrm[3 * m + 1], n2 = nrm[3 * m + 2];
    const double len = sqrt(n0 * n0 + n1 * n1 + n2 * n2);
    if (!(len > 0.0) || !isfinite(len)) {
        n[0] = n[1] = n[2] = 0.0;
        return 0.0;
    }
    n[0] = n0 / len;
    n[1] = n1 / len;
    n[2] = n2 / len;
    return (double)alpha[m];
}

// stats2 (after the model is built): [max ω, Σ α, Σ ||y - ȳ||², Σ nn-distance, n_degenerate, Σ √(1+α)]
__device__ __forceinline__ void model_stats_body(const float* __restrict__ xyz, const float* __restrict__ nrm, const float* __restrict__ alpha,
                       const float* __restrict__ nnd, const int* __restrict__ degen, int64_t M,
                       const double* __restrict__ stats1, double* blockpart, double* out, unsigned* counter) {
    double v[6] = {-INFINITY, 0.0, 0.0, 0.0, 0.0, 0.0};
    const double yb[3] = {stats1[6] / M, stats1[7] / M, stats1[8] / M};
    for (int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; m < M; m += (int64_t)gridDim.x * blockDim.x) {
        double n[3];
        const double a = model_of(nrm, alpha, m, n);
        v[0] = fmax(v[0], 0.5 * log2(1.0 + a));
        v[1] += a;
        v[5] += sqrt(1.0 + a);
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            const double d = (double)xyz[3 * m + i] - yb[i];
            v[2] = fma(d, d, v[2]);
        }
        if (nnd) v[3] += nnd[m];
        if (degen) v[4] += degen[m];
    }
    block_reduce_store<6, 1, kRedThreads>(v, blockpart, out, counter);
}
__global__ void __launch_bounds__(kRedThreads)
    model_stats_kernel(const float* __restrict__ xyz, const float* __restrict__ nrm, const float* __restrict__ alpha,
                       const float* __restrict__ nnd, const int* __restrict__ degen, int64_t M,
                       const double* __restrict__ stats1, double* blockpart, double* out, unsigned* counter) {
    model_stats_body(xyz, nrm, alpha, nnd, degen, M, stats1, blockpart, out, counter);
}

// Header: AABB, centroid, V (margin per side; a zero-extent axis is floored at the mean
// nearest-neighbour spacing when known, else at sqrt(area/M) of the other two axes), extent.
__device__ __forceinline__ void header_body(TargetHeader* hdr, int64_t M, const double* stats1, const double* stats2,
                              double margin, int have_nn) {
    TargetHeader h;
    h.M = M;
    h.M_pad = ((M + kTgtPadMultiple - 1) / kTgtPadMultiple) * kTgtPadMultiple;
    h.omega_ref = stats2[0];
    double ext[3], e2 = 0.0;
    for (int a = 0; a < 3; ++a) {
        h.aabb_lo[a] = -stats1[a];
        h.aabb_hi[a] = stats1[3 + a];
        ext[a] = h.aabb_hi[a] - h.aabb_lo[a];
        e2 += ext[a] * ext[a];
        h.ybar[a] = stats1[6 + a] / (double)M;
    }
    h.extent = sqrt(e2);
    double floor_s;
    if (have_nn) {
        floor_s = stats2[3] / (double)M;
    } else {
        double area = 1.0;
        int nz = 0;
        for (int a = 0; a < 3; ++a)
            if (ext[a] > 0.0) { area *= ext[a]; ++nz; }
        floor_s = nz >= 2 ? sqrt(area / (double)M) : (nz == 1 ? area / (double)M : 1.0);
    }
    double V = 1.0;
    for (int a = 0; a < 3; ++a) V *= (ext[a] > 0.0 ? ext[a] : floor_s) * (1.0 + 2.0 * margin);
    h.volume = V;
    h.syy = stats2[2];
    h.alpha_sum = stats2[1];
    h.spc = stats2[5] / (double)M;   // uniform prior π(m) = 1/M
    h.n_degenerate = (int64_t)stats2[4];
    h.magic = kTargetMagic;
    h.prior = 0;
    h.pad_[0] = h.pad_[1] = 0;
    *hdr = h;
    // the rest of the 256-byte header region is zero (the prepared target's bytes are fully defined)
    uint32_t* tail = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(hdr) + sizeof(TargetHeader));
    for (size_t i = 0; i < (kHeaderBytes - sizeof(TargetHeader)) / 4; ++i) tail[i] = 0u;
}
__global__ void header_kernel(TargetHeader* hdr, int64_t M, const double* stats1, const double* stats2,
                              double margin, int have_nn) {
    header_body(hdr, M, stats1, stats2, margin, have_nn);
}

// ---- slot order: a Morton (Z-order) curve over the AABB ----------------------------------------------
// 21 bits per axis of the AABB's enclosing cube; ties (one cell) keep the input order (stable radix sort).
__device__ __forceinline__ uint64_t morton_spread(uint64_t x) {
    x &= 0x1fffffull;
    x = (x | (x << 32)) & 0x1f00000000ffffull;
    x = (x | (x << 16)) & 0x1f0000ff0000ffull;
    x = (x | (x << 8)) & 0x100f00f00f00f00full;
    x = (x | (x << 4)) & 0x10c30c30c30c30c3ull;
    x = (x | (x << 2)) & 0x1249249249249249ull;
    return x;
}
__device__ __forceinline__ void morton_keys_body(const float* __restrict__ xyz, int64_t M, const double* __restrict__ stats1,
                                   uint64_t* __restrict__ keys, int* __restrict__ ids) {
    const int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (m >= M) return;
    const double lo[3] = {-stats1[0], -stats1[1], -stats1[2]};
    const double side = fmax(fmax(stats1[3] + stats1[0], stats1[4] + stats1[1]), stats1[5] + stats1[2]);
    const double sc = side > 0.0 ? 2097151.0 / side : 0.0;
    uint64_t k = 0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        double q = floor(((double)xyz[3 * m + a] - lo[a]) * sc);
        q = q < 0.0 ? 0.0 : (q > 2097151.0 ? 2097151.0 : q);
        k |= morton_spread((uint64_t)q) << a;
    }
    keys[m] = k;
    ids[m] = (int)m;
}
__global__ void morton_keys_kernel(const float* __restrict__ xyz, int64_t M, const double* __restrict__ stats1,
                                   uint64_t* __restrict__ keys, int* __restrict__ ids) {
    morton_keys_body(xyz, M, stats1, keys, ids);
}
// slot_of[perm[s]] = s (the inverse permutation, kept in the target for lsgcpd_target_set_prior)
__device__ __forceinline__ void slot_inverse_body(const int* __restrict__ perm, int64_t M, int64_t M_pad, int32_t* __restrict__ slot_of) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s < M) slot_of[perm[s]] = (int32_t)s;
    else if (s < M_pad) slot_of[s] = -1;
}
__global__ void slot_inverse_kernel(const int* __restrict__ perm, int64_t M, int64_t M_pad, int32_t* __restrict__ slot_of) {
    slot_inverse_body(perm, M, M_pad, slot_of);
}

// Packed per-target record in slot order (FP64 arithmetic, FP32 storage); padding targets contribute nothing.
__device__ __forceinline__ void pack_record_body(const float* __restrict__ xyz, const float* __restrict__ nrm,
                                 const float* __restrict__ alpha, const int* __restrict__ perm, int64_t M,
                                 int64_t M_pad, const double* __restrict__ stats2, float* __restrict__ body) {
    const int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;   // slot
    if (m >= M_pad) return;
    // pair-interleaved layout: slot m is lane (m & 1) of pair m >> 1; field f at pair*32 + 2f + lane
    float* o = body + (m >> 1) * (2 * kTgtFloats) + (m & 1);
    float f[kTgtFloats];
    if (m >= M) {
        // far away (τ overflows to a huge value → weight 0 in both normaliser modes) and ω̄ = -inf
        f[0] = f[1] = f[2] = 1e18f;
        f[3] = -INFINITY;
        for (int i = 4; i < kTgtFloats; ++i) f[i] = 0.f;
    } else {
        const int64_t i = perm[m];
        double n[3];
        const double a = model_of(nrm, alpha, i, n);
        const double y0 = xyz[3 * i], y1 = xyz[3 * i + 1], y2 = xyz[3 * i + 2];
        const double sa = sqrt(a);
        const double ny = n[0] * y0 + n[1] * y1 + n[2] * y2;
        f[0] = (float)y0; f[1] = (float)y1; f[2] = (float)y2;
        f[3] = (float)(0.5 * log2(1.0 + a) - stats2[0]);
        f[4] = (float)(sa * n[0]); f[5] = (float)(sa * n[1]); f[6] = (float)(sa * n[2]);
        f[7] = (float)(a * n[0] * n[0]); f[8] = (float)(a * n[0] * n[1]); f[9] = (float)(a * n[0] * n[2]);
        f[10] = (float)(a * n[1] * n[1]); f[11] = (float)(a * n[1] * n[2]); f[12] = (float)(a * n[2] * n[2]);
        f[13] = (float)(a * ny * n[0]); f[14] = (float)(a * ny * n[1]); f[15] = (float)(a * ny * n[2]);
    }
#pragma unroll
    for (int i = 0; i < kTgtFloats; ++i) o[2 * i] = f[i];
}
__global__ void pack_body_kernel(const float* __restrict__ xyz, const float* __restrict__ nrm,
                                 const float* __restrict__ alpha, const int* __restrict__ perm, int64_t M,
                                 int64_t M_pad, const double* __restrict__ stats2, float* __restrict__ body) {
    pack_record_body(xyz, nrm, alpha, perm, M, M_pad, stats2, body);
}

// Tensor-core section: core fields (tile-centred) and the hi/lo TF32 feature blocks (see common.cuh).
__device__ __forceinline__ float tf32_rna(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}
// y - c is exactly representable in FP32 (FP64 TwoSum: the double difference is exact, then it fits a float)
__device__ __forceinline__ bool exact_diff_f32(float y, float c) {
    const double a = y, b = -(double)c;
    const double s = __dadd_rn(a, b);
    const double bb = __dsub_rn(s, a);
    const double err = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
    return err == 0.0 && (double)(float)s == s;
}
// One CTA of kTcTile threads per tile, one thread per slot.
__device__ __forceinline__ void pack_tc_body(const float* __restrict__ xyz, const float* __restrict__ nrm, const float* __restrict__ alpha,
                   const int* __restrict__ perm, int64_t M, const double* __restrict__ stats2, float* __restrict__ tc) {
    __shared__ float s_lo[3][kTcTile], s_hi[3][kTcTile];
    __shared__ int s_bad[3];
    __shared__ double s_r[kTcTile], s_a[kTcTile];
    const int64_t tile = blockIdx.x;
    const int jt = threadIdx.x;
    const int64_t m = tile * kTcTile + jt;
    const bool real = m < M;
    char* base = reinterpret_cast<char*>(tc) + tile * kTcTileBytes;
    float* core = reinterpret_cast<float*>(base) + (jt >> 1) * 16 + (jt & 1);
    float y[3] = {0.f, 0.f, 0.f};
    double n[3] = {0.0, 0.0, 0.0}, a = 0.0;
    if (real) {
        const int64_t i = perm[m];
        a = model_of(nrm, alpha, i, n);
        for (int k = 0; k < 3; ++k) y[k] = xyz[3 * i + k];
    }
    // tile centre c: the FP32 midpoint of the real targets' box, per axis, kept only if every y - c is exact
    for (int k = 0; k < 3; ++k) {
        s_lo[k][jt] = real ? y[k] : INFINITY;
        s_hi[k][jt] = real ? y[k] : -INFINITY;
    }
    if (jt < 3) s_bad[jt] = 0;
    __syncthreads();
    for (int w = kTcTile / 2; w > 0; w >>= 1) {
        if (jt < w)
            for (int k = 0; k < 3; ++k) {
                s_lo[k][jt] = fminf(s_lo[k][jt], s_lo[k][jt + w]);
                s_hi[k][jt] = fmaxf(s_hi[k][jt], s_hi[k][jt + w]);
            }
        __syncthreads();
    }
    float c[3];
    for (int k = 0; k < 3; ++k) {
        const float lo = s_lo[k][0], hi = s_hi[k][0];
        c[k] = (lo <= hi) ? (float)(0.5 * ((double)lo + (double)hi)) : 0.f;
    }
    __syncthreads();
    for (int k = 0; k < 3; ++k)
        if (real && !exact_diff_f32(y[k], c[k])) atomicOr(&s_bad[k], 1);
    __syncthreads();
    for (int k = 0; k < 3; ++k)
        if (s_bad[k]) c[k] = 0.f;
    float yc[3];
    double r2 = 0.0;
    for (int k = 0; k < 3; ++k) {
        yc[k] = real ? y[k] - c[k] : 1e18f;   // exact by construction; padding far away
        r2 += real ? (double)yc[k] * (double)yc[k] : 0.0;
    }
    s_r[jt] = sqrt(r2);
    s_a[jt] = a;
    __syncthreads();
    for (int w = kTcTile / 2; w > 0; w >>= 1) {
        if (jt < w) {
            s_r[jt] = fmax(s_r[jt], s_r[jt + w]);
            s_a[jt] = fmax(s_a[jt], s_a[jt + w]);
        }
        __syncthreads();
    }
    const float E = (float)(s_r[0] * sqrt(1.0 + s_a[0]));   // rounded; the gate compares it with a margin
    float cf[8];
    float F[16];
    for (int i = 0; i < 16; ++i) F[i] = 0.f;
    if (!real) {
        cf[0] = cf[1] = cf[2] = 1e18f;
        cf[3] = -INFINITY;
        cf[4] = cf[5] = cf[6] = 0.f;
    } else {
        const double sa = sqrt(a);
        const double y0 = y[0], y1 = y[1], y2 = y[2];
        const double ny = n[0] * y0 + n[1] * y1 + n[2] * y2;
        cf[0] = yc[0]; cf[1] = yc[1]; cf[2] = yc[2];
        cf[3] = (float)(0.5 * log2(1.0 + a) - stats2[0]);
        cf[4] = (float)(sa * n[0]); cf[5] = (float)(sa * n[1]); cf[6] = (float)(sa * n[2]);
        F[0] = 1.f; F[1] = y[0]; F[2] = y[1]; F[3] = y[2];
        F[4] = (float)(a * n[0] * n[0]); F[5] = (float)(a * n[0] * n[1]); F[6] = (float)(a * n[0] * n[2]);
        F[7] = (float)(a * n[1] * n[1]); F[8] = (float)(a * n[1] * n[2]); F[9] = (float)(a * n[2] * n[2]);
        F[10] = (float)(a * ny * n[0]); F[11] = (float)(a * ny * n[1]); F[12] = (float)(a * ny * n[2]);
    }
    // tile meta in the spare field of targets 0..4: c_0, c_1, c_2, E_tile, R_tile (rounded up)
    const float Rt = __double2float_ru(s_r[0]);
    cf[7] = jt < 3 ? c[jt] : (jt == 3 ? E : (jt == 4 ? Rt : 0.f));
    for (int f = 0; f < 8; ++f) core[2 * f] = cf[f];
    const int s = jt / 8, j = jt % 8;
    for (int f = 0; f < 16; ++f) {
        const int off = kTcBOff + 1024 * s + (f / 8) * 256 + (j / 4) * 128 + (f % 8) * 16 + (j % 4) * 4;
        const float hi = tf32_rna(F[f]);
        *reinterpret_cast<float*>(base + off) = hi;              // rows 0-15 of the K-step block: F_hi
        // rows 16-31: F_lo = F - F_hi (exact in FP32), rounded to nearest TF32 so that the MMA (which reads
        // TF32 operands truncated) sees it exactly: no truncation bias on the lo product
        *reinterpret_cast<float*>(base + off + 512) = tf32_rna(F[f] - hi);
    }
}
__global__ void __launch_bounds__(kTcTile)
    pack_tc_kernel(const float* __restrict__ xyz, const float* __restrict__ nrm, const float* __restrict__ alpha,
                   const int* __restrict__ perm, int64_t M, const double* __restrict__ stats2, float* __restrict__ tc) {
    pack_tc_body(xyz, nrm, alpha, perm, M, stats2, tc);
}

// ---- grid kNN ------------------------------------------------------------------------------------
struct Grid {
    double lo[3];
    double h;
    int dim[3];
};

__device__ __forceinline__ int cell_coord(double p, double lo, double h, int dim) {
    int c = (int)floor((p - lo) / h);
    return c < 0 ? 0 : (c >= dim ? dim - 1 : c);
}

__device__ __forceinline__ void cell_keys_body(const float* __restrict__ xyz, int64_t M, Grid g, int* keys, int* ids) {
    const int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (m >= M) return;
    const int cx = cell_coord(xyz[3 * m], g.lo[0], g.h, g.dim[0]);
    const int cy = cell_coord(xyz[3 * m + 1], g.lo[1], g.h, g.dim[1]);
    const int cz = cell_coord(xyz[3 * m + 2], g.lo[2], g.h, g.dim[2]);
    keys[m] = (cx * g.dim[1] + cy) * g.dim[2] + cz;
    ids[m] = (int)m;
}
__global__ void cell_keys_kernel(const float* __restrict__ xyz, int64_t M, Grid g, int* keys, int* ids) {
    cell_keys_body(xyz, M, g, keys, ids);
}

// A grid's points in its cell order, padded to 16 B: the searches read a cell's points contiguously.
__device__ __forceinline__ void gather_pts_body(const float* __restrict__ xyz, const int* __restrict__ sids, int64_t M,
                                  float4* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= M) return;
    const int64_t j = sids[i];
    out[i] = make_float4(xyz[3 * j], xyz[3 * j + 1], xyz[3 * j + 2], 0.f);
}
__global__ void gather_pts_kernel(const float* __restrict__ xyz, const int* __restrict__ sids, int64_t M,
                                  float4* __restrict__ out) {
    gather_pts_body(xyz, sids, M, out);
}

__device__ __forceinline__ void cell_ranges_body(const int* __restrict__ skeys, int64_t M, int* cstart, int* cend) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= M) return;
    const int k = skeys[i];
    if (i == 0 || skeys[i - 1] != k) cstart[k] = (int)i;
    if (i == M - 1 || skeys[i + 1] != k) cend[k] = (int)i + 1;
}
__global__ void cell_ranges_kernel(const int* __restrict__ skeys, int64_t M, int* cstart, int* cend) {
    cell_ranges_body(skeys, M, cstart, cend);
}

// One thread per target point: exact k nearest (self included), ties → lower id, by ring search
// over grid cells until the k-th distance is below the distance to the unsearched region.
// Then the centred scatter, a cyclic Jacobi eigen-solve (FP64) and α (Eq. 3, tanh form).
__device__ inline void jacobi3(double A[3][3], double V[3][3]) {
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) V[i][j] = (i == j) ? 1.0 : 0.0;
    for (int sweep = 0; sweep < 16; ++sweep) {
        const double off = A[0][1] * A[0][1] + A[0][2] * A[0][2] + A[1][2] * A[1][2];
        const double dia = A[0][0] * A[0][0] + A[1][1] * A[1][1] + A[2][2] * A[2][2];
        if (!(off > 1e-36 * dia) ) break;
        for (int p = 0; p < 2; ++p)
            for (int q = p + 1; q < 3; ++q) {
                const double apq = A[p][q];
                if (apq == 0.0) continue;
                const double theta = (A[q][q] - A[p][p]) / (2.0 * apq);
                const double tt = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
                const double c = 1.0 / sqrt(tt * tt + 1.0), s = tt * c;
                for (int k = 0; k < 3; ++k) {  // A ← Jᵀ A J
                    const double akp = A[k][p], akq = A[k][q];
                    A[k][p] = c * akp - s * akq;
                    A[k][q] = s * akp + c * akq;
                }
                for (int k = 0; k < 3; ++k) {
                    const double apk = A[p][k], aqk = A[q][k];
                    A[p][k] = c * apk - s * aqk;
                    A[q][k] = s * apk + c * aqk;
                }
                for (int k = 0; k < 3; ++k) {
                    const double vkp = V[k][p], vkq = V[k][q];
                    V[k][p] = c * vkp - s * vkq;
                    V[k][q] = s * vkp + c * vkq;
                }
            }
    }
}

// Exact k nearest neighbours of p (self included, ties → lower id) by ring search over the cells of `g`:
// rings r = 0, 1, … until the k-th distance is below the distance to the unsearched region.  Gives up
// (returns false) after ring rmax; the caller then restarts on a coarser grid.
__device__ __forceinline__ bool ring_search(const float4* __restrict__ pts, double p0, double p1, double p2,
                                            const Grid& g, const int* __restrict__ sids,
                                            const int* __restrict__ cstart, const int* __restrict__ cend, int k,
                                            int rmax, double* bd, int* bi, int& cnt) {
    const int c0 = cell_coord(p0, g.lo[0], g.h, g.dim[0]);
    const int c1 = cell_coord(p1, g.lo[1], g.h, g.dim[1]);
    const int c2 = cell_coord(p2, g.lo[2], g.h, g.dim[2]);
    cnt = 0;
    for (int r = 0; r <= rmax; ++r) {
        const int x0 = c0 - r, x1 = c0 + r, y0 = c1 - r, y1 = c1 + r, z0 = c2 - r, z1 = c2 + r;
        for (int cx = max(x0, 0); cx <= min(x1, g.dim[0] - 1); ++cx)
            for (int cy = max(y0, 0); cy <= min(y1, g.dim[1] - 1); ++cy) {
                const bool edge_xy = (cx == x0 || cx == x1 || cy == y0 || cy == y1);
                for (int cz = max(z0, 0); cz <= min(z1, g.dim[2] - 1); ++cz) {
                    if (!edge_xy && cz != z0 && cz != z1) continue;  // only the shell of radius r
                    const int key = (cx * g.dim[1] + cy) * g.dim[2] + cz;
                    const int s = cstart[key];
                    if (s < 0) continue;
                    if (cnt == k) {   // skip a cell whose box is farther than the k-th distance (border cells
                                      // are open outwards: they hold the clamped points beyond the grid)
                        const int cc3[3] = {cx, cy, cz};
                        const double pp[3] = {p0, p1, p2};
                        double d2 = 0.0;
                        for (int a = 0; a < 3; ++a) {
                            const double lo = g.lo[a] + cc3[a] * g.h, hi = lo + g.h;
                            double e = 0.0;
                            if (pp[a] < lo && cc3[a] > 0) e = lo - pp[a];
                            else if (pp[a] > hi && cc3[a] < g.dim[a] - 1) e = pp[a] - hi;
                            d2 = fma(e, e, d2);
                        }
                        if (d2 > bd[k - 1]) continue;
                    }
                    const int e = cend[key];
                    for (int i = s; i < e; ++i) {
                        const int j = sids[i];
                        const float4 q = pts[i];   // the grid's points in cell order: a cell is contiguous
                        const double dx = (double)q.x - p0, dy = (double)q.y - p1, dz = (double)q.z - p2;
                        const double d = dx * dx + dy * dy + dz * dz;
                        if (cnt == k && !(d < bd[k - 1] || (d == bd[k - 1] && j < bi[k - 1]))) continue;
                        int pos = cnt < k ? cnt : k - 1;
                        while (pos > 0 && (d < bd[pos - 1] || (d == bd[pos - 1] && j < bi[pos - 1]))) {
                            bd[pos] = bd[pos - 1];
                            bi[pos] = bi[pos - 1];
                            --pos;
                        }
                        bd[pos] = d;
                        bi[pos] = j;
                        if (cnt < k) ++cnt;
                    }
                }
            }
        // distance from p to the unsearched region (sides that reach the grid border are closed)
        double bound = INFINITY;
        const double pc[3] = {p0, p1, p2};
        const int cc[3] = {c0, c1, c2};
        bool all_covered = true;
        for (int a = 0; a < 3; ++a) {
            if (cc[a] - r > 0) {
                bound = fmin(bound, pc[a] - (g.lo[a] + (cc[a] - r) * g.h));
                all_covered = false;
            }
            if (cc[a] + r < g.dim[a] - 1) {
                bound = fmin(bound, g.lo[a] + (cc[a] + r + 1) * g.h - pc[a]);
                all_covered = false;
            }
        }
        if (all_covered) return true;
        if (cnt == k && bd[k - 1] < bound * bound) return true;
    }
    return false;
}

// Outputs of target m from its k nearest neighbours bi[0..k) (ascending distance bd): the nearest other point
// distance, the centred scatter, a cyclic Jacobi eigen-solve (FP64), n, κ and α (Eq. 3, tanh form).
__device__ __noinline__ void finish_point(const float* __restrict__ xyz, int64_t m, const double* bd, const int* bi,
                                          int k, float alpha_max, float lambda, float* __restrict__ nrm_out,
                                          float* __restrict__ kappa_out, float* __restrict__ alpha_out,
                                          int* __restrict__ knn_out, float* __restrict__ nnd_out,
                                          int* __restrict__ degen_out) {
    // neighbour ids, nearest other point distance
    double nn = 0.0;
    for (int i = 0; i < k; ++i) {
        if (knn_out) knn_out[m * k + i] = bi[i];
        if (bi[i] != (int)m && nn == 0.0) nn = sqrt(bd[i]);
    }
    if (nn == 0.0) {
        for (int i = 0; i < k; ++i)
            if (bi[i] != (int)m) { nn = sqrt(bd[i]); break; }
    }
    nnd_out[m] = (float)nn;
    // centred scatter of the k neighbours
    double mean[3] = {0.0, 0.0, 0.0};
    for (int i = 0; i < k; ++i)
        for (int a = 0; a < 3; ++a) mean[a] += (double)xyz[3 * (int64_t)bi[i] + a];
    for (int a = 0; a < 3; ++a) mean[a] /= k;
    double C[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
    for (int i = 0; i < k; ++i) {
        double d[3];
        for (int a = 0; a < 3; ++a) d[a] = (double)xyz[3 * (int64_t)bi[i] + a] - mean[a];
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) C[a][b] += d[a] * d[b];
    }
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) C[a][b] /= k;
    const double trace = C[0][0] + C[1][1] + C[2][2];
    double n[3] = {0.0, 0.0, 1.0};
    double kappa = 1.0 / 3.0;
    int degenerate = 1;
    if (trace > 0.0) {
        degenerate = 0;
        double V[3][3];
        jacobi3(C, V);
        int imin = 0;
        for (int a = 1; a < 3; ++a)
            if (C[a][a] < C[imin][imin]) imin = a;
        const double lmin = C[imin][imin];
        const double tr2 = C[0][0] + C[1][1] + C[2][2];
        kappa = lmin / tr2;
        double nrm = 0.0;
        for (int a = 0; a < 3; ++a) { n[a] = V[a][imin]; nrm += n[a] * n[a]; }
        nrm = sqrt(nrm);
        for (int a = 0; a < 3; ++a) n[a] /= nrm;
    }
    kappa = fmin(fmax(kappa, 1e-12), 1.0 / 3.0);
    const double alpha = (double)alpha_max * tanh(0.5 * (double)lambda * (1.0 / kappa - 3.0));
    for (int a = 0; a < 3; ++a) nrm_out[3 * m + a] = (float)n[a];
    kappa_out[m] = (float)kappa;
    alpha_out[m] = (float)alpha;
    degen_out[m] = degenerate;}

// Up to three grids: the bulk grid (fine cells over the robust box, when the AABB is inflated by outliers),
// the fine one (≈ one point per cell of the AABB volume) and a grid 4× coarser.  A point tries them in that
// order, giving up on the first two after kFineRings rings; points in sparse regions (isolated outliers, far
// LiDAR returns) thus end on the coarse grid instead of scanning O(r³) fine cells.  Every search is exact,
// so the result does not depend on which one finished.
__device__ __forceinline__ void knn_surface_body(const float* __restrict__ xyz, int64_t M, Grid g, const int* __restrict__ sids,
                       const int* __restrict__ cstart, const int* __restrict__ cend, Grid gc,
                       const int* __restrict__ sids_c, const int* __restrict__ cstart_c,
                       const int* __restrict__ cend_c, Grid gb, const int* __restrict__ sids_b,
                       const int* __restrict__ cstart_b, const int* __restrict__ cend_b, int use_bulk, int k,
                       float alpha_max, float lambda,
                       float* __restrict__ nrm_out, float* __restrict__ kappa_out, float* __restrict__ alpha_out,
                       int* __restrict__ knn_out, float* __restrict__ nnd_out, int* __restrict__ degen_out,
                       int* __restrict__ hard, int* __restrict__ nhard, const float4* __restrict__ pts_f,
                       const float4* __restrict__ pts_b) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= M) return;
    // threads take the points in cell order (of the grid searched first): a warp's points share cells, so
    // their searches visit the same cells and take similar time
    const int64_t m = (int64_t)(use_bulk ? sids_b[i] : sids[i]);
    const double p0 = xyz[3 * m], p1 = xyz[3 * m + 1], p2 = xyz[3 * m + 2];
    double bd[kMaxK];
    int bi[kMaxK];
    int cnt = 0;
    if (!(use_bulk && ring_search(pts_b, p0, p1, p2, gb, sids_b, cstart_b, cend_b, k, kFineRings, bd, bi, cnt)) &&
        !ring_search(pts_f, p0, p1, p2, g, sids, cstart, cend, k, kFineRings, bd, bi, cnt)) {
        hard[atomicAdd(nhard, 1)] = (int)m;   // knn_hard_kernel: one warp per such point on the coarse grid
        return;
    }
    finish_point(xyz, m, bd, bi, k, alpha_max, lambda, nrm_out, kappa_out, alpha_out, knn_out, nnd_out, degen_out);
}
__global__ void __launch_bounds__(128)
    knn_surface_kernel(const float* __restrict__ xyz, int64_t M, Grid g, const int* __restrict__ sids,
                       const int* __restrict__ cstart, const int* __restrict__ cend, Grid gc,
                       const int* __restrict__ sids_c, const int* __restrict__ cstart_c,
                       const int* __restrict__ cend_c, Grid gb, const int* __restrict__ sids_b,
                       const int* __restrict__ cstart_b, const int* __restrict__ cend_b, int use_bulk, int k,
                       float alpha_max, float lambda,
                       float* __restrict__ nrm_out, float* __restrict__ kappa_out, float* __restrict__ alpha_out,
                       int* __restrict__ knn_out, float* __restrict__ nnd_out, int* __restrict__ degen_out,
                       int* __restrict__ hard, int* __restrict__ nhard, const float4* __restrict__ pts_f,
                       const float4* __restrict__ pts_b) {
    knn_surface_body(xyz, M, g, sids, cstart, cend, gc, sids_c, cstart_c, cend_c, gb, sids_b, cstart_b, cend_b, use_bulk, k, alpha_max, lambda, nrm_out, kappa_out, alpha_out, knn_out, nnd_out, degen_out, hard, nhard, pts_f, pts_b);
}

// The points whose search left the first two grids (isolated outliers, far returns): one warp per point on the
// coarse grid.  Ring by ring, the lanes split the shell's points (cell by cell, each cell's points strided over
// the warp), each keeping its own k best (distance, id);
// the warp then merges the 32 lists (k rounds of a warp-wide lexicographic minimum) into the ring's k best,
// whose k-th distance prunes the next rings' cells and decides the stop exactly as ring_search does.  Lane 0
// finishes the point.  Same result as the one-thread search (exact k nearest, ties → lower id).
__device__ __forceinline__ void knn_hard_body(const float* __restrict__ xyz, Grid g, const int* __restrict__ sids, const int* __restrict__ cstart,
                    const int* __restrict__ cend, int k, float alpha_max, float lambda, float* __restrict__ nrm_out,
                    float* __restrict__ kappa_out, float* __restrict__ alpha_out, int* __restrict__ knn_out,
                    float* __restrict__ nnd_out, int* __restrict__ degen_out, const int* __restrict__ hard,
                    const int* __restrict__ nhard, const float4* __restrict__ pts) {
    __shared__ double sd[4][kMaxK];
    __shared__ int si[4][kMaxK];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int nw = (int)((gridDim.x * blockDim.x) >> 5);
    const int nh = *nhard;
    for (int h = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5); h < nh; h += nw) {
        const int64_t m = hard[h];
        const double p0 = xyz[3 * m], p1 = xyz[3 * m + 1], p2 = xyz[3 * m + 2];
        const double pp[3] = {p0, p1, p2};
        const int c0 = cell_coord(p0, g.lo[0], g.h, g.dim[0]);
        const int c1 = cell_coord(p1, g.lo[1], g.h, g.dim[1]);
        const int c2 = cell_coord(p2, g.lo[2], g.h, g.dim[2]);
        const int cc[3] = {c0, c1, c2};
        double bd[kMaxK];
        int bi[kMaxK];
        int cnt = 0;
        double gk = INFINITY;   // the warp's k-th distance so far (after the last merge)
        for (int r = 0;; ++r) {
            const int x0 = max(c0 - r, 0), x1 = min(c0 + r, g.dim[0] - 1);
            const int y0 = max(c1 - r, 0), y1 = min(c1 + r, g.dim[1] - 1);
            const int z0 = max(c2 - r, 0), z1 = min(c2 + r, g.dim[2] - 1);
            const int nx = x1 - x0 + 1, ny = y1 - y0 + 1, nz = z1 - z0 + 1;
            const int64_t ncube = (int64_t)nx * ny * nz;
            // 32 cube cells at a time, one per lane; then every lane scans a share of each kept cell's points
            // (a dense cell is split over the warp instead of stalling one lane)
            for (int64_t q0 = 0; q0 < ncube; q0 += 32) {
                const int64_t q = q0 + lane;
                int s0 = -1, e0 = -1;
                if (q < ncube) {
                    const int cx = x0 + (int)(q / ((int64_t)ny * nz));
                    const int cy = y0 + (int)((q / nz) % ny);
                    const int cz = z0 + (int)(q % nz);
                    const bool shell = cx == c0 - r || cx == c0 + r || cy == c1 - r || cy == c1 + r ||
                                       cz == c2 - r || cz == c2 + r;   // interior cells: earlier rings
                    const int key = (cx * g.dim[1] + cy) * g.dim[2] + cz;
                    if (shell && cstart[key] >= 0) {
                        const int cell[3] = {cx, cy, cz};
                        double d2c = 0.0;
                        for (int a = 0; a < 3; ++a) {
                            const double lo = g.lo[a] + cell[a] * g.h, hi = lo + g.h;
                            double e = 0.0;
                            if (pp[a] < lo && cell[a] > 0) e = lo - pp[a];
                            else if (pp[a] > hi && cell[a] < g.dim[a] - 1) e = pp[a] - hi;
                            d2c = fma(e, e, d2c);
                        }
                        if (!(d2c > gk)) {
                            s0 = cstart[key];
                            e0 = cend[key];
                        }
                    }
                }
                unsigned todo = __ballot_sync(0xffffffffu, s0 >= 0);
                while (todo) {
                    const int src = __ffs(todo) - 1;
                    todo &= todo - 1;
                    const int a0 = __shfl_sync(0xffffffffu, s0, src), a1 = __shfl_sync(0xffffffffu, e0, src);
                    for (int t = a0 + lane; t < a1; t += 32) {
                        const int j = sids[t];
                        const float4 q = pts[t];
                        const double dx = (double)q.x - p0, dy = (double)q.y - p1, dz = (double)q.z - p2;
                        const double d = dx * dx + dy * dy + dz * dz;
                        if (cnt == k && !(d < bd[k - 1] || (d == bd[k - 1] && j < bi[k - 1]))) continue;
                        int pos = cnt < k ? cnt : k - 1;
                        while (pos > 0 && (d < bd[pos - 1] || (d == bd[pos - 1] && j < bi[pos - 1]))) {
                            bd[pos] = bd[pos - 1];
                            bi[pos] = bi[pos - 1];
                            --pos;
                        }
                        bd[pos] = d;
                        bi[pos] = j;
                        if (cnt < k) ++cnt;
                    }
                }
            }
            // merge the lanes' lists: k rounds of a warp-wide minimum over the lanes' next entries
            int head = 0, total = 0;
            for (int t = 0; t < k; ++t) {
                double d = head < cnt ? bd[head] : INFINITY;
                int id = head < cnt ? bi[head] : 0x7fffffff;
                for (int o = 16; o > 0; o >>= 1) {
                    const double od = __shfl_xor_sync(0xffffffffu, d, o);
                    const int oid = __shfl_xor_sync(0xffffffffu, id, o);
                    if (od < d || (od == d && oid < id)) {
                        d = od;
                        id = oid;
                    }
                }
                if (head < cnt && bd[head] == d && bi[head] == id) ++head;
                if (lane == 0) {
                    sd[wib][t] = d;
                    si[wib][t] = id;
                }
                if (d < INFINITY) ++total;
            }
            __syncwarp();
            if (total == k) gk = sd[wib][k - 1];
            // stop as ring_search does: every cell searched, or the k-th distance inside the searched box
            double bound = INFINITY;
            bool all_covered = true;
            for (int a = 0; a < 3; ++a) {
                if (cc[a] - r > 0) {
                    bound = fmin(bound, pp[a] - (g.lo[a] + (cc[a] - r) * g.h));
                    all_covered = false;
                }
                if (cc[a] + r < g.dim[a] - 1) {
                    bound = fmin(bound, g.lo[a] + (cc[a] + r + 1) * g.h - pp[a]);
                    all_covered = false;
                }
            }
            if (all_covered || (total == k && gk < bound * bound)) break;
            __syncwarp();
        }
        if (lane == 0) {
            double fd[kMaxK];
            int fi[kMaxK];
            for (int t = 0; t < k; ++t) {
                fd[t] = sd[wib][t];
                fi[t] = si[wib][t];
            }
            finish_point(xyz, m, fd, fi, k, alpha_max, lambda, nrm_out, kappa_out, alpha_out, knn_out, nnd_out,
                         degen_out);
        }
        __syncwarp();
    }
}
__global__ void __launch_bounds__(128)
    knn_hard_kernel(const float* __restrict__ xyz, Grid g, const int* __restrict__ sids, const int* __restrict__ cstart,
                    const int* __restrict__ cend, int k, float alpha_max, float lambda, float* __restrict__ nrm_out,
                    float* __restrict__ kappa_out, float* __restrict__ alpha_out, int* __restrict__ knn_out,
                    float* __restrict__ nnd_out, int* __restrict__ degen_out, const int* __restrict__ hard,
                    const int* __restrict__ nhard, const float4* __restrict__ pts) {
    knn_hard_body(xyz, g, sids, cstart, cend, k, alpha_max, lambda, nrm_out, kappa_out, alpha_out, knn_out, nnd_out, degen_out, hard, nhard, pts);
}

// ---- host side -------------------------------------------------------------------------------------
struct PrepLayout {
    size_t blockpart, stats1, stats2, counter, keys, ids, skeys, sids, cstart, cend, nrm, kappa, alpha, nnd,
        degen, cub_tmp, cub_bytes, total;
    size_t skeys_c, sids_c, cstart_c, cend_c;   // the 4× coarser grid of the kNN search
    size_t skeys_b, sids_b, cstart_b, cend_b;   // the bulk grid (fine cells over the robust box)
    size_t hard;                                // points left to the coarse grid (knn_hard_kernel)
    size_t pts_f, pts_c, pts_b;                 // float4 copies of the points in each grid's cell order
    size_t mkeys, mkeys_s, mids, mperm, mcub, mcub_bytes;   // the Morton sort of the slot order
};
static size_t al(size_t x) { return (x + 255) & ~size_t(255); }
constexpr int64_t kMaxCells = 1 << 22;
// dense-grid cell cap of an M-point cloud: 128 cells per point (a volume-filling cloud needs ~64 at a quarter of
// the mean spacing), at least 2^16, at most 2^22 — small clouds get small workspaces
static int64_t cell_cap(int64_t M) {
    const int64_t c = 128 * M;
    return c < (1 << 16) ? (1 << 16) : (c > kMaxCells ? kMaxCells : c);
}
static int64_t cell_cap_coarse(int64_t M) { return 2 * cell_cap(M) / (kCoarse * kCoarse * kCoarse); }

static size_t cub_sort_bytes(int64_t M) {
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const int*)nullptr, (int*)nullptr, (const int*)nullptr,
                                    (int*)nullptr, (int)M, 0, 22);
    return bytes;
}

static size_t cub_morton_bytes(int64_t M) {
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const uint64_t*)nullptr, (uint64_t*)nullptr, (const int*)nullptr,
                                    (int*)nullptr, (int)M, 0, 63);
    return bytes;
}

static PrepLayout prep_layout(int64_t M, bool with_knn) {
    PrepLayout L;
    size_t o = 0;
    L.mkeys = o; o += al(sizeof(uint64_t) * M);
    L.mkeys_s = o; o += al(sizeof(uint64_t) * M);
    L.mids = o; o += al(sizeof(int) * M);
    L.mperm = o; o += al(sizeof(int) * M);
    L.mcub_bytes = cub_morton_bytes(M);
    L.mcub = o; o += al(L.mcub_bytes);
    L.blockpart = o; o += al(sizeof(double) * kRedBlocks * 16);
    L.stats1 = o; o += al(sizeof(double) * 16);
    L.stats2 = o; o += al(sizeof(double) * 16);
    L.counter = o; o += al(sizeof(unsigned) * 4);
    L.nrm = o; o += al(sizeof(float) * 3 * M);
    L.kappa = o; o += al(sizeof(float) * M);
    L.alpha = o; o += al(sizeof(float) * M);
    L.nnd = o; o += al(sizeof(float) * M);
    L.degen = o; o += al(sizeof(int) * M);
    if (with_knn) {
        L.keys = o; o += al(sizeof(int) * M);
        L.ids = o; o += al(sizeof(int) * M);
        L.skeys = o; o += al(sizeof(int) * M);
        L.sids = o; o += al(sizeof(int) * M);
        L.cstart = o; o += al(sizeof(int) * cell_cap(M));
        L.cend = o; o += al(sizeof(int) * cell_cap(M));
        L.skeys_c = o; o += al(sizeof(int) * M);
        L.sids_c = o; o += al(sizeof(int) * M);
        L.cstart_c = o; o += al(sizeof(int) * cell_cap_coarse(M));
        L.cend_c = o; o += al(sizeof(int) * cell_cap_coarse(M));
        L.hard = o; o += al(sizeof(int) * (M + 1));   // [0] = count, then the point ids
        L.pts_f = o; o += al(sizeof(float4) * M);       // each grid's points in its cell order
        L.pts_c = o; o += al(sizeof(float4) * M);
        L.pts_b = o; o += al(sizeof(float4) * M);
        L.skeys_b = o; o += al(sizeof(int) * M);
        L.sids_b = o; o += al(sizeof(int) * M);
        L.cstart_b = o; o += al(sizeof(int) * cell_cap(M));
        L.cend_b = o; o += al(sizeof(int) * cell_cap(M));
        L.cub_bytes = cub_sort_bytes(M);
        L.cub_tmp = o; o += al(L.cub_bytes);
    } else {
        L.keys = L.ids = L.skeys = L.sids = L.cstart = L.cend = L.cub_tmp = L.cub_bytes = 0;
        L.skeys_c = L.sids_c = L.cstart_c = L.cend_c = 0;
        L.skeys_b = L.sids_b = L.cstart_b = L.cend_b = L.hard = 0;
        L.pts_f = L.pts_c = L.pts_b = 0;
    }
    L.total = o;
    return L;
}

size_t prepare_ws_bytes(int64_t M) { return prep_layout(M, true).total; }

// ---- source order for the E step (DESIGN §8 "far points") ---------------------------------------------
// lsgcpd_register runs on a Morton-ordered copy of the source (and of its confidences): a warp's points are
// then spatially compact, so for most target tiles all of them are far from the tile and the warp takes the
// cheaper centred residual.  The registration is a sum over points: the order changes only FP summation.
// Device-side only (no host synchronisation): the source box from cloud_stats, keys, a stable radix sort, gather.
__global__ void source_gather_kernel(const float* __restrict__ src, const float* __restrict__ phi,
                                     const int* __restrict__ perm, int64_t N, float* __restrict__ out,
                                     float* __restrict__ phi_out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    const int64_t j = perm[i];
    out[3 * i] = src[3 * j];
    out[3 * i + 1] = src[3 * j + 1];
    out[3 * i + 2] = src[3 * j + 2];
    if (phi) phi_out[i] = phi[j];
}
struct SrcSortLayout {
    size_t keys, keys_s, ids, perm, part, stats, ctr, cub, total;
    size_t cub_bytes;
};
static SrcSortLayout src_sort_layout(int64_t N) {
    SrcSortLayout L;
    size_t o = 0;
    L.keys = o; o += al(sizeof(uint64_t) * N);
    L.keys_s = o; o += al(sizeof(uint64_t) * N);
    L.ids = o; o += al(sizeof(int) * N);
    L.perm = o; o += al(sizeof(int) * N);
    L.part = o; o += al(sizeof(double) * kRedBlocks * 16);
    L.stats = o; o += al(sizeof(double) * 16);
    L.ctr = o; o += al(sizeof(unsigned) * 4);
    L.cub_bytes = cub_morton_bytes(N);
    L.cub = o; o += al(L.cub_bytes);
    L.total = o;
    return L;
}
size_t source_sort_ws_bytes(int64_t N) { return src_sort_layout(N).total; }
int source_sort_launch(const float* src, const float* phi, int64_t N, float* out, float* phi_out, void* d_ws,
                       cudaStream_t stream) {
    const SrcSortLayout L = src_sort_layout(N);
    char* ws = static_cast<char*>(d_ws);
    unsigned* ctr = reinterpret_cast<unsigned*>(ws + L.ctr);
    double* stats = reinterpret_cast<double*>(ws + L.stats);
    LSG_CUDA(cudaMemsetAsync(ctr, 0, sizeof(unsigned) * 4, stream));
    cloud_stats_kernel<<<kRedBlocks, kRedThreads, 0, stream>>>(src, N, reinterpret_cast<double*>(ws + L.part), stats, ctr);
    uint64_t* k = reinterpret_cast<uint64_t*>(ws + L.keys);
    int* ids = reinterpret_cast<int*>(ws + L.ids);
    int* perm = reinterpret_cast<int*>(ws + L.perm);
    morton_keys_kernel<<<(unsigned)((N + 255) / 256), 256, 0, stream>>>(src, N, stats, k, ids);
    size_t cb = L.cub_bytes;
    LSG_CUDA(cub::DeviceRadixSort::SortPairs(ws + L.cub, cb, k, reinterpret_cast<uint64_t*>(ws + L.keys_s), ids, perm,
                                             (int)N, 0, 63, stream));
    source_gather_kernel<<<(unsigned)((N + 255) / 256), 256, 0, stream>>>(src, phi, perm, N, out, phi_out);
    LSG_CUDA(cudaGetLastError());
    return 0;
}
size_t pack_ws_bytes(int64_t M) { return prep_layout(M, false).total; }

// Model statistics, header and the two packed sections of one target (async; st1 = its cloud statistics).
static int finish_launch(const float* d_xyz, const float* nrm, const float* alpha, const float* nnd, const int* degen,
                         int64_t M, double margin, char* ws, const PrepLayout& L, const double* st1, void* d_target,
                         cudaStream_t stream) {
    double* bp = reinterpret_cast<double*>(ws + L.blockpart);
    double* st2 = reinterpret_cast<double*>(ws + L.stats2);
    unsigned* ctr = reinterpret_cast<unsigned*>(ws + L.counter);
    model_stats_kernel<<<kRedBlocks, kRedThreads, 0, stream>>>(d_xyz, nrm, alpha, nnd, degen, M, st1, bp, st2, ctr);
    TargetHeader* hdr = reinterpret_cast<TargetHeader*>(d_target);
    header_kernel<<<1, 1, 0, stream>>>(hdr, M, st1, st2, margin, nnd != nullptr ? 1 : 0);
    const int64_t M_pad = pad_targets(M);
    // slot order: Morton sort of the points (stable), its inverse kept in the target
    uint64_t* mk = reinterpret_cast<uint64_t*>(ws + L.mkeys);
    uint64_t* mks = reinterpret_cast<uint64_t*>(ws + L.mkeys_s);
    int* mid = reinterpret_cast<int*>(ws + L.mids);
    int* perm = reinterpret_cast<int*>(ws + L.mperm);
    morton_keys_kernel<<<(unsigned)((M + 255) / 256), 256, 0, stream>>>(d_xyz, M, st1, mk, mid);
    size_t cb = L.mcub_bytes;
    LSG_CUDA(cub::DeviceRadixSort::SortPairs(ws + L.mcub, cb, mk, mks, mid, perm, (int)M, 0, 63, stream));
    slot_inverse_kernel<<<(unsigned)((M_pad + 255) / 256), 256, 0, stream>>>(perm, M, M_pad,
                                                                            target_slots(d_target, M_pad));
    pack_body_kernel<<<(unsigned)((M_pad + 255) / 256), 256, 0, stream>>>(d_xyz, nrm, alpha, perm, M, M_pad, st2,
                                                                          target_body(d_target));
    pack_tc_kernel<<<(unsigned)(M_pad / kTcTile), kTcTile, 0, stream>>>(d_xyz, nrm, alpha, perm, M, st2,
                                                                       target_tc(d_target, M_pad));
    LSG_CUDA(cudaGetLastError());
    return 0;
}

// Host summary and final checks of a finished target, from its header (already copied to the host).
static int info_from_header(const TargetHeader& h, int64_t M, bool knn, lsgcpd_target_info* info) {
    if (info) {
        info->volume = h.volume;
        info->extent = h.extent;
        for (int a = 0; a < 3; ++a) {
            info->aabb_lo[a] = h.aabb_lo[a];
            info->aabb_hi[a] = h.aabb_hi[a];
        }
        info->alpha_mean = h.alpha_sum / (double)M;
        info->n_degenerate = h.n_degenerate;
    }
    LSG_CHECK(isfinite(h.extent) && isfinite(h.ybar[0]) && isfinite(h.ybar[1]) && isfinite(h.ybar[2]), LSGCPD_EINVAL,
              "non-finite coordinate in the target cloud");
    LSG_CHECK(h.extent > 0.0 || !knn, LSGCPD_EDEGENERATE, "degenerate target: all points coincide");
    LSG_CHECK(isfinite(h.volume) && h.volume > 0.0, LSGCPD_EDEGENERATE, "degenerate target: zero working volume");
    return 0;
}

static int finish_target(const float* d_xyz, const float* nrm, const float* alpha, const float* nnd, const int* degen,
                         int64_t M, double margin, char* ws, const PrepLayout& L, void* d_target,
                         lsgcpd_target_info* info, cudaStream_t stream) {
    int rc = finish_launch(d_xyz, nrm, alpha, nnd, degen, M, margin, ws, L,
                           reinterpret_cast<const double*>(ws + L.stats1), d_target, stream);
    if (rc) return rc;
    TargetHeader h;
    LSG_CUDA(cudaMemcpyAsync(&h, d_target, sizeof(h), cudaMemcpyDeviceToHost, stream));
    LSG_CUDA(cudaStreamSynchronize(stream));
    return info_from_header(h, M, nnd != nullptr, info);
}

int pack_target_impl(const float* d_xyz, const float* d_nrm, const float* d_alpha, int64_t M, double margin,
                     void* d_target, void* d_ws, lsgcpd_target_info* info, cudaStream_t stream) {
    const PrepLayout L = prep_layout(M, false);
    char* ws = static_cast<char*>(d_ws);
    LSG_CUDA(cudaMemsetAsync(ws + L.counter, 0, sizeof(unsigned) * 4, stream));
    cloud_stats_kernel<<<kRedBlocks, kRedThreads, 0, stream>>>(d_xyz, M, reinterpret_cast<double*>(ws + L.blockpart),
                                                              reinterpret_cast<double*>(ws + L.stats1),
                                                              reinterpret_cast<unsigned*>(ws + L.counter));
    return finish_target(d_xyz, d_nrm, d_alpha, nullptr, nullptr, M, margin, ws, L, d_target, info, stream);
}

// kNN grids, sorts, the searches, the surface fit and the packed model of one target, from its cloud statistics
// s1 (host copy) and st1 (device copy).  Async: no host synchronisation.
// The three kNN grids of a target from its cloud statistics s1 (host copy), and the host checks.
struct GridPlan {
    Grid g, gc, gb;
    int use_bulk;
    int64_t ncells, ncells_c, ncells_b;
};
static int plan_grids(const double* s1, int64_t M, GridPlan& P) {
    // grid: cell size from the AABB volume per point (≈ 1 point per cell for a volume-filling cloud)
    Grid& g = P.g;
    double ext[3], ext_b[3], maxe = 0.0;
    for (int a = 0; a < 3; ++a) {
        g.lo[a] = -s1[a];
        ext[a] = s1[3 + a] + s1[a];
        maxe = fmax(maxe, ext[a]);
    }
    // fmax/fmin skip NaN, so a NaN coordinate shows only in the coordinate sums
    LSG_CHECK(isfinite(s1[6]) && isfinite(s1[7]) && isfinite(s1[8]) && isfinite(maxe), LSGCPD_EINVAL,
              "non-finite coordinate in the target cloud");
    LSG_CHECK(maxe > 0.0, LSGCPD_EDEGENERATE, "degenerate target: all points coincide");
    const double floor_e = maxe * 1e-3;
    double h = cbrt(fmax(ext[0], floor_e) * fmax(ext[1], floor_e) * fmax(ext[2], floor_e) / (double)M) / LSG_KNN_FINE;
    for (;;) {
        int64_t cells = 1;
        for (int a = 0; a < 3; ++a) {
            g.dim[a] = (int)fmin(floor(ext[a] / h) + 1.0, 1024.0);
            cells *= g.dim[a];
        }
        if (cells <= cell_cap(M)) break;
        h *= 1.25;
    }
    g.h = h;
    // the bulk grid: the same cell rule over mean ± 2.5 sd per axis (clipped to the AABB; points outside are
    // clamped into its border cells, which keeps every search exact).  Used first when that box is under a
    // quarter of the AABB volume — a cloud whose AABB is inflated by sparse outliers (the LiDAR config's
    // 100 m box), where AABB-sized cells would hold hundreds of the dense points.
    P.gb = g;
    Grid& gb = P.gb;
    double vb = 1.0, va = 1.0;
    for (int a = 0; a < 3; ++a) {
        const double mean = s1[6 + a] / (double)M;
        const double sd = sqrt(fmax(s1[9 + a] / (double)M - mean * mean, 0.0));
        const double lo = fmax(-s1[a], mean - 2.5 * sd), hi = fmin(s1[3 + a], mean + 2.5 * sd);
        gb.lo[a] = lo;
        ext_b[a] = fmax(hi - lo, floor_e);
        vb *= ext_b[a];
        va *= fmax(ext[a], floor_e);
    }
    P.use_bulk = (vb * 4.0 < va) ? 1 : 0;
    if (P.use_bulk) {
        double hb = cbrt(vb / (double)M) / LSG_KNN_FINE;
        for (;;) {
            int64_t cells = 1;
            for (int a = 0; a < 3; ++a) {
                gb.dim[a] = (int)fmin(floor(ext_b[a] / hb) + 1.0, 1024.0);
                cells *= gb.dim[a];
            }
            if (cells <= cell_cap(M)) break;
            hb *= 1.25;
        }
        gb.h = hb;
    }
    P.gc = g;
    P.gc.h = g.h * kCoarse;
    for (int a = 0; a < 3; ++a) P.gc.dim[a] = (g.dim[a] + kCoarse - 1) / kCoarse;
    P.ncells = (int64_t)g.dim[0] * g.dim[1] * g.dim[2];
    P.ncells_c = (int64_t)P.gc.dim[0] * P.gc.dim[1] * P.gc.dim[2];
    P.ncells_b = P.use_bulk ? (int64_t)gb.dim[0] * gb.dim[1] * gb.dim[2] : 0;
    LSG_CHECK(P.ncells_c <= cell_cap_coarse(M), LSGCPD_EINVAL, "coarse grid too large (%lld cells)",
              (long long)P.ncells_c);
    return 0;
}

static int prep_build(const float* d_xyz, int64_t M, const lsgcpd_prep_params& p, const double* s1, const double* st1,
                      void* d_target, char* ws, const PrepLayout& L, const lsgcpd_annotations* ann,
                      cudaStream_t stream) {
    GridPlan P;
    const int prc = plan_grids(s1, M, P);
    if (prc) return prc;
    const Grid &g = P.g, &gc = P.gc, &gb = P.gb;
    const int use_bulk = P.use_bulk;
    int* keys = reinterpret_cast<int*>(ws + L.keys);
    int* ids = reinterpret_cast<int*>(ws + L.ids);
    int* skeys = reinterpret_cast<int*>(ws + L.skeys);
    int* sids = reinterpret_cast<int*>(ws + L.sids);
    int* cstart = reinterpret_cast<int*>(ws + L.cstart);
    int* cend = reinterpret_cast<int*>(ws + L.cend);
    const unsigned nb = (unsigned)((M + 255) / 256);
    cell_keys_kernel<<<nb, 256, 0, stream>>>(d_xyz, M, g, keys, ids);
    size_t cub_bytes = L.cub_bytes;
    LSG_CUDA(cub::DeviceRadixSort::SortPairs(ws + L.cub_tmp, cub_bytes, keys, skeys, ids, sids, (int)M, 0, 22, stream));
    const int64_t ncells = (int64_t)g.dim[0] * g.dim[1] * g.dim[2];
    LSG_CUDA(cudaMemsetAsync(cstart, 0xff, sizeof(int) * ncells, stream));
    LSG_CUDA(cudaMemsetAsync(cend, 0xff, sizeof(int) * ncells, stream));
    cell_ranges_kernel<<<nb, 256, 0, stream>>>(skeys, M, cstart, cend);
    float4* pts_f = reinterpret_cast<float4*>(ws + L.pts_f);
    gather_pts_kernel<<<nb, 256, 0, stream>>>(d_xyz, sids, M, pts_f);
    // the coarse grid (keys and ids scratch reused: the fine sort has consumed them)
    int* skeys_c = reinterpret_cast<int*>(ws + L.skeys_c);
    int* sids_c = reinterpret_cast<int*>(ws + L.sids_c);
    int* cstart_c = reinterpret_cast<int*>(ws + L.cstart_c);
    int* cend_c = reinterpret_cast<int*>(ws + L.cend_c);
    cell_keys_kernel<<<nb, 256, 0, stream>>>(d_xyz, M, gc, keys, ids);
    cub_bytes = L.cub_bytes;
    LSG_CUDA(cub::DeviceRadixSort::SortPairs(ws + L.cub_tmp, cub_bytes, keys, skeys_c, ids, sids_c, (int)M, 0, 22,
                                             stream));
    const int64_t ncells_c = P.ncells_c;
    LSG_CUDA(cudaMemsetAsync(cstart_c, 0xff, sizeof(int) * ncells_c, stream));
    LSG_CUDA(cudaMemsetAsync(cend_c, 0xff, sizeof(int) * ncells_c, stream));
    cell_ranges_kernel<<<nb, 256, 0, stream>>>(skeys_c, M, cstart_c, cend_c);
    float4* pts_c = reinterpret_cast<float4*>(ws + L.pts_c);
    gather_pts_kernel<<<nb, 256, 0, stream>>>(d_xyz, sids_c, M, pts_c);
    float4* pts_b = reinterpret_cast<float4*>(ws + L.pts_b);
    int* sids_b = reinterpret_cast<int*>(ws + L.sids_b);
    int* cstart_b = reinterpret_cast<int*>(ws + L.cstart_b);
    int* cend_b = reinterpret_cast<int*>(ws + L.cend_b);
    if (use_bulk) {
        int* skeys_b = reinterpret_cast<int*>(ws + L.skeys_b);
        cell_keys_kernel<<<nb, 256, 0, stream>>>(d_xyz, M, gb, keys, ids);
        cub_bytes = L.cub_bytes;
        LSG_CUDA(cub::DeviceRadixSort::SortPairs(ws + L.cub_tmp, cub_bytes, keys, skeys_b, ids, sids_b, (int)M, 0, 22,
                                                 stream));
        const int64_t ncells_b = (int64_t)gb.dim[0] * gb.dim[1] * gb.dim[2];
        LSG_CUDA(cudaMemsetAsync(cstart_b, 0xff, sizeof(int) * ncells_b, stream));
        LSG_CUDA(cudaMemsetAsync(cend_b, 0xff, sizeof(int) * ncells_b, stream));
        cell_ranges_kernel<<<nb, 256, 0, stream>>>(skeys_b, M, cstart_b, cend_b);
        gather_pts_kernel<<<nb, 256, 0, stream>>>(d_xyz, sids_b, M, pts_b);
    }
    float* nrm = ann && ann->d_normals ? ann->d_normals : reinterpret_cast<float*>(ws + L.nrm);
    float* kap = ann && ann->d_kappa ? ann->d_kappa : reinterpret_cast<float*>(ws + L.kappa);
    float* alp = ann && ann->d_alpha ? ann->d_alpha : reinterpret_cast<float*>(ws + L.alpha);
    int* knn = ann ? ann->d_knn : nullptr;
    float* nnd = reinterpret_cast<float*>(ws + L.nnd);
    int* degen = reinterpret_cast<int*>(ws + L.degen);
    int* nhard = reinterpret_cast<int*>(ws + L.hard);
    LSG_CUDA(cudaMemsetAsync(nhard, 0, sizeof(int), stream));
    knn_surface_kernel<<<(unsigned)((M + 127) / 128), 128, 0, stream>>>(d_xyz, M, g, sids, cstart, cend, gc, sids_c,
                                                                        cstart_c, cend_c, gb, sids_b, cstart_b, cend_b,
                                                                        use_bulk, p.knn_k, p.alpha_max, p.lambda, nrm,
                                                                        kap, alp, knn, nnd, degen, nhard + 1, nhard,
                                                                        pts_f, pts_b);
    knn_hard_kernel<<<(unsigned)(4 * 148), 128, 0, stream>>>(d_xyz, gc, sids_c, cstart_c, cend_c, p.knn_k, p.alpha_max,
                                                             p.lambda, nrm, kap, alp, knn, nnd, degen, nhard + 1, nhard,
                                                             pts_c);
    LSG_CUDA(cudaGetLastError());
    return finish_launch(d_xyz, nrm, alp, nnd, degen, M, p.volume_margin, ws, L, st1, d_target, stream);
}

int prepare_target_impl(const float* d_xyz, int64_t M, const lsgcpd_prep_params& p, void* d_target, void* d_ws,
                        lsgcpd_target_info* info, const lsgcpd_annotations* ann, cudaStream_t stream) {
    const PrepLayout L = prep_layout(M, true);
    char* ws = static_cast<char*>(d_ws);
    double* bp = reinterpret_cast<double*>(ws + L.blockpart);
    double* st1 = reinterpret_cast<double*>(ws + L.stats1);
    unsigned* ctr = reinterpret_cast<unsigned*>(ws + L.counter);
    LSG_CUDA(cudaMemsetAsync(ctr, 0, sizeof(unsigned) * 4, stream));
    cloud_stats_kernel<<<kRedBlocks, kRedThreads, 0, stream>>>(d_xyz, M, bp, st1, ctr);
    double s1[12];
    LSG_CUDA(cudaMemcpyAsync(s1, st1, sizeof(s1), cudaMemcpyDeviceToHost, stream));
    LSG_CUDA(cudaStreamSynchronize(stream));
    int rc = prep_build(d_xyz, M, p, s1, st1, d_target, ws, L, ann, stream);
    if (rc) return rc;
    TargetHeader h;
    LSG_CUDA(cudaMemcpyAsync(&h, d_target, sizeof(h), cudaMemcpyDeviceToHost, stream));
    LSG_CUDA(cudaStreamSynchronize(stream));
    return info_from_header(h, M, true, info);
}

// ---- lsgcpd_prepare_batch (NEXT-3 workloads): every stage launched once per wave of targets ------------
// The per-target chain above is ~35 launches and memsets; for hundreds of small clouds the host launch rate, not
// the GPU, set the time (550 clouds of 3,500 points: 70 ms, tools/prep_batch_time.py).  Here every stage runs
// once per wave of targets, blockIdx.y = the target within the wave, through the same device
// bodies with the same block decomposition per target (gridDim.x, blockIdx.x and thread roles unchanged), and the
// radix sorts become segmented sorts of the wave's concatenated keys (stable: the same permutations).  So each
// target is built byte for byte as lsgcpd_prepare_target builds it (tests/test_gpu_prepare.py).  A wave holds up
// to 64 targets (wave_size), each with a job region of the largest cloud's PrepLayout.
struct PrepJob {
    const float* xyz;
    int64_t M, M_pad;
    Grid g, gc, gb;
    int use_bulk;
    int64_t ncells, ncells_c, ncells_b;
    int64_t off;               // first entry of this target in its wave's concatenated sort buffers
    char* ws;                  // its workspace region (the PrepLayout of the largest cloud)
    const double* st1;         // its cloud statistics (device)
    TargetHeader* hdr;         // the target's sections
    float* body;
    float* tc;
    int32_t* slots;
};
struct WaveBufs {              // concatenated over a wave's targets: wave_span entries each
    int *kin, *vin;            // cell keys / point ids of the grid being built
    int *ks[3], *vs[3];        // sorted (keys, ids) of the fine, coarse and bulk grids
    uint64_t *mkin, *mkout;    // Morton keys
    int *mvin, *mvout;         // Morton ids → slot permutation
};
// targets per wave: up to 64, their job regions within ~512 MB of workspace (a 3,500-point cloud's region is
// ≈ 7.7 MB, dominated by the dense cell arrays), and a wave's sort buffers indexable by int
static int wave_size(int64_t mmax) {
    const size_t region = al(prep_layout(mmax, true).total);
    int64_t P = (int64_t)((size_t)512 << 20) / (int64_t)region;
    P = P < 1 ? 1 : (P > 64 ? 64 : P);
    while (P > 1 && P * mmax >= ((int64_t)1 << 31)) --P;
    return (int)P;
}

__global__ void __launch_bounds__(kRedThreads)
    cloud_stats_batch(const float* const* xyz, const int64_t* M, int b0, double* part, double* out, unsigned* ctr) {
    const int b = b0 + blockIdx.y;
    cloud_stats_body(xyz[b], M[b], part + (int64_t)b * kRedBlocks * 16, out + 16 * (int64_t)b, ctr + 4 * b);
}
// which: 0 fine, 1 coarse, 2 bulk grid
__device__ __forceinline__ const Grid& job_grid(const PrepJob& j, int which) {
    return which == 0 ? j.g : (which == 1 ? j.gc : j.gb);
}
__device__ __forceinline__ int* job_cstart(const PrepJob& j, const PrepLayout& L, int which) {
    return reinterpret_cast<int*>(j.ws + (which == 0 ? L.cstart : (which == 1 ? L.cstart_c : L.cstart_b)));
}
__device__ __forceinline__ int* job_cend(const PrepJob& j, const PrepLayout& L, int which) {
    return reinterpret_cast<int*>(j.ws + (which == 0 ? L.cend : (which == 1 ? L.cend_c : L.cend_b)));
}
__device__ __forceinline__ float4* job_pts(const PrepJob& j, const PrepLayout& L, int which) {
    return reinterpret_cast<float4*>(j.ws + (which == 0 ? L.pts_f : (which == 1 ? L.pts_c : L.pts_b)));
}
__global__ void cell_keys_batch(const PrepJob* __restrict__ J, WaveBufs W, int which) {
    const PrepJob& j = J[blockIdx.y];
    if (which == 2 && !j.use_bulk) return;
    cell_keys_body(j.xyz, j.M, job_grid(j, which), W.kin + j.off, W.vin + j.off);
}
// the dense cell arrays to -1 (the memset 0xff of the single-target chain); also clears the hard-point count and
// the model-statistics counter of the job region (the single-target chain zeroes it before its cloud statistics;
// block_reduce_store leaves it at 0 after each use)
__global__ void fill_cells_batch(const PrepJob* __restrict__ J, PrepLayout L, int which) {
    const PrepJob& j = J[blockIdx.y];
    if (which == 2 && !j.use_bulk) return;
    const int64_t n = which == 0 ? j.ncells : (which == 1 ? j.ncells_c : j.ncells_b);
    int* cs = job_cstart(j, L, which);
    int* ce = job_cend(j, L, which);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        cs[i] = -1;
        ce[i] = -1;
    }
    if (which == 0 && blockIdx.x == 0 && threadIdx.x == 0) {
        *reinterpret_cast<int*>(j.ws + L.hard) = 0;
        *reinterpret_cast<unsigned*>(j.ws + L.counter) = 0u;
    }
}
__global__ void cell_ranges_batch(const PrepJob* __restrict__ J, PrepLayout L, WaveBufs W, int which) {
    const PrepJob& j = J[blockIdx.y];
    if (which == 2 && !j.use_bulk) return;
    cell_ranges_body(W.ks[which] + j.off, j.M, job_cstart(j, L, which), job_cend(j, L, which));
}
__global__ void gather_pts_batch(const PrepJob* __restrict__ J, PrepLayout L, WaveBufs W, int which) {
    const PrepJob& j = J[blockIdx.y];
    if (which == 2 && !j.use_bulk) return;
    gather_pts_body(j.xyz, W.vs[which] + j.off, j.M, job_pts(j, L, which));
}
__global__ void __launch_bounds__(128)
    knn_surface_batch(const PrepJob* __restrict__ J, PrepLayout L, WaveBufs W, int k, float alpha_max, float lambda) {
    const PrepJob& j = J[blockIdx.y];
    if ((int64_t)blockIdx.x * blockDim.x >= j.M) return;
    char* ws = j.ws;
    int* nhard = reinterpret_cast<int*>(ws + L.hard);
    knn_surface_body(j.xyz, j.M, j.g, W.vs[0] + j.off, job_cstart(j, L, 0), job_cend(j, L, 0), j.gc,
                     W.vs[1] + j.off, job_cstart(j, L, 1), job_cend(j, L, 1), j.gb, W.vs[2] + j.off,
                     job_cstart(j, L, 2), job_cend(j, L, 2), j.use_bulk, k, alpha_max, lambda,
                     reinterpret_cast<float*>(ws + L.nrm), reinterpret_cast<float*>(ws + L.kappa),
                     reinterpret_cast<float*>(ws + L.alpha), nullptr, reinterpret_cast<float*>(ws + L.nnd),
                     reinterpret_cast<int*>(ws + L.degen), nhard + 1, nhard, job_pts(j, L, 0), job_pts(j, L, 2));
}
__global__ void __launch_bounds__(128)
    knn_hard_batch(const PrepJob* __restrict__ J, PrepLayout L, WaveBufs W, int k, float alpha_max, float lambda) {
    const PrepJob& j = J[blockIdx.y];
    char* ws = j.ws;
    const int* nhard = reinterpret_cast<const int*>(ws + L.hard);
    knn_hard_body(j.xyz, j.gc, W.vs[1] + j.off, job_cstart(j, L, 1), job_cend(j, L, 1), k, alpha_max, lambda,
                  reinterpret_cast<float*>(ws + L.nrm), reinterpret_cast<float*>(ws + L.kappa),
                  reinterpret_cast<float*>(ws + L.alpha), nullptr, reinterpret_cast<float*>(ws + L.nnd),
                  reinterpret_cast<int*>(ws + L.degen), nhard + 1, nhard, job_pts(j, L, 1));
}
__global__ void __launch_bounds__(kRedThreads) model_stats_batch(const PrepJob* __restrict__ J, PrepLayout L) {
    const PrepJob& j = J[blockIdx.y];
    char* ws = j.ws;
    model_stats_body(j.xyz, reinterpret_cast<const float*>(ws + L.nrm), reinterpret_cast<const float*>(ws + L.alpha),
                     reinterpret_cast<const float*>(ws + L.nnd), reinterpret_cast<const int*>(ws + L.degen), j.M,
                     j.st1, reinterpret_cast<double*>(ws + L.blockpart), reinterpret_cast<double*>(ws + L.stats2),
                     reinterpret_cast<unsigned*>(ws + L.counter));
}
__global__ void header_batch(const PrepJob* __restrict__ J, PrepLayout L, double margin) {
    const PrepJob& j = J[blockIdx.y];
    header_body(j.hdr, j.M, j.st1, reinterpret_cast<const double*>(j.ws + L.stats2), margin, 1);
}
__global__ void morton_keys_batch(const PrepJob* __restrict__ J, WaveBufs W) {
    const PrepJob& j = J[blockIdx.y];
    morton_keys_body(j.xyz, j.M, j.st1, W.mkin + j.off, W.mvin + j.off);
}
__global__ void slot_inverse_batch(const PrepJob* __restrict__ J, WaveBufs W) {
    const PrepJob& j = J[blockIdx.y];
    slot_inverse_body(W.mvout + j.off, j.M, j.M_pad, j.slots);
}
__global__ void pack_record_batch(const PrepJob* __restrict__ J, PrepLayout L, WaveBufs W) {
    const PrepJob& j = J[blockIdx.y];
    pack_record_body(j.xyz, reinterpret_cast<const float*>(j.ws + L.nrm), reinterpret_cast<const float*>(j.ws + L.alpha),
                     W.mvout + j.off, j.M, j.M_pad, reinterpret_cast<const double*>(j.ws + L.stats2), j.body);
}
__global__ void __launch_bounds__(kTcTile) pack_tc_batch(const PrepJob* __restrict__ J, PrepLayout L, WaveBufs W) {
    const PrepJob& j = J[blockIdx.y];
    if ((int64_t)blockIdx.x >= j.M_pad / kTcTile) return;   // the whole CTA: no thread reaches the body's barriers
    pack_tc_body(j.xyz, reinterpret_cast<const float*>(j.ws + L.nrm), reinterpret_cast<const float*>(j.ws + L.alpha),
                 W.mvout + j.off, j.M, reinterpret_cast<const double*>(j.ws + L.stats2), j.tc);
}

// Workspace of lsgcpd_prepare_batch: [stats B×16 | cloud partials B×kRedBlocks×16 | counters B×4 | jobs B |
// segment offsets 3×B | cloud pointers + sizes B | wave sort buffers | cub temp | wave job regions]
struct BatchWs {
    size_t stats, part, ctr, jobs, seg, xyzp, msz, wave, cub, regions, total;
    int P;
    int64_t span;              // entries per wave sort buffer (P × largest cloud)
    size_t cub_bytes;
};
static BatchWs batch_ws(const int64_t* M, int B) {
    int64_t mmax = 1;
    for (int b = 0; b < B; ++b) mmax = M[b] > mmax ? M[b] : mmax;
    BatchWs w;
    w.P = wave_size(mmax);
    if (w.P > B) w.P = B;
    w.span = (int64_t)w.P * mmax;
    size_t c1 = 0, c2 = 0;
    cub::DeviceSegmentedRadixSort::SortPairs(nullptr, c1, (const int*)nullptr, (int*)nullptr, (const int*)nullptr,
                                             (int*)nullptr, (int)w.span, w.P, (const int*)nullptr, (const int*)nullptr,
                                             0, 22);
    cub::DeviceSegmentedRadixSort::SortPairs(nullptr, c2, (const uint64_t*)nullptr, (uint64_t*)nullptr,
                                             (const int*)nullptr, (int*)nullptr, (int)w.span, w.P, (const int*)nullptr,
                                             (const int*)nullptr, 0, 63);
    w.cub_bytes = c1 > c2 ? c1 : c2;
    size_t o = 0;
    w.stats = o; o += al(sizeof(double) * 16 * (size_t)B);
    w.part = o; o += al(sizeof(double) * kRedBlocks * 16 * (size_t)B);
    w.ctr = o; o += al(sizeof(unsigned) * 4 * (size_t)B);
    w.jobs = o; o += al(sizeof(PrepJob) * (size_t)B);
    w.seg = o; o += al(sizeof(int) * 3 * (size_t)B);
    w.xyzp = o; o += al(sizeof(float*) * (size_t)B);
    w.msz = o; o += al(sizeof(int64_t) * (size_t)B);
    w.wave = o; o += al((sizeof(int) * 8 + sizeof(uint64_t) * 2 + sizeof(int) * 2) * (size_t)w.span);
    w.cub = o; o += al(w.cub_bytes);
    w.regions = o; o += (size_t)w.P * al(prep_layout(mmax, true).total);
    w.total = o;
    return w;
}
size_t prepare_batch_ws_bytes(const int64_t* M, int B) { return batch_ws(M, B).total; }

int prepare_batch_impl(const float* const* xyz, const int64_t* M, int B, const lsgcpd_prep_params& p,
                       void* const* targets, void* d_ws, lsgcpd_target_info* info, cudaStream_t stream) {
    const BatchWs w = batch_ws(M, B);
    int64_t mmax = 1;
    for (int b = 0; b < B; ++b) mmax = M[b] > mmax ? M[b] : mmax;
    const PrepLayout L = prep_layout(mmax, true);
    char* ws = static_cast<char*>(d_ws);
    double* stats = reinterpret_cast<double*>(ws + w.stats);
    // 1. every cloud's statistics in one launch per 65,535 clouds; one host synchronisation
    LSG_CUDA(cudaMemsetAsync(ws + w.ctr, 0, sizeof(unsigned) * 4 * (size_t)B, stream));
    LSG_CUDA(cudaMemcpyAsync(ws + w.xyzp, xyz, sizeof(float*) * (size_t)B, cudaMemcpyHostToDevice, stream));
    LSG_CUDA(cudaMemcpyAsync(ws + w.msz, M, sizeof(int64_t) * (size_t)B, cudaMemcpyHostToDevice, stream));
    for (int b0 = 0; b0 < B; b0 += 65535) {
        const int nb = B - b0 < 65535 ? B - b0 : 65535;
        cloud_stats_batch<<<dim3(kRedBlocks, nb), kRedThreads, 0, stream>>>(
            reinterpret_cast<const float* const*>(ws + w.xyzp), reinterpret_cast<const int64_t*>(ws + w.msz), b0,
            reinterpret_cast<double*>(ws + w.part), stats, reinterpret_cast<unsigned*>(ws + w.ctr));
    }
    std::vector<double> hs(16 * (size_t)B);
    LSG_CUDA(cudaMemcpyAsync(hs.data(), stats, sizeof(double) * hs.size(), cudaMemcpyDeviceToHost, stream));
    LSG_CUDA(cudaStreamSynchronize(stream));
    // 2. every target's grids (host checks, naming the problem), its wave slot and segment
    std::vector<PrepJob> jobs(B);
    std::vector<int> seg(3 * (size_t)B);   // [begin | end | end of the bulk segment (empty without a bulk grid)]
    int64_t off = 0;
    for (int b = 0; b < B; ++b) {
        GridPlan P;
        const int rc = plan_grids(hs.data() + 16 * (size_t)b, M[b], P);
        if (rc) {
            char msg[1024];
            snprintf(msg, sizeof(msg), "problem %d: %s", b, lsgcpd_last_error());
            set_error("%s", msg);
            return rc;
        }
        if (b % w.P == 0) off = 0;
        PrepJob& j = jobs[b];
        j.xyz = xyz[b];
        j.M = M[b];
        j.M_pad = pad_targets(M[b]);
        j.g = P.g;
        j.gc = P.gc;
        j.gb = P.gb;
        j.use_bulk = P.use_bulk;
        j.ncells = P.ncells;
        j.ncells_c = P.ncells_c;
        j.ncells_b = P.ncells_b;
        j.off = off;
        j.ws = ws + w.regions + (size_t)(b % w.P) * al(L.total);
        j.st1 = stats + 16 * (size_t)b;
        j.hdr = reinterpret_cast<TargetHeader*>(targets[b]);
        j.body = target_body(targets[b]);
        j.tc = target_tc(targets[b], j.M_pad);
        j.slots = target_slots(targets[b], j.M_pad);
        seg[b] = (int)off;
        seg[B + b] = (int)(off + M[b]);
        seg[2 * (size_t)B + b] = (int)(P.use_bulk ? off + M[b] : off);
        off += M[b];
    }
    PrepJob* d_jobs = reinterpret_cast<PrepJob*>(ws + w.jobs);
    int* d_seg = reinterpret_cast<int*>(ws + w.seg);
    LSG_CUDA(cudaMemcpyAsync(d_jobs, jobs.data(), sizeof(PrepJob) * (size_t)B, cudaMemcpyHostToDevice, stream));
    LSG_CUDA(cudaMemcpyAsync(d_seg, seg.data(), sizeof(int) * seg.size(), cudaMemcpyHostToDevice, stream));
    WaveBufs W;
    {
        char* q = ws + w.wave;
        auto take = [&](size_t elem) { char* r = q; q += elem * (size_t)w.span; return r; };
        W.kin = reinterpret_cast<int*>(take(sizeof(int)));
        W.vin = reinterpret_cast<int*>(take(sizeof(int)));
        for (int g = 0; g < 3; ++g) {
            W.ks[g] = reinterpret_cast<int*>(take(sizeof(int)));
            W.vs[g] = reinterpret_cast<int*>(take(sizeof(int)));
        }
        W.mkin = reinterpret_cast<uint64_t*>(take(sizeof(uint64_t)));
        W.mkout = reinterpret_cast<uint64_t*>(take(sizeof(uint64_t)));
        W.mvin = reinterpret_cast<int*>(take(sizeof(int)));
        W.mvout = reinterpret_cast<int*>(take(sizeof(int)));
    }
    // 3. the waves: every stage once per wave (stream order separates the waves' uses of the job regions)
    for (int b0 = 0; b0 < B; b0 += w.P) {
        const int n = B - b0 < w.P ? B - b0 : w.P;
        const PrepJob* J = d_jobs + b0;
        int64_t wm = 1, wspan = 0, wcells = 1, wpad = kTcTile;
        for (int b = b0; b < b0 + n; ++b) {
            wm = M[b] > wm ? M[b] : wm;
            wspan += M[b];
            wcells = jobs[b].ncells > wcells ? jobs[b].ncells : wcells;
            wpad = jobs[b].M_pad > wpad ? jobs[b].M_pad : wpad;
        }
        const unsigned nb = (unsigned)((wm + 255) / 256);
        const unsigned nfill = (unsigned)std::min<int64_t>((wcells + 255) / 256, 1024);
        const int* beg = d_seg + b0;
        const int* end = d_seg + B + b0;
        const int* endb = d_seg + 2 * (size_t)B + b0;
        for (int g = 0; g < 3; ++g) {
            if (g == 2) {
                bool any = false;
                for (int b = b0; b < b0 + n; ++b) any = any || jobs[b].use_bulk;
                if (!any) break;
            }
            cell_keys_batch<<<dim3(nb, n), 256, 0, stream>>>(J, W, g);
            size_t cb = w.cub_bytes;
            LSG_CUDA(cub::DeviceSegmentedRadixSort::SortPairs(ws + w.cub, cb, W.kin, W.ks[g], W.vin, W.vs[g], (int)wspan,
                                                              n, beg, g == 2 ? endb : end, 0, 22, stream));
            fill_cells_batch<<<dim3(nfill, n), 256, 0, stream>>>(J, L, g);
            cell_ranges_batch<<<dim3(nb, n), 256, 0, stream>>>(J, L, W, g);
            gather_pts_batch<<<dim3(nb, n), 256, 0, stream>>>(J, L, W, g);
        }
        knn_surface_batch<<<dim3((unsigned)((wm + 127) / 128), n), 128, 0, stream>>>(J, L, W, p.knn_k, p.alpha_max,
                                                                                    p.lambda);
        knn_hard_batch<<<dim3(8, n), 128, 0, stream>>>(J, L, W, p.knn_k, p.alpha_max, p.lambda);
        model_stats_batch<<<dim3(kRedBlocks, n), kRedThreads, 0, stream>>>(J, L);
        header_batch<<<dim3(1, n), 1, 0, stream>>>(J, L, p.volume_margin);
        morton_keys_batch<<<dim3(nb, n), 256, 0, stream>>>(J, W);
        size_t cb = w.cub_bytes;
        LSG_CUDA(cub::DeviceSegmentedRadixSort::SortPairs(ws + w.cub, cb, W.mkin, W.mkout, W.mvin, W.mvout, (int)wspan,
                                                          n, beg, end, 0, 63, stream));
        const unsigned np = (unsigned)((wpad + 255) / 256);
        slot_inverse_batch<<<dim3(np, n), 256, 0, stream>>>(J, W);
        pack_record_batch<<<dim3(np, n), 256, 0, stream>>>(J, L, W);
        pack_tc_batch<<<dim3((unsigned)(wpad / kTcTile), n), kTcTile, 0, stream>>>(J, L, W);
        LSG_CUDA(cudaGetLastError());
    }
    // 4. every header, one host synchronisation
    std::vector<TargetHeader> hh(B);
    for (int b = 0; b < B; ++b)
        LSG_CUDA(cudaMemcpyAsync(&hh[b], targets[b], sizeof(TargetHeader), cudaMemcpyDeviceToHost, stream));
    LSG_CUDA(cudaStreamSynchronize(stream));
    for (int b = 0; b < B; ++b) {
        const int rc = info_from_header(hh[b], M[b], true, info ? info + b : nullptr);
        if (rc) {
            char msg[1024];
            snprintf(msg, sizeof(msg), "problem %d: %s", b, lsgcpd_last_error());
            set_error("%s", msg);
            return rc;
        }
    }
    return 0;
}

// ---- confidence filtering (Eq. 8) ----------------------------------------------------------
// Component prior π(m) = φ(y_m)/Σφ folds into the per-target log2 weight: ω_m = ½log2(1+α_m) + log2(M π(m))
// (the E step's constant keeps ln((1-w)/M)), re-referenced to ω_ref = max_m ω_m.  α_m = tr(α n nᵀ) is read
// back from the packed model, so the call is idempotent (it never compounds an earlier prior).
__device__ __forceinline__ double packed_alpha(const float* __restrict__ body, int64_t m) {
    const float* b = body + (m >> 1) * (2 * kTgtFloats) + (m & 1);
    return (double)b[2 * 7] + (double)b[2 * 10] + (double)b[2 * 12];   // W_xx + W_yy + W_zz
}

__global__ void __launch_bounds__(kRedThreads)
    prior_sum_kernel(const float* __restrict__ phi, int64_t M, double* blockpart, double* out, unsigned* counter) {
    double v[4] = {-INFINITY, -INFINITY, 0.0, 0.0};   // [max φ, -min φ, Σ φ, #invalid]
    for (int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; m < M; m += (int64_t)gridDim.x * blockDim.x) {
        const double f = phi[m];
        if (isfinite(f) && f >= 0.0) {
            v[0] = fmax(v[0], f);
            v[1] = fmax(v[1], -f);
            v[2] += f;
        } else {
            v[3] += 1.0;
        }
    }
    block_reduce_store<4, 2, kRedThreads>(v, blockpart, out, counter);
}

// out: [max ω, Σ π √(1+α)]
__global__ void __launch_bounds__(kRedThreads)
    prior_stats_kernel(const float* __restrict__ phi, const float* __restrict__ body, const int32_t* __restrict__ slot_of,
                       int64_t M, const double* __restrict__ sums, double* blockpart, double* out, unsigned* counter) {
    double v[2] = {-INFINITY, 0.0};
    const double inv = 1.0 / sums[2];
    for (int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; m < M; m += (int64_t)gridDim.x * blockDim.x) {
        const double pi = (double)phi[m] * inv;
        const double a = packed_alpha(body, slot_of[m]);
        if (pi > 0.0) v[0] = fmax(v[0], 0.5 * log2(1.0 + a) + log2((double)M * pi));
        v[1] += pi * sqrt(1.0 + a);
    }
    block_reduce_store<2, 1, kRedThreads>(v, blockpart, out, counter);
}

__global__ void prior_write_kernel(const float* __restrict__ phi, float* __restrict__ body, float* __restrict__ tc,
                                   const int32_t* __restrict__ slot_of, int64_t M, const double* __restrict__ sums,
                                   const double* __restrict__ stats, TargetHeader* hdr) {
    const int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (m == 0) {
        hdr->omega_ref = stats[0];
        hdr->spc = stats[1];
        hdr->prior = (sums[0] != -sums[1]) ? 1u : 0u;   // max φ ≠ min φ: non-uniform
    }
    if (m >= M) return;
    const double pi = (double)phi[m] / sums[2];
    const int64_t sl = slot_of[m];
    const double a = packed_alpha(body, sl);
    const float om = pi > 0.0 ? (float)(0.5 * log2(1.0 + a) + log2((double)M * pi) - stats[0]) : -INFINITY;
    body[(sl >> 1) * (2 * kTgtFloats) + (sl & 1) + 2 * 3] = om;
    const int64_t tile = sl / kTcTile;
    const int jt = (int)(sl % kTcTile);
    float* core = reinterpret_cast<float*>(reinterpret_cast<char*>(tc) + tile * kTcTileBytes) + (jt >> 1) * 16 + (jt & 1);
    core[2 * 3] = om;
}

size_t prior_ws_bytes(int64_t M) {
    (void)M;
    return al(sizeof(double) * kRedBlocks * 4) + al(sizeof(double) * 8) + al(sizeof(unsigned) * 4);   // K ≤ 4
}

int set_prior_impl(void* d_target, int64_t M, const float* d_phi, void* d_ws, double* h_spc, cudaStream_t stream) {
    char* ws = static_cast<char*>(d_ws);
    double* bp = reinterpret_cast<double*>(ws);
    double* st = reinterpret_cast<double*>(ws + al(sizeof(double) * kRedBlocks * 4));
    unsigned* ctr = reinterpret_cast<unsigned*>(ws + al(sizeof(double) * kRedBlocks * 4) + al(sizeof(double) * 8));
    LSG_CUDA(cudaMemsetAsync(ctr, 0, sizeof(unsigned) * 4, stream));
    prior_sum_kernel<<<kRedBlocks, kRedThreads, 0, stream>>>(d_phi, M, bp, st, ctr);
    double sums[4];
    LSG_CUDA(cudaMemcpyAsync(sums, st, sizeof(sums), cudaMemcpyDeviceToHost, stream));
    LSG_CUDA(cudaStreamSynchronize(stream));
    LSG_CHECK(sums[3] == 0.0, LSGCPD_EINVAL, "%lld target confidences are negative or non-finite", (long long)sums[3]);
    LSG_CHECK(sums[2] > 0.0 && isfinite(sums[2]), LSGCPD_EINVAL, "all target confidences are zero");
    const int64_t M_pad = pad_targets(M);
    float* body = target_body(d_target);
    const int32_t* slot_of = target_slots(d_target, M_pad);
    prior_stats_kernel<<<kRedBlocks, kRedThreads, 0, stream>>>(d_phi, body, slot_of, M, st, bp, st + 4, ctr);
    prior_write_kernel<<<(unsigned)((M + 255) / 256), 256, 0, stream>>>(d_phi, body, target_tc(d_target, M_pad),
                                                                        slot_of, M, st, st + 4,
                                                                        reinterpret_cast<TargetHeader*>(d_target));
    LSG_CUDA(cudaGetLastError());
    if (h_spc) {
        LSG_CUDA(cudaMemcpyAsync(h_spc, st + 5, sizeof(double), cudaMemcpyDeviceToHost, stream));
        LSG_CUDA(cudaStreamSynchronize(stream));
    }
    return 0;
}

// ---- confidence truncation and the depth error model (reading R23) ----------------------------
__global__ void select_flags_kernel(const float* __restrict__ phi, int64_t n, float thr, int* __restrict__ flags) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) flags[i] = phi[i] >= thr ? 1 : 0;
}
__global__ void select_scatter_kernel(const float* __restrict__ xyz, const float* __restrict__ phi, int64_t n,
                                      const int* __restrict__ flags, const int* __restrict__ pos,
                                      float* __restrict__ xyz_out, float* __restrict__ phi_out, int64_t* count) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (i == n - 1) *count = (int64_t)pos[i] + flags[i];
    if (!flags[i]) return;
    const int64_t o = pos[i];
    xyz_out[3 * o] = xyz[3 * i];
    xyz_out[3 * o + 1] = xyz[3 * i + 1];
    xyz_out[3 * o + 2] = xyz[3 * i + 2];
    if (phi_out) phi_out[o] = phi[i];
}

static size_t scan_tmp_bytes(int64_t n) {
    size_t b = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, b, (const int*)nullptr, (int*)nullptr, (int)n);
    return b;
}
size_t select_ws_bytes(int64_t n) {
    return al(sizeof(int) * n) * 2 + al(sizeof(int64_t)) + al(scan_tmp_bytes(n));
}

int select_confident_impl(const float* d_xyz, const float* d_phi, int64_t n, float threshold, float* d_xyz_out,
                          float* d_phi_out, int64_t* h_n_out, void* d_ws, cudaStream_t stream) {
    char* ws = static_cast<char*>(d_ws);
    int* flags = reinterpret_cast<int*>(ws);
    int* pos = reinterpret_cast<int*>(ws + al(sizeof(int) * n));
    int64_t* cnt = reinterpret_cast<int64_t*>(ws + 2 * al(sizeof(int) * n));
    void* tmp = ws + 2 * al(sizeof(int) * n) + al(sizeof(int64_t));
    size_t tb = scan_tmp_bytes(n);
    const unsigned g = (unsigned)((n + 255) / 256);
    select_flags_kernel<<<g, 256, 0, stream>>>(d_phi, n, threshold, flags);
    LSG_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, flags, pos, (int)n, stream));
    select_scatter_kernel<<<g, 256, 0, stream>>>(d_xyz, d_phi, n, flags, pos, d_xyz_out, d_phi_out, cnt);
    LSG_CUDA(cudaGetLastError());
    LSG_CUDA(cudaMemcpyAsync(h_n_out, cnt, sizeof(int64_t), cudaMemcpyDeviceToHost, stream));
    LSG_CUDA(cudaStreamSynchronize(stream));
    return 0;
}

// φ = e_min / e(z), e(z) = c0 + c1 z² of the camera-frame depth z (the point's third coordinate),
// e_min = e(z_min); clipped to [0, 1].
__global__ void depth_confidence_kernel(const float* __restrict__ xyz, int64_t n, double c0, double c1, double zmin,
                                        float* __restrict__ phi) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double z = xyz[3 * i + 2];
    const double f = (c0 + c1 * zmin * zmin) / (c0 + c1 * z * z);
    phi[i] = (float)fmin(fmax(isfinite(f) ? f : 0.0, 0.0), 1.0);
}
void depth_confidence_launch(const float* d_xyz, int64_t n, double c0, double c1, double z_min, float* d_phi,
                             cudaStream_t stream) {
    depth_confidence_kernel<<<(unsigned)((n + 255) / 256), 256, 0, stream>>>(d_xyz, n, c0, c1, z_min, d_phi);
}

}  // namespace lsg
