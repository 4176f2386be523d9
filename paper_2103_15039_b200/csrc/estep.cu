// Fused LSG-CPD E step for sm_100a (the hot path).
//
// For every source point x_n and every target component m (Eq. 5 with the Eq. 2
// densities; P never materialised — prior art P:266-304 is the matrix form):
//   r = x̂_n - y_m,  τ = ||r||² + α_m (n_m·r)²  (= σ² d_mn),  l̄ = ω̄_m - k2 τ  (log2 weight)
//   p = 2^{l̄ - μ}  with μ ≡ 0 (fixed mode: all l̄ ≤ 0 and the outlier term bounds the sum from
//   below) or a running max (flash-softmax style, rescaling the accumulators on a raise).
//   Accumulate S = Σp, Σp y, Σp W, Σp b, Σp τ (14 floats per point, registers).
// Work decomposition: stream-K over units (source block of kB points, target tile of kTT
// targets); every persistent CTA owns a contiguous unit range and writes one partial per source
// block it touches; the merge kernel combines partials (log-sum-exp) and adds the outlier term.
// Target tiles are staged in shared memory by 1-D TMA bulk copies (cp.async.bulk) through a
// kStages-deep mbarrier ring fed by a dedicated producer warp; consumer warps read each target
// as 4 broadcast LDS.128.  Source points live in registers as FP32 hi/lo pairs of x̂ (FP64).
#include "common.cuh"
#include "kernels.h"

namespace lsg {

constexpr int kTT = 64;                  // targets per pipeline stage (4 KB)
constexpr int kStages = 6;
constexpr int kNCW = 8;                  // consumer warps
constexpr int kPPT = 2;                  // source points per consumer thread
constexpr int kB = kNCW * 32 * kPPT;     // source points per block (512)
constexpr int kThreads = (kNCW + 1) * 32;
constexpr int kPartF = 16;               // partial: S, Sy[3], SW[6], Sb[3], Sτ, μ, 0

struct PointAcc {
    float S, yx, yy, yz, w0, w1, w2, w3, w4, w5, bx, by, bz, tau;
};

__device__ __forceinline__ void acc_zero(PointAcc& a) {
    a.S = a.yx = a.yy = a.yz = a.w0 = a.w1 = a.w2 = a.w3 = a.w4 = a.w5 = a.bx = a.by = a.bz = a.tau = 0.f;
}
__device__ __forceinline__ void acc_scale(PointAcc& a, float s) {
    a.S *= s; a.yx *= s; a.yy *= s; a.yz *= s; a.w0 *= s; a.w1 *= s; a.w2 *= s; a.w3 *= s; a.w4 *= s;
    a.w5 *= s; a.bx *= s; a.by *= s; a.bz *= s; a.tau *= s;
}
__device__ __forceinline__ void acc_add(PointAcc& a, float p, float tau, const float4& T0, const float4& T1,
                                        const float4& T2, const float4& T3) {
    a.S += p;
    a.yx = fmaf(p, T0.x, a.yx);
    a.yy = fmaf(p, T0.y, a.yy);
    a.yz = fmaf(p, T0.z, a.yz);
    a.w0 = fmaf(p, T1.w, a.w0);
    a.w1 = fmaf(p, T2.x, a.w1);
    a.w2 = fmaf(p, T2.y, a.w2);
    a.w3 = fmaf(p, T2.z, a.w3);
    a.w4 = fmaf(p, T2.w, a.w4);
    a.w5 = fmaf(p, T3.x, a.w5);
    a.bx = fmaf(p, T3.y, a.bx);
    a.by = fmaf(p, T3.z, a.by);
    a.bz = fmaf(p, T3.w, a.bz);
    a.tau = fmaf(p, tau, a.tau);
}

// τ = ||r||² + (ñ·r)² with r = (hi - y) + lo: the subtraction of two nearby FP32 values is exact,
// so r is accurate relative to ||r|| rather than ||x̂||.
__device__ __forceinline__ float pair_tau(float hx, float hy, float hz, float lx, float ly, float lz,
                                          const float4& T0, const float4& T1) {
    const float rx = __fadd_rn(__fsub_rn(hx, T0.x), lx);
    const float ry = __fadd_rn(__fsub_rn(hy, T0.y), ly);
    const float rz = __fadd_rn(__fsub_rn(hz, T0.z), lz);
    const float q = fmaf(T1.z, rz, fmaf(T1.y, ry, T1.x * rx));
    return fmaf(q, q, fmaf(rz, rz, fmaf(ry, ry, rx * rx)));
}

// ---- mbarrier / bulk-copy PTX wrappers --------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// ---- setup: per-call constants (lsgcpd_estep path) ---------------------------------------
__global__ void estep_setup_kernel(IterState* st, const TargetHeader* hdr, double r0, double r1, double r2,
                                   double r3, double r4, double r5, double r6, double r7, double r8, double t0,
                                   double t1, double t2, double sigma2, double w, double V, int64_t M,
                                   int consistent) {
    const double R[9] = {r0, r1, r2, r3, r4, r5, r6, r7, r8};
    const double t[3] = {t0, t1, t2};
    IterState s;
    make_state(s, R, t, sigma2, w, V, M, hdr->omega_ref, consistent);
    s.extent = hdr->extent;
    s.active = 1;
    s.iter = 0;
    s.status = 0;
    s.no_mass = 0;
    s.last_step_rot = s.last_step_trans = 0.0;
    *st = s;
}

// ---- the fused E-step kernel -------------------------------------------------------------
template <bool kLiteral>
__global__ void __launch_bounds__(kThreads, 2)
    estep_kernel(const float* __restrict__ tgt, const float* __restrict__ src, int64_t N,
                 const IterState* __restrict__ st, Sched sc, float* __restrict__ part) {
    __shared__ __align__(128) float4 tiles[kStages][kTT * 4];
    __shared__ __align__(8) uint64_t full_bar[kStages];
    __shared__ __align__(8) uint64_t empty_bar[kStages];

    if (!st->active) return;
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t g = blockIdx.x;
    const int64_t u0 = sched_start(sc, g), u1 = sched_start(sc, g + 1);
    if (u0 >= u1) return;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], kNCW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == kNCW) {
        // ---------------- producer warp: TMA bulk copies of target tiles ----------------
        if (lane == 0) {
            int64_t it = 0;
            for (int64_t u = u0; u < u1; ++u, ++it) {
                const int s = (int)(it % kStages);
                const uint32_t ph = (uint32_t)((it / kStages) & 1);
                mbar_wait(&empty_bar[s], ph ^ 1);
                const int64_t tile = u % sc.T;
                mbar_arrive_expect_tx(&full_bar[s], kTT * kTgtFloats * 4);
                bulk_g2s(&tiles[s][0], tgt + tile * (int64_t)kTT * kTgtFloats, kTT * kTgtFloats * 4, &full_bar[s]);
            }
        }
        return;
    }

    // ---------------- consumer warps ----------------
    const int tid = threadIdx.x;  // 0 .. kNCW*32-1
    const float k2 = st->k2;
    const bool fixed = st->fixed != 0;
    const float Lo_f = (float)st->Lo;
    double Rm[9], tv[3];
#pragma unroll
    for (int i = 0; i < 9; ++i) Rm[i] = st->R[i];
#pragma unroll
    for (int i = 0; i < 3; ++i) tv[i] = st->t[i];

    PointAcc acc[kPPT];
    float hx[kPPT], hy[kPPT], hz[kPPT], lx[kPPT], ly[kPPT], lz[kPPT], mu[kPPT];
    int64_t cur_blk = -1;

    auto load_points = [&](int64_t j) {
#pragma unroll
        for (int k = 0; k < kPPT; ++k) {
            const int64_t n = j * kB + k * (kNCW * 32) + tid;
            double x0 = 0.0, x1 = 0.0, x2 = 0.0;
            if (n < N) {
                x0 = src[3 * n];
                x1 = src[3 * n + 1];
                x2 = src[3 * n + 2];
            }
            const double X0 = fma(Rm[0], x0, fma(Rm[1], x1, fma(Rm[2], x2, tv[0])));
            const double X1 = fma(Rm[3], x0, fma(Rm[4], x1, fma(Rm[5], x2, tv[1])));
            const double X2 = fma(Rm[6], x0, fma(Rm[7], x1, fma(Rm[8], x2, tv[2])));
            hx[k] = __double2float_rn(X0);
            hy[k] = __double2float_rn(X1);
            hz[k] = __double2float_rn(X2);
            lx[k] = __double2float_rn(X0 - (double)hx[k]);
            ly[k] = __double2float_rn(X1 - (double)hy[k]);
            lz[k] = __double2float_rn(X2 - (double)hz[k]);
            acc_zero(acc[k]);
            mu[k] = fixed ? 0.f : (isinf(Lo_f) ? -1e30f : Lo_f);
        }
    };
    auto flush = [&](int64_t j) {
        const int64_t slot = j * sc.kmax + (g - sched_owner(sc, j * sc.T));
        float* base = part + slot * (int64_t)kPartF * kB;
#pragma unroll
        for (int k = 0; k < kPPT; ++k) {
            const int b = k * (kNCW * 32) + tid;
            const PointAcc& a = acc[k];
            base[0 * kB + b] = a.S;
            base[1 * kB + b] = a.yx;
            base[2 * kB + b] = a.yy;
            base[3 * kB + b] = a.yz;
            base[4 * kB + b] = a.w0;
            base[5 * kB + b] = a.w1;
            base[6 * kB + b] = a.w2;
            base[7 * kB + b] = a.w3;
            base[8 * kB + b] = a.w4;
            base[9 * kB + b] = a.w5;
            base[10 * kB + b] = a.bx;
            base[11 * kB + b] = a.by;
            base[12 * kB + b] = a.bz;
            base[13 * kB + b] = a.tau;
            base[14 * kB + b] = mu[k];
            base[15 * kB + b] = 0.f;
        }
    };

    int64_t it = 0;
    for (int64_t u = u0; u < u1; ++u, ++it) {
        const int64_t j = u / sc.T;
        if (j != cur_blk) {
            if (cur_blk >= 0) flush(cur_blk);
            cur_blk = j;
            load_points(j);
        }
        const int s = (int)(it % kStages);
        mbar_wait(&full_bar[s], (uint32_t)((it / kStages) & 1));
        const float4* tl = &tiles[s][0];
        if (fixed) {
#pragma unroll 4
            for (int m = 0; m < kTT; ++m) {
                const float4 T0 = tl[4 * m + 0], T1 = tl[4 * m + 1], T2 = tl[4 * m + 2], T3 = tl[4 * m + 3];
#pragma unroll
                for (int k = 0; k < kPPT; ++k) {
                    const float tau = pair_tau(hx[k], hy[k], hz[k], lx[k], ly[k], lz[k], T0, T1);
                    const float e = kLiteral ? -k2 * tau : fmaf(-k2, tau, T0.w);
                    const float p = ex2_approx(e);
                    acc_add(acc[k], p, tau, T0, T1, T2, T3);
                }
            }
        } else {
            for (int m = 0; m < kTT; ++m) {
                const float4 T0 = tl[4 * m + 0], T1 = tl[4 * m + 1], T2 = tl[4 * m + 2], T3 = tl[4 * m + 3];
#pragma unroll
                for (int k = 0; k < kPPT; ++k) {
                    const float tau = pair_tau(hx[k], hy[k], hz[k], lx[k], ly[k], lz[k], T0, T1);
                    const float e = kLiteral ? -k2 * tau : fmaf(-k2, tau, T0.w);
                    if (e > mu[k]) {
                        acc_scale(acc[k], ex2_approx(mu[k] - e));
                        mu[k] = e;
                    }
                    const float p = ex2_approx(e - mu[k]);
                    acc_add(acc[k], p, tau, T0, T1, T2, T3);
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty_bar[s]);
    }
    if (cur_blk >= 0) flush(cur_blk);
}

// ---- merge: log-sum-exp over partials + outlier term → 16-float record -------------------
__global__ void estep_merge_kernel(const float* __restrict__ part, int64_t N, const IterState* __restrict__ st,
                                   Sched sc, float* __restrict__ rec) {
    if (!st->active) return;
    const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= N) return;
    const int64_t j = n / kB;
    const int b = (int)(n % kB);
    const int64_t g0 = sched_owner(sc, j * sc.T);
    const int64_t g1 = sched_owner(sc, (j + 1) * sc.T - 1);
    const int64_t nk = g1 - g0 + 1;
    double mustar = st->Lo;  // -inf when w == 0
    for (int64_t k = 0; k < nk; ++k) {
        const float* base = part + (j * sc.kmax + k) * (int64_t)kPartF * kB;
        mustar = fmax(mustar, (double)base[14 * kB + b]);
    }
    double a[14];
#pragma unroll
    for (int f = 0; f < 14; ++f) a[f] = 0.0;
    for (int64_t k = 0; k < nk; ++k) {
        const float* base = part + (j * sc.kmax + k) * (int64_t)kPartF * kB;
        const double sc_k = exp2((double)base[14 * kB + b] - mustar);
#pragma unroll
        for (int f = 0; f < 14; ++f) a[f] += sc_k * (double)base[f * kB + b];
    }
    const double O = (st->w > 0.0) ? exp2(st->Lo - mustar) : 0.0;
    const double Z = a[0] + O;
    const double iz = 1.0 / Z;
    float* r = rec + n * LSGCPD_REC;
    float4 o0, o1, o2, o3;
    o0.x = (float)(a[0] * iz);
    o0.y = (float)(a[1] * iz);
    o0.z = (float)(a[2] * iz);
    o0.w = (float)(a[3] * iz);
    o1.x = (float)(a[4] * iz);
    o1.y = (float)(a[5] * iz);
    o1.z = (float)(a[6] * iz);
    o1.w = (float)(a[7] * iz);
    o2.x = (float)(a[8] * iz);
    o2.y = (float)(a[9] * iz);
    o2.z = (float)(a[10] * iz);
    o2.w = (float)(a[11] * iz);
    o3.x = (float)(a[12] * iz);
    o3.y = (float)(a[13] * iz / st->sigma2);
    o3.z = (float)(st->C1 + 0.69314718055994530942 * (st->omega_ref + mustar + log2(Z)));
    o3.w = (float)(O * iz);
    reinterpret_cast<float4*>(r)[0] = o0;
    reinterpret_cast<float4*>(r)[1] = o1;
    reinterpret_cast<float4*>(r)[2] = o2;
    reinterpret_cast<float4*>(r)[3] = o3;
}

// ---- host-side planning and launch ---------------------------------------------------------
static int g_num_sms = 0;
static int g_occ = 0;

int estep_plan(int64_t M_pad, int64_t N, Sched* sc) {
    if (g_num_sms == 0) {
        int dev;
        LSG_CUDA(cudaGetDevice(&dev));
        LSG_CUDA(cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev));
        int occ = 0;
        LSG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, estep_kernel<false>, kThreads, 0));
        g_occ = occ > 0 ? occ : 1;
    }
    Sched s;
    s.nblk = (N + kB - 1) / kB;
    s.T = M_pad / kTT;
    s.U = s.nblk * s.T;
    const int64_t slots = (int64_t)g_num_sms * g_occ;
    s.G = s.U < slots ? s.U : slots;
    if (s.G < 1) s.G = 1;
    int64_t kmax = 1;
    for (int64_t j = 0; j < s.nblk; ++j) {
        const int64_t k = sched_owner(s, (j + 1) * s.T - 1) - sched_owner(s, j * s.T) + 1;
        if (k > kmax) kmax = k;
    }
    s.kmax = kmax;
    *sc = s;
    return 0;
}

size_t estep_partial_bytes(const Sched& s) { return (size_t)s.nblk * s.kmax * kPartF * kB * sizeof(float); }

// Upper bound of the partial buffer for any device (used by the *_workspace_bytes queries).
size_t estep_partial_bytes_bound(int64_t M_pad, int64_t N, int64_t max_ctas) {
    const int64_t nblk = (N + kB - 1) / kB;
    const int64_t T = M_pad / kTT;
    const int64_t U = nblk * T;
    const int64_t G = U < max_ctas ? U : max_ctas;
    const int64_t kmax = (T * G + U - 1) / U + 1;
    return (size_t)nblk * kmax * kPartF * kB * sizeof(float);
}

void estep_launch_setup(IterState* st, const void* d_target, const double* R, const double* t, double sigma2,
                        double w, double V, int64_t M, int consistent, cudaStream_t stream) {
    estep_setup_kernel<<<1, 1, 0, stream>>>(st, reinterpret_cast<const TargetHeader*>(d_target), R[0], R[1], R[2],
                                             R[3], R[4], R[5], R[6], R[7], R[8], t[0], t[1], t[2], sigma2, w, V, M,
                                             consistent);
}

void estep_launch(const void* d_target, const float* d_src, int64_t N, const IterState* st, const Sched& sc,
                  float* part, float* rec, int consistent, cudaStream_t stream) {
    const float* body = target_body(d_target);
    if (consistent)
        estep_kernel<false><<<(unsigned)sc.G, kThreads, 0, stream>>>(body, d_src, N, st, sc, part);
    else
        estep_kernel<true><<<(unsigned)sc.G, kThreads, 0, stream>>>(body, d_src, N, st, sc, part);
    const int mt = 256;
    estep_merge_kernel<<<(unsigned)((N + mt - 1) / mt), mt, 0, stream>>>(part, N, st, sc, rec);
}

}  // namespace lsg
