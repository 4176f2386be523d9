// Fused LSG-CPD E step for sm_100a (the hot path).
//
// For every source point x_n and every target component m (Eq. 5 with the Eq. 2
// densities; P is never materialised — the matrix form of P:266-304 is prior art):
//   r = x̂_n - y_m,  τ = ||r||² + α_m (n_m·r)²  (= σ² d_mn),  l̄ = ω̄_m - k2 τ  (log2 weight)
//   p = 2^{l̄ - μ}  with μ ≡ 0 (fixed mode: every l̄ ≤ 0 and the outlier term bounds the sum from
//   below) or a per-point running max (two-pass per tile, rescaling the accumulators on a raise).
//   Accumulate S = Σp, Σp y, Σp W, Σp b, Σp τ (14 numbers per point).
// Accuracy: each tile's 64 targets are summed into fresh registers, then folded into the running
// sums with Kahan compensation, so the FP32 rounding error does not grow with M.
// Work decomposition: stream-K over units (source block of B points, target tile of kTT targets);
// each persistent CTA owns a contiguous unit range and writes one partial per source block it
// touches; the merge kernel combines partials (log-sum-exp, FP64) and adds the outlier term once.
// Target tiles are staged in shared memory by 1-D TMA bulk copies (cp.async.bulk) through a
// kStages-deep mbarrier ring fed by a producer warp; consumers read targets with broadcast
// LDS.128.  Source points live in registers as FP32 hi/lo pairs of x̂ (computed in FP64).
// Arithmetic: packed f32x2 (FFMA2/FADD2/FMUL2) over two source points per instruction with the
// target field as a broadcast operand (PACKED), or scalar FP32 (reference variant).
#include "common.cuh"
#include "kernels.h"

namespace lsg {

constexpr int kTT = 64;                  // targets per pipeline stage (4 KB)
constexpr int kStages = 6;
constexpr int kPartF = 16;               // partial: S, Sy[3], SW[6], Sb[3], Sτ, μ, 0
constexpr int kAcc = 14;

// ---- accumulators ------------------------------------------------------------------------------
// A register "lane" of type T is float (scalar mode) or float2 (two source points).
template <typename T>
struct Acc {
    T v[kAcc];  // S, yx, yy, yz, W0..W5, bx, by, bz, τ
};

__device__ __forceinline__ float2 bc(float v) { return make_float2(v, v); }
__device__ __forceinline__ float vadd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float2 vadd(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float vsub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float2 vsub(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
__device__ __forceinline__ float vmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float2 vmul(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float vfma(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ float2 vfma(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float splat(float v, float) { return v; }
__device__ __forceinline__ float2 splat(float v, float2) { return bc(v); }
__device__ __forceinline__ float vzero(float) { return 0.f; }
__device__ __forceinline__ float2 vzero(float2) { return make_float2(0.f, 0.f); }

template <typename T>
__device__ __forceinline__ void acc_zero(Acc<T>& a) {
#pragma unroll
    for (int i = 0; i < kAcc; ++i) a.v[i] = vzero(T());
}
template <typename T>
__device__ __forceinline__ void acc_scale(Acc<T>& a, T s) {
#pragma unroll
    for (int i = 0; i < kAcc; ++i) a.v[i] = vmul(a.v[i], s);
}
// R += L with Kahan compensation C (true running sum ≈ R - C).
template <typename T>
__device__ __forceinline__ void acc_fold(Acc<T>& R, Acc<T>& C, const Acc<T>& L) {
#pragma unroll
    for (int i = 0; i < kAcc; ++i) {
        const T y = vsub(L.v[i], C.v[i]);
        const T t = vadd(R.v[i], y);
        C.v[i] = vsub(vsub(t, R.v[i]), y);
        R.v[i] = t;
    }
}

// Target m of a tile, unpacked from the pair-interleaved layout: float4 k of a pair block holds
// {f_a, f_b, (f+1)_a, (f+1)_b} for fields f = 2k.
struct Tgt {
    float y0, y1, y2, om, n0, n1, n2, w0, w1, w2, w3, w4, w5, b0, b1, b2;
};
__device__ __forceinline__ void load_pair(const float4* tp, Tgt& a, Tgt& b) {
    const float4 v0 = tp[0], v1 = tp[1], v2 = tp[2], v3 = tp[3], v4 = tp[4], v5 = tp[5], v6 = tp[6], v7 = tp[7];
    a = {v0.x, v0.z, v1.x, v1.z, v2.x, v2.z, v3.x, v3.z, v4.x, v4.z, v5.x, v5.z, v6.x, v6.z, v7.x, v7.z};
    b = {v0.y, v0.w, v1.y, v1.w, v2.y, v2.w, v3.y, v3.w, v4.y, v4.w, v5.y, v5.w, v6.y, v6.w, v7.y, v7.w};
}

// τ = ||r||² + (ñ·r)² with r = (hi - y) + lo: the subtraction of two nearby FP32 values is exact,
// so r is accurate relative to ||r|| rather than ||x̂||.
template <typename T>
__device__ __forceinline__ T pair_tau(const T (&h)[3], const T (&l)[3], const Tgt& t) {
    const T rx = vadd(vsub(h[0], splat(t.y0, T())), l[0]);
    const T ry = vadd(vsub(h[1], splat(t.y1, T())), l[1]);
    const T rz = vadd(vsub(h[2], splat(t.y2, T())), l[2]);
    const T q = vfma(splat(t.n2, T()), rz, vfma(splat(t.n1, T()), ry, vmul(splat(t.n0, T()), rx)));
    return vfma(q, q, vfma(rz, rz, vfma(ry, ry, vmul(rx, rx))));
}
template <typename T>
__device__ __forceinline__ void acc_add(Acc<T>& a, T p, T tau, const Tgt& t) {
    a.v[0] = vadd(a.v[0], p);
    a.v[1] = vfma(p, splat(t.y0, T()), a.v[1]);
    a.v[2] = vfma(p, splat(t.y1, T()), a.v[2]);
    a.v[3] = vfma(p, splat(t.y2, T()), a.v[3]);
    a.v[4] = vfma(p, splat(t.w0, T()), a.v[4]);
    a.v[5] = vfma(p, splat(t.w1, T()), a.v[5]);
    a.v[6] = vfma(p, splat(t.w2, T()), a.v[6]);
    a.v[7] = vfma(p, splat(t.w3, T()), a.v[7]);
    a.v[8] = vfma(p, splat(t.w4, T()), a.v[8]);
    a.v[9] = vfma(p, splat(t.w5, T()), a.v[9]);
    a.v[10] = vfma(p, splat(t.b0, T()), a.v[10]);
    a.v[11] = vfma(p, splat(t.b1, T()), a.v[11]);
    a.v[12] = vfma(p, splat(t.b2, T()), a.v[12]);
    a.v[13] = vfma(p, tau, a.v[13]);
}
__device__ __forceinline__ float vex2(float e) { return ex2_approx(e); }
__device__ __forceinline__ float2 vex2(float2 e) { return make_float2(ex2_approx(e.x), ex2_approx(e.y)); }
__device__ __forceinline__ float vmaxs(float a, float b) { return fmaxf(a, b); }
__device__ __forceinline__ float2 vmaxs(float2 a, float2 b) { return make_float2(fmaxf(a.x, b.x), fmaxf(a.y, b.y)); }
__device__ __forceinline__ float lane_of(float v, int) { return v; }
__device__ __forceinline__ float lane_of(float2 v, int i) { return i ? v.y : v.x; }
__device__ __forceinline__ void set_lane(float& v, int, float x) { v = x; }
__device__ __forceinline__ void set_lane(float2& v, int i, float x) {
    if (i) v.y = x; else v.x = x;
}

template <bool kLiteral, typename T>
__device__ __forceinline__ T log_weight(T tau, const Tgt& t, float k2) {
    return kLiteral ? vmul(splat(-k2, T()), tau) : vfma(splat(-k2, T()), tau, splat(t.om, T()));
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
// Producer-side wait: the thread is suspended until the phase flips (or the time hint elapses)
// instead of spinning and stealing issue slots from the consumer warps of its SM sub-partition.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAITS_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
        "@!P1 bra WAITS_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(1000000u)
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
// PPT source points per consumer thread (PPT / W register lanes of type float or float2),
// NCW consumer warps + 1 producer warp per CTA.
template <int PPT, int NCW, int MINB, bool PACKED, bool kLiteral>
__global__ void __launch_bounds__((NCW + 1) * 32, MINB)
    estep_kernel(const float* __restrict__ tgt, const float* __restrict__ src, int64_t N,
                 const IterState* __restrict__ st, Sched sc, float* __restrict__ part) {
    using T = typename std::conditional<PACKED, float2, float>::type;
    constexpr int W = PACKED ? 2 : 1;        // source points per register lane
    constexpr int NL = PPT / W;              // register lanes per thread
    static_assert(PPT % W == 0, "PPT must be a multiple of the lane width");
    constexpr int kBlk = NCW * 32 * PPT;
    constexpr int kTileF4 = kTT * kTgtFloats / 4;   // float4 per tile
    __shared__ __align__(128) float4 tiles[kStages * kTileF4];
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
            mbar_init(&empty_bar[s], NCW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == NCW) {
        // ---------------- producer warp: TMA bulk copies of target tiles ----------------
        if (lane == 0) {
            int64_t it = 0;
            for (int64_t u = u0; u < u1; ++u, ++it) {
                const int s = (int)(it % kStages);
                const uint32_t ph = (uint32_t)((it / kStages) & 1);
                mbar_wait_sleep(&empty_bar[s], ph ^ 1);
                const int64_t tile = u % sc.T;
                mbar_arrive_expect_tx(&full_bar[s], kTT * kTgtFloats * 4);
                bulk_g2s(&tiles[s * kTileF4], tgt + tile * (int64_t)kTT * kTgtFloats, kTT * kTgtFloats * 4,
                         &full_bar[s]);
            }
        }
        return;
    }

    // ---------------- consumer warps ----------------
    const int tid = threadIdx.x;  // 0 .. NCW*32-1
    const float k2 = st->k2;
    const bool fixed = st->fixed != 0;
    const float Lo_f = (float)st->Lo;
    double Rm[9], tv[3];
#pragma unroll
    for (int i = 0; i < 9; ++i) Rm[i] = st->R[i];
#pragma unroll
    for (int i = 0; i < 3; ++i) tv[i] = st->t[i];

    Acc<T> R[NL], C[NL];
    T h[NL][3], l[NL][3], mu[NL];
    int64_t cur_blk = -1;

    // point k of register lane L is local point (L*W + k)*(NCW*32) + tid
    auto load_points = [&](int64_t j) {
#pragma unroll
        for (int L = 0; L < NL; ++L) {
#pragma unroll
            for (int k = 0; k < W; ++k) {
                const int64_t n = j * kBlk + (int64_t)(L * W + k) * (NCW * 32) + tid;
                double x0 = 0.0, x1 = 0.0, x2 = 0.0;
                if (n < N) {
                    x0 = src[3 * n];
                    x1 = src[3 * n + 1];
                    x2 = src[3 * n + 2];
                }
                const double X[3] = {fma(Rm[0], x0, fma(Rm[1], x1, fma(Rm[2], x2, tv[0]))),
                                     fma(Rm[3], x0, fma(Rm[4], x1, fma(Rm[5], x2, tv[1]))),
                                     fma(Rm[6], x0, fma(Rm[7], x1, fma(Rm[8], x2, tv[2])))};
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    const float hi = __double2float_rn(X[a]);
                    set_lane(h[L][a], k, hi);
                    set_lane(l[L][a], k, __double2float_rn(X[a] - (double)hi));
                }
                set_lane(mu[L], k, fixed ? 0.f : (isinf(Lo_f) ? -1e30f : Lo_f));
            }
            acc_zero(R[L]);
            acc_zero(C[L]);
        }
    };
    auto flush = [&](int64_t j) {
        const int64_t slot = j * sc.kmax + (g - sched_owner(sc, j * sc.T));
        float* base = part + slot * (int64_t)kPartF * kBlk;
#pragma unroll
        for (int L = 0; L < NL; ++L)
#pragma unroll
            for (int k = 0; k < W; ++k) {
                const int b = (L * W + k) * (NCW * 32) + tid;
#pragma unroll
                for (int f = 0; f < kAcc; ++f)
                    base[f * kBlk + b] = __fsub_rn(lane_of(R[L].v[f], k), lane_of(C[L].v[f], k));
                base[14 * kBlk + b] = lane_of(mu[L], k);
                base[15 * kBlk + b] = 0.f;
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
        const float4* tl = &tiles[s * kTileF4];
        Acc<T> Lt[NL];
#pragma unroll
        for (int L = 0; L < NL; ++L) acc_zero(Lt[L]);
        if (fixed) {
#pragma unroll 2
            for (int pr = 0; pr < kTT / 2; ++pr) {
                Tgt ta, tb;
                load_pair(tl + 8 * pr, ta, tb);
#pragma unroll
                for (int hsel = 0; hsel < 2; ++hsel) {
                    const Tgt& t = hsel ? tb : ta;
#pragma unroll
                    for (int L = 0; L < NL; ++L) {
                        const T tau = pair_tau(h[L], l[L], t);
                        const T p = vex2(log_weight<kLiteral>(tau, t, k2));
                        acc_add(Lt[L], p, tau, t);
                    }
                }
            }
        } else {
            // pass 1: tile maximum of the log weights per point; rescale the running sums on a raise
            T tmax[NL];
#pragma unroll
            for (int L = 0; L < NL; ++L) tmax[L] = splat(-INFINITY, T());
            for (int pr = 0; pr < kTT / 2; ++pr) {
                Tgt ta, tb;
                load_pair(tl + 8 * pr, ta, tb);
#pragma unroll
                for (int hsel = 0; hsel < 2; ++hsel) {
                    const Tgt& t = hsel ? tb : ta;
#pragma unroll
                    for (int L = 0; L < NL; ++L)
                        tmax[L] = vmaxs(tmax[L], log_weight<kLiteral>(pair_tau(h[L], l[L], t), t, k2));
                }
            }
#pragma unroll
            for (int L = 0; L < NL; ++L) {
                T f = splat(1.f, T());
                bool raise = false;
#pragma unroll
                for (int k = 0; k < W; ++k) {
                    const float m_old = lane_of(mu[L], k), m_new = fmaxf(m_old, lane_of(tmax[L], k));
                    if (m_new > m_old) {
                        set_lane(f, k, ex2_approx(m_old - m_new));
                        set_lane(mu[L], k, m_new);
                        raise = true;
                    }
                }
                if (raise) {
                    acc_scale(R[L], f);
                    acc_scale(C[L], f);
                }
            }
            // pass 2: accumulate with the (now fixed) per-point maximum
            for (int pr = 0; pr < kTT / 2; ++pr) {
                Tgt ta, tb;
                load_pair(tl + 8 * pr, ta, tb);
#pragma unroll
                for (int hsel = 0; hsel < 2; ++hsel) {
                    const Tgt& t = hsel ? tb : ta;
#pragma unroll
                    for (int L = 0; L < NL; ++L) {
                        const T tau = pair_tau(h[L], l[L], t);
                        const T p = vex2(vsub(log_weight<kLiteral>(tau, t, k2), mu[L]));
                        acc_add(Lt[L], p, tau, t);
                    }
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty_bar[s]);
#pragma unroll
        for (int L = 0; L < NL; ++L) acc_fold(R[L], C[L], Lt[L]);
    }
    if (cur_blk >= 0) flush(cur_blk);
}

// ---- merge: log-sum-exp over partials + outlier term → 16-float record -------------------
__global__ void estep_merge_kernel(const float* __restrict__ part, int64_t N, const IterState* __restrict__ st,
                                   Sched sc, float* __restrict__ rec) {
    if (!st->active) return;
    const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= N) return;
    const int64_t kB = sc.B;
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
    double a[kAcc];
#pragma unroll
    for (int f = 0; f < kAcc; ++f) a[f] = 0.0;
    for (int64_t k = 0; k < nk; ++k) {
        const float* base = part + (j * sc.kmax + k) * (int64_t)kPartF * kB;
        const double sc_k = exp2((double)base[14 * kB + b] - mustar);
#pragma unroll
        for (int f = 0; f < kAcc; ++f) a[f] += sc_k * (double)base[f * kB + b];
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
// Kernel variants (points per thread, consumer warps, min CTAs/SM, packed).  LSGCPD_ESTEP_VARIANT
// selects one (tuning/benchmarking); the default is the fastest measured on B200.
struct Variant {
    int ppt, ncw, minb, packed;
    const void* fn[2];  // [literal]
};
#define LSG_VARIANT(P, W, B, X) \
    {P, W, B, X, {(const void*)estep_kernel<P, W, B, X, false>, (const void*)estep_kernel<P, W, B, X, true>}}
static const Variant kVariants[] = {
    LSG_VARIANT(2, 16, 1, true), LSG_VARIANT(2, 8, 2, true), LSG_VARIANT(4, 8, 1, true), LSG_VARIANT(2, 12, 1, true),
    LSG_VARIANT(4, 4, 2, true),  LSG_VARIANT(2, 8, 2, false), LSG_VARIANT(1, 16, 1, false),
};
constexpr int kNumVariants = sizeof(kVariants) / sizeof(kVariants[0]);
constexpr int kDefaultVariant = 3;   // packed, 2 points/thread, 12 consumer warps (tools/estep_speed.py)

static int variant_index() {
    const char* e = getenv("LSGCPD_ESTEP_VARIANT");
    int v = e ? atoi(e) : kDefaultVariant;
    return (v >= 0 && v < kNumVariants) ? v : kDefaultVariant;
}

static int g_num_sms = 0;
static int g_occ[kNumVariants] = {0};

int estep_plan(int64_t M_pad, int64_t N, Sched* sc) {
    const int vi = variant_index();
    const Variant& V = kVariants[vi];
    if (g_num_sms == 0) {
        int dev;
        LSG_CUDA(cudaGetDevice(&dev));
        LSG_CUDA(cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev));
    }
    if (g_occ[vi] == 0) {
        int occ = 0;
        LSG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, V.fn[0], (V.ncw + 1) * 32, 0));
        g_occ[vi] = occ > 0 ? occ : 1;
    }
    Sched s;
    s.variant = vi;
    s.B = (int64_t)V.ppt * V.ncw * 32;
    s.nblk = (N + s.B - 1) / s.B;
    s.T = M_pad / kTT;
    s.U = s.nblk * s.T;
    const int64_t slots = (int64_t)g_num_sms * g_occ[vi];
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

size_t estep_partial_bytes(const Sched& s) { return (size_t)s.nblk * s.kmax * kPartF * s.B * sizeof(float); }

void estep_launch_setup(IterState* st, const void* d_target, const double* R, const double* t, double sigma2,
                        double w, double V, int64_t M, int consistent, cudaStream_t stream) {
    estep_setup_kernel<<<1, 1, 0, stream>>>(st, reinterpret_cast<const TargetHeader*>(d_target), R[0], R[1], R[2],
                                             R[3], R[4], R[5], R[6], R[7], R[8], t[0], t[1], t[2], sigma2, w, V, M,
                                             consistent);
}

void estep_launch(const void* d_target, const float* d_src, int64_t N, const IterState* st, const Sched& sc,
                  float* part, float* rec, int consistent, cudaStream_t stream) {
    const float* body = target_body(d_target);
    const Variant& V = kVariants[sc.variant];
    Sched scv = sc;
    void* args[] = {(void*)&body, (void*)&d_src, (void*)&N, (void*)&st, (void*)&scv, (void*)&part};
    cudaLaunchKernel(V.fn[consistent ? 0 : 1], dim3((unsigned)sc.G), dim3((V.ncw + 1) * 32), args, 0, stream);
    const int mt = 256;
    estep_merge_kernel<<<(unsigned)((N + mt - 1) / mt), mt, 0, stream>>>(part, N, st, sc, rec);
}

}  // namespace lsg
