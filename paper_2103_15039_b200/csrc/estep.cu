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
#include <string.h>

#include "common.cuh"
#include "estep_dev.cuh"
#include "kernels.h"

namespace lsg {

// ---- setup: per-call constants (lsgcpd_estep path) ---------------------------------------
__global__ void estep_setup_kernel(IterState* st, const TargetHeader* hdr, double r0, double r1, double r2,
                                   double r3, double r4, double r5, double r6, double r7, double r8, double t0,
                                   double t1, double t2, double sigma2, double w, double V, int64_t M,
                                   int consistent, double eta) {
    const double R[9] = {r0, r1, r2, r3, r4, r5, r6, r7, r8};
    const double t[3] = {t0, t1, t2};
    IterState s;
    make_state(s, R, t, sigma2, w, V, M, hdr->omega_ref, consistent, eta, hdr->spc);
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
                 const IterState* __restrict__ st, Sched sc, float* __restrict__ part, int skip_fixed) {
    using T = typename std::conditional<PACKED, float2, float>::type;
    constexpr int W = PACKED ? 2 : 1;        // source points per register lane
    constexpr int NL = PPT / W;              // register lanes per thread
    static_assert(PPT % W == 0, "PPT must be a multiple of the lane width");
    constexpr int kBlk = NCW * 32 * PPT;
    constexpr int kTileF4 = kTT * kTgtFloats / 4;   // float4 per tile
    __shared__ __align__(128) float4 tiles[kStages * kTileF4];
    __shared__ __align__(8) uint64_t full_bar[kStages];
    __shared__ __align__(8) uint64_t empty_bar[kStages];

    if (!st->active || (skip_fixed && st->fixed)) return;
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

// ---- tensor-core (tcgen05) variant --------------------------------------------------------------
// The 13 target-feature accumulations Σ_m p_mn F_m (F = 1, y, α n nᵀ, α(n·y)n) are a dense K = M
// contraction D[points × 16] += P[points × K] · F[K × 16].  The CUDA cores compute p per pair (τ, e,
// MUFU.EX2) and Σ p τ; p is split into TF32 hi + lo (p_hi = p with the low 13 mantissa bits cleared,
// p_lo = p - p_hi exactly) and written to TMEM as the A operand; one elected thread per warpgroup
// issues tcgen05.mma.kind::tf32 (A from TMEM, B = F_hi / F_lo from shared memory, D in TMEM):
// D += A_hi F_hi + A_lo F_hi + A_hi F_lo (3×TF32 ≈ FP32 products).  D is drained to registers and
// Kahan-folded after every 64-target tile (FP32 error independent of M).  Fixed-max mode only; the
// running-max mode (w = 0 or tiny w) is served by the CUDA-core kernel.
// TC kernel configuration: NWG consumer warpgroups (128 TMEM lanes each), RB row blocks (points) per
// thread, MW MMA-issuing warps.  TMEM per warpgroup: RB × (D 32 + A 2 buffers × 16) = 64·RB columns.
template <int NWG, int RB, int MW>
struct TcCfg {
    static constexpr int kNCW = 4 * NWG;
    static constexpr int kThreads = (kNCW + 1 + MW) * 32;
    static constexpr int kWGCols = 64 * RB;
    static constexpr int kBlk = NWG * 128 * RB;
    static constexpr size_t kSmem = (size_t)26 * kNCW * 32 * RB * sizeof(float);   // Kahan R, C
    static_assert(NWG * kWGCols <= kTcCols, "TMEM columns");
    static_assert(kThreads <= 1024, "threads");
    static_assert(NWG % MW == 0, "MMA warps must split the warpgroups evenly");
};
// Warp roles: 4·NWG consumer warps (NWG warpgroups × 128 TMEM lanes), 1 TMA producer warp, MW MMA warps.
// Per warpgroup mbarriers: afull[b] (4 warp arrivals: A buffer b written), aempty[b] (MMA commit: buffer
// b consumed), dfull (commit after a tile's last MMAs: D ready), dfree (4 arrivals: D drained).
// The running Kahan sums live in shared memory (touched once per tile), leaving registers for
// in-flight pairs: the kernel is latency-bound on the τ → e → ex2 chain, so warps matter.
template <int NWG, int RB, int MW, bool kLiteral>
__global__ void __launch_bounds__(TcCfg<NWG, RB, MW>::kThreads, 1)
    estep_tc_kernel(const char* __restrict__ tc, const float* __restrict__ src, int64_t N,
                    const IterState* __restrict__ st, Sched sc, float* __restrict__ part) {
    using Cfg = TcCfg<NWG, RB, MW>;
    constexpr int kNCW = Cfg::kNCW;
    constexpr int kBlk = Cfg::kBlk;
    constexpr int kWGCols = Cfg::kWGCols;
    constexpr int kChunks = kTcTile / kTcChunk;
    // static shared memory for the TMA stages (link-time constant addresses: the MMA warps' B
    // descriptors become immediates); dynamic shared memory for the Kahan running sums
    __shared__ __align__(1024) char tiles_st[kTcStages][kTcTileBytes];
    extern __shared__ __align__(16) char dsmem[];
    float* smRC = reinterpret_cast<float*>(dsmem);   // [26][RB × consumer threads]
    __shared__ __align__(8) uint64_t full_bar[kTcStages];
    __shared__ __align__(8) uint64_t empty_bar[kTcStages];
    __shared__ __align__(8) uint64_t afull[NWG][2], aempty[NWG][2], dfull[NWG], dfree[NWG];
    __shared__ uint32_t tmem_base_sh;

    if (!st->active || !st->fixed) return;
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t g = blockIdx.x;
    const int64_t u0 = sched_start(sc, g), u1 = sched_start(sc, g + 1);
    if (u0 >= u1) return;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                     "r"((uint32_t)kTcCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (threadIdx.x == 32) {
        for (int s = 0; s < kTcStages; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], kNCW);
        }
        for (int w = 0; w < NWG; ++w) {
            mbar_init(&afull[w][0], 4);
            mbar_init(&afull[w][1], 4);
            mbar_init(&aempty[w][0], 1);
            mbar_init(&aempty[w][1], 1);
            mbar_init(&dfull[w], 1);
            mbar_init(&dfree[w], 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_sh;
    if (tmem != 0u) __trap();   // 512 columns = the whole TMEM: the allocation must start at lane 0, column 0

    if (warp == kNCW) {
        // ---------------- producer warp: TMA bulk copies of 10-KB tensor-core tiles ----------------
        if (lane == 0) {
            int64_t it = 0;
            for (int64_t u = u0; u < u1; ++u, ++it) {
                const int s = (int)(it % kTcStages);
                const uint32_t ph = (uint32_t)((it / kTcStages) & 1);
                mbar_wait_sleep(&empty_bar[s], ph ^ 1);
                const int64_t tile = u % sc.T;
                mbar_arrive_expect_tx(&full_bar[s], kTcTileBytes);
                bulk_g2s(&tiles_st[s][0], tc + tile * (int64_t)kTcTileBytes, kTcTileBytes, &full_bar[s]);
            }
        }
        return;
    }
    if (warp > kNCW) {
        // ---------------- MMA warps: warp-uniform loop, one elected lane issues tcgen05.mma ----------------
        // per warpgroup w, row block rb, K step c:  D[:, 0:32] (+)= A_hi · [F_hi | F_lo]   (N = 32)
        //                                           D[:, 0:16]  += A_lo · F_hi             (N = 16)
        // The CTA owns all 512 TMEM columns, so every TMEM operand is a compile-time constant.
        const int mw = warp - kNCW - 1;
        constexpr int kWPer = NWG / MW;
        uint32_t aph[kWPer][2] = {}, fph[kWPer] = {};
        for (int64_t ub = u0; ub < u1; ub += kTcStages) {
            const uint32_t round_ph = (uint32_t)(((ub - u0) / kTcStages) & 1);
#pragma unroll
            for (int s = 0; s < kTcStages; ++s) {   // stage index is a compile-time constant
                if (ub + s >= u1) break;
                mbar_wait(&full_bar[s], round_ph);
#pragma unroll
                for (int c = 0; c < kChunks; ++c) {
                    const int buf = c & 1;   // kChunks is even: the buffer parity restarts every tile
                    const uint64_t b32 = bdesc(smem_u32(&tiles_st[s][0]) + kTcBOff + 1024 * c);
#pragma unroll
                    for (int wi = 0; wi < kWPer; ++wi) {
                        const int w = mw * kWPer + wi;
                        if (c == 0 && (ub + s) > u0) {   // D must be drained before it is overwritten
                            mbar_wait(&dfree[w], fph[wi]);
                            fph[wi] ^= 1u;
                        }
                        mbar_wait(&afull[w][buf], aph[wi][buf]);
                        aph[wi][buf] ^= 1u;
                        tc_fence_after();
                        if (elect_one()) {
                            const uint32_t colD = (uint32_t)(w * kWGCols);
                            const uint32_t colA = colD + 32 * RB + buf * 16 * RB;
#pragma unroll
                            for (int rb = 0; rb < RB; ++rb) {
                                mma_tf32_ts(colD + rb * 32, colA + rb * 16, b32, kTcIdesc32, c == 0 ? 0u : 1u);
                                mma_tf32_ts(colD + rb * 32, colA + rb * 16 + 8, b32, kTcIdesc16, 1u);
                            }
                            mma_commit(&aempty[w][buf]);
                            if (c == kChunks - 1) mma_commit(&dfull[w]);
                        }
                        __syncwarp();
                    }
                }
            }
        }
        return;
    }

    // ---------------- consumers: warpgroup wg, TMEM lane quadrant q ----------------
    // Each thread owns one point in each of its RB 128-row blocks; f32x2 instructions cover two
    // consecutive TARGETS, so {p_m, p_m+1} pairs go straight into consecutive A columns of TMEM.
    const int wg = warp >> 2, q = warp & 3;
    const int tw = q * 32 + lane;                      // thread (= TMEM lane) within the warpgroup
    const int tid = threadIdx.x;                       // consumer thread id (smem column)
    const uint32_t tl = tmem + ((uint32_t)(q * 32) << 16);
    const uint32_t colD0 = (uint32_t)(wg * kWGCols), colA0 = colD0 + 32 * RB;
    const uint32_t aempty_a[2] = {smem_u32(&aempty[wg][0]), smem_u32(&aempty[wg][1])};
    const uint32_t afull_a[2] = {smem_u32(&afull[wg][0]), smem_u32(&afull[wg][1])};
    const float k2 = st->k2;
    const float2 nk2 = bc(-k2);
    double Rm[9], tv[3];
#pragma unroll
    for (int i = 0; i < 9; ++i) Rm[i] = st->R[i];
#pragma unroll
    for (int i = 0; i < 3; ++i) tv[i] = st->t[i];

    float h[RB][3], l[RB][3];
    float Rt[RB], Ct[RB];
    int64_t cur_blk = -1;
    uint32_t eph[2] = {0u, 0u}, dph = 0u;
    bool used[2] = {false, false};
    uint32_t cc = 0;
    constexpr int kRC = kNCW * 32 * RB;

    auto load_points = [&](int64_t j) {
#pragma unroll
        for (int k = 0; k < RB; ++k) {
            const int64_t n = j * kBlk + (wg * RB + k) * 128 + tw;
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
                h[k][a] = __double2float_rn(X[a]);
                l[k][a] = __double2float_rn(X[a] - (double)h[k][a]);
            }
            Rt[k] = Ct[k] = 0.f;
#pragma unroll
            for (int f = 0; f < 26; ++f) smRC[f * kRC + k * (kNCW * 32) + tid] = 0.f;
        }
    };
    auto flush = [&](int64_t j) {
        const int64_t slot = j * sc.kmax + (g - sched_owner(sc, j * sc.T));
        float* base = part + slot * (int64_t)kPartF * kBlk;
#pragma unroll
        for (int k = 0; k < RB; ++k) {
            const int b = (wg * RB + k) * 128 + tw;
            const int rc = k * (kNCW * 32) + tid;
#pragma unroll
            for (int f = 0; f < 13; ++f) base[f * kBlk + b] = __fsub_rn(smRC[f * kRC + rc], smRC[(13 + f) * kRC + rc]);
            base[13 * kBlk + b] = __fsub_rn(Rt[k], Ct[k]);
            base[14 * kBlk + b] = 0.f;
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
        const int s = (int)(it % kTcStages);
        mbar_wait(&full_bar[s], (uint32_t)((it / kTcStages) & 1));
        const float4* core = reinterpret_cast<const float4*>(&tiles_st[s][0]);
        float2 Lt[RB];
#pragma unroll
        for (int k = 0; k < RB; ++k) Lt[k] = make_float2(0.f, 0.f);   // Σ p τ, {even, odd} targets
#pragma unroll 1
        for (int c = 0; c < kChunks; ++c, ++cc) {
            const int buf = (int)(cc & 1u);
            if (used[buf]) {                 // wait until the MMAs of two chunks ago released this A buffer
                asm volatile(
                    "{\n"
                    ".reg .pred P1;\n"
                    "WAITE_%=:\n"
                    "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
                    "@!P1 bra WAITE_%=;\n"
                    "}\n" ::"r"(aempty_a[buf]),
                    "r"(eph[buf])
                    : "memory");
                eph[buf] ^= 1u;
                tc_fence_after();
            }
            used[buf] = true;
#ifdef LSG_TC_DIAG
            float2 sink = make_float2(0.f, 0.f);
#endif
#pragma unroll
            for (int pp = 0; pp < 4; ++pp) {
                const int pr = c * 4 + pp;   // target pair within the tile
                const float4 v0 = core[4 * pr], v1 = core[4 * pr + 1], v2 = core[4 * pr + 2], v3 = core[4 * pr + 3];
                // v0 = {y0a, y0b, y1a, y1b}, v1 = {y2a, y2b, ωa, ωb}, v2 = {n0a, n0b, n1a, n1b}, v3 = {n2a, n2b, -, -}
#pragma unroll
                for (int rb = 0; rb < RB; ++rb) {
                    const float2 rx = __fadd2_rn(__fadd2_rn(bc(h[rb][0]), make_float2(-v0.x, -v0.y)), bc(l[rb][0]));
                    const float2 ry = __fadd2_rn(__fadd2_rn(bc(h[rb][1]), make_float2(-v0.z, -v0.w)), bc(l[rb][1]));
                    const float2 rz = __fadd2_rn(__fadd2_rn(bc(h[rb][2]), make_float2(-v1.x, -v1.y)), bc(l[rb][2]));
                    const float2 qv = __ffma2_rn(make_float2(v3.x, v3.y), rz,
                                                 __ffma2_rn(make_float2(v2.z, v2.w), ry,
                                                            __fmul2_rn(make_float2(v2.x, v2.y), rx)));
                    const float2 tau = __ffma2_rn(qv, qv, __ffma2_rn(rz, rz, __ffma2_rn(ry, ry, __fmul2_rn(rx, rx))));
                    const float2 e = kLiteral ? __fmul2_rn(nk2, tau) : __ffma2_rn(nk2, tau, make_float2(v1.z, v1.w));
                    const float2 p = make_float2(ex2_approx(e.x), ex2_approx(e.y));
                    Lt[rb] = __ffma2_rn(p, tau, Lt[rb]);
                    const float2 hi = make_float2(__uint_as_float(__float_as_uint(p.x) & 0xFFFFE000u),
                                                  __uint_as_float(__float_as_uint(p.y) & 0xFFFFE000u));
                    const float2 lo = __fadd2_rn(p, make_float2(-hi.x, -hi.y));
                    // row block rb, A columns: [hi of targets 0-7 | lo of targets 0-7] of this K step
#ifdef LSG_TC_DIAG
                    sink = __fadd2_rn(sink, __fadd2_rn(hi, lo));
#else
                    tmem_st2(tl + colA0 + buf * 16 * RB + rb * 16 + 2 * pp, hi);
                    tmem_st2(tl + colA0 + buf * 16 * RB + rb * 16 + 8 + 2 * pp, lo);
#endif
                }
            }
#ifdef LSG_TC_DIAG
            Lt[0].x += sink.x + sink.y;
#else
            tmem_wait_st();
            tc_fence_before();
#endif
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(afull_a[buf]) : "memory");
        }
        // tile done: wait for D, drain it, free D and the smem stage, Kahan-fold into shared memory
        mbar_wait(&dfull[wg], dph);
        dph ^= 1u;
        tc_fence_after();
        uint32_t dh[RB][16], dl[RB][16];
#pragma unroll
        for (int rb = 0; rb < RB; ++rb) {
            tmem_ld16(tl + colD0 + rb * 32, dh[rb]);        // hi·hi + lo·hi
            tmem_ld16(tl + colD0 + rb * 32 + 16, dl[rb]);   // hi·lo
        }
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
            mbar_arrive(&dfree[wg]);
            mbar_arrive(&empty_bar[s]);
        }
#pragma unroll
        for (int rb = 0; rb < RB; ++rb) {
            const int rc = rb * (kNCW * 32) + tid;
#pragma unroll
            for (int f = 0; f < 13; ++f) {
                const float L = __uint_as_float(dh[rb][f]) + __uint_as_float(dl[rb][f]);
                const float R = smRC[f * kRC + rc], C = smRC[(13 + f) * kRC + rc];
                const float y = L - C;
                const float t = R + y;
                smRC[(13 + f) * kRC + rc] = (t - R) - y;
                smRC[f * kRC + rc] = t;
            }
            const float L = Lt[rb].x + Lt[rb].y;
            const float y = L - Ct[rb];
            const float t = Rt[rb] + y;
            Ct[rb] = (t - Rt[rb]) - y;
            Rt[rb] = t;
        }
    }
    if (cur_blk >= 0) flush(cur_blk);
    // all MMAs of this warpgroup completed (dfull of the last tile was awaited); release TMEM
    tc_fence_before();
    named_bar_sync(1, kNCW * 32);
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"((uint32_t)kTcCols)
                     : "memory");
    }
}

// ---- tensor-core E step, second generation ---------------------------------------------------------
// Same arithmetic as estep_tc_kernel; the pipeline is restructured so that the consumer warps never wait
// on the tensor core in steady state (ncu of the first generation: 22 % of warp samples in local-memory
// round trips for the runtime-indexed A-buffer state, 8 % waiting for D after every tile):
//  * the chunk loop is unrolled by two, so the A buffer, every mbarrier parity and every TMEM column are
//    compile-time constants (no local memory, one uniform TMEM base per warp);
//  * D is double-buffered and a single 16-column accumulator: D += A_hi·F_hi + A_lo·F_hi + A_hi·F_lo
//    (three N = 16 MMAs per K step); tile t's D is drained after the second chunk of tile t + 1, by when
//    its MMAs have long completed;
//  * drained tile sums go into a plain FP32 running sum S1 (one add), which is Kahan-folded into the
//    (R, C) running sums every kTc2Fold tiles: the FP32 error stays independent of M at a quarter of
//    the per-tile cost;
//  * unit → (source block, tile) bookkeeping is incremental (no 64-bit division per tile).
// TMEM per warpgroup: D 2 × 16·RB columns, A 2 × 16·RB columns (hi 8 | lo 8 per row block).
constexpr int kTc2Fold = 16;
template <int NWG, int RB, bool kSelf, int MW>
struct Tc2Cfg {
    static constexpr int kNCW = 4 * NWG;
    // consumers + TMA producer warp + MW MMA warps (none if each warpgroup issues its own MMAs)
    static constexpr int kThreads = (kNCW + 1 + (kSelf ? 0 : MW)) * 32;
    static_assert(NWG % MW == 0, "MMA warps must split the warpgroups evenly");
    static constexpr int kWGCols = 64 * RB;
    static constexpr int kBlk = NWG * 128 * RB;
    static constexpr int kSmF = 39;                    // S1[13], R[13], C[13] per point
    static constexpr size_t kSmem = (size_t)kSmF * kNCW * 32 * RB * sizeof(float);
    static_assert(NWG * kWGCols <= kTcCols, "TMEM columns");
    static_assert(kThreads <= 1024, "threads");
};
static_assert(kTcStages == 4, "stage arithmetic below assumes 4 stages");

template <int NWG, int RB, bool kLiteral, bool kStX8, bool kSelf, int MW, int NT>
__global__ void __launch_bounds__(Tc2Cfg<NWG, RB, kSelf, MW>::kThreads, 1)
    estep_tc2_kernel(const char* __restrict__ tc, const float* __restrict__ src, int64_t N,
                     const IterState* __restrict__ st, Sched sc, float* __restrict__ part) {
    using Cfg = Tc2Cfg<NWG, RB, kSelf, MW>;
    constexpr int kNCW = Cfg::kNCW;
    constexpr int kBlk = Cfg::kBlk;
    constexpr int kWGCols = Cfg::kWGCols;
    constexpr int kChunks = kTcTile / kTcChunk;
    static_assert(kChunks % 2 == 0, "chunks per tile must be even");
    constexpr int kNF = 13;   // D features kept: 1, y, W, b
    // D accumulates NT consecutive tiles of one source block (a "D group") before it is drained; a group
    // also ends at a block boundary and at the end of the CTA's range.  With MMA warps, a stage is
    // released by the consumers when they finish reading it plus one tcgen05.commit per MMA warp.
    static_assert(!kSelf || NT == 1, "self-issuing warpgroups drain every tile");
    __shared__ __align__(1024) char tiles_st[kTcStages][kTcTileBytes];
    extern __shared__ __align__(16) char dsmem[];
    float* smS = reinterpret_cast<float*>(dsmem);   // [3 kNF][RB × consumer threads]: S1, R, C
    __shared__ __align__(8) uint64_t full_bar[kTcStages];
    __shared__ __align__(8) uint64_t empty_bar[kTcStages];
    __shared__ __align__(8) uint64_t afull[NWG][2], aempty[NWG][2], dfull[NWG][2], dfree[NWG][2];
    __shared__ uint32_t tmem_base_sh;

    if (!st->active || !st->fixed) return;
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t g = blockIdx.x;
    const int64_t u0 = sched_start(sc, g), u1 = sched_start(sc, g + 1);
    if (u0 >= u1) return;
    const int64_t nunits = u1 - u0;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                     "r"((uint32_t)kTcCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (threadIdx.x == 32) {
        for (int s = 0; s < kTcStages; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], kSelf ? kNCW : kNCW + MW);
        }
        for (int w = 0; w < NWG; ++w)
            for (int b = 0; b < 2; ++b) {
                mbar_init(&afull[w][b], 4);
                mbar_init(&aempty[w][b], 1);
                mbar_init(&dfull[w][b], 1);
                mbar_init(&dfree[w][b], 4);
            }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_sh;
    if (tmem != 0u) __trap();   // 512 columns = the whole TMEM: the allocation must start at column 0

    if (warp == kNCW) {
        // ---------------- producer warp: TMA bulk copies of the 10-KB tensor-core tiles ----------------
        if (lane == 0) {
            int64_t tile = u0 % sc.T;
            for (int64_t it = 0; it < nunits; ++it) {
                const int s = (int)(it & 3);
                mbar_wait_sleep(&empty_bar[s], (uint32_t)(((it >> 2) & 1) ^ 1));
                mbar_arrive_expect_tx(&full_bar[s], kTcTileBytes);
                bulk_g2s(&tiles_st[s][0], tc + tile * (int64_t)kTcTileBytes, kTcTileBytes, &full_bar[s]);
                if (++tile == sc.T) tile = 0;
            }
        }
        return;
    }
    if (!kSelf && warp > kNCW) {
        // ---------------- MMA warp: one elected lane issues tcgen05.mma for every warpgroup ----------------
        // D[db] (+)= A_hi·F_hi, += A_lo·F_hi, += A_hi·F_lo per row block and K step (N = 16 each).
        // Parities: the k-th completion of a barrier has parity k & 1; A buffer b of K step c of any tile
        // is used for the (4·it + c/2)-th time, so its parity is the constant (c >> 1) & 1.
        const uint32_t tiles0 = smem_u32(&tiles_st[0][0]) + kTcBOff;
        constexpr int kWPer = NWG / MW;
        const int w0 = (warp - kNCW - 1) * kWPer;   // this MMA warp serves warpgroups [w0, w0 + kWPer)
        int64_t tile = u0 % sc.T, grp = 0;
        int tig = 0;                                  // tile index within the current D group
        for (int64_t it = 0; it < nunits; ++it) {
            const int s = (int)(it & 3);
            const int db = (int)(grp & 1);
            const bool first = tig == 0;
            const bool last = tig + 1 == NT || tile + 1 == sc.T || it + 1 == nunits;
            const uint32_t dpar = (uint32_t)(((grp >> 1) & 1) ^ 1);   // completion (grp>>1) - 1 of dfree[db]
            mbar_wait_sleep(&full_bar[s], (uint32_t)((it >> 2) & 1));
            const uint32_t bbase = tiles0 + (uint32_t)s * kTcTileBytes;
#pragma unroll
            for (int c = 0; c < kChunks; ++c) {
                const int ab = c & 1;
                const uint64_t bhi = bdesc(bbase + 1024 * c), blo = bdesc(bbase + 1024 * c + 512);
#pragma unroll
                for (int wi = 0; wi < kWPer; ++wi) {
                    const int w = w0 + wi;
                    if (c == 0 && first) mbar_wait_sleep(&dfree[w][db], dpar);
                    mbar_wait_sleep(&afull[w][ab], (uint32_t)((c >> 1) & 1));
                    tc_fence_after();
                    if (elect_one()) {
                        const uint32_t colD = (uint32_t)(w * kWGCols + db * 16 * RB);
                        const uint32_t colA = (uint32_t)(w * kWGCols + 32 * RB + ab * 16 * RB);
#ifndef LSG_TC2_NOMMA   // diagnostic builds only (tools/build_diag.sh)
#pragma unroll
                        for (int rb = 0; rb < RB; ++rb) {
                            mma_tf32_ts(colD + rb * 16, colA + rb * 16, bhi, kTcIdesc16, (c == 0 && first) ? 0u : 1u);
                            mma_tf32_ts(colD + rb * 16, colA + rb * 16 + 8, bhi, kTcIdesc16, 1u);
                            mma_tf32_ts(colD + rb * 16, colA + rb * 16, blo, kTcIdesc16, 1u);
                        }
#endif
                        mma_commit(&aempty[w][ab]);
                        if (c == kChunks - 1 && last) mma_commit(&dfull[w][db]);
                        if (c == kChunks - 1 && wi == kWPer - 1) mma_commit(&empty_bar[s]);   // stage s read
                    }
                    __syncwarp();
                }
            }
            if (last) {
                tig = 0;
                ++grp;
            } else {
                ++tig;
            }
            if (++tile == sc.T) tile = 0;
        }
        return;
    }

    // ---------------- consumers: warpgroup wg, TMEM lane quadrant q ----------------
    const int wg = warp >> 2, q = warp & 3;
    const int tw = q * 32 + lane;
    const int tid = threadIdx.x;
    const uint32_t tl = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(wg * kWGCols);
    const float k2 = st->k2;
    const float2 nk2 = bc(-k2);
    double Rm[9], tv[3];
#pragma unroll
    for (int i = 0; i < 9; ++i) Rm[i] = st->R[i];
#pragma unroll
    for (int i = 0; i < 3; ++i) tv[i] = st->t[i];
    constexpr int kRC = kNCW * 32 * RB;

    float2 h[RB][3], l[RB][3];   // x̂ as FP32 hi/lo, broadcast to both f32x2 lanes (two targets per instruction)
    float Rt[RB], Ct[RB];
    int nfold = 0;

    auto load_points = [&](int64_t j) {
#pragma unroll
        for (int k = 0; k < RB; ++k) {
            const int64_t n = j * kBlk + (wg * RB + k) * 128 + tw;
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
                h[k][a] = bc(hi);
                l[k][a] = bc(__double2float_rn(X[a] - (double)hi));
            }
            Rt[k] = Ct[k] = 0.f;
#pragma unroll
            for (int f = 0; f < Cfg::kSmF; ++f) smS[f * kRC + k * (kNCW * 32) + tid] = 0.f;
        }
        nfold = 0;
    };
    // Kahan-fold S1 into (R, C) and clear S1
    auto fold_s1 = [&]() {
#pragma unroll
        for (int rb = 0; rb < RB; ++rb) {
            const int rc = rb * (kNCW * 32) + tid;
#pragma unroll
            for (int f = 0; f < kNF; ++f) {
                const float L = smS[f * kRC + rc];
                const float R = smS[(kNF + f) * kRC + rc], C = smS[(2 * kNF + f) * kRC + rc];
                const float y = L - C;
                const float t = R + y;
                smS[(2 * kNF + f) * kRC + rc] = (t - R) - y;
                smS[(kNF + f) * kRC + rc] = t;
                smS[f * kRC + rc] = 0.f;
            }
        }
        nfold = 0;
    };
    // drain D group `gd` (all its MMAs are complete once dfull fires), release D (and, self-issuing, the
    // stage of its single tile `itd`)
    auto drain = [&](int64_t gd, int64_t itd) {
        const int db = (int)(gd & 1);
        mbar_wait_sleep(&dfull[wg][db], (uint32_t)((gd >> 1) & 1));
        tc_fence_after();
        uint32_t d[RB][16];
#pragma unroll
        for (int rb = 0; rb < RB; ++rb) tmem_ld16(tl + (uint32_t)(db * 16 * RB + rb * 16), d[rb]);
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
            if (!kSelf) mbar_arrive(&dfree[wg][db]);   // self-issue: the next chunk-0 barrier orders it
            if (kSelf) mbar_arrive(&empty_bar[itd & 3]);
        }
#pragma unroll
        for (int rb = 0; rb < RB; ++rb) {
            const int rc = rb * (kNCW * 32) + tid;
#pragma unroll
            for (int f = 0; f < kNF; ++f) smS[f * kRC + rc] += __uint_as_float(d[rb][f]);
        }
        if (++nfold == kTc2Fold) fold_s1();
    };
    auto flush = [&](int64_t j) {
        fold_s1();
        const int64_t slot = j * sc.kmax + (g - sched_owner(sc, j * sc.T));
        float* base = part + slot * (int64_t)kPartF * kBlk;
#pragma unroll
        for (int k = 0; k < RB; ++k) {
            const int b = (wg * RB + k) * 128 + tw;
            const int rc = k * (kNCW * 32) + tid;
#pragma unroll
            for (int f = 0; f < 13; ++f)
                base[f * kBlk + b] = __fsub_rn(smS[(kNF + f) * kRC + rc], smS[(2 * kNF + f) * kRC + rc]);
            base[13 * kBlk + b] = __fsub_rn(Rt[k], Ct[k]);
            base[14 * kBlk + b] = 0.f;
            base[15 * kBlk + b] = 0.f;
        }
    };

    uint32_t cur_b = 0, cur_db = 0;   // self-issue: B operand base of the current stage, D buffer
    // one K step (8 targets = 4 target pairs) for buffer AB: residual, τ, ex2, Σpτ, TF32 split → TMEM A
    auto chunk = [&](const float4* core, int c, float2 (&Lt)[RB], auto ABc) {
        constexpr int AB = decltype(ABc)::value;
        // wait for the MMAs of this buffer's previous use (K step c - 2): parity of completion 4·it + c/2 - 1
        const uint32_t apar = (uint32_t)(((c >> 1) & 1) ^ 1);
        if (!kStX8) {
            mbar_wait_sleep(&aempty[wg][AB], apar);
            tc_fence_after();
        }
        uint32_t av[RB][16];   // A row of this K step: TF32 hi of the 8 targets, then lo
#pragma unroll
        for (int pp = 0; pp < 4; ++pp) {
            const int pr = c * 4 + pp;
            const float4 v0 = core[4 * pr], v1 = core[4 * pr + 1], v2 = core[4 * pr + 2], v3 = core[4 * pr + 3];
#pragma unroll
            for (int rb = 0; rb < RB; ++rb) {
                const float2 rx = __fadd2_rn(__fadd2_rn(h[rb][0], make_float2(-v0.x, -v0.y)), l[rb][0]);
                const float2 ry = __fadd2_rn(__fadd2_rn(h[rb][1], make_float2(-v0.z, -v0.w)), l[rb][1]);
                const float2 rz = __fadd2_rn(__fadd2_rn(h[rb][2], make_float2(-v1.x, -v1.y)), l[rb][2]);
                const float2 qv = __ffma2_rn(make_float2(v3.x, v3.y), rz,
                                             __ffma2_rn(make_float2(v2.z, v2.w), ry, __fmul2_rn(make_float2(v2.x, v2.y), rx)));
                const float2 tau = __ffma2_rn(qv, qv, __ffma2_rn(rz, rz, __ffma2_rn(ry, ry, __fmul2_rn(rx, rx))));
                const float2 e = kLiteral ? __fmul2_rn(nk2, tau) : __ffma2_rn(nk2, tau, make_float2(v1.z, v1.w));
                const float2 p = make_float2(ex2_approx(e.x), ex2_approx(e.y));
                Lt[rb] = __ffma2_rn(p, tau, Lt[rb]);
                const float2 hi = make_float2(__uint_as_float(__float_as_uint(p.x) & 0xFFFFE000u),
                                              __uint_as_float(__float_as_uint(p.y) & 0xFFFFE000u));
                const float2 lo = __fadd2_rn(p, make_float2(-hi.x, -hi.y));
                if (kStX8) {
                    av[rb][2 * pp] = __float_as_uint(hi.x);
                    av[rb][2 * pp + 1] = __float_as_uint(hi.y);
                    av[rb][8 + 2 * pp] = __float_as_uint(lo.x);
                    av[rb][8 + 2 * pp + 1] = __float_as_uint(lo.y);
                } else {
                    tmem_st2(tl + (uint32_t)(32 * RB + AB * 16 * RB + rb * 16 + 2 * pp), hi);
                    tmem_st2(tl + (uint32_t)(32 * RB + AB * 16 * RB + rb * 16 + 8 + 2 * pp), lo);
                }
            }
        }
        if (kStX8) {
            // the A buffer is needed only now: the MMAs of its previous use had this chunk's math to finish
            mbar_wait_sleep(&aempty[wg][AB], apar);
            tc_fence_after();
#ifndef LSG_TC2_NOSTTM
#pragma unroll
            for (int rb = 0; rb < RB; ++rb) tmem_st16(tl + (uint32_t)(32 * RB + AB * 16 * RB + rb * 16), av[rb]);
#else
            float sink = 0.f;
#pragma unroll
            for (int rb = 0; rb < RB; ++rb)
#pragma unroll
                for (int k = 0; k < 16; ++k) sink += __uint_as_float(av[rb][k]);
            Lt[0].x += sink * 1e-30f;
#endif
        }
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (!kSelf) {
            if (lane == 0) mbar_arrive(&afull[wg][AB]);
        } else {
            // the warpgroup's four warps meet at a named barrier (two ids, alternating with the A buffer, so
            // a warp one K step ahead cannot complete the wrong phase); warp 0 then issues the MMAs
            const int bid = 2 + 2 * wg + AB;
            if (q != 0) {
                named_bar_arrive(bid, 128);
            } else {
                named_bar_sync(bid, 128);
                tc_fence_after();
                if (elect_one()) {
                    const uint64_t bhi = bdesc(cur_b + 1024 * c), blo = bdesc(cur_b + 1024 * c + 512);
                    const uint32_t colD = (uint32_t)(wg * kWGCols) + cur_db * 16 * RB;
                    constexpr uint32_t kColA = 32 * RB + AB * 16 * RB;
#pragma unroll
                    for (int rb = 0; rb < RB; ++rb) {
                        mma_tf32_ts(colD + rb * 16, (uint32_t)(wg * kWGCols) + kColA + rb * 16, bhi, kTcIdesc16,
                                    c == 0 ? 0u : 1u);
                        mma_tf32_ts(colD + rb * 16, (uint32_t)(wg * kWGCols) + kColA + rb * 16 + 8, bhi, kTcIdesc16, 1u);
                        mma_tf32_ts(colD + rb * 16, (uint32_t)(wg * kWGCols) + kColA + rb * 16, blo, kTcIdesc16, 1u);
                    }
                    mma_commit(&aempty[wg][AB]);
                    if (c == kChunks - 1) mma_commit(&dfull[wg][cur_db]);
                }
                __syncwarp();
            }
        }
    };

    int64_t j = u0 / sc.T, tile = u0 % sc.T;
    load_points(j);
    bool pending = false;   // the previous D group has not been drained yet
    int64_t grp = 0, pend_g = 0, pend_it = 0;
    int tig = 0;
    for (int64_t it = 0; it < nunits; ++it) {
        mbar_wait_sleep(&full_bar[it & 3], (uint32_t)((it >> 2) & 1));
        cur_b = smem_u32(&tiles_st[0][0]) + kTcBOff + (uint32_t)(it & 3) * kTcTileBytes;
        cur_db = (uint32_t)(grp & 1);
        const float4* core = reinterpret_cast<const float4*>(&tiles_st[it & 3][0]);
        float2 Lt[RB];
#pragma unroll
        for (int k = 0; k < RB; ++k) Lt[k] = make_float2(0.f, 0.f);
#ifndef LSG_TC2_UNROLL
#define LSG_TC2_UNROLL 1
#endif
#define LSG_PRAGMA(x) _Pragma(#x)
#define LSG_UNROLL(n) LSG_PRAGMA(unroll n)
        LSG_UNROLL(LSG_TC2_UNROLL)
        for (int c = 0; c < kChunks; c += 2) {
            chunk(core, c, Lt, std::integral_constant<int, 0>());
            chunk(core, c + 1, Lt, std::integral_constant<int, 1>());
            if (c == 0 && pending) {
                drain(pend_g, pend_it);
                pending = false;
            }
        }
        if (!kSelf) {   // this warp is done reading the stage's core data
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty_bar[it & 3]);
        }
#pragma unroll
        for (int rb = 0; rb < RB; ++rb) {
            const float L = Lt[rb].x + Lt[rb].y;
            const float y = L - Ct[rb];
            const float t = Rt[rb] + y;
            Ct[rb] = (t - Rt[rb]) - y;
            Rt[rb] = t;
        }
        const bool block_end = tile + 1 == sc.T || it + 1 == nunits;
        const bool last = tig + 1 == NT || block_end;
        if (last) {
            if (block_end) {   // source block (or the CTA's range) ends here: drain and flush now
                drain(grp, it);
                flush(j);
            } else {
                pending = true;
                pend_g = grp;
                pend_it = it;
            }
            tig = 0;
            ++grp;
        } else {
            ++tig;
        }
        if (++tile == sc.T) {
            tile = 0;
            ++j;
            if (it + 1 < nunits) load_points(j);
        }
    }
    // all MMAs of this warpgroup completed (dfull of the last tile was awaited); release TMEM
    tc_fence_before();
    named_bar_sync(1, kNCW * 32);
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"((uint32_t)kTcCols)
                     : "memory");
    }
}

// ---- merge: log-sum-exp over partials + outlier term → 16-float record -------------------
// With per-point confidences (Eq. 8) the outlier weight is w_n = 1 - (1 - w0) φ(x_n), so the
// outlier log2-weight and the density constant are per point:
//   C1_n = ln((1 - w_n)/M) - 1.5 ln(2πσ²) = C1 + ln((1 - w_n)/(1 - w0)),
//   L_o,n = (ln(w_n/V) - C1_n)/ln2 - ω_ref;   w_n = 1 → the point is all outlier (P_out = 1, ln p = -ln V).
// The pair kernels do not depend on w_n (the fixed-max mode needs L_o,n ≥ L_o, true since w_n ≥ w0).
// One CTA (16 warps) merges 32 points (merge_tile32) and stores their records as one contiguous 2-KB row.
__global__ void __launch_bounds__(kMergePts * 16)
    estep_merge_kernel(const float* __restrict__ part, int64_t N, const IterState* __restrict__ st, Sched sc,
                       float* __restrict__ rec, const float* __restrict__ phi) {
    if (!st->active) return;
    __shared__ float tile[kMergePts][LSGCPD_REC + 1];
    __shared__ double a0s[kMergePts];
    const int64_t n0 = (int64_t)blockIdx.x * kMergePts;
    merge_tile32(part, N, n0, st, sc, phi, tile, a0s);
    __syncthreads();
    const int p = threadIdx.x / LSGCPD_REC, g = threadIdx.x % LSGCPD_REC;
    if (n0 + p < N) rec[(n0 + p) * LSGCPD_REC + g] = tile[p][g];
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
    LSG_VARIANT(4, 4, 2, true),  LSG_VARIANT(2, 8, 2, false), LSG_VARIANT(1, 16, 1, false), LSG_VARIANT(2, 16, 1, true),
    LSG_VARIANT(2, 14, 1, true), LSG_VARIANT(2, 8, 1, true), LSG_VARIANT(2, 2, 8, true), LSG_VARIANT(1, 2, 8, false),
    LSG_VARIANT(2, 1, 8, true),
};
constexpr int kNumVariants = sizeof(kVariants) / sizeof(kVariants[0]);
constexpr int kDefaultVariant = 3;   // packed, 2 points/thread, 12 consumer warps (tools/estep_speed.py)

static int variant_index() {
    const char* e = getenv("LSGCPD_ESTEP_VARIANT");
    int v = e ? atoi(e) : kDefaultVariant;
    return (v >= 0 && v < kNumVariants) ? v : kDefaultVariant;
}
// Tensor-core E step (fixed-max mode) paired with a CUDA-core variant of the same block size for the
// running-max mode.  LSGCPD_TC=0 disables it; LSGCPD_TC_VARIANT picks the configuration.
struct TcVariant {
    int nwg, rb, mw, pair_variant;
    int threads, blk;
    size_t smem;
    const void* fn[2];
};
#define LSG_TC(NWG, RB, MW, PV)                                                                           \
    {NWG, RB, MW, PV, TcCfg<NWG, RB, MW>::kThreads, TcCfg<NWG, RB, MW>::kBlk, TcCfg<NWG, RB, MW>::kSmem, \
     {(const void*)estep_tc_kernel<NWG, RB, MW, false>, (const void*)estep_tc_kernel<NWG, RB, MW, true>}}
#define LSG_TC2N(NWG, RB, X8, SELF, MW, NT, PV)                                                      \
    {NWG, RB, MW, PV, Tc2Cfg<NWG, RB, SELF, MW>::kThreads, Tc2Cfg<NWG, RB, SELF, MW>::kBlk,          \
     Tc2Cfg<NWG, RB, SELF, MW>::kSmem,                                                               \
     {(const void*)estep_tc2_kernel<NWG, RB, false, X8, SELF, MW, NT>,                               \
      (const void*)estep_tc2_kernel<NWG, RB, true, X8, SELF, MW, NT>}}
#define LSG_TC2M(NWG, RB, X8, SELF, MW, PV) LSG_TC2N(NWG, RB, X8, SELF, MW, 1, PV)
#define LSG_TC2(NWG, RB, X8, SELF, PV) LSG_TC2M(NWG, RB, X8, SELF, 1, PV)
static const TcVariant kTcVariants[] = {
    LSG_TC(4, 2, 2, 0),   // 16 consumer warps, 2 points/thread (1024-point blocks) — CUDA-core variant 0
    LSG_TC(6, 1, 2, 3),   // 24 consumer warps, 1 point/thread (768) — variant 3
    LSG_TC(7, 1, 1, 8),   // 28 consumer warps (896) — variant 8
    LSG_TC(4, 1, 2, 9),   // 16 consumer warps, 1 point/thread (512) — variant 9
    LSG_TC(4, 2, 4, 0),   // as 0 with one MMA warp per warpgroup
    LSG_TC(4, 2, 1, 0),   // as 0 with a single MMA warp
    LSG_TC(2, 4, 1, 0),   // 8 consumer warps, 4 points/thread (1024)
    LSG_TC(3, 2, 1, 3),   // 12 consumer warps, 2 points/thread (768)
    // second generation (estep_tc2_kernel): one MMA warp, double-buffered D
    LSG_TC2(3, 2, false, false, 3),   // 8: 12 consumer warps × 2 points (768), per-pair TMEM stores
    LSG_TC2(3, 2, true, false, 3),    // 9: as 8 with two x8 TMEM stores per row block and K step
    LSG_TC2(4, 2, true, false, 0),    // 10: 16 consumer warps × 2 points (1024)
    LSG_TC2(2, 4, true, false, 0),    // 11: 8 consumer warps × 4 points (1024)
    LSG_TC2(6, 1, true, false, 3),    // 12: 24 consumer warps × 1 point (768)
    LSG_TC2(6, 1, false, false, 3),   // 13: as 12 with per-pair TMEM stores
    LSG_TC2(2, 2, true, false, 9),    // 14: 8 consumer warps × 2 points (512)
    // each warpgroup issues its own MMAs (no MMA warp)
    LSG_TC2(3, 2, true, true, 3),     // 15: as 9
    LSG_TC2(4, 2, true, true, 0),     // 16: as 10
    LSG_TC2(2, 4, true, true, 0),     // 17: as 11
    LSG_TC2(6, 1, true, true, 3),     // 18: as 12
    // one MMA warp per warpgroup
    LSG_TC2M(3, 2, true, false, 3, 3),   // 19: as 9
    LSG_TC2M(6, 1, true, false, 3, 3),   // 20: as 12, one MMA warp per two warpgroups
    LSG_TC2M(2, 2, true, false, 2, 9),   // 21: as 14
    // D accumulated over NT tiles before each drain
    LSG_TC2N(3, 2, true, false, 3, 2, 3),   // 22: as 19, NT = 2
    LSG_TC2N(3, 2, true, false, 3, 4, 3),   // 23: as 19, NT = 4
    LSG_TC2N(3, 2, true, false, 3, 8, 3),   // 24: as 19, NT = 8
    LSG_TC2N(3, 2, true, false, 3, 16, 3),  // 25: as 19, NT = 16
};
constexpr int kNumTcVariants = sizeof(kTcVariants) / sizeof(kTcVariants[0]);
// LSGCPD_TC: unset = automatic (tensor cores unless the problem is too small), 0 = off, 1 = forced on
static int tc_mode() {
    const char* e = getenv("LSGCPD_TC");
    return e ? (atoi(e) != 0 ? 1 : 0) : 2;
}
constexpr int kDefaultTcVariant = 23;  // tc2, 12 consumer warps × 2 points, one MMA warp per warpgroup, D over 4 tiles (tools/tc_speed.py)
static int tc_variant_index() {
    const char* e = getenv("LSGCPD_TC_VARIANT");
    int v = e ? atoi(e) : kDefaultTcVariant;
    return (v >= 0 && v < kNumTcVariants) ? v : kDefaultTcVariant;
}

static int g_num_sms = 0;
static int g_occ[kNumVariants] = {0};

constexpr int kMidVariant = 9, kMidBlk = 2 * 8 * 32;   // packed, 2 points/thread, 8 consumer warps: 512-point blocks
constexpr int kSmallVariant = 12;
constexpr int64_t kSplitBytes = 48ll << 20;   // tensor-core sections above this are swept in two halves   // one consumer warp, 64-point blocks: problems too small to fill the GPU

int estep_plan(int64_t M_pad, int64_t N, Sched* sc) {
    const int tvi = tc_variant_index();
    const int mode = tc_mode();
    bool tc = mode != 0;
    int vi = tc ? kTcVariants[tvi].pair_variant : variant_index();
    if (g_num_sms == 0) {
        int dev;
        LSG_CUDA(cudaGetDevice(&dev));
        LSG_CUDA(cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev));
    }
    if (mode == 2 && !getenv("LSGCPD_ESTEP_VARIANT")) {
        // small problems (tiny / object configs): too few (block, tile) units for one CTA per SM with the
        // big blocks — use the small-block CUDA-core kernel so every SM gets work
        const int64_t units_big = (N + kTcVariants[tvi].blk - 1) / kTcVariants[tvi].blk * (M_pad / kTT);
        if (units_big < 2 * (int64_t)g_num_sms) {
            // 512-point blocks once they give ~3/4 of a unit per SM, else 64-point blocks (the most CTAs):
            // tools/small_path_sweep.py — 1,000 points 38 µs per EM iteration with 64-point blocks, 2,000 / 3,500
            // points 44 / 56 µs with 512-point blocks (64-point: 51 / 72; tensor cores: 50 / 59)
            tc = false;
            const int64_t units_mid = (N + kMidBlk - 1) / kMidBlk * (M_pad / kTT);
            vi = 4 * units_mid >= 3 * (int64_t)g_num_sms ? kMidVariant : kSmallVariant;
        }
    }
    const Variant& V = kVariants[vi];
    if (g_occ[vi] == 0) {
        int occ = 0;
        LSG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, V.fn[0], (V.ncw + 1) * 32, 0));
        g_occ[vi] = occ > 0 ? occ : 1;
    }
    Sched s;
    memset(&s, 0, sizeof(s));
    s.variant = tc ? -1 - vi : vi;   // negative: tensor-core kernel + CUDA-core variant for running max
    s.tc_variant = tvi;
    s.B = (int64_t)V.ppt * V.ncw * 32;
    s.nblk = (N + s.B - 1) / s.B;
    // a tensor-core section larger than ~48 MB is swept in two halves, one launch each, so every CTA reads
    // tiles of the same half at a time and the half stays in L2 (the whole section re-read from HBM otherwise;
    // DESIGN §7 "DRAM traffic").  M_pad is a multiple of 256 targets, so the tile count is even.
    const char* he = getenv("LSGCPD_HALVES");
    const bool split = tc && (M_pad / kTT) * (int64_t)kTcTileBytes > kSplitBytes && !(he && he[0] == '1');
    s.halves = split ? 2 : 1;
    s.T = M_pad / kTT / s.halves;
    s.U = s.nblk * s.T;
    const int64_t slots = (int64_t)g_num_sms * (tc ? 1 : g_occ[vi]);   // the TC kernel holds all TMEM: 1 CTA/SM
    s.G = s.U < slots ? s.U : slots;
    if (s.G < 1) s.G = 1;
    int64_t kmax = 1;
    for (int64_t j = 0; j < s.nblk; ++j) {
        const int64_t k = sched_owner(s, (j + 1) * s.T - 1) - sched_owner(s, j * s.T) + 1;
        if (k > kmax) kmax = k;
    }
    s.kmax = kmax;
    s.hstride = s.nblk * s.kmax * (int64_t)kPartF * s.B;
    *sc = s;
    return 0;
}

size_t estep_partial_bytes(const Sched& s) { return (size_t)s.halves * s.hstride * sizeof(float); }

void estep_launch_setup(IterState* st, const void* d_target, const double* R, const double* t, double sigma2,
                        double w, double V, int64_t M, int consistent, double eta, cudaStream_t stream) {
    estep_setup_kernel<<<1, 1, 0, stream>>>(st, reinterpret_cast<const TargetHeader*>(d_target), R[0], R[1], R[2],
                                             R[3], R[4], R[5], R[6], R[7], R[8], t[0], t[1], t[2], sigma2, w, V, M,
                                             consistent, eta);
}

void estep_launch(const void* d_target, const float* d_src, int64_t N, const IterState* st, const Sched& sc,
                  float* part, float* rec, int consistent, const float* phi, cudaStream_t stream, int merge) {
    const bool tc = sc.variant < 0;
    const Variant& V = kVariants[tc ? -1 - sc.variant : sc.variant];
    Sched scv = sc;
    int skip_fixed = tc ? 1 : 0;
    const int64_t M_pad = sc.T * kTT * sc.halves;
    for (int h = 0; h < sc.halves; ++h) {   // one sweep per half of the targets (sc.T tiles each)
        const float* body = target_body(d_target) + (int64_t)h * sc.T * kTT * kTgtFloats;
        float* parth = part + (int64_t)h * sc.hstride;
        void* args[] = {(void*)&body, (void*)&d_src, (void*)&N, (void*)&st, (void*)&scv, (void*)&parth,
                        (void*)&skip_fixed};
        if (tc) {
            const char* tcb = reinterpret_cast<const char*>(target_tc(d_target, M_pad)) +
                              (int64_t)h * sc.T * kTcTileBytes;
            const TcVariant& TV = kTcVariants[sc.tc_variant];
            static bool attr_set[kNumTcVariants] = {};
            if (!attr_set[sc.tc_variant]) {
                cudaFuncSetAttribute(TV.fn[0], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TV.smem);
                cudaFuncSetAttribute(TV.fn[1], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TV.smem);
                attr_set[sc.tc_variant] = true;
            }
            void* targs[] = {(void*)&tcb, (void*)&d_src, (void*)&N, (void*)&st, (void*)&scv, (void*)&parth};
            cudaLaunchKernel(TV.fn[consistent ? 0 : 1], dim3((unsigned)sc.G), dim3(TV.threads), targs, TV.smem,
                             stream);
        }
        cudaLaunchKernel(V.fn[consistent ? 0 : 1], dim3((unsigned)sc.G), dim3((V.ncw + 1) * 32), args, 0, stream);
    }
    if (!merge) return;
    estep_merge_kernel<<<(unsigned)((N + kMergePts - 1) / kMergePts), kMergePts * 16, 0, stream>>>(part, N, st, sc,
                                                                                                 rec, phi);
}

}  // namespace lsg
