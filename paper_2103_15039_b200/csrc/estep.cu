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

#include <mutex>

#include "common.cuh"
#include "estep_dev.cuh"
#include "kernels.h"

namespace lsg {

// ---- setup: per-call constants (lsgcpd_estep path) ---------------------------------------
// The target header is checked here (no host synchronisation): a buffer that is not a prepared target of M
// points leaves the state inactive with status EINVAL, and the merge writes an all-NaN record.
__global__ void estep_setup_kernel(IterState* st, const TargetHeader* hdr, double r0, double r1, double r2,
                                   double r3, double r4, double r5, double r6, double r7, double r8, double t0,
                                   double t1, double t2, double sigma2, double w, double V, int64_t M,
                                   int consistent, double eta) {
    const double R[9] = {r0, r1, r2, r3, r4, r5, r6, r7, r8};
    const double t[3] = {t0, t1, t2};
    IterState s;
    const bool ok = hdr->magic == kTargetMagic && hdr->M == M;
    make_state(s, R, t, sigma2, w, V, M, ok ? hdr->omega_ref : 0.0, consistent, eta, ok ? hdr->spc : 1.0);
    s.extent = ok ? hdr->extent : 0.0;
    s.active = ok ? 1 : 0;
    s.iter = 0;
    s.status = ok ? 0 : LSGCPD_EINVAL;
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

// ---- tensor-core (tcgen05) E step --------------------------------------------------------------------
// The 13 target-feature accumulations Σ_m p_mn F_m (F = 1, y, α n nᵀ, α(n·y)n) are a dense K = M
// contraction D[points × 16] += P[points × K] · F[K × 16] (not the K = 3 cross term).  The CUDA cores
// compute p per pair (residual, τ, e, MUFU.EX2) and Σ p τ; p is split into TF32 hi + lo (p_hi = p with the
// low 13 mantissa bits cleared, p_lo = p - p_hi exactly) and written to TMEM as the A operand; one MMA warp
// per warpgroup issues tcgen05.mma.kind::tf32 (A from TMEM, B = F_hi / F_lo from shared memory, D in TMEM):
// D += A_hi F_hi + A_lo F_hi + A_hi F_lo (3×TF32 ≈ FP32 products).  Fixed-max mode only; the running-max
// mode (w = 0 or tiny w) is served by the CUDA-core kernel.
// Pipeline (no consumer ever waits on the tensor core in steady state):
//  * per warpgroup two A buffers (afull: 4 warp arrivals, aempty: MMA commit) and two D buffers (dfull:
//    commit after a D group's last MMAs, dfree: 4 arrivals after the drain); the chunk loop is unrolled by
//    two, so every A-buffer index, mbarrier parity and TMEM column is a compile-time constant;
//  * D accumulates kNT consecutive tiles of one source block (a "D group", which also ends at a block
//    boundary); group g is drained after the second K step of group g + 1's first tile, when its MMAs have
//    long completed; drained sums go into a plain FP32 running sum S1 that is Kahan-folded into (R, C)
//    every kTcFold drains (FP32 error independent of M; the MMA accumulation over kNT = 4 tiles keeps a
//    10× margin to the parity bar);
//  * a shared-memory stage is released by the 12 consumer warps' arrivals plus one tcgen05.commit per MMA
//    warp (its B operand read), independent of the drain.
// Per tile the consumers pick the residual mode (tile_cheap): the tile-centred residual (13 FP32 lane-ops
// per pair) on compact tiles, the hi/lo residual (16) on the others — estep_dev.cuh, DESIGN §8.
// Warp roles: 12 consumer warps (3 warpgroups × 128 TMEM lanes, 2 points per thread = 768-point blocks),
// 1 TMA producer warp, 3 MMA warps.  TMEM per warpgroup: D 2 × 32 + A 2 × 32 columns; 384 of 512 used
// (the CTA allocates all 512: one CTA per SM).
constexpr int kTcFold = 16;
#ifndef LSG_TC_NWG
#define LSG_TC_NWG 3
#define LSG_TC_RB 2
#endif

#ifndef LSG_TC_NT
#define LSG_TC_NT 4
#endif
#ifndef LSG_TC_MW
#define LSG_TC_MW LSG_TC_NWG   // MMA-issuing warps (each serves NWG / MW consumer warpgroups)
#endif
constexpr int kNWG = LSG_TC_NWG, kRB = LSG_TC_RB, kNT = LSG_TC_NT, kTcMW = LSG_TC_MW;
static_assert(kNWG % kTcMW == 0, "MMA warps must split the warpgroups evenly");
constexpr int kTcNCW = 4 * kNWG;                      // consumer warps
constexpr int kTcHelpers = (1 + kTcMW + 3) / 4 * 4;   // producer + MMA warps, padded to a whole warpgroup
constexpr int kTcThreads = (kTcNCW + kTcHelpers) * 32;
constexpr int kTcWGCols = 64 * kRB;
constexpr int kTcBlk = kNWG * 128 * kRB;              // 768 source points per block
constexpr int kTcSmF = 39;                            // S1[13], R[13], C[13] per point
constexpr size_t kTcSmem = (size_t)kTcSmF * kTcNCW * 32 * kRB * sizeof(float);
static_assert(kNWG * kTcWGCols <= kTcCols, "TMEM columns");
// setmaxnreg only moves registers within the CTA's launch allocation (launch registers per thread × threads):
// a larger request would block forever
constexpr int kTcLaunchRegs = (65536 / kTcThreads) / 8 * 8 > 255 ? 255 : (65536 / kTcThreads) / 8 * 8;
static_assert(LSG_MAXNREG == 0 ||
                  kTcNCW * 32 * LSG_MAXNREG + kTcHelpers * 32 * LSG_MAXNREG_LO <= kTcLaunchRegs * kTcThreads,
              "register split: consumer warpgroups + the helper warpgroup within the CTA's register allocation");
static_assert(kTcStages == 4, "stage arithmetic below assumes 4 stages");

template <bool kLiteral>
__global__ void __launch_bounds__(kTcThreads, 1)
    estep_tc_kernel(const char* __restrict__ tc, const float* __restrict__ src, int64_t N,
                    const IterState* __restrict__ st, Sched sc, float* __restrict__ part) {
    constexpr int NWG = kNWG, RB = kRB, NT = kNT;
    constexpr int kNCW = kTcNCW;
    constexpr int kBlk = kTcBlk;
    constexpr int kWGCols = kTcWGCols;
    constexpr int kChunks = kTcTile / kTcChunk;
    static_assert(kChunks % 2 == 0, "chunks per tile must be even");
    constexpr int kNF = 13;   // D features kept: 1, y, W, b
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
            mbar_init(&empty_bar[s], kNCW + kTcMW);
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

    if (warp >= kNCW) {   // warpgroup 3: the TMA producer warp and the MMA warps
    if (LSG_MAXNREG > 0) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(LSG_MAXNREG_LO));
    if (warp == kNCW) {
        // ---------------- producer warp: TMA bulk copies of the 10-KB tensor-core tiles ----------------
        if (lane == 0) {
            int64_t tile = u0 % sc.T;
            for (int64_t it = 0; it < nunits; ++it) {
                const int s = (int)(it & 3);
                LSG_PWAIT(&empty_bar[s], (uint32_t)(((it >> 2) & 1) ^ 1));
                mbar_arrive_expect_tx(&full_bar[s], kTcTileBytes);
                bulk_g2s(&tiles_st[s][0], tc + tile * (int64_t)kTcTileBytes, kTcTileBytes, &full_bar[s]);
                if (++tile == sc.T) tile = 0;
            }
        }
        return;
    }
    if (warp > kNCW + kTcMW) return;   // padding warps of the helper warpgroup
    if (warp > kNCW) {
        // ---------------- MMA warp: one elected lane issues the tcgen05.mma of its warpgroup(s) ----------------
        // D[db] (+)= A_hi·F_hi, += A_lo·F_hi, += A_hi·F_lo per row block and K step (N = 16 each).
        // Parities: the k-th completion of a barrier has parity k & 1; A buffer b of K step c of any tile
        // is used for the (4·it + c/2)-th time, so its parity is the constant (c >> 1) & 1.
        const uint32_t tiles0 = smem_u32(&tiles_st[0][0]) + kTcBOff;
        constexpr int kWPer = NWG / kTcMW;
        const int w0 = (warp - kNCW - 1) * kWPer;   // this MMA warp serves warpgroups [w0, w0 + kWPer)
        int64_t tile = u0 % sc.T, grp = 0;
        int tig = 0;   // tile index within the current D group
        for (int64_t it = 0; it < nunits; ++it) {
            const int s = (int)(it & 3);
            const int db = (int)(grp & 1);
            const bool first = tig == 0;
            const bool last = tig + 1 == NT || tile + 1 == sc.T || it + 1 == nunits;
            const uint32_t dpar = (uint32_t)(((grp >> 1) & 1) ^ 1);   // completion (grp>>1) - 1 of dfree[db]
            LSG_MWAIT(&full_bar[s], (uint32_t)((it >> 2) & 1));
            const uint32_t bbase = tiles0 + (uint32_t)s * kTcTileBytes;
#if LSG_PAIRED
            // one hand-off per pair of K steps (both A buffers): afull[w][0] / aempty[w][0], parity k & 1
#pragma unroll
            for (int k = 0; k < kChunks / 2; ++k) {
#pragma unroll
                for (int wi = 0; wi < kWPer; ++wi) {
                    const int w = w0 + wi;
                    if (k == 0 && first) LSG_MWAIT(&dfree[w][db], dpar);
                    LSG_MWAIT(&afull[w][0], (uint32_t)(k & 1));
                    tc_fence_after();
                    if (elect_one()) {
                        const uint32_t colD = (uint32_t)(w * kWGCols + db * 16 * RB);
#pragma unroll
                        for (int ab = 0; ab < 2; ++ab) {
                            const int c = 2 * k + ab;
                            const uint64_t bhi = bdesc(bbase + 1024 * c), blo = bdesc(bbase + 1024 * c + 512);
                            const uint32_t colA = (uint32_t)(w * kWGCols + 32 * RB + ab * 16 * RB);
#pragma unroll
                            for (int rb = 0; rb < RB; ++rb) {
                                mma_tf32_ts(colD + rb * 16, colA + rb * 16, bhi, kTcIdesc16,
                                            (c == 0 && first) ? 0u : 1u);
                                mma_tf32_ts(colD + rb * 16, colA + rb * 16 + 8, bhi, kTcIdesc16, 1u);
                                mma_tf32_ts(colD + rb * 16, colA + rb * 16, blo, kTcIdesc16, 1u);
                            }
                        }
                        mma_commit(&aempty[w][0]);
                        if (k == kChunks / 2 - 1 && last) mma_commit(&dfull[w][db]);
                        // stage s's B operand read by this warp's MMAs
                        if (k == kChunks / 2 - 1 && wi == kWPer - 1) mma_commit(&empty_bar[s]);
                    }
                    __syncwarp();
                }
            }
#else
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
#pragma unroll
                        for (int rb = 0; rb < RB; ++rb) {
                            mma_tf32_ts(colD + rb * 16, colA + rb * 16, bhi, kTcIdesc16, (c == 0 && first) ? 0u : 1u);
                            mma_tf32_ts(colD + rb * 16, colA + rb * 16 + 8, bhi, kTcIdesc16, 1u);
                            mma_tf32_ts(colD + rb * 16, colA + rb * 16, blo, kTcIdesc16, 1u);
                        }
                        mma_commit(&aempty[w][ab]);
                        if (c == kChunks - 1 && last) mma_commit(&dfull[w][db]);
                        // stage s's B operand read by this warp's MMAs
                        if (c == kChunks - 1 && wi == kWPer - 1) mma_commit(&empty_bar[s]);
                    }
                    __syncwarp();
                }
            }
#endif
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

    }   // warpgroup 3
    if (LSG_MAXNREG > 0) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(LSG_MAXNREG));

    // ---------------- consumers: warpgroup wg, TMEM lane quadrant q ----------------
    const int wg = warp >> 2, q = warp & 3;
    const int tw = q * 32 + lane;
    const int tid = threadIdx.x;
    const uint32_t tl = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(wg * kWGCols);
    const float2 nk2 = bc(-st->k2);
    const float gate = sc.gate_g * (float)sqrt(st->sigma2);
    double Rm[9], tv[3];
#pragma unroll
    for (int i = 0; i < 9; ++i) Rm[i] = st->R[i];
#pragma unroll
    for (int i = 0; i < 3; ++i) tv[i] = st->t[i];
    constexpr int kRC = kNCW * 32 * RB;

    float h[RB][3], l[RB][3];   // x̂ as FP32 hi/lo (computed in FP64)
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
                h[k][a] = __double2float_rn(X[a]);
                l[k][a] = __double2float_rn(X[a] - (double)h[k][a]);
            }
            Rt[k] = Ct[k] = 0.f;
#pragma unroll
            for (int f = 0; f < kTcSmF; ++f) smS[f * kRC + k * (kNCW * 32) + tid] = 0.f;
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
    // drain D group `gd` (all its MMAs are complete once dfull fires) and release D
    auto drain = [&](int64_t gd) {
        const int db = (int)(gd & 1);
        mbar_wait_sleep(&dfull[wg][db], (uint32_t)((gd >> 1) & 1));
        tc_fence_after();
        uint32_t d[RB][16];
#pragma unroll
        for (int rb = 0; rb < RB; ++rb) tmem_ld16(tl + (uint32_t)(db * 16 * RB + rb * 16), d[rb]);
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&dfree[wg][db]);
#pragma unroll
        for (int rb = 0; rb < RB; ++rb) {
            const int rc = rb * (kNCW * 32) + tid;
#pragma unroll
            for (int f = 0; f < kNF; ++f) smS[f * kRC + rc] += __uint_as_float(d[rb][f]);
        }
        if (++nfold == kTcFold) fold_s1();
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
    // one K step for A buffer AB: the pair math (tc_chunk_pairs), then the A rows into TMEM
    auto chunk = [&](const float4* core, int c, const float2 (&xa)[RB][3], const float2 (&xb)[RB][3],
                     float2 (&Lt)[RB], auto ABc, auto cheapc) {
        constexpr int AB = decltype(ABc)::value;
        uint32_t av[RB][16];
        tc_chunk_pairs<kLiteral, decltype(cheapc)::value, RB>(core, c, xa, xb, nk2, Lt, av);
        // the A buffer is needed only now: the MMAs of its previous use (K step c - 2) had this chunk's math
        // to finish (parity of completion 4·it + c/2 - 1)
        mbar_wait_sleep(&aempty[wg][AB], (uint32_t)(((c >> 1) & 1) ^ 1));
        tc_fence_after();
#pragma unroll
        for (int rb = 0; rb < RB; ++rb) tmem_st16(tl + (uint32_t)(32 * RB + AB * 16 * RB + rb * 16), av[rb]);
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&afull[wg][AB]);
    };

    // two K steps (both A buffers) per hand-off: one aempty wait, one wait::st, one afull arrival per pair
    auto chunk_pair = [&](const float4* core, int k, const float2 (&xa)[RB][3], const float2 (&xb)[RB][3],
                          float2 (&Lt)[RB], auto PARc, auto cheapc) {
        constexpr uint32_t PAR = decltype(PARc)::value;
        uint32_t av0[RB][16], av1[RB][16];
        tc_chunk_pairs<kLiteral, decltype(cheapc)::value, RB>(core, 2 * k, xa, xb, nk2, Lt, av0);
        tc_chunk_pairs<kLiteral, decltype(cheapc)::value, RB>(core, 2 * k + 1, xa, xb, nk2, Lt, av1);
        LSG_CWAIT(&aempty[wg][0], PAR ^ 1u);   // the MMAs of the previous pair are complete
        tc_fence_after();
#pragma unroll
        for (int rb = 0; rb < RB; ++rb) tmem_st16(tl + (uint32_t)(32 * RB + rb * 16), av0[rb]);
#pragma unroll
        for (int rb = 0; rb < RB; ++rb) tmem_st16(tl + (uint32_t)(32 * RB + 16 * RB + rb * 16), av1[rb]);
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&afull[wg][0]);
    };

    int64_t j = u0 / sc.T, tile = u0 % sc.T;
    load_points(j);
    bool pending = false;   // the previous D group has not been drained yet
    int64_t grp = 0, pend_g = 0;
    int tig = 0;
    for (int64_t it = 0; it < nunits; ++it) {
        LSG_CWAIT(&full_bar[it & 3], (uint32_t)((it >> 2) & 1));
        const float4* core = reinterpret_cast<const float4*>(&tiles_st[it & 3][0]);
        float2 Lt[RB];
#pragma unroll
        for (int k = 0; k < RB; ++k) Lt[k] = make_float2(0.f, 0.f);
        const TileMeta tm = tile_meta(core);
        auto run_tile = [&](auto cheapc) {
            float2 xa[RB][3], xb[RB][3];
            tile_points<decltype(cheapc)::value, RB>(h, l, tm, xa, xb);
#if LSG_PAIRED
#pragma unroll 1
            for (int k = 0; k < kChunks / 2; k += 2) {
                chunk_pair(core, k, xa, xb, Lt, std::integral_constant<uint32_t, 0>(), cheapc);
                if (k == 0 && pending && tig >= kDrainLag) {
                    drain(pend_g);
                    pending = false;
                }
                chunk_pair(core, k + 1, xa, xb, Lt, std::integral_constant<uint32_t, 1>(), cheapc);
            }
#else
            LSG_UNROLL(LSG_TC_UNROLL)
            for (int c = 0; c < kChunks; c += 2) {
                chunk(core, c, xa, xb, Lt, std::integral_constant<int, 0>(), cheapc);
                chunk(core, c + 1, xa, xb, Lt, std::integral_constant<int, 1>(), cheapc);
                if (c == 0 && pending && tig >= kDrainLag) {
                    drain(pend_g);
                    pending = false;
                }
            }
#endif
        };
        if (tile_cheap(tm, gate) || (sc.far_rule && warp_far<RB>(h, l, tm))) run_tile(std::true_type());
        else run_tile(std::false_type());
        __syncwarp();   // this warp is done reading the stage's core data
        if (lane == 0) mbar_arrive(&empty_bar[it & 3]);
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
                if (pending) {
                    drain(pend_g);
                    pending = false;
                }
                drain(grp);
                flush(j);
            } else {
                pending = true;
                pend_g = grp;
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
    // all MMAs of this warpgroup completed (dfull of the last group was awaited); release TMEM
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
    if (!st->active) {
        if (st->status == LSGCPD_EINVAL) {   // the target did not match (estep_setup_kernel): all-NaN record
            const int64_t i = (int64_t)blockIdx.x * kMergePts * LSGCPD_REC + threadIdx.x;
            if (i < N * LSGCPD_REC) rec[i] = __int_as_float(0x7fc00000);
        }
        return;
    }
    __shared__ float tile[kMergePts][LSGCPD_REC + 1];
    __shared__ double a0s[kMergePts];
    const int64_t n0 = (int64_t)blockIdx.x * kMergePts;
    merge_tile32(part, N, n0, st, sc, phi, tile, a0s);
    __syncthreads();
    const int p = threadIdx.x / LSGCPD_REC, g = threadIdx.x % LSGCPD_REC;
    if (n0 + p < N) rec[(n0 + p) * LSGCPD_REC + g] = tile[p][g];
}


// ---- host-side planning and launch ---------------------------------------------------------
// CUDA-core kernel configurations (points per thread, consumer warps, min CTAs/SM, packed):
//   0  768-point blocks (12 consumer warps): the running-max mode of large problems, and LSGCPD_TC=0
//   1  512-point blocks (8 warps): problems too small to fill the GPU with 768-point tensor-core blocks
//   2  64-point blocks (1 warp, 8 CTAs/SM): the smallest problems (most CTAs per problem)
// tools/small_path_sweep.py picked the small-problem rule.
struct Variant {
    int ppt, ncw, minb, packed;
    const void* fn[2];  // [literal]
};
#define LSG_VARIANT(P, W, B, X) \
    {P, W, B, X, {(const void*)estep_kernel<P, W, B, X, false>, (const void*)estep_kernel<P, W, B, X, true>}}
static const Variant kVariants[] = {LSG_VARIANT(kTcBlk / (kTcNCW * 32), kTcNCW, 1, true), LSG_VARIANT(2, 8, 1, true),
                                    LSG_VARIANT(2, 1, 8, true)};
constexpr int kNumVariants = sizeof(kVariants) / sizeof(kVariants[0]);
constexpr int kBigVariant = 0, kMidVariant = 1, kSmallVariant = 2;
constexpr int kMidBlk = 2 * 8 * 32;
static_assert(kTcBlk % (kTcNCW * 32) == 0, "the running-max partner of the tensor-core kernel uses its block size");
constexpr int64_t kSplitBytes = 48ll << 20;   // tensor-core sections above this are swept in two halves

// Per-device facts (SM count, occupancies) and one-time function attributes, set up once per device under a
// lock (a thread may move between devices; function attributes are per device).
struct DevInfo {
    bool ready = false;
    int nsm = 0;
    int occ[kNumVariants] = {};
};
static std::mutex g_dev_mu;
static DevInfo g_dev[64];

static int device_info(const DevInfo** out) {
    int dev;
    LSG_CUDA(cudaGetDevice(&dev));
    LSG_CHECK(dev >= 0 && dev < 64, LSGCPD_ECUDA, "device ordinal %d out of range", dev);
    std::lock_guard<std::mutex> lk(g_dev_mu);
    DevInfo& d = g_dev[dev];
    if (!d.ready) {
        LSG_CUDA(cudaDeviceGetAttribute(&d.nsm, cudaDevAttrMultiProcessorCount, dev));
        for (int v = 0; v < kNumVariants; ++v) {
            int occ = 0;
            LSG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kVariants[v].fn[0],
                                                                   (kVariants[v].ncw + 1) * 32, 0));
            d.occ[v] = occ > 0 ? occ : 1;
        }
        LSG_CUDA(cudaFuncSetAttribute((const void*)estep_tc_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)kTcSmem));
        LSG_CUDA(cudaFuncSetAttribute((const void*)estep_tc_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)kTcSmem));
        d.ready = true;
    }
    *out = &d;
    return 0;
}

int sm_count() {
    const DevInfo* d = nullptr;
    return device_info(&d) ? 0 : d->nsm;
}

int estep_plan(int64_t M_pad, int64_t N, Sched* sc) {
    const Options& op = options();
    const int mode = op.tc.load();   // 0 off, 1 forced, 2 automatic
    const int forced = op.estep_variant.load();
    const DevInfo* di = nullptr;
    const int rc = device_info(&di);
    if (rc) return rc;
    bool tc = mode != 0;
    int vi = (forced >= 0 && forced < kNumVariants) ? forced : kBigVariant;
    if (tc) vi = kBigVariant;
    if (mode == 2 && forced < 0) {
        // small problems (tiny / object configs): too few (block, tile) units for one CTA per SM with the
        // big blocks — use the small-block CUDA-core kernel so every SM gets work
        const int64_t units_big = (N + kTcBlk - 1) / kTcBlk * (M_pad / kTT);
        if (units_big < 2 * (int64_t)di->nsm) {
            // 512-point blocks once they give ~3/4 of a unit per SM, else 64-point blocks (the most CTAs):
            // tools/small_path_sweep.py — 1,000 points 38 µs per EM iteration with 64-point blocks, 2,000 / 3,500
            // points 44 / 56 µs with 512-point blocks (64-point: 51 / 72; tensor cores: 50 / 59)
            tc = false;
            const int64_t units_mid = (N + kMidBlk - 1) / kMidBlk * (M_pad / kTT);
            vi = 4 * units_mid >= 3 * (int64_t)di->nsm ? kMidVariant : kSmallVariant;
        }
    }
    const Variant& V = kVariants[vi];
    Sched s;
    memset(&s, 0, sizeof(s));
    s.variant = tc ? -1 - vi : vi;   // negative: tensor-core kernel + CUDA-core variant for running max
    s.tc_variant = 0;
    s.B = (int64_t)V.ppt * V.ncw * 32;
    s.nblk = (N + s.B - 1) / s.B;
    // a tensor-core section larger than ~48 MB is swept in two halves, one launch each, so every CTA reads
    // tiles of the same half at a time and the half stays in L2 (the whole section re-read from HBM otherwise;
    // DESIGN §7 "DRAM traffic").  M_pad is a multiple of 256 targets, so the tile count is even.
    const int hv = op.halves.load();
    const bool split = tc && (M_pad / kTT) * (int64_t)kTcTileBytes > kSplitBytes && hv != 1;
    s.halves = split ? 2 : 1;
    s.gate_g = op.tile_gate.load();
    s.far_rule = op.far_rule.load() ? 1 : 0;
    s.T = M_pad / kTT / s.halves;
    s.U = s.nblk * s.T;
    const int64_t slots = (int64_t)di->nsm * (tc ? 1 : di->occ[vi]);   // the TC kernel holds all TMEM: 1 CTA/SM
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

int estep_launch(const void* d_target, const float* d_src, int64_t N, const IterState* st, const Sched& sc,
                 float* part, float* rec, int consistent, const float* phi, cudaStream_t stream, int merge) {
    const bool tc = sc.variant < 0;
    const Variant& V = kVariants[tc ? -1 - sc.variant : sc.variant];
    Sched scv = sc;
    int skip_fixed = tc ? 1 : 0;
    const int64_t M_pad = sc.T * kTT * sc.halves;
    for (int h = 0; h < sc.halves; ++h) {   // one sweep per half of the targets (sc.T tiles each)
        const float* body = target_body(d_target) + (int64_t)h * sc.T * kTT * kTgtFloats;
        float* parth = part + (int64_t)h * sc.hstride;
        if (tc) {
            const char* tcb = reinterpret_cast<const char*>(target_tc(d_target, M_pad)) +
                              (int64_t)h * sc.T * kTcTileBytes;
            void* targs[] = {(void*)&tcb, (void*)&d_src, (void*)&N, (void*)&st, (void*)&scv, (void*)&parth};
            const void* fn = consistent ? (const void*)estep_tc_kernel<false> : (const void*)estep_tc_kernel<true>;
            LSG_CUDA(cudaLaunchKernel(fn, dim3((unsigned)sc.G), dim3(kTcThreads), targs, kTcSmem, stream));
        }
        void* args[] = {(void*)&body, (void*)&d_src, (void*)&N, (void*)&st, (void*)&scv, (void*)&parth,
                        (void*)&skip_fixed};
        LSG_CUDA(cudaLaunchKernel(V.fn[consistent ? 0 : 1], dim3((unsigned)sc.G), dim3((V.ncw + 1) * 32), args, 0,
                                  stream));
    }
    if (!merge) return 0;
    estep_merge_kernel<<<(unsigned)((N + kMergePts - 1) / kMergePts), kMergePts * 16, 0, stream>>>(part, N, st, sc,
                                                                                                 rec, phi);
    LSG_CUDA(cudaGetLastError());
    return 0;
}

// ---- options (read once from the environment; lsgcpd_set_option changes them at run time) ----------------
static int env_int(const char* name, int dflt) {
    const char* e = getenv(name);
    return e && *e ? atoi(e) : dflt;
}
Options::Options() {
    const char* t = getenv("LSGCPD_TC");
    tc.store(t && *t ? (atoi(t) != 0 ? 1 : 0) : 2);
    estep_variant.store(env_int("LSGCPD_ESTEP_VARIANT", -1));
    halves.store(env_int("LSGCPD_HALVES", 0));
    no_fuse.store(env_int("LSGCPD_NO_FUSE", 0));
    graph_cache.store(env_int("LSGCPD_GRAPH_CACHE", 1));
    no_graph.store(env_int("LSGCPD_NO_GRAPH", 0));
    const char* g = getenv("LSGCPD_TILE_GATE");
    tile_gate.store(g && *g ? (float)atof(g) : kDefaultTileGate);
    far_rule.store(env_int("LSGCPD_FAR_RULE", 1));
    sort_source.store(env_int("LSGCPD_SORT_SOURCE", 1));
}
Options& options() {
    static Options o;   // thread-safe one-time initialisation (C++11 magic static)
    return o;
}

}  // namespace lsg
