// Batched E step for many small registrations in one launch (paper-scale
// 3.5k-5k-point pairs; the §4.1 sweeps of 30 runs).
//
// Same per-pair arithmetic as the single-problem CUDA-core kernel (estep.cu, P:189-193 / Eq. 5 with the
// Eq. 2 densities): r = (hi - y) + lo, τ = ||r||² + (ñ·r)², p = 2^{ω̄ - k2 τ} (fixed max) or with a
// per-point running max (per problem), 14 Kahan-folded accumulators per point.  What is new is the work
// decomposition: the units (source block, target tile) of ALL problems are concatenated and split
// stream-K over one persistent grid, so B problems of 1k-10k points fill the 148 SMs that one of them
// alone cannot (a 5k × 5k E step is 25 M pairs ≈ 20 µs of one B200, less than its launch latency).
// Each CTA walks its unit range in order; when the problem changes it flushes the current block's
// partial, reloads the problem's constants (k2, pose, fixed/running-max mode) and source points, and the
// TMA producer switches to that problem's target.  Problems that finished (IterState.active = 0) are
// skipped by producer and consumers alike.
#include <mutex>

#include "common.cuh"
#include "estep_dev.cuh"
#include "kernels.h"

namespace lsg {

constexpr int kBPPT = 2;                     // source points per consumer thread (one f32x2 lane)
constexpr int kBNCW = 12;                    // consumer warps
constexpr int kBMinB = 1;                    // CTAs per SM
constexpr int kBBlk = kBPPT * kBNCW * 32;    // 768 source points per block (= the tensor-core kernel's)

int batch_block_points() { return kBBlk; }
size_t batch_partial_floats(int64_t nblk, int64_t kmax) { return (size_t)nblk * kmax * kPartF * kBBlk; }

// first problem whose unit range contains u (binary search over unit0)
__device__ __forceinline__ int find_problem_unit(const BatchProblem* __restrict__ bp, int B, int64_t u) {
    int lo = 0, hi = B - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (bp[mid].unit0 <= u) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}
__device__ __forceinline__ int find_problem_point(const BatchProblem* __restrict__ bp, int B, int64_t p) {
    int lo = 0, hi = B - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (bp[mid].pt0 <= p) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// Cursor over the concatenated unit space: (problem b, block j, tile i) for the CTA's units in order.
struct BatchCursor {
    int b;
    int64_t j, tile;
    __device__ void start(const BatchProblem* bp, int B, int64_t u) {
        b = find_problem_unit(bp, B, u);
        const int64_t lu = u - bp[b].unit0;
        j = lu / bp[b].T;
        tile = lu % bp[b].T;
    }
    // jump to the last unit of the current problem (the caller's loop step then enters the next problem):
    // skipping a problem costs one step instead of one per unit
    __device__ void to_last(const BatchProblem* bp, int64_t& u) {
        const BatchProblem& P = bp[b];
        j = P.nblk - 1;
        tile = P.T - 1;
        u = P.unit0 + P.nblk * P.T - 1;
    }
    __device__ void next(const BatchProblem* bp) {
        if (++tile == bp[b].T) {
            tile = 0;
            if (++j == bp[b].nblk) {   // every problem has ≥ 1 block (N ≥ 1, checked on the host)
                j = 0;
                ++b;
            }
        }
    }
};

// Which problems a batched E-step kernel serves: mode 0 = every active problem (CUDA cores only),
// 1 = active problems in the running-max mode (the tensor-core kernel takes the fixed-max ones).
__device__ __forceinline__ bool serves(const IterState& s, int mode) {
    return s.active && (mode == 0 || !s.fixed);
}

template <bool kLiteral>
__global__ void __launch_bounds__((kBNCW + 1) * 32, kBMinB)
    estep_batch_kernel(const BatchProblem* __restrict__ bp, int B, const IterState* __restrict__ st, Sched sc,
                       float* __restrict__ part, int mode) {
    using T = float2;
    constexpr int NL = kBPPT / 2;
    constexpr int kTileF4 = kTT * kTgtFloats / 4;
    __shared__ __align__(128) float4 tiles[kStages * kTileF4];
    __shared__ __align__(8) uint64_t full_bar[kStages];
    __shared__ __align__(8) uint64_t empty_bar[kStages];

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t g = blockIdx.x;
    const int64_t u0 = sched_start(sc, g), u1 = sched_start(sc, g + 1);
    if (u0 >= u1) return;
    {   // nothing to serve in this CTA's range (e.g. mode 1 while every problem is in the fixed-max mode)
        const int b0 = find_problem_unit(bp, B, u0), b1 = find_problem_unit(bp, B, u1 - 1);
        bool any = false;
        for (int b = b0; b <= b1 && !any; ++b) any = serves(st[b], mode);
        if (!any) return;
    }

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], kBNCW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == kBNCW) {
        // producer: TMA bulk copies of the current problem's target tiles (inactive problems skipped)
        if (lane == 0) {
            BatchCursor cur;
            cur.start(bp, B, u0);
            int64_t it = 0;
            for (int64_t u = u0; u < u1; ++u, cur.next(bp)) {
                if (!serves(st[cur.b], mode)) { cur.to_last(bp, u); continue; }
                const int s = (int)(it % kStages);
                const uint32_t ph = (uint32_t)((it / kStages) & 1);
                mbar_wait_sleep(&empty_bar[s], ph ^ 1);
                mbar_arrive_expect_tx(&full_bar[s], kTT * kTgtFloats * 4);
                bulk_g2s(&tiles[s * kTileF4], bp[cur.b].body + cur.tile * (int64_t)kTT * kTgtFloats,
                         kTT * kTgtFloats * 4, &full_bar[s]);
                ++it;
            }
        }
        return;
    }

    const int tid = threadIdx.x;
    Acc<T> R[NL], C[NL];
    T h[NL][3], l[NL][3], mu[NL];
    float k2 = 0.f;
    bool fixed = true;
    int cur_b = -1;
    int64_t cur_j = -1;

    auto load_points = [&](int b, int64_t j) {
        const IterState* s = st + b;
        k2 = s->k2;
        fixed = s->fixed != 0;
        const float Lo_f = (float)s->Lo;
        double Rm[9], tv[3];
#pragma unroll
        for (int i = 0; i < 9; ++i) Rm[i] = s->R[i];
#pragma unroll
        for (int i = 0; i < 3; ++i) tv[i] = s->t[i];
        const float* src = bp[b].src;
        const int64_t N = bp[b].N;
#pragma unroll
        for (int L = 0; L < NL; ++L) {
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const int64_t n = j * kBBlk + (int64_t)(L * 2 + k) * (kBNCW * 32) + tid;
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
    auto flush = [&](int b, int64_t j) {
        const BatchProblem& P = bp[b];
        const int64_t slot = j * sc.kmax + (g - sched_owner(sc, P.unit0 + j * P.T));
        float* base = part + P.part0 + slot * (int64_t)kPartF * kBBlk;
#pragma unroll
        for (int L = 0; L < NL; ++L)
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const int bb = (L * 2 + k) * (kBNCW * 32) + tid;
#pragma unroll
                for (int f = 0; f < kAcc; ++f) base[f * kBBlk + bb] = __fsub_rn(lane_of(R[L].v[f], k), lane_of(C[L].v[f], k));
                base[14 * kBBlk + bb] = lane_of(mu[L], k);
                base[15 * kBBlk + bb] = 0.f;
            }
    };

    BatchCursor cur;
    cur.start(bp, B, u0);
    int64_t it = 0;
    for (int64_t u = u0; u < u1; ++u, cur.next(bp)) {
        if (!serves(st[cur.b], mode)) { cur.to_last(bp, u); continue; }
        if (cur.b != cur_b || cur.j != cur_j) {
            if (cur_b >= 0) flush(cur_b, cur_j);
            cur_b = cur.b;
            cur_j = cur.j;
            load_points(cur_b, cur_j);
        }
        const int s = (int)(it % kStages);
        mbar_wait(&full_bar[s], (uint32_t)((it / kStages) & 1));
        ++it;
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
                for (int k = 0; k < 2; ++k) {
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
    if (cur_b >= 0) flush(cur_b, cur_j);
}

// ---- batched tensor-core E step ---------------------------------------------------------------------
// estep_tc_kernel's pipeline (TMA producer, one MMA warp per warpgroup, TF32 3-term split of p into TMEM,
// D accumulated over NT tiles, Kahan-folded drains) walking the concatenated units of the problems that are
// active and in the fixed-max mode.  A D group also ends where a source block (hence a problem) ends.
constexpr int kBTNWG = 3, kBTRB = 2, kBTMW = 3, kBTNT = 4;
constexpr int kBTNCW = 4 * kBTNWG;
constexpr int kBTThreads = (kBTNCW + 1 + kBTMW) * 32;
// register split (setmaxnreg): the producer / MMA warps walk the problem list (BatchCursor) with 48 registers
// (a few spills outside their waits), each consumer thread gets 152 (tools/batch_speed.py: 144/72 → 152/48
// +1.5 %, 160/32 +1.3 %; gpurun_out/r04f)
#ifndef LSG_BT_REG_HI
#define LSG_BT_REG_HI 152
#define LSG_BT_REG_LO 48
#endif
constexpr int kBTRegHi = LSG_MAXNREG > 0 ? LSG_BT_REG_HI : 0, kBTRegLo = LSG_BT_REG_LO;
static_assert(kBTRegHi == 0 || (kBTThreads == 512 && 384 * kBTRegHi + 128 * kBTRegLo <= 65536),
              "register split: 3 consumer warpgroups + warpgroup 3");
constexpr int kBTWGCols = 64 * kBTRB;
constexpr int kBTSmF = 39;
constexpr size_t kBTSmem = (size_t)kBTSmF * kBTNCW * 32 * kBTRB * sizeof(float);
static_assert(kBTNWG * 128 * kBTRB == kBBlk, "both batched kernels use one block size");

__device__ __forceinline__ bool serves_tc(const IterState& s) { return s.active && s.fixed; }

template <bool kLiteral>
__global__ void __launch_bounds__(kBTThreads, 1)
    estep_batch_tc_kernel(const BatchProblem* __restrict__ bp, int B, const IterState* __restrict__ st, Sched sc,
                          float* __restrict__ part) {
    constexpr int NWG = kBTNWG, RB = kBTRB, MW = kBTMW, NT = kBTNT;
    constexpr int kNCW = kBTNCW, kBlk = kBBlk, kWGCols = kBTWGCols;
    constexpr int kChunks = kTcTile / kTcChunk;
    constexpr int kNF = 13;
    __shared__ __align__(1024) char tiles_st[kTcStages][kTcTileBytes];
    extern __shared__ __align__(16) char dsmem[];
    float* smS = reinterpret_cast<float*>(dsmem);
    __shared__ __align__(8) uint64_t full_bar[kTcStages];
    __shared__ __align__(8) uint64_t empty_bar[kTcStages];
    __shared__ __align__(8) uint64_t afull[NWG][2], aempty[NWG][2], dfull[NWG][2], dfree[NWG][2];
    __shared__ uint32_t tmem_base_sh;

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t g = blockIdx.x;
    const int64_t u0 = sched_start(sc, g), u1 = sched_start(sc, g + 1);
    if (u0 >= u1) return;
    // does this CTA have any unit to serve?  (all roles must agree before TMEM is allocated)
    {
        BatchCursor c0;
        c0.start(bp, B, u0);
        const BatchCursor cl = c0;
        bool any = false;
        // the range spans problems c0.b .. the problem of u1 - 1
        const int b1 = find_problem_unit(bp, B, u1 - 1);
        for (int b = cl.b; b <= b1 && !any; ++b) any = serves_tc(st[b]);
        if (!any) return;
    }

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                     "r"((uint32_t)kTcCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (threadIdx.x == 32) {
        for (int s = 0; s < kTcStages; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], kNCW + MW);
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
    if (tmem != 0u) __trap();

    if (warp >= kNCW) {   // warpgroup 3: the TMA producer warp and the MMA warps (registers to the consumers)
    if (kBTRegHi > 0) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(kBTRegLo));
    if (warp == kNCW) {
        // producer: TMA bulk copies of the served problems' tensor-core tiles
        if (lane == 0) {
            BatchCursor cur;
            cur.start(bp, B, u0);
            int64_t it = 0;
            for (int64_t u = u0; u < u1; ++u, cur.next(bp)) {
                if (!serves_tc(st[cur.b])) { cur.to_last(bp, u); continue; }
                const int s = (int)(it & 3);
                mbar_wait_sleep(&empty_bar[s], (uint32_t)(((it >> 2) & 1) ^ 1));
                mbar_arrive_expect_tx(&full_bar[s], kTcTileBytes);
                bulk_g2s(&tiles_st[s][0], bp[cur.b].tc + cur.tile * (int64_t)kTcTileBytes, kTcTileBytes, &full_bar[s]);
                ++it;
            }
        }
        return;
    }
    if (warp > kNCW) {
        // MMA warp for warpgroup w (see estep_tc_kernel); groups end at NT tiles or a block end
        const uint32_t tiles0 = smem_u32(&tiles_st[0][0]) + kTcBOff;
        const int w = warp - kNCW - 1;
        BatchCursor cur;
        cur.start(bp, B, u0);
        int64_t it = 0, grp = 0;
        int tig = 0;
        for (int64_t u = u0; u < u1; ++u, cur.next(bp)) {
            if (!serves_tc(st[cur.b])) { cur.to_last(bp, u); continue; }
            const int s = (int)(it & 3);
            const int db = (int)(grp & 1);
            const bool first = tig == 0;
            const bool last = tig + 1 == NT || cur.tile + 1 == bp[cur.b].T || u + 1 == u1;
            const uint32_t dpar = (uint32_t)(((grp >> 1) & 1) ^ 1);
            mbar_wait_sleep(&full_bar[s], (uint32_t)((it >> 2) & 1));
            const uint32_t bbase = tiles0 + (uint32_t)s * kTcTileBytes;
#if LSG_PAIRED
#pragma unroll
            for (int k = 0; k < kChunks / 2; ++k) {   // one hand-off per pair of K steps (see estep.cu)
                if (k == 0 && first) mbar_wait_sleep(&dfree[w][db], dpar);
                mbar_wait_sleep(&afull[w][0], (uint32_t)(k & 1));
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
                            mma_tf32_ts(colD + rb * 16, colA + rb * 16, bhi, kTcIdesc16, (c == 0 && first) ? 0u : 1u);
                            mma_tf32_ts(colD + rb * 16, colA + rb * 16 + 8, bhi, kTcIdesc16, 1u);
                            mma_tf32_ts(colD + rb * 16, colA + rb * 16, blo, kTcIdesc16, 1u);
                        }
                    }
                    mma_commit(&aempty[w][0]);
                    if (k == kChunks / 2 - 1 && last) mma_commit(&dfull[w][db]);
                    if (k == kChunks / 2 - 1) mma_commit(&empty_bar[s]);
                }
                __syncwarp();
            }
#else
#pragma unroll
            for (int c = 0; c < kChunks; ++c) {
                const int ab = c & 1;
                const uint64_t bhi = bdesc(bbase + 1024 * c), blo = bdesc(bbase + 1024 * c + 512);
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
                    if (c == kChunks - 1) mma_commit(&empty_bar[s]);
                }
                __syncwarp();
            }
#endif
            if (last) {
                tig = 0;
                ++grp;
            } else {
                ++tig;
            }
            ++it;
        }
        return;
    }
    }   // warpgroup 3
    if (kBTRegHi > 0) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(kBTRegHi));

    // consumers
    const int wg = warp >> 2, q = warp & 3;
    const int tw = q * 32 + lane;
    const int tid = threadIdx.x;
    const uint32_t tl = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(wg * kWGCols);
    constexpr int kRC = kNCW * 32 * RB;
    float h[RB][3], l[RB][3];   // x̂ as FP32 hi/lo
    float Rt[RB], Ct[RB];
    float k2 = 0.f, gate = 0.f;
    float2 nk2 = bc(0.f);
    int nfold = 0;

    auto load_points = [&](int b, int64_t j) {
        const IterState* s = st + b;
        k2 = s->k2;
        nk2 = bc(-k2);
        gate = sc.gate_g * (float)sqrt(s->sigma2);
        double Rm[9], tv[3];
#pragma unroll
        for (int i = 0; i < 9; ++i) Rm[i] = s->R[i];
#pragma unroll
        for (int i = 0; i < 3; ++i) tv[i] = s->t[i];
        const float* src = bp[b].src;
        const int64_t N = bp[b].N;
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
            for (int f = 0; f < kBTSmF; ++f) smS[f * kRC + k * (kNCW * 32) + tid] = 0.f;
        }
        nfold = 0;
    };
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
        if (++nfold == 16) fold_s1();
    };
    auto flush = [&](int b, int64_t j) {
        fold_s1();
        const BatchProblem& P = bp[b];
        const int64_t slot = j * sc.kmax + (g - sched_owner(sc, P.unit0 + j * P.T));
        float* base = part + P.part0 + slot * (int64_t)kPartF * kBlk;
#pragma unroll
        for (int k = 0; k < RB; ++k) {
            const int bb = (wg * RB + k) * 128 + tw;
            const int rc = k * (kNCW * 32) + tid;
#pragma unroll
            for (int f = 0; f < 13; ++f)
                base[f * kBlk + bb] = __fsub_rn(smS[(kNF + f) * kRC + rc], smS[(2 * kNF + f) * kRC + rc]);
            base[13 * kBlk + bb] = __fsub_rn(Rt[k], Ct[k]);
            base[14 * kBlk + bb] = 0.f;
            base[15 * kBlk + bb] = 0.f;
        }
    };
    // one K step (tile-centred or hi/lo residual, estep_dev.cuh), then the A rows into TMEM
    auto chunk = [&](const float4* core, int c, const float2 (&xa)[RB][3], const float2 (&xb)[RB][3],
                     float2 (&Lt)[RB], auto ABc, auto cheapc) {
        constexpr int AB = decltype(ABc)::value;
        uint32_t av[RB][16];
        tc_chunk_pairs<kLiteral, decltype(cheapc)::value, RB>(core, c, xa, xb, nk2, Lt, av);
        mbar_wait_sleep(&aempty[wg][AB], (uint32_t)(((c >> 1) & 1) ^ 1));
        tc_fence_after();
#pragma unroll
        for (int rb = 0; rb < RB; ++rb) tmem_st16(tl + (uint32_t)(32 * RB + AB * 16 * RB + rb * 16), av[rb]);
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&afull[wg][AB]);
    };

    auto chunk_pair = [&](const float4* core, int k, const float2 (&xa)[RB][3], const float2 (&xb)[RB][3],
                          float2 (&Lt)[RB], auto PARc, auto cheapc) {
        constexpr uint32_t PAR = decltype(PARc)::value;
        uint32_t av0[RB][16], av1[RB][16];
        tc_chunk_pairs<kLiteral, decltype(cheapc)::value, RB>(core, 2 * k, xa, xb, nk2, Lt, av0);
        tc_chunk_pairs<kLiteral, decltype(cheapc)::value, RB>(core, 2 * k + 1, xa, xb, nk2, Lt, av1);
        LSG_CWAIT(&aempty[wg][0], PAR ^ 1u);
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

    BatchCursor cur;
    cur.start(bp, B, u0);
    int cur_b = -1;
    int64_t cur_j = -1, it = 0, grp = 0, pend_g = 0;
    int tig = 0;
    bool pending = false;
    for (int64_t u = u0; u < u1; ++u, cur.next(bp)) {
        if (!serves_tc(st[cur.b])) { cur.to_last(bp, u); continue; }
        if (cur.b != cur_b || cur.j != cur_j) {   // previous block fully drained and flushed at its end
            cur_b = cur.b;
            cur_j = cur.j;
            load_points(cur_b, cur_j);
        }
        const int s = (int)(it & 3);
        LSG_CWAIT(&full_bar[s], (uint32_t)((it >> 2) & 1));
        const float4* core = reinterpret_cast<const float4*>(&tiles_st[s][0]);
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
#pragma unroll 1
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
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty_bar[s]);
#pragma unroll
        for (int rb = 0; rb < RB; ++rb) {
            const float L = Lt[rb].x + Lt[rb].y;
            const float y = L - Ct[rb];
            const float t = Rt[rb] + y;
            Ct[rb] = (t - Rt[rb]) - y;
            Rt[rb] = t;
        }
        const bool block_end = cur.tile + 1 == bp[cur.b].T || u + 1 == u1;
        const bool last = tig + 1 == NT || block_end;
        if (last) {
            if (block_end) {
                if (pending) {
                    drain(pend_g);
                    pending = false;
                }
                drain(grp);
                flush(cur_b, cur_j);
            } else {
                pending = true;
                pend_g = grp;
            }
            tig = 0;
            ++grp;
        } else {
            ++tig;
        }
        ++it;
    }
    tc_fence_before();
    named_bar_sync(1, kNCW * 32);
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"((uint32_t)kTcCols)
                     : "memory");
    }
}

// merge: one thread per point of the concatenated record
__global__ void estep_batch_merge_kernel(const BatchProblem* __restrict__ bp, int B, const IterState* __restrict__ st,
                                         Sched sc, const float* __restrict__ part, float* __restrict__ rec,
                                         int64_t Ntot) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= Ntot) return;
    const int b = find_problem_point(bp, B, p);
    const BatchProblem& P = bp[b];
    if (!st[b].active) return;
    const int64_t n = p - P.pt0;
    const int64_t j = n / kBBlk;
    const int64_t g0 = sched_owner(sc, P.unit0 + j * P.T);
    const int64_t g1 = sched_owner(sc, P.unit0 + (j + 1) * P.T - 1);
    merge_point(part + P.part0 + j * sc.kmax * (int64_t)kPartF * kBBlk, g1 - g0 + 1, kBBlk, (int)(n % kBBlk), st + b,
                P.conf ? P.conf + n : nullptr, rec + p * LSGCPD_REC);
}

// Per-problem fields that live in the target header (read on the device: no host round trip per problem):
// V (unless the caller gave one), extent, ω_ref, Σπ√(1+α); err[b] = 1 bad target, 2 priors with the literal form.
__global__ void batch_fill_kernel(BatchProblem* bp, int B, int consistent, int* err) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    BatchProblem& P = bp[b];
    const TargetHeader* h = reinterpret_cast<const TargetHeader*>(P.target);
    int e = 0;
    if (h->magic != kTargetMagic || h->M != P.M) e = 1;
    else if (!consistent && h->prior) e = 2;
    err[b] = e;
    if (e) return;
    if (!(P.volume > 0.0)) P.volume = h->volume;
    P.extent = h->extent;
    P.omega_ref = consistent ? h->omega_ref : 0.0;
    P.spc = h->spc;
}
void batch_fill_launch(BatchProblem* bp, int B, int consistent, int* err, cudaStream_t stream) {
    batch_fill_kernel<<<(B + 127) / 128, 128, 0, stream>>>(bp, B, consistent, err);
}

// tensor cores for the fixed-max problems unless the tc option is 0 (CUDA cores only)
static int batch_tc_mode() { return options().tc.load() != 0 ? 1 : 0; }
static std::mutex g_battr_mu;
static bool g_battr[64];   // per device: the tensor-core kernel's shared-memory attribute is set

void estep_batch_launch(const BatchProblem* bp, int B, const Sched& sc, const IterState* st, float* part, float* rec,
                        int64_t Ntot, int consistent, cudaStream_t stream) {
    const int tc = batch_tc_mode();
    if (tc) {
        int dev = 0;
        cudaGetDevice(&dev);
        std::lock_guard<std::mutex> lk(g_battr_mu);
        if (dev >= 0 && dev < 64 && !g_battr[dev]) {
            cudaFuncSetAttribute((const void*)estep_batch_tc_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)kBTSmem);
            cudaFuncSetAttribute((const void*)estep_batch_tc_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)kBTSmem);
            g_battr[dev] = true;
        }
        if (consistent)
            estep_batch_tc_kernel<false><<<(unsigned)sc.G, kBTThreads, kBTSmem, stream>>>(bp, B, st, sc, part);
        else
            estep_batch_tc_kernel<true><<<(unsigned)sc.G, kBTThreads, kBTSmem, stream>>>(bp, B, st, sc, part);
    }
    if (consistent)
        estep_batch_kernel<false><<<(unsigned)sc.G, (kBNCW + 1) * 32, 0, stream>>>(bp, B, st, sc, part, tc);
    else
        estep_batch_kernel<true><<<(unsigned)sc.G, (kBNCW + 1) * 32, 0, stream>>>(bp, B, st, sc, part, tc);
    const int mt = 256;
    estep_batch_merge_kernel<<<(unsigned)((Ntot + mt - 1) / mt), mt, 0, stream>>>(bp, B, st, sc, part, rec, Ntot);
}

}  // namespace lsg
