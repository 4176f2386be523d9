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
#include "common.cuh"
#include "estep_dev.cuh"
#include "kernels.h"

namespace lsg {

constexpr int kBPPT = 2;                     // source points per consumer thread (one f32x2 lane)
constexpr int kBNCW = 4;                     // consumer warps
constexpr int kBMinB = 4;                    // CTAs per SM
constexpr int kBBlk = kBPPT * kBNCW * 32;    // 256 source points per block

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

template <bool kLiteral>
__global__ void __launch_bounds__((kBNCW + 1) * 32, kBMinB)
    estep_batch_kernel(const BatchProblem* __restrict__ bp, int B, const IterState* __restrict__ st, Sched sc,
                       float* __restrict__ part) {
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
                if (!st[cur.b].active) continue;
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
        if (!st[cur.b].active) continue;
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

void estep_batch_launch(const BatchProblem* bp, int B, const Sched& sc, const IterState* st, float* part, float* rec,
                        int64_t Ntot, int consistent, cudaStream_t stream) {
    if (consistent)
        estep_batch_kernel<false><<<(unsigned)sc.G, (kBNCW + 1) * 32, 0, stream>>>(bp, B, st, sc, part);
    else
        estep_batch_kernel<true><<<(unsigned)sc.G, (kBNCW + 1) * 32, 0, stream>>>(bp, B, st, sc, part);
    const int mt = 256;
    estep_batch_merge_kernel<<<(unsigned)((Ntot + mt - 1) / mt), mt, 0, stream>>>(bp, B, st, sc, part, rec, Ntot);
}

}  // namespace lsg
