// Device helpers shared by the E-step kernels (estep.cu: single problem; batch.cu: many small
// problems in one launch).  Product path only.
#pragma once
#include <type_traits>

#include "common.cuh"

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
// Diagnostic: helper-warp waits with a fixed back-off instead of the suspend-time hint (LSG_PROD_NS: the TMA
// producer; LSG_MMA_NS: the MMA warps).  Test the phase, else sleep NS nanoseconds, repeat.
template <int NS>
__device__ __forceinline__ void mbar_wait_backoff(uint64_t* bar, uint32_t parity) {
    const uint32_t a = smem_u32(bar);
    for (;;) {
        uint32_t ok;
        asm volatile(
            "{\n"
            ".reg .pred P1;\n"
            "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
            "selp.u32 %0, 1, 0, P1;\n"
            "}\n"
            : "=r"(ok)
            : "r"(a), "r"(parity)
            : "memory");
        if (ok) break;
        __nanosleep(NS);
    }
}
#ifdef LSG_PROD_NS
#define LSG_PWAIT mbar_wait_backoff<LSG_PROD_NS>
#else
#define LSG_PWAIT mbar_wait_sleep
#endif
#ifdef LSG_MMA_NS
#define LSG_MWAIT mbar_wait_backoff<LSG_MMA_NS>
#else
#define LSG_MWAIT mbar_wait_sleep
#endif
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}


// ---- tcgen05 / TMEM helpers (tensor-core E-step kernels) ----------------------------------------
constexpr int kTcStages = 4;
constexpr int kTcCols = 512;                  // TMEM columns allocated (the whole TMEM: base column 0)
constexpr int kTcChunk = 8;                   // targets per A buffer (one K step)
// D group g is drained at the start of tile kDrainLag of group g + 1 (its MMAs long complete, and the slowest
// warp of the warpgroup is no longer on the critical path); group g + 2 reuses its D buffer only after that
// Tensor-core E-step configuration shared by estep.cu and batch.cu
#ifndef LSG_PAIRED
#define LSG_PAIRED 1   // one A-buffer hand-off per pair of K steps (tools/estep_time.py: +2.7 %)
#endif
#ifndef LSG_TC_UNROLL
#define LSG_TC_UNROLL 2   // chunk-pair loop unrolled by two (tools/estep_time.py: +1 %)
#endif
// Register split between the warp roles (setmaxnreg, per warpgroup): warpgroup 3 (producer + MMA warps) keeps
// 32 registers, each consumer thread gets 160 instead of the launch's 128 — the whole register file
// (384·160 + 128·32 = 65536).  ILP in the pair math: 128 → 152 +1.7 %, → 160 +2.4 % more (tools/estep_time.py)
#ifndef LSG_MAXNREG
#define LSG_MAXNREG 160
#define LSG_MAXNREG_LO 32
#endif
// consumer-side barrier waits (A buffer free, stage full): a plain try_wait spin — the waits are short and a
// suspended consumer wakes later than it could issue (+0.8 %, tools/estep_time.py); the producer and MMA warps keep
// the suspend-time hint so their polling does not take issue slots from the consumers
#ifndef LSG_CONSUMER_SLEEP
#define LSG_CWAIT mbar_wait
#else
#define LSG_CWAIT mbar_wait_sleep
#endif
#define LSG_PRAGMA(x) _Pragma(#x)
#define LSG_UNROLL(n) LSG_PRAGMA(unroll n)
#ifndef LSG_DRAIN_LAG
#define LSG_DRAIN_LAG 1
#endif
constexpr int kDrainLag = LSG_DRAIN_LAG;
// instruction descriptor: D F32, A/B TF32, K-major A and B, M = 128, N = 16
constexpr uint32_t kTcIdesc16 = (1u << 4) | (2u << 7) | (2u << 10) | ((16u >> 3) << 17) | ((128u >> 4) << 24);

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
        "%14, %15, %16};" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
        : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr)
        : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void mma_tf32_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                            uint32_t enable_d) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n"
        "}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(enable_d)
        : "memory");
}
__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile(
        "{\n"
        ".reg .pred P;\n"
        "elect.sync _|P, 0xffffffff;\n"
        "selp.u32 %0, 1, 0, P;\n"
        "}\n"
        : "=r"(pred));
    return pred != 0;
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
// UMMA shared-memory descriptor: K-major, no swizzle, LBO = 128 B, SBO = 256 B, version 1 (sm_100).
__device__ __forceinline__ uint64_t bdesc(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)(128u >> 4) << 16) | ((uint64_t)(256u >> 4) << 32) |
           ((uint64_t)1 << 46);
}


// ---- tensor-core consumers: per-tile residual setup and the pair math of one K step ------------------
// Tile-centred residual.  The core holds y' = y - c exactly (c: the tile centre, per axis).
//  * cheap tiles (E_tile ≤ gate): x' = fl((hi - c) + lo) once per (point, tile); r = x' - y' costs 3 FP32
//    lane-ops per pair.  Its rounding error is ≈ ε(|x'| + |r|) ≤ ε(R_tile + 2|r|), i.e. the hi/lo error plus
//    a term in R_tile that the gate bounds relative to σ.
//  * other tiles: (xh, xl) = TwoSum(hi, -c) + lo, r = (xh - y') + xl — the hi/lo residual of round 1, exact
//    to ≈ ε|r| whatever the tile's size (outlier-laden tiles, large targets far from their centre).
struct TileMeta {
    float c[3];
    float E;
    float R;
};
__device__ __forceinline__ TileMeta tile_meta(const float4* core) {
    const float4 a = core[3], b = core[7], e = core[11];   // spare fields of targets 0..4 (see common.cuh)
    return {{a.z, a.w, b.z}, b.w, e.z};
}
template <bool kCheap, int RB>
__device__ __forceinline__ void tile_points(const float (&h)[RB][3], const float (&l)[RB][3], const TileMeta& tm,
                                            float2 (&xa)[RB][3], float2 (&xb)[RB][3]) {
#pragma unroll
    for (int rb = 0; rb < RB; ++rb)
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            if (kCheap) {
                xa[rb][a] = bc(__fadd_rn(__fsub_rn(h[rb][a], tm.c[a]), l[rb][a]));
            } else {
                const float hi = h[rb][a], nc = -tm.c[a];
                const float s = __fadd_rn(hi, nc);
                const float bb = __fsub_rn(s, hi);
                const float err = __fadd_rn(__fsub_rn(hi, __fsub_rn(s, bb)), __fsub_rn(nc, bb));
                xa[rb][a] = bc(s);
                xb[rb][a] = bc(__fadd_rn(l[rb][a], err));
            }
        }
}
// One K step (8 targets = 4 target pairs): residual, τ, ex2, Σpτ, TF32 split of p → the A row of each row
// block (hi of the 8 targets, then lo).  Cheap tiles: 13 FP32 lane-ops per pair; other tiles: 16.
template <bool kLiteral, bool kCheap, int RB>
__device__ __forceinline__ void tc_chunk_pairs(const float4* __restrict__ core, int c, const float2 (&xa)[RB][3],
                                               const float2 (&xb)[RB][3], float2 nk2, float2 (&Lt)[RB],
                                               uint32_t (&av)[RB][16]) {
#pragma unroll
    for (int pp = 0; pp < 4; ++pp) {
        const int pr = c * 4 + pp;
        const float4 v0 = core[4 * pr], v1 = core[4 * pr + 1], v2 = core[4 * pr + 2], v3 = core[4 * pr + 3];
#pragma unroll
        for (int rb = 0; rb < RB; ++rb) {
            float2 rx = __fadd2_rn(xa[rb][0], make_float2(-v0.x, -v0.y));
            float2 ry = __fadd2_rn(xa[rb][1], make_float2(-v0.z, -v0.w));
            float2 rz = __fadd2_rn(xa[rb][2], make_float2(-v1.x, -v1.y));
            if (!kCheap) {
                rx = __fadd2_rn(rx, xb[rb][0]);
                ry = __fadd2_rn(ry, xb[rb][1]);
                rz = __fadd2_rn(rz, xb[rb][2]);
            }
            const float2 qv = __ffma2_rn(make_float2(v3.x, v3.y), rz,
                                         __ffma2_rn(make_float2(v2.z, v2.w), ry, __fmul2_rn(make_float2(v2.x, v2.y), rx)));
            const float2 tau = __ffma2_rn(qv, qv, __ffma2_rn(rz, rz, __ffma2_rn(ry, ry, __fmul2_rn(rx, rx))));
            const float2 e = kLiteral ? __fmul2_rn(nk2, tau) : __ffma2_rn(nk2, tau, make_float2(v1.z, v1.w));
            const float2 p = make_float2(ex2_approx(e.x), ex2_approx(e.y));
            Lt[rb] = __ffma2_rn(p, tau, Lt[rb]);
            const uint32_t hx = __float_as_uint(p.x) & 0xFFFFE000u, hy = __float_as_uint(p.y) & 0xFFFFE000u;
            const float2 lo = __fadd2_rn(p, make_float2(-__uint_as_float(hx), -__uint_as_float(hy)));
            av[rb][2 * pp] = hx;
            av[rb][2 * pp + 1] = hy;
            av[rb][8 + 2 * pp] = __float_as_uint(lo.x);
            av[rb][8 + 2 * pp + 1] = __float_as_uint(lo.y);
        }
    }
}
// the tile's residual mode: centred when E_tile ≤ gate (gate = gate_g·σ, uniform over the CTA)
__device__ __forceinline__ bool tile_cheap(const TileMeta& tm, float gate) { return tm.E <= gate; }
// ... or, per warp, when every point of the warp is at least 2 R_tile from the tile centre (DESIGN §8 "far
// points"): then |r| ≥ |x'| - R_tile ≥ |x'|/2 for every pair, so the centred residual's extra rounding
// ε|x'| is at most 2ε|r| — the hi/lo residual's relative accuracy up to a small factor, whatever σ is
#ifndef LSG_FAR_K2
#define LSG_FAR_K2 4.01f   // (2 R_tile)² with a margin: |r| ≥ |x'| - R_tile ≥ |x'|/2
#endif
template <int RB>
__device__ __forceinline__ bool warp_far(const float (&h)[RB][3], const float (&l)[RB][3], const TileMeta& tm) {
    bool far = true;
#pragma unroll
    for (int rb = 0; rb < RB; ++rb) {
        float d2 = 0.f;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const float x = __fadd_rn(__fsub_rn(h[rb][a], tm.c[a]), l[rb][a]);
            d2 = __fmaf_rn(x, x, d2);
        }
        far = far && d2 >= LSG_FAR_K2 * tm.R * tm.R;
    }
    return __all_sync(0xffffffffu, far);
}

// One point of the split-M merge: the nk partials of its source block start at `blk` (slot stride
// kPartF·kB floats, field stride kB, point index b), `phi` → φ(x_n) or NULL, record row `r`.
__device__ inline void merge_point(const float* __restrict__ blk, int64_t nk, int64_t kB, int b,
                                   const IterState* __restrict__ st, const float* __restrict__ phi,
                                   float* __restrict__ r) {
    double wn = st->w, C1n = st->C1, Lon = st->Lo;
    if (phi) {
        const double f = fmin(fmax((double)*phi, 0.0), 1.0);
        wn = 1.0 - (1.0 - st->w) * f;
        if (!(wn < 1.0)) {
            float4* r4 = reinterpret_cast<float4*>(r);
            r4[0] = r4[1] = r4[2] = make_float4(0.f, 0.f, 0.f, 0.f);
            r4[3] = make_float4(0.f, 0.f, (float)(-log(st->volume)), 1.f);
            return;
        }
        C1n = st->C1 + log((1.0 - wn) / (1.0 - st->w));
        Lon = wn > 0.0 ? (log(wn / st->volume) - C1n) * 1.4426950408889634074 - st->omega_ref : -INFINITY;
    }
    // reference max over the segments' maxima (all 0 in the fixed-max mode: no rescaling needed)
    double mustar = -INFINITY;
#pragma unroll 4
    for (int64_t k = 0; k < nk; ++k) {
        const float* base = blk + k * (int64_t)kPartF * kB;
        mustar = fmax(mustar, (double)base[14 * kB + b]);
    }
    if (wn > 0.0) mustar = fmax(mustar, fmin(Lon, 0.0));   // keep the outlier term representable
    double a[kAcc];
#pragma unroll
    for (int f = 0; f < kAcc; ++f) a[f] = 0.0;
#pragma unroll 2
    for (int64_t k = 0; k < nk; ++k) {
        const float* base = blk + k * (int64_t)kPartF * kB;
        const double muk = (double)base[14 * kB + b];
        const double sc_k = (muk == mustar) ? 1.0 : exp2(muk - mustar);
#pragma unroll
        for (int f = 0; f < kAcc; ++f) a[f] = fma(sc_k, (double)base[f * kB + b], a[f]);
    }
    const double O = (wn > 0.0) ? exp2(Lon - mustar) : 0.0;
    const double Z = a[0] + O;
    const double iz = 1.0 / Z;
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
    o3.z = (float)(C1n + 0.69314718055994530942 * (st->omega_ref + mustar + log2(Z)));
    o3.w = (float)(O * iz);
    reinterpret_cast<float4*>(r)[0] = o0;
    reinterpret_cast<float4*>(r)[1] = o1;
    reinterpret_cast<float4*>(r)[2] = o2;
    reinterpret_cast<float4*>(r)[3] = o3;
}

// Merge of the 32 points n0..n0+31 (n0 a multiple of 32, so all in one source block) by 16 warps: warp f
// produces record float f, so every partial load is a coalesced 128-B row (32 consecutive points of one
// accumulator) and each point's serial chain is 1/16 of merge_point's.  The arithmetic is merge_point's,
// operation for operation (bit-identical records).  All 512 threads call it; tile[p][f] is valid after the
// caller's next __syncthreads().
constexpr int kMergePts = 32;
__device__ inline void merge_tile32(const float* __restrict__ part, int64_t N, int64_t n0,
                                    const IterState* __restrict__ st, const Sched& sc, const float* __restrict__ phi,
                                    float (*tile)[LSGCPD_REC + 1], double* a0s) {
    const int f = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t n = n0 + lane;
    const int64_t kB = sc.B;   // a multiple of 32
    const int64_t j = n0 / kB;
    const int b = (int)(n0 - j * kB) + lane;
    const int nk = (int)(sched_owner(sc, (j + 1) * sc.T - 1) - sched_owner(sc, j * sc.T) + 1);
    const float* blk = part + j * sc.kmax * (int64_t)kPartF * kB + b;
    const bool ok = n < N;
    double wn = st->w, C1n = st->C1, Lon = st->Lo;
    if (ok && phi) {
        const double fi = fmin(fmax((double)phi[n], 0.0), 1.0);
        wn = 1.0 - (1.0 - st->w) * fi;
        if (wn < 1.0) {
            C1n = st->C1 + log((1.0 - wn) / (1.0 - st->w));
            Lon = wn > 0.0 ? (log(wn / st->volume) - C1n) * 1.4426950408889634074 - st->omega_ref : -INFINITY;
        }
    }
    double mustar = -INFINITY, a = 0.0;
    if (ok) {
        if (st->fixed) {
            // fixed-max mode: every segment's max is 0 and so is the reference (max(0, min(L_o, 0)) = 0), every
            // scale factor is 1 — the plain sum, as the general path computes it, without the pass over the maxima
            mustar = 0.0;
            if (f < kAcc)
                for (int h = 0; h < sc.halves; ++h) {
                    const float* bh = blk + h * sc.hstride;
#pragma unroll 4
                    for (int k = 0; k < nk; ++k) a = fma(1.0, (double)bh[(int64_t)k * kPartF * kB + f * kB], a);
                }
        } else {
            for (int h = 0; h < sc.halves; ++h) {   // the segments of every half of the targets (Sched::halves)
                const float* bh = blk + h * sc.hstride;
#pragma unroll 4
                for (int k = 0; k < nk; ++k) mustar = fmax(mustar, (double)bh[(int64_t)k * kPartF * kB + 14 * kB]);
            }
            if (wn > 0.0) mustar = fmax(mustar, fmin(Lon, 0.0));
            if (f < kAcc) {
                for (int h = 0; h < sc.halves; ++h) {
                    const float* bh = blk + h * sc.hstride;
#pragma unroll 4
                    for (int k = 0; k < nk; ++k) {
                        const float* base = bh + (int64_t)k * kPartF * kB;
                        const double muk = (double)base[14 * kB];
                        const double sc_k = (muk == mustar) ? 1.0 : exp2(muk - mustar);
                        a = fma(sc_k, (double)base[f * kB], a);
                    }
                }
            }
        }
    }
    if (f == 0) a0s[lane] = a;
    __syncthreads();
    float out = 0.f;
    if (ok) {
        if (!(wn < 1.0)) {   // all outlier
            out = f == 14 ? (float)(-log(st->volume)) : (f == 15 ? 1.f : 0.f);
        } else {
            const double O = (wn > 0.0) ? exp2(Lon - mustar) : 0.0;
            const double Z = a0s[lane] + O;
            const double iz = 1.0 / Z;
            if (f < 13) out = (float)(a * iz);
            else if (f == 13) out = (float)(a * iz / st->sigma2);
            else if (f == 14) out = (float)(C1n + 0.69314718055994530942 * (st->omega_ref + mustar + log2(Z)));
            else out = (float)(O * iz);
        }
    }
    tile[lane][f] = out;
}

}  // namespace lsg
