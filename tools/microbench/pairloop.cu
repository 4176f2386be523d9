// Microbenchmark: the CUDA-core part of the tensor-core E step in isolation (residual with hi/lo,
// τ, e, ex2, Σpτ, TF32 split of p) over broadcast shared-memory targets, no TMEM / MMA / barriers.
// Reports pairs per clock per SM for several warp counts and points per thread: the ceiling the
// E-step consumer code can reach on this SM.
// MODE 3: tile-centred residual (13 lane-ops); MODE 4: expanded residual (11 lane-ops).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pairloop pairloop.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float2 bc(float v) { return make_float2(v, v); }
__device__ __forceinline__ float ex2a(float x) { float y; asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }

constexpr int kTgt = 1024;   // targets in shared memory (pair-interleaved, 32 B per target)
constexpr int kReps = 64;

template <int RB, int MODE>
__global__ void pairloop(const float4* __restrict__ gt, float* out, long long* cyc, float k2) {
    constexpr int kS = MODE == 4 ? 5 : 4;   // float4 per target pair (mode 4: + |y'|², -ñ·y')
    __shared__ float4 core[kTgt / 2 * 5];
    for (int i = threadIdx.x; i < kTgt / 2 * kS; i += blockDim.x) core[i] = gt[i];
    __syncthreads();
    float h[RB][3], l[RB][3];
    for (int rb = 0; rb < RB; ++rb)
        for (int a = 0; a < 3; ++a) { h[rb][a] = 0.01f * (threadIdx.x % 7 + a + rb); l[rb][a] = 1e-9f * a; }
    float2 Lt[RB];
    for (int rb = 0; rb < RB; ++rb) Lt[rb] = make_float2(0.f, 0.f);
    unsigned sink = 0;
    const float2 nk2 = bc(-k2);
    long long t0 = clock64();
    for (int rep = 0; rep < kReps; ++rep) {
#pragma unroll 4
        for (int pr = 0; pr < kTgt / 2; ++pr) {
            const float4 v0 = core[kS * pr], v1 = core[kS * pr + 1], v2 = core[kS * pr + 2], v3 = core[kS * pr + 3];
#pragma unroll
            for (int rb = 0; rb < RB; ++rb) {
                if (MODE == 4) {   // expanded residual: τ = |x'|² + |y'|² - 2x'·y' + (ñ·x' - ñ·y')², 11 lane-ops
                    const float4 v4 = core[kS * pr + 4];
                    float2 s2 = __fadd2_rn(bc(l[rb][0]), make_float2(v4.x, v4.y));
                    s2 = __ffma2_rn(bc(-2.f * h[rb][0]), make_float2(v0.x, v0.y), s2);
                    s2 = __ffma2_rn(bc(-2.f * h[rb][1]), make_float2(v0.z, v0.w), s2);
                    s2 = __ffma2_rn(bc(-2.f * h[rb][2]), make_float2(v1.x, v1.y), s2);
                    float2 qv = __ffma2_rn(bc(h[rb][0]), make_float2(v2.x, v2.y), make_float2(v4.z, v4.w));
                    qv = __ffma2_rn(bc(h[rb][1]), make_float2(v2.z, v2.w), qv);
                    qv = __ffma2_rn(bc(h[rb][2]), make_float2(v3.x, v3.y), qv);
                    const float2 tau = __ffma2_rn(qv, qv, s2);
                    const float2 e = __ffma2_rn(nk2, tau, make_float2(v1.z, v1.w));
                    const float2 p = make_float2(ex2a(e.x), ex2a(e.y));
                    Lt[rb] = __ffma2_rn(p, tau, Lt[rb]);
                    const unsigned hx = __float_as_uint(p.x) & 0xFFFFE000u, hy = __float_as_uint(p.y) & 0xFFFFE000u;
                    const float2 lo = __fadd2_rn(p, make_float2(-__uint_as_float(hx), -__uint_as_float(hy)));
                    sink ^= hx ^ hy ^ __float_as_uint(lo.x) ^ __float_as_uint(lo.y);
                    continue;
                }
                const float2 rx = MODE == 3 ? __fadd2_rn(bc(h[rb][0]), make_float2(-v0.x, -v0.y))
                                            : __fadd2_rn(__fadd2_rn(bc(h[rb][0]), make_float2(-v0.x, -v0.y)), bc(l[rb][0]));
                const float2 ry = MODE == 3 ? __fadd2_rn(bc(h[rb][1]), make_float2(-v0.z, -v0.w))
                                            : __fadd2_rn(__fadd2_rn(bc(h[rb][1]), make_float2(-v0.z, -v0.w)), bc(l[rb][1]));
                const float2 rz = MODE == 3 ? __fadd2_rn(bc(h[rb][2]), make_float2(-v1.x, -v1.y))
                                            : __fadd2_rn(__fadd2_rn(bc(h[rb][2]), make_float2(-v1.x, -v1.y)), bc(l[rb][2]));
                const float2 qv = __ffma2_rn(make_float2(v3.x, v3.y), rz,
                                             __ffma2_rn(make_float2(v2.z, v2.w), ry, __fmul2_rn(make_float2(v2.x, v2.y), rx)));
                const float2 tau = __ffma2_rn(qv, qv, __ffma2_rn(rz, rz, __ffma2_rn(ry, ry, __fmul2_rn(rx, rx))));
                const float2 e = __ffma2_rn(nk2, tau, make_float2(v1.z, v1.w));
                if (MODE == 2) { Lt[rb] = __fadd2_rn(Lt[rb], e); continue; }          // no MUFU
                const float2 p = make_float2(ex2a(e.x), ex2a(e.y));
                Lt[rb] = __ffma2_rn(p, tau, Lt[rb]);
                if (MODE == 1) { sink ^= __float_as_uint(p.x) ^ __float_as_uint(p.y); continue; }   // no split
                const unsigned hx = __float_as_uint(p.x) & 0xFFFFE000u, hy = __float_as_uint(p.y) & 0xFFFFE000u;
                const float2 lo = __fadd2_rn(p, make_float2(-__uint_as_float(hx), -__uint_as_float(hy)));
                sink ^= hx ^ hy ^ __float_as_uint(lo.x) ^ __float_as_uint(lo.y);
            }
        }
    }
    long long t1 = clock64();
    float s = 0.f;
    for (int rb = 0; rb < RB; ++rb) s += Lt[rb].x + Lt[rb].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s + (float)(sink & 1);
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int RB, int MODE>
void run(int warps, const float4* gt, float* out, long long* cyc, int nsm) {
    const int thr = warps * 32;
    pairloop<RB, MODE><<<nsm, thr>>>(gt, out, cyc, 721.f);
    cudaDeviceSynchronize();
    pairloop<RB, MODE><<<nsm, thr>>>(gt, out, cyc, 721.f);
    cudaDeviceSynchronize();
    long long c[1024];
    cudaMemcpy(c, cyc, nsm * sizeof(long long), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < nsm; ++i) avg += c[i];
    avg /= nsm;
    const double pairs = (double)thr * RB * kTgt * kReps;   // per SM
    printf("mode=%d RB=%d warps=%2d  %.3f pairs/clk/SM  (%.3e pairs/s at 1965 MHz x %d SMs)\n", MODE, RB, warps,
           pairs / avg, pairs / avg * 1.965e9 * nsm, nsm);
}


// Variant: f32x2 over TWO SOURCE POINTS per instruction with the target's fields broadcast (the
// CUDA-core kernel's packing), RBP point pairs per thread; same per-pair math as mode 0.
template <int RBP>
__global__ void pairloop_pts(const float4* __restrict__ gt, float* out, long long* cyc, float k2) {
    __shared__ float4 core[kTgt / 2 * 4];
    for (int i = threadIdx.x; i < kTgt / 2 * 4; i += blockDim.x) core[i] = gt[i];
    __syncthreads();
    float2 h[RBP][3], l[RBP][3];
    for (int rb = 0; rb < RBP; ++rb)
        for (int a = 0; a < 3; ++a) {
            h[rb][a] = make_float2(0.01f * (threadIdx.x % 7 + a + rb), 0.011f * (threadIdx.x % 5 + a));
            l[rb][a] = make_float2(1e-9f * a, 2e-9f * a);
        }
    float2 Lt[RBP];
    for (int rb = 0; rb < RBP; ++rb) Lt[rb] = make_float2(0.f, 0.f);
    unsigned sink = 0;
    const float2 nk2 = bc(-k2);
    long long t0 = clock64();
    for (int rep = 0; rep < kReps; ++rep) {
#pragma unroll 2
        for (int pr = 0; pr < kTgt / 2; ++pr) {
            const float4 v0 = core[4 * pr], v1 = core[4 * pr + 1], v2 = core[4 * pr + 2], v3 = core[4 * pr + 3];
#pragma unroll
            for (int ts = 0; ts < 2; ++ts) {   // the two targets of the pair block
                const float y0 = ts ? v0.y : v0.x, y1 = ts ? v0.w : v0.z, y2 = ts ? v1.y : v1.x, om = ts ? v1.w : v1.z;
                const float n0 = ts ? v2.y : v2.x, n1 = ts ? v2.w : v2.z, n2 = ts ? v3.y : v3.x;
#pragma unroll
                for (int rb = 0; rb < RBP; ++rb) {
                    const float2 rx = __fadd2_rn(__fadd2_rn(h[rb][0], bc(-y0)), l[rb][0]);
                    const float2 ry = __fadd2_rn(__fadd2_rn(h[rb][1], bc(-y1)), l[rb][1]);
                    const float2 rz = __fadd2_rn(__fadd2_rn(h[rb][2], bc(-y2)), l[rb][2]);
                    const float2 qv = __ffma2_rn(bc(n2), rz, __ffma2_rn(bc(n1), ry, __fmul2_rn(bc(n0), rx)));
                    const float2 tau = __ffma2_rn(qv, qv, __ffma2_rn(rz, rz, __ffma2_rn(ry, ry, __fmul2_rn(rx, rx))));
                    const float2 e = __ffma2_rn(nk2, tau, bc(om));
                    const float2 p = make_float2(ex2a(e.x), ex2a(e.y));
                    Lt[rb] = __ffma2_rn(p, tau, Lt[rb]);
                    const unsigned hx = __float_as_uint(p.x) & 0xFFFFE000u, hy = __float_as_uint(p.y) & 0xFFFFE000u;
                    const float2 lo = __fadd2_rn(p, make_float2(-__uint_as_float(hx), -__uint_as_float(hy)));
                    sink ^= hx ^ hy ^ __float_as_uint(lo.x) ^ __float_as_uint(lo.y);
                }
            }
        }
    }
    long long t1 = clock64();
    float s = 0.f;
    for (int rb = 0; rb < RBP; ++rb) s += Lt[rb].x + Lt[rb].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s + (float)(sink & 1);
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int RBP>
void run_pts(int warps, const float4* gt, float* out, long long* cyc, int nsm) {
    const int thr = warps * 32;
    for (int r = 0; r < 2; ++r) { pairloop_pts<RBP><<<nsm, thr>>>(gt, out, cyc, 721.f); cudaDeviceSynchronize(); }
    long long c[1024];
    cudaMemcpy(c, cyc, nsm * sizeof(long long), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < nsm; ++i) avg += c[i];
    avg /= nsm;
    const double pairs = (double)thr * 2 * RBP * kTgt * kReps;
    printf("points-packed RBP=%d warps=%2d  %.3f pairs/clk/SM\n", RBP, warps, pairs / avg);
}

int main() {
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    float4* gt; float* out; long long* cyc;
    cudaMalloc(&gt, kTgt / 2 * 5 * sizeof(float4));
    cudaMalloc(&out, 1024 * 1024 * sizeof(float));
    cudaMalloc(&cyc, 1024 * sizeof(long long));
    float4 hbuf[kTgt / 2 * 5];
    for (int i = 0; i < kTgt / 2 * 5; ++i) hbuf[i] = make_float4(0.013f * (i % 17), 0.011f * (i % 13), -0.5f, 0.3f);
    cudaMemcpy(gt, hbuf, sizeof(hbuf), cudaMemcpyHostToDevice);
    for (int w : {8, 12, 16, 24, 32}) run<2, 0>(w, gt, out, cyc, nsm);
    for (int w : {12, 16, 24}) run<1, 0>(w, gt, out, cyc, nsm);
    for (int w : {8, 12, 16}) run<4, 0>(w, gt, out, cyc, nsm);
    for (int w : {12, 16}) run<2, 1>(w, gt, out, cyc, nsm);
    for (int w : {12, 16}) run<2, 2>(w, gt, out, cyc, nsm);
    for (int w : {12, 16}) run_pts<1>(w, gt, out, cyc, nsm);
    for (int w : {8, 12}) run_pts<2>(w, gt, out, cyc, nsm);
    // round 2: the tile-centred residual (13 FP32 lane-ops per pair + ex2 + TF32 split)
    for (int w : {8, 12, 16, 20, 24, 32}) run<2, 3>(w, gt, out, cyc, nsm);
    for (int w : {12, 16, 24, 32}) run<1, 3>(w, gt, out, cyc, nsm);
    for (int w : {8, 12, 16}) run<4, 3>(w, gt, out, cyc, nsm);
    // the expanded residual on very compact tiles (11 FP32 lane-ops per pair + ex2 + TF32 split)
    for (int w : {8, 12, 16, 24, 32}) run<2, 4>(w, gt, out, cyc, nsm);
    for (int w : {12, 16, 24}) run<1, 4>(w, gt, out, cyc, nsm);
    for (int w : {8, 12}) run<4, 4>(w, gt, out, cyc, nsm);
    return 0;
}
