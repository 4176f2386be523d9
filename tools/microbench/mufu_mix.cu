// Microbenchmark: how MUFU.EX2 interleaves with packed (FFMA2) and scalar (FFMA) FP32 work.
// Each thread runs 8 independent chains; per iteration 16 FP32 instructions (f32x2 or scalar x2 = same
// lane-ops) and K ex2.  Prints lane-ops/clk/SM and ex2/clk/SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mufu_mix mufu_mix.cu
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float ex2a(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
constexpr int ITERS = 2048;
template <int K, bool PACKED>
__global__ void mix(float* out, long long* cyc, float a) {
    float2 x[8];
    for (int c = 0; c < 8; ++c) x[c] = make_float2(threadIdx.x * 1e-3f + c, c * 0.5f);
    float m[8];
    for (int c = 0; c < 8; ++c) m[c] = -0.001f * c;
    const float2 A = make_float2(a, a), B = make_float2(1e-7f, 1e-7f);
    long long t0 = clock64();
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            if (PACKED) {
                x[c] = __ffma2_rn(x[c], A, B);
                x[c] = __ffma2_rn(x[c], A, B);
            } else {
                x[c].x = fmaf(x[c].x, a, 1e-7f); x[c].y = fmaf(x[c].y, a, 1e-7f);
                x[c].x = fmaf(x[c].x, a, 1e-7f); x[c].y = fmaf(x[c].y, a, 1e-7f);
            }
        }
#pragma unroll
        for (int k = 0; k < K; ++k) m[k % 8] = ex2a(m[k % 8] * 0.5f - 1.f);
    }
    long long t1 = clock64();
    float s = 0;
    for (int c = 0; c < 8; ++c) s += x[c].x + x[c].y + m[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int K, bool P>
void run(int warps, float* out, long long* cyc, int nsm) {
    for (int r = 0; r < 2; ++r) { mix<K, P><<<nsm, warps * 32>>>(out, cyc, 0.999f); cudaDeviceSynchronize(); }
    long long c[1024]; cudaMemcpy(c, cyc, nsm * 8, cudaMemcpyDeviceToHost);
    double avg = 0; for (int i = 0; i < nsm; ++i) avg += c[i]; avg /= nsm;
    const double thr = warps * 32.0;
    printf("%s K=%2d warps=%2d: FP32 lane-ops/clk/SM %.1f (of 128)  ex2/clk/SM %.2f (of 16)\n", P ? "ffma2" : "ffma ", K,
           warps, thr * ITERS * 32 / avg, thr * ITERS * K / avg);
}
int main() {
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    float* out; long long* cyc; cudaMalloc(&out, 1 << 22); cudaMalloc(&cyc, 8192);
    run<0, true>(16, out, cyc, nsm); run<0, false>(16, out, cyc, nsm);
    run<1, true>(16, out, cyc, nsm); run<1, false>(16, out, cyc, nsm);
    run<2, true>(16, out, cyc, nsm); run<2, false>(16, out, cyc, nsm);
    run<4, true>(16, out, cyc, nsm); run<4, false>(16, out, cyc, nsm);
    run<8, true>(16, out, cyc, nsm); run<8, false>(16, out, cyc, nsm);
    run<2, true>(32, out, cyc, nsm); run<2, false>(32, out, cyc, nsm);
    return 0;
}
