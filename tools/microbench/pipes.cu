// Pipe-throughput microbenchmark for the E-step design (FFMA, FFMA2, MUFU.EX2, mixes).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipes pipes.cu
#include <cstdio>
#include <cuda_runtime.h>

#define ITERS 4096
#define CHAINS 8

__global__ void k_ffma(float* out, float a, float b, long long* cyc) {
  float x[CHAINS];
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-3f + c;
  long long t0 = clock64();
  #pragma unroll 4
  for (int i = 0; i < ITERS; ++i) {
    #pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = fmaf(x[c], a, b);
  }
  long long t1 = clock64();
  float s = 0; for (int c = 0; c < CHAINS; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__device__ __forceinline__ unsigned long long ffma2(unsigned long long x, unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(x), "l"(a), "l"(b));
  return d;
}

__global__ void k_ffma2(float* out, float a, float b, long long* cyc) {
  unsigned long long x[CHAINS];
  float2 af = make_float2(a, a), bf = make_float2(b, b);
  unsigned long long A = *reinterpret_cast<unsigned long long*>(&af);
  unsigned long long B = *reinterpret_cast<unsigned long long*>(&bf);
  for (int c = 0; c < CHAINS; ++c) { float2 v = make_float2(threadIdx.x * 1e-3f + c, c); x[c] = *reinterpret_cast<unsigned long long*>(&v); }
  long long t0 = clock64();
  #pragma unroll 4
  for (int i = 0; i < ITERS; ++i) {
    #pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = ffma2(x[c], A, B);
  }
  long long t1 = clock64();
  float s = 0; for (int c = 0; c < CHAINS; ++c) { float2 v = *reinterpret_cast<float2*>(&x[c]); s += v.x + v.y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }

__global__ void k_ex2(float* out, float a, float b, long long* cyc) {
  float x[CHAINS];
  for (int c = 0; c < CHAINS; ++c) x[c] = -(threadIdx.x * 1e-3f + c) * 1e-3f;
  long long t0 = clock64();
  #pragma unroll 4
  for (int i = 0; i < ITERS; ++i) {
    #pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = ex2(x[c]) * a;   // 1 MUFU + 1 FMUL
  }
  long long t1 = clock64();
  float s = 0; for (int c = 0; c < CHAINS; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// 1 ex2 per K FFMAs (K template), independent chains: measures the mix.
template <int K>
__global__ void k_mix(float* out, float a, float b, long long* cyc) {
  float x[CHAINS], acc[CHAINS][K];
  for (int c = 0; c < CHAINS; ++c) { x[c] = -(threadIdx.x * 1e-3f + c) * 1e-3f; for (int k = 0; k < K; ++k) acc[c][k] = k; }
  long long t0 = clock64();
  #pragma unroll 2
  for (int i = 0; i < ITERS / 4; ++i) {
    #pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
      float p = ex2(x[c]);
      #pragma unroll
      for (int k = 0; k < K; ++k) acc[c][k] = fmaf(p, a, acc[c][k]);
      x[c] = x[c] * 0.999f;
    }
  }
  long long t1 = clock64();
  float s = 0; for (int c = 0; c < CHAINS; ++c) for (int k = 0; k < K; ++k) s += acc[c][k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

typedef void (*kfn)(float*, float, float, long long*);

static void run(const char* name, kfn f, double ops_per_inner, int blocks, int threads) {
  float* out; long long* cyc; cudaMalloc(&out, sizeof(float) * blocks * threads); cudaMalloc(&cyc, sizeof(long long) * blocks);
  f<<<blocks, threads>>>(out, 0.999f, 1e-4f, cyc);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  f<<<blocks, threads>>>(out, 0.999f, 1e-4f, cyc);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long* h = new long long[blocks]; cudaMemcpy(h, cyc, sizeof(long long) * blocks, cudaMemcpyDeviceToHost);
  double mc = 0; for (int i = 0; i < blocks; ++i) mc += h[i]; mc /= blocks;
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double total = ops_per_inner * (double)blocks * threads;
  double per_sm_clk = total / sms / mc;   // assumes all blocks co-resident (1 wave)
  printf("%-10s blocks=%d thr=%d  %.3f ms  %.3e ops/s  ~%.2f ops/clk/SM (avg block cycles %.0f => %.0f MHz)\n",
         name, blocks, threads, ms, total / (ms * 1e-3), per_sm_clk, mc, mc / (ms * 1e3));
  cudaFree(out); cudaFree(cyc); delete[] h;
  cudaError_t err = cudaGetLastError(); if (err) printf("err %s\n", cudaGetErrorString(err));
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs=%d clockRate=%d kHz\n", sms, clk);
  for (int occ = 2; occ <= 4; occ *= 2) {
    int blocks = sms * occ, thr = 256;
    run("ffma", k_ffma, (double)ITERS * CHAINS, blocks, thr);
    run("ffma2", k_ffma2, (double)ITERS * CHAINS * 2, blocks, thr);
    run("ex2", k_ex2, (double)ITERS * CHAINS, blocks, thr);
    run("mix4", k_mix<4>, (double)(ITERS / 4) * CHAINS, blocks, thr);
    run("mix8", k_mix<8>, (double)(ITERS / 4) * CHAINS, blocks, thr);
    run("mix16", k_mix<16>, (double)(ITERS / 4) * CHAINS, blocks, thr);
  }
  return 0;
}
