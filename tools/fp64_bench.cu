// FP64 throughput on B200: DFMA (FP64 pipe) vs DMMA m8n8k4 (FP64 tensor
// path) vs both interleaved in the same warps.  Answers whether the sweep's
// dense 4x4 complex ops could gain from DMMA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_bench tools/fp64_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

__global__ void k_dfma(double* out, double s) {
  double a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], s, 1e-12);
  }
  double t = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) t += a[i];
  if (t == 1.2345) out[threadIdx.x] = t;
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__global__ void k_dmma(double* out, double s) {
  double c[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i] = 0;
  const double a = threadIdx.x * 1e-9 + s, b = s * 0.5;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) dmma(c[2 * i], c[2 * i + 1], a, b);
  }
  double t = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) t += c[i];
  if (t == 1.2345) out[threadIdx.x] = t;
}

__global__ void k_mixed(double* out, double s) {
  double c[8], x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    c[i] = 0;
    x[i] = threadIdx.x * 1e-9 + i;
  }
  const double a = threadIdx.x * 1e-9 + s, b = s * 0.5;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) dmma(c[2 * i], c[2 * i + 1], a, b);
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], s, 1e-12);
  }
  double t = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) t += c[i] + x[i];
  if (t == 1.2345) out[threadIdx.x] = t;
}

template <typename F>
float run(F f, int blocks, int threads) {
  double* out;
  cudaMalloc(&out, 1 << 20);
  f<<<blocks, threads>>>(out, 0.999);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  f<<<blocks, threads>>>(out, 0.999);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaFree(out);
  return ms;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int warps : {4, 8, 16}) {
    const int blocks = sms * 2, threads = 32 * warps / 2 * 1;
    const double nthreads = (double)blocks * threads;
    float t1 = run(k_dfma, blocks, threads);
    const double dfma_flops = nthreads * ITERS * 8 * 2;
    float t2 = run(k_dmma, blocks, threads);
    const double dmma_flops = nthreads / 32 * ITERS * 4 * 8 * 8 * 4 * 2;  // warps x mma x m*n*k x 2
    float t3 = run(k_mixed, blocks, threads);
    printf("warps/SM %2d: DFMA %.1f TF/s (%.2f ms) | DMMA %.1f TF/s (%.2f ms) | mixed %.1f TF/s (%.2f ms, "
           "DFMA-only time %.2f + DMMA-only %.2f)\n",
           warps, dfma_flops / t1 / 1e9, t1, dmma_flops / t2 / 1e9, t2, (dfma_flops + dmma_flops) / t3 / 1e9,
           t3, t1, t2);
  }
  return 0;
}
