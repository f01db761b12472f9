// Throughput probe: FP64 tensor-core mma.sync m8n8k4 (DMMA) vs scalar DFMA on
// this GPU. Decides whether the QV sweep's 2-qubit blocks should run on DMMA.
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void k_dmma(double* out, int iters, double s) {
  double a = s + threadIdx.x * 1e-9, b = s - threadIdx.x * 1e-9;
  double c[CH][2];
#pragma unroll
  for (int j = 0; j < CH; ++j) { c[j][0] = j; c[j][1] = -j; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < CH; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
  }
  double t = 0;
#pragma unroll
  for (int j = 0; j < CH; ++j) t += c[j][0] + c[j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

template <int CH>
__global__ void k_dfma(double* out, int iters, double s) {
  double a = s + threadIdx.x * 1e-9, b = s - threadIdx.x * 1e-9;
  double c[CH];
#pragma unroll
  for (int j = 0; j < CH; ++j) c[j] = j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < CH; ++j) c[j] = fma(a, c[j], b);
  }
  double t = 0;
#pragma unroll
  for (int j = 0; j < CH; ++j) t += c[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

// Both pipes at once: half the chains DMMA, the other half DFMA.
template <int CH>
__global__ void k_mix(double* out, int iters, double s) {
  double a = s + threadIdx.x * 1e-9, b = s - threadIdx.x * 1e-9;
  double c[CH][2], f[CH * 4];
#pragma unroll
  for (int j = 0; j < CH; ++j) { c[j][0] = j; c[j][1] = -j; }
#pragma unroll
  for (int j = 0; j < CH * 4; ++j) f[j] = j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < CH; ++j) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
#pragma unroll
      for (int q = 0; q < 4; ++q) f[j * 4 + q] = fma(a, f[j * 4 + q], b);
    }
  }
  double t = 0;
#pragma unroll
  for (int j = 0; j < CH; ++j) t += c[j][0] + c[j][1];
#pragma unroll
  for (int j = 0; j < CH * 4; ++j) t += f[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, sizeof(double) * sms * 16 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4096;
  for (int warps : {4, 8, 16, 32}) {
    int nt = warps * 32; int grid = sms;
    float ms;
    // DMMA: 512 flop per warp-instruction
    k_dmma<8><<<grid, nt>>>(out, 16, 1.0); cudaDeviceSynchronize();
    cudaEventRecord(e0); k_dmma<8><<<grid, nt>>>(out, iters, 1.0); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double fl = 512.0 * 8 * iters * warps * grid;
    printf("warps/SM %2d  DMMA m8n8k4: %.1f TF/s\n", warps, fl / ms / 1e9);
    k_dfma<8><<<grid, nt>>>(out, 16, 1.0); cudaDeviceSynchronize();
    cudaEventRecord(e0); k_dfma<8><<<grid, nt>>>(out, iters, 1.0); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    fl = 2.0 * 8 * iters * (double)nt * grid;
    printf("warps/SM %2d  DFMA        : %.1f TF/s\n", warps, fl / ms / 1e9);
    k_mix<4><<<grid, nt>>>(out, 16, 1.0); cudaDeviceSynchronize();
    cudaEventRecord(e0); k_mix<4><<<grid, nt>>>(out, iters, 1.0); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    fl = (512.0 * 4 * warps + 2.0 * 16 * nt) * iters * grid;
    printf("warps/SM %2d  DMMA+DFMA   : %.1f TF/s\n", warps, fl / ms / 1e9);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
