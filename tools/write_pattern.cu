// HBM write bandwidth by store pattern and warps per SM (one B200): the
// broadcast sweep of QFT-30 writes 256-byte runs (lanes on address bits 0-3
// and one high bit) from 8 warps per SM; is that pattern or occupancy bound?
#include <cstdio>
#include <cuda_runtime.h>

typedef unsigned long long u64;

template <int M>
__device__ __forceinline__ void st_m(double2* p, double2 v) {
  if (M == 0) asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
  if (M == 1) asm volatile("st.global.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
  if (M == 2) asm volatile("st.global.L1::no_allocate.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
}
#define st_cs st_m<MODE>

// contiguous: each warp instruction writes 512 contiguous bytes
template <int MODE>
__global__ void k_contig(double2* s, u64 n) {
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (; i < n; i += stride) st_cs(s + i, make_double2(1.0, 0.0));
}

// tile pattern: tile id = bits 4..19, lanes = bits 0-3 and bit 20, other
// thread bits 21-23, 16 registers on bits 24-27, 4 broadcast copies on 28-29
template <int MODE>
__global__ void k_tile(double2* s, int ntiles, int bcast) {
  const int t = threadIdx.x;
  const u64 dt = (u64)(t & 15) | ((u64)((t >> 4) & 15) << 20);
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const u64 base = (u64)tile << 4;
    double2 v = make_double2(tile, t);
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const u64 a = base | dt | ((u64)r << 24);
      if (bcast) {
#pragma unroll
        for (int f = 0; f < 4; ++f) st_cs(s + (a | ((u64)f << 28)), v);
      } else {
        st_cs(s + a, v);
      }
    }
  }
}

template <int MODE>
void run(const char* tag) {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const u64 n = 1ull << 30;
  double2* s;
  cudaMalloc(&s, n * sizeof(double2));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  for (int warps : {8, 16, 32, 64}) {
    int nt = 32 * warps > 1024 ? 1024 : 32 * warps;
    int grid = sms * (32 * warps / nt);
    k_contig<MODE><<<grid, nt>>>(s, n);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) k_contig<MODE><<<grid, nt>>>(s, n);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%s contiguous  warps/SM %2d: %.0f GB/s\n", tag, warps, 5.0 * 16 * n / (ms / 1e3) / 1e9);
  }
  for (int ctas : {1, 2, 4}) {  // 256 threads per CTA = 8 warps
    int grid = sms * ctas;
    k_tile<MODE><<<grid, 256>>>(s, 1 << 16, 1);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) k_tile<MODE><<<grid, 256>>>(s, 1 << 16, 1);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%s tile x4 bcast  warps/SM %2d: %.0f GB/s\n", tag, 8 * ctas, 5.0 * 16 * n / (ms / 1e3) / 1e9);
    k_tile<MODE><<<grid, 256>>>(s, 1 << 16, 0);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) k_tile<MODE><<<grid, 256>>>(s, 1 << 16, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%s tile no bcast  warps/SM %2d: %.0f GB/s\n", tag, 8 * ctas, 5.0 * 16 * (n >> 2) / (ms / 1e3) / 1e9);
  }
  cudaFree(s);
}

int main() {
  run<0>("st.cs");
  run<1>("st.wb");
  run<2>("st.noalloc");
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
