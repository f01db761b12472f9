// Shared helpers for libsvb200 (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "svb200.h"

namespace svb {

// ---- error reporting (thread-local message, C-ABI status codes) ----------
void set_error(const char* fmt, ...);
int cuda_status(cudaError_t e, const char* what);

#define SVB_CHECK_LAUNCH(what)                                   \
  do {                                                           \
    cudaError_t _e = cudaGetLastError();                         \
    if (_e != cudaSuccess) return ::svb::cuda_status(_e, what);  \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// SM count of the current device (cached per device): grids are sized in
// multiples of it (persistent kernels: one CTA per SM)
int num_sms();

// ---- complex128 arithmetic on double2 ------------------------------------
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) {
  return make_double2(a.x + b.x, a.y + b.y);
}
__device__ __forceinline__ double2 csub(double2 a, double2 b) {
  return make_double2(a.x - b.x, a.y - b.y);
}
// acc + a*b
__device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 acc) {
  return make_double2(fma(a.x, b.x, fma(-a.y, b.y, acc.x)),
                      fma(a.x, b.y, fma(a.y, b.x, acc.y)));
}

__device__ __forceinline__ double2 ld_c(const svb_c128* p) {
  return *reinterpret_cast<const double2*>(p);
}
__device__ __forceinline__ double2 ldg_c(const svb_c128* p) {
  return __ldg(reinterpret_cast<const double2*>(p));
}

// streaming 128-bit global load / store (state is touched once per sweep)
__device__ __forceinline__ double2 ld_stream(const double2* p) {
  double2 r;
  asm volatile("ld.global.cs.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}
__device__ __forceinline__ void st_stream(double2* p, double2 v) {
  asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
}

// insert a zero bit at position `pos` (LSB-indexed) of x
__host__ __device__ __forceinline__ uint64_t insert_zero(uint64_t x, int pos) {
  uint64_t low = x & ((uint64_t(1) << pos) - 1);
  return ((x >> pos) << (pos + 1)) | low;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// block-wide sum; result valid on thread 0. `red` must hold blockDim/32 doubles
__device__ __forceinline__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double s = 0.0;
  if (wid == 0) {
    const int nw = (blockDim.x + 31) >> 5;
    s = lane < nw ? red[lane] : 0.0;
    s = warp_sum(s);
  }
  return s;
}

}  // namespace svb
