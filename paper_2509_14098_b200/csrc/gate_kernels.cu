// Per-gate kernels: the GPU twin of the reference's compiled core
// (svpart/kernels/_core.pyx:7-106).  They back the inner plugin API
// (svpart.kernels.apply_gate / apply_diagonal) and the dense
// oracle_simulate path; the fused sweep kernel (sweep.cu) is the hot path.
#include <stdarg.h>
#include <string.h>

#include "common.cuh"

namespace svb {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int cuda_status(cudaError_t e, const char* what) {
  set_error("%s: %s", what, cudaGetErrorString(e));
  return SVB_ECUDA;
}

int num_sms() {
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  if (cache[dev] == 0) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    cache[dev] = n;
  }
  return cache[dev];
}

namespace {

struct GateGeom {
  int p;
  int ins[16];          // ascending LSB-indexed positions for zero insertion
  uint64_t offs_slot[16];  // 1 << ibit[slot]
};

// Decode (bits, p, L) into zero-insertion order and slot strides.
int make_geom(const int64_t* bits, int p, int L, GateGeom& g) {
  g.p = p;
  uint64_t seen = 0;
  for (int i = 0; i < p; ++i) {
    if (bits[i] < 0 || bits[i] >= L) {
      set_error("bit %lld out of range for L=%d", (long long)bits[i], L);
      return SVB_EINVAL;
    }
    int ib = L - 1 - (int)bits[i];
    if (seen >> ib & 1) {
      set_error("bit %lld repeated", (long long)bits[i]);
      return SVB_EINVAL;
    }
    seen |= uint64_t(1) << ib;
    g.offs_slot[i] = uint64_t(1) << ib;
  }
  int k = 0;
  for (int b = 0; b < 64 && k < p; ++b)
    if (seen >> b & 1) g.ins[k++] = b;
  return SVB_OK;
}

int log2_exact(int64_t n, int* L) {
  if (n <= 0 || (n & (n - 1))) {
    set_error("block length %lld is not a power of two", (long long)n);
    return SVB_EINVAL;
  }
  int l = 0;
  while ((int64_t(1) << l) < n) ++l;
  *L = l;
  return SVB_OK;
}

__device__ __forceinline__ uint64_t group_base(uint64_t k, const GateGeom& g) {
  for (int i = 0; i < g.p; ++i) k = insert_zero(k, g.ins[i]);
  return k;
}

// register path, p <= 3: one thread per amplitude group
template <int P>
__global__ void __launch_bounds__(256) k_gate_small(double2* __restrict__ blocks, int L,
                                                    uint64_t total_groups, GateGeom g,
                                                    const svb_c128* __restrict__ mat) {
  constexpr int DIM = 1 << P;
  __shared__ double2 m[DIM * DIM];
  for (int i = threadIdx.x; i < DIM * DIM; i += blockDim.x) m[i] = ldg_c(mat + i);
  __syncthreads();
  uint64_t offs[DIM];
#pragma unroll
  for (int t = 0; t < DIM; ++t) {
    uint64_t o = 0;
#pragma unroll
    for (int i = 0; i < P; ++i)
      if ((t >> (P - 1 - i)) & 1) o += g.offs_slot[i];
    offs[t] = o;
  }
  const uint64_t per_row = (uint64_t(1) << L) >> P;
  for (uint64_t gid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; gid < total_groups;
       gid += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t row = gid / per_row, k = gid - row * per_row;
    double2* base = blocks + (row << L) + group_base(k, g);
    double2 x[DIM], y[DIM];
#pragma unroll
    for (int t = 0; t < DIM; ++t) x[t] = base[offs[t]];
#pragma unroll
    for (int t = 0; t < DIM; ++t) {
      double2 acc = make_double2(0.0, 0.0);
#pragma unroll
      for (int j = 0; j < DIM; ++j) acc = cfma(m[t * DIM + j], x[j], acc);
      y[t] = acc;
    }
#pragma unroll
    for (int t = 0; t < DIM; ++t) base[offs[t]] = y[t];
  }
}

// shared-memory path for wide gates: one block per group, thread t owns row t
__global__ void k_gate_wide(double2* __restrict__ blocks, int L, uint64_t total_groups,
                            GateGeom g, const svb_c128* __restrict__ mat) {
  extern __shared__ double2 xs[];
  const int dim = 1 << g.p;
  const int t = threadIdx.x;
  uint64_t off_t = 0;
  for (int i = 0; i < g.p; ++i)
    if ((t >> (g.p - 1 - i)) & 1) off_t += g.offs_slot[i];
  const uint64_t per_row = (uint64_t(1) << L) >> g.p;
  for (uint64_t gid = blockIdx.x; gid < total_groups; gid += gridDim.x) {
    uint64_t row = gid / per_row, k = gid - row * per_row;
    double2* base = blocks + (row << L) + group_base(k, g);
    __syncthreads();
    xs[t] = base[off_t];
    __syncthreads();
    double2 acc = make_double2(0.0, 0.0);
    const svb_c128* mrow = mat + (uint64_t)t * dim;
    for (int j = 0; j < dim; ++j) acc = cfma(ldg_c(mrow + j), xs[j], acc);
    base[off_t] = acc;
  }
}

// diagonal: one thread per amplitude, table in shared memory
__global__ void k_diag(double2* __restrict__ blocks, uint64_t total, GateGeom g, int L,
                       const svb_c128* __restrict__ diag) {
  extern __shared__ double2 dt[];
  const int dim = 1 << g.p;
  for (int i = threadIdx.x; i < dim; i += blockDim.x) dt[i] = ldg_c(diag + i);
  __syncthreads();
  int ib[16];
  for (int i = 0; i < g.p; ++i) ib[i] = __ffsll((long long)g.offs_slot[i]) - 1;
  const uint64_t lmask = (uint64_t(1) << L) - 1;
  for (uint64_t f = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; f < total;
       f += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t loc = f & lmask;
    int idx = 0;
    for (int i = 0; i < g.p; ++i) idx = (idx << 1) | int((loc >> ib[i]) & 1);
    blocks[f] = cmul(blocks[f], dt[idx]);
  }
}

int grid_for(uint64_t work, int threads) {
  uint64_t b = (work + threads - 1) / threads;
  uint64_t cap = (uint64_t)num_sms() * 16;
  if (b > cap) b = cap;
  return b ? (int)b : 1;
}

}  // namespace
}  // namespace svb

using namespace svb;

extern "C" int svb_abi_version(void) { return 1; }
extern "C" const char* svb_last_error(void) { return g_err; }
extern "C" void svb_abi_sizes(size_t* op, size_t* cterm, size_t* desc) {
  *op = sizeof(svb_op);
  *cterm = sizeof(svb_cterm);
  *desc = sizeof(svb_sweep_desc);
}

extern "C" int svb_apply_gate(svb_c128* blocks, int64_t ranks, int64_t n, const svb_c128* matrix,
                              int64_t dim, const int64_t* bits, int p, int max_width,
                              void* stream) {
  if (p < 0 || p > max_width || dim != (int64_t(1) << p)) {
    set_error("gate wider than %d qubits or matrix shape mismatch", max_width);
    return SVB_EINVAL;
  }
  int L;
  if (int rc = log2_exact(n, &L)) return rc;
  if (p > 10) {
    set_error("gate width %d exceeds device kernel limit 10", p);
    return SVB_ERANGE;
  }
  if (p == 0)  // a 0-qubit gate is a scalar: same as a length-1 diagonal
    return svb_apply_diagonal(blocks, ranks, n, matrix, 1, bits, 0, max_width, stream);
  if (p > L) {
    set_error("gate wider than the %d-bit block", L);
    return SVB_EINVAL;
  }
  GateGeom g;
  if (int rc = make_geom(bits, p, L, g)) return rc;
  if (ranks == 0) return SVB_OK;
  uint64_t groups = (uint64_t)ranks * ((uint64_t)n >> p);
  cudaStream_t st = as_stream(stream);
  double2* b = reinterpret_cast<double2*>(blocks);
  switch (p) {
    case 1: k_gate_small<1><<<grid_for(groups, 256), 256, 0, st>>>(b, L, groups, g, matrix); break;
    case 2: k_gate_small<2><<<grid_for(groups, 256), 256, 0, st>>>(b, L, groups, g, matrix); break;
    case 3: k_gate_small<3><<<grid_for(groups, 256), 256, 0, st>>>(b, L, groups, g, matrix); break;
    default: {
      int blocks_n = (int)(groups < (uint64_t)num_sms() * 32 ? groups : (uint64_t)num_sms() * 32);
      size_t smem = sizeof(double2) << p;
      k_gate_wide<<<blocks_n, 1 << p, smem, st>>>(b, L, groups, g, matrix);
    }
  }
  SVB_CHECK_LAUNCH("svb_apply_gate");
  return SVB_OK;
}

extern "C" int svb_apply_diagonal(svb_c128* blocks, int64_t ranks, int64_t n, const svb_c128* diag,
                                  int64_t dim, const int64_t* bits, int p, int max_width,
                                  void* stream) {
  if (p < 0 || p > max_width || dim != (int64_t(1) << p)) {
    set_error("gate wider than %d qubits or diagonal shape mismatch", max_width);
    return SVB_EINVAL;
  }
  int L;
  if (int rc = log2_exact(n, &L)) return rc;
  if (p > 12) {
    set_error("diagonal width %d exceeds device kernel limit 12", p);
    return SVB_ERANGE;
  }
  GateGeom g;
  if (int rc = make_geom(bits, p, L, g)) return rc;
  uint64_t total = (uint64_t)ranks * (uint64_t)n;
  if (!total) return SVB_OK;
  k_diag<<<grid_for(total, 256), 256, sizeof(double2) << p, as_stream(stream)>>>(
      reinterpret_cast<double2*>(blocks), total, g, L, diag);
  SVB_CHECK_LAUNCH("svb_apply_diagonal");
  return SVB_OK;
}
