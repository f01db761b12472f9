// Reductions: squared norm (drift check, svpart/executor.py:220-222) and the
// phase-aligned max deviation of compare() (executor.py:361-372).
#include "common.cuh"

namespace svb {
namespace {

constexpr int kThreads = 256;

__global__ void k_norm2(const double2* __restrict__ x, int64_t n, double* out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double2 v = x[i];
    s = fma(v.x, v.x, fma(v.y, v.y, s));
  }
  s = block_sum(s, red);
  if (threadIdx.x == 0) atomicAdd(out, s);
}

struct WI {
  double w;
  int64_t i;
};

// larger weight wins; ties go to the smaller index (numpy argmax = first).
// NaN is the largest weight, as in numpy's argmax: a NaN amplitude makes the
// phase and the result NaN (executor.py:361-372 then fails `compare < tol`)
__device__ __forceinline__ WI better(WI a, WI b) {
  const bool an = a.w != a.w, bn = b.w != b.w;
  if (an || bn) return (an && bn) ? (b.i < a.i ? b : a) : (bn ? b : a);
  if (b.w > a.w || (b.w == a.w && b.i < a.i)) return b;
  return a;
}

// max that keeps a NaN (numpy's max propagates it; fmax would drop it)
__device__ __forceinline__ double nmax(double m, double v) { return (v > m || v != v) ? v : m; }

__device__ __forceinline__ double cabs_(double2 z) { return hypot(z.x, z.y); }

__global__ void k_argmax_w(const double2* __restrict__ a, const double2* __restrict__ b, int64_t n,
                           WI* part) {
  __shared__ WI sh[kThreads];
  WI best{-1.0, INT64_MAX};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    best = better(best, WI{__dmul_rn(cabs_(a[i]), cabs_(b[i])), i});
  }
  sh[threadIdx.x] = best;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] = better(sh[threadIdx.x], sh[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

// reduce partials, derive phi, then max |a - phi b| per block
__global__ void k_maxdev(const double2* __restrict__ a, const double2* __restrict__ b, int64_t n,
                         const WI* part, int nparts, double* dpart) {
  __shared__ WI sh[kThreads];
  __shared__ double2 phi_s;
  WI best{-1.0, INT64_MAX};
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) best = better(best, part[i]);
  sh[threadIdx.x] = best;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] = better(sh[threadIdx.x], sh[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    double2 phi = make_double2(1.0, 0.0);
    if (sh[0].w > 0.0) {
      const double2 ak = a[sh[0].i], bk = b[sh[0].i];
      // z = a_k * conj(b_k); phi = z / |z|, with numpy's (uncontracted) rounding
      const double2 z = make_double2(__dadd_rn(__dmul_rn(ak.x, bk.x), __dmul_rn(ak.y, bk.y)),
                                     __dsub_rn(__dmul_rn(ak.y, bk.x), __dmul_rn(ak.x, bk.y)));
      const double az = cabs_(z);
      phi = make_double2(z.x / az, z.y / az);
    }
    phi_s = phi;
  }
  __syncthreads();
  const double2 phi = phi_s;
  double m = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double2 bi = b[i], ai = a[i];
    const double2 pb = make_double2(__dsub_rn(__dmul_rn(phi.x, bi.x), __dmul_rn(phi.y, bi.y)),
                                    __dadd_rn(__dmul_rn(phi.x, bi.y), __dmul_rn(phi.y, bi.x)));
    m = nmax(m, cabs_(make_double2(__dsub_rn(ai.x, pb.x), __dsub_rn(ai.y, pb.y))));
  }
  __shared__ double shm[kThreads];
  shm[threadIdx.x] = m;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) shm[threadIdx.x] = nmax(shm[threadIdx.x], shm[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) dpart[blockIdx.x] = shm[0];
}

__global__ void k_max_final(const double* dpart, int nparts, double* out) {
  __shared__ double shm[kThreads];
  double m = 0.0;
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) m = nmax(m, dpart[i]);
  shm[threadIdx.x] = m;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) shm[threadIdx.x] = nmax(shm[threadIdx.x], shm[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = shm[0];
}

// ---- distributed compare (one shard per process) ---------------------------
// Shard element i has storage index base + i; its basis index (numpy argmax
// tie-break) is the bit permutation perm[storage bit] -> basis bit, applied
// with 8-bit chunk tables.
struct Perm {
  int nchunks;
  uint64_t lut[6 * 256];
};

struct WI2 {
  double w;
  int64_t bi;  // basis index (tie-break)
  int64_t li;  // shard index
};

__device__ __forceinline__ WI2 better2(WI2 a, WI2 b) {
  const bool an = a.w != a.w, bn = b.w != b.w;
  if (an || bn) return (an && bn) ? (b.bi < a.bi ? b : a) : (bn ? b : a);
  if (b.w > a.w || (b.w == a.w && b.bi < a.bi)) return b;
  return a;
}

__global__ void k_argmax_basis(const double2* __restrict__ a, const double2* __restrict__ b, int64_t n,
                               uint64_t base, const __grid_constant__ Perm pm, WI2* part) {
  __shared__ uint64_t lut[6 * 256];
  for (int i = threadIdx.x; i < pm.nchunks * 256; i += blockDim.x) lut[i] = pm.lut[i];
  __syncthreads();
  WI2 best{-1.0, INT64_MAX, 0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t f = base + (uint64_t)i;
    uint64_t bi = 0;
    for (int c = 0; c < pm.nchunks; ++c) bi |= lut[c * 256 + ((f >> (8 * c)) & 255)];
    best = better2(best, WI2{__dmul_rn(cabs_(a[i]), cabs_(b[i])), (int64_t)bi, i});
  }
  __shared__ WI2 sh[kThreads];
  sh[threadIdx.x] = best;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] = better2(sh[threadIdx.x], sh[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

// out[0] = w, out[1] = basis index (as double bits), out[2..3] = a_k conj(b_k)
__global__ void k_argmax_final(const double2* __restrict__ a, const double2* __restrict__ b,
                               const WI2* part, int nparts, double* out) {
  __shared__ WI2 sh[kThreads];
  WI2 best{-1.0, INT64_MAX, 0};
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) best = better2(best, part[i]);
  sh[threadIdx.x] = best;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] = better2(sh[threadIdx.x], sh[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const WI2 w = sh[0];
    const double2 ak = a[w.li], bk = b[w.li];
    out[0] = w.w;
    reinterpret_cast<int64_t*>(out)[1] = w.bi;
    out[2] = __dadd_rn(__dmul_rn(ak.x, bk.x), __dmul_rn(ak.y, bk.y));
    out[3] = __dsub_rn(__dmul_rn(ak.y, bk.x), __dmul_rn(ak.x, bk.y));
  }
}

__global__ void k_maxdev_phi(const double2* __restrict__ a, const double2* __restrict__ b, int64_t n,
                             double2 phi, double* dpart) {
  double m = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double2 bi = b[i], ai = a[i];
    const double2 pb = make_double2(__dsub_rn(__dmul_rn(phi.x, bi.x), __dmul_rn(phi.y, bi.y)),
                                    __dadd_rn(__dmul_rn(phi.x, bi.y), __dmul_rn(phi.y, bi.x)));
    m = nmax(m, cabs_(make_double2(__dsub_rn(ai.x, pb.x), __dsub_rn(ai.y, pb.y))));
  }
  __shared__ double shm[kThreads];
  shm[threadIdx.x] = m;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) shm[threadIdx.x] = nmax(shm[threadIdx.x], shm[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) dpart[blockIdx.x] = shm[0];
}

int nblocks(int64_t n) {
  int64_t b = (n + kThreads - 1) / kThreads;
  if (b > num_sms() * 8) b = num_sms() * 8;
  return b > 0 ? (int)b : 1;
}

}  // namespace
}  // namespace svb

using namespace svb;

extern "C" int svb_norm2(const svb_c128* x, int64_t n, double* out, void* stream) {
  if (n < 0) return SVB_EINVAL;
  if (n == 0) return SVB_OK;
  k_norm2<<<nblocks(n), kThreads, 0, as_stream(stream)>>>(reinterpret_cast<const double2*>(x), n,
                                                          out);
  SVB_CHECK_LAUNCH("svb_norm2");
  return SVB_OK;
}

extern "C" size_t svb_compare_scratch_bytes(int64_t n) {
  const int nb = nblocks(n);
  return sizeof(WI) * nb + sizeof(double) * nb;
}

extern "C" int svb_compare(const svb_c128* a, const svb_c128* b, int64_t n, double* out,
                           void* scratch, void* stream) {
  if (n <= 0) {
    set_error("compare: empty vectors");
    return SVB_EINVAL;
  }
  const int nb = nblocks(n);
  WI* part = static_cast<WI*>(scratch);
  double* dpart = reinterpret_cast<double*>(part + nb);
  cudaStream_t st = as_stream(stream);
  auto A = reinterpret_cast<const double2*>(a);
  auto B = reinterpret_cast<const double2*>(b);
  k_argmax_w<<<nb, kThreads, 0, st>>>(A, B, n, part);
  k_maxdev<<<nb, kThreads, 0, st>>>(A, B, n, part, nb, dpart);
  k_max_final<<<1, kThreads, 0, st>>>(dpart, nb, out);
  SVB_CHECK_LAUNCH("svb_compare");
  return SVB_OK;
}

extern "C" int svb_shard_argmax(const svb_c128* a, const svb_c128* b, int64_t n, uint64_t base, int nbits,
                                const int32_t* perm, double* out, void* scratch, void* stream) {
  if (n <= 0 || nbits < 0 || nbits > 48) {
    set_error("shard_argmax: bad arguments (n=%lld, nbits=%d)", (long long)n, nbits);
    return SVB_EINVAL;
  }
  Perm pm;
  pm.nchunks = (nbits + 7) / 8;
  if (pm.nchunks == 0) pm.nchunks = 1;
  for (int c = 0; c < pm.nchunks; ++c)
    for (int v = 0; v < 256; ++v) {
      uint64_t d = 0;
      for (int j = 0; j < 8; ++j) {
        const int sb = 8 * c + j;
        if (sb < nbits && ((v >> j) & 1)) {
          if (perm[sb] < 0 || perm[sb] >= 64) {
            set_error("shard_argmax: bad perm entry %d", perm[sb]);
            return SVB_EINVAL;
          }
          d |= uint64_t(1) << perm[sb];
        }
      }
      pm.lut[c * 256 + v] = d;
    }
  const int nb = nblocks(n);
  WI2* part = static_cast<WI2*>(scratch);
  cudaStream_t st = as_stream(stream);
  auto A = reinterpret_cast<const double2*>(a);
  auto B = reinterpret_cast<const double2*>(b);
  k_argmax_basis<<<nb, kThreads, 0, st>>>(A, B, n, base, pm, part);
  k_argmax_final<<<1, kThreads, 0, st>>>(A, B, part, nb, out);
  SVB_CHECK_LAUNCH("svb_shard_argmax");
  return SVB_OK;
}

extern "C" int svb_shard_maxdev(const svb_c128* a, const svb_c128* b, int64_t n, double phi_re,
                                double phi_im, double* out, void* scratch, void* stream) {
  if (n <= 0) {
    set_error("shard_maxdev: empty shard");
    return SVB_EINVAL;
  }
  const int nb = nblocks(n);
  double* dpart = static_cast<double*>(scratch);
  cudaStream_t st = as_stream(stream);
  k_maxdev_phi<<<nb, kThreads, 0, st>>>(reinterpret_cast<const double2*>(a),
                                        reinterpret_cast<const double2*>(b), n,
                                        make_double2(phi_re, phi_im), dpart);
  k_max_final<<<1, kThreads, 0, st>>>(dpart, nb, out);
  SVB_CHECK_LAUNCH("svb_shard_maxdev");
  return SVB_OK;
}

extern "C" size_t svb_shard_scratch_bytes(int64_t n) {
  return sizeof(WI2) * nblocks(n) + 64;
}
