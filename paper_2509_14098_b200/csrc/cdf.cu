// numpy-identical measurement sampling on the device (svpart/executor.py:375-383).
//
// The reference evaluates
//     probs = np.abs(dense) ** 2;  probs = probs / probs.sum()
//     rng.choice(2^d, shots, p=probs)
// which numpy runs as cdf = probs.cumsum(); cdf /= cdf[-1];
// idx = cdf.searchsorted(rng.random(shots), side="right").  Every step is
// reproduced here bit for bit:
//   * |z| is numpy's complex absolute (SIMD loops: L * sqrt(fma(r, r, 1)),
//     L = max(|re|,|im|), r = min/L), squared with one multiply;
//   * probs.sum() is numpy's pairwise summation (blocks of 128 summed with
//     8 accumulators, halves combined recursively);
//   * cumsum is a SEQUENTIAL sum, c_i = fl(c_{i-1} + q_i).  It is evaluated
//     exactly without a sequential pass over 2^d elements: while c stays in
//     one binade [2^e, 2^(e+1)), fl(c + q) = c + k*ulp_e with the integer k
//     = q/ulp_e rounded to nearest (ties to even on the running sum's
//     parity), so a chunk of B elements acts on c as m -> m + a[m & 1]
//     (m = c/ulp_e).  Chunks are classified in parallel from an approximate
//     prefix; one warp then walks the chunks in order from the exact start,
//     applying a chunk's integers when it provably stays in its binade
//     (checked with the exact value) and adding its elements one by one
//     otherwise (the ~60 binade crossings).  The walk yields the exact c at
//     every chunk end;
//   * each shot binary-searches the chunk ends, then re-adds the elements
//     of its chunk from the exact chunk start (hardware fl adds are numpy's
//     adds) and compares fl(c_i / c_last) with its uniform.
#include "common.cuh"

namespace svb {
namespace {

constexpr int kChunkLog2 = 13;  // elements per chunk of the CDF walk

struct DepositLut {
  int nchunks;
  uint64_t lut[6 * 256];  // index chunk -> destination bits
};

// numpy's complex absolute value (SIMD path: hypot by scaling with an FMA)
__device__ __forceinline__ double numpy_cabs(double2 z) {
  const double ax = fabs(z.x), ay = fabs(z.y);
  const double L = fmax(ax, ay), S = fmin(ax, ay);
  if (L == 0.0) return 0.0;
  if (isinf(L)) return L;
  const double r = __ddiv_rn(S, L);
  return __dmul_rn(L, __dsqrt_rn(__fma_rn(r, r, 1.0)));
}

__global__ void k_probs_numpy(const double2* __restrict__ a, uint64_t n, const __grid_constant__ DepositLut lut_in,
                              double* __restrict__ out) {
  __shared__ uint64_t lut[6 * 256];
  for (int i = threadIdx.x; i < lut_in.nchunks * 256; i += blockDim.x) lut[i] = lut_in.lut[i];
  __syncthreads();
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < n; t += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t j = 0;
    for (int c = 0; c < lut_in.nchunks; ++c) j |= lut[c * 256 + ((t >> (8 * c)) & 255)];
    const double m = numpy_cabs(a[t]);
    out[j] = __dmul_rn(m, m);
  }
}

__global__ void k_deposit_scatter(const double* __restrict__ src, uint64_t n, const __grid_constant__ DepositLut lut_in,
                                  uint64_t or_val, double* __restrict__ dst) {
  __shared__ uint64_t lut[6 * 256];
  for (int i = threadIdx.x; i < lut_in.nchunks * 256; i += blockDim.x) lut[i] = lut_in.lut[i];
  __syncthreads();
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < n; t += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t j = or_val;
    for (int c = 0; c < lut_in.nchunks; ++c) j |= lut[c * 256 + ((t >> (8 * c)) & 255)];
    dst[j] = src[t];
  }
}

// numpy pairwise sum of one 128-element block (8 accumulators)
__device__ double pw_block128(const double* x) {
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = x[j];
  for (int i = 8; i < 128; i += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], x[i + j]);
  }
  return __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                   __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
}

// numpy pairwise sum of a short array (n <= 128)
__device__ double pw_small(const double* x, int64_t n) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; ++i) res = __dadd_rn(res, x[i]);
    return res;
  }
  double r[8];
  for (int j = 0; j < 8; ++j) r[j] = x[j];
  int64_t i = 8;
  for (; i < n - (n % 8); i += 8)
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], x[i + j]);
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __dadd_rn(res, x[i]);
  return res;
}

// 256 leaves (128 elements each) per block, reduced in the recursion's
// left/right order: the block result is the pairwise sum of its 2^15 elements
__global__ void k_pw_leaves(const double* __restrict__ x, int64_t nleaves, double* __restrict__ part) {
  __shared__ double sh[256];
  const int64_t leaf = blockIdx.x * 256ll + threadIdx.x;
  sh[threadIdx.x] = leaf < nleaves ? pw_block128(x + leaf * 128) : 0.0;
  __syncthreads();
  for (int w = 2; w <= 256; w <<= 1) {
    if ((threadIdx.x & (w - 1)) == 0) sh[threadIdx.x] = __dadd_rn(sh[threadIdx.x], sh[threadIdx.x + w / 2]);
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

// pairwise tree over npart (a power of two) partial sums, in place
__global__ void k_pw_tree(double* part, int64_t npart) {
  for (int64_t w = 2; w <= npart; w <<= 1) {
    for (int64_t i = threadIdx.x * w; i < npart; i += (int64_t)blockDim.x * w)
      part[i] = __dadd_rn(part[i], part[i + w / 2]);
    __syncthreads();
  }
}

__global__ void k_pw_small(const double* x, int64_t n, double* out) { *out = pw_small(x, n); }

__global__ void k_div_scalar(double* __restrict__ x, int64_t n, const double* __restrict__ d) {
  const double s = *d;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = __ddiv_rn(x[i], s);
}

// approximate chunk totals (any order)
__global__ void k_chunk_tot(const double* __restrict__ q, int64_t n, int64_t B, double* __restrict__ tot) {
  __shared__ double red[32];
  const int64_t k = blockIdx.x;
  double s = 0.0;
  for (int64_t i = k * B + threadIdx.x; i < min(n, (k + 1) * B); i += blockDim.x) s += q[i];
  s = block_sum(s, red);
  if (threadIdx.x == 0) tot[k] = s;
}

struct ChunkFn {
  long long a0, a1;  // integer increment of m for start parity 0 / 1
  int e;             // binade of c the increments assume
  int simple;        // 0: add the elements one by one in the walk
};

__device__ __forceinline__ void inc_of(double q, int e, long long& k, int& cls) {
  // f = q / ulp_e exactly (power-of-two scaling); k = floor(f); cls: 0 round
  // down, 1 round up, 2 tie
  const double f = ldexp(q, 52 - e);
  const double fl_ = trunc(f);
  const double fr = f - fl_;
  k = (long long)fl_;
  cls = fr < 0.5 ? 0 : (fr > 0.5 ? 1 : 2);
}

// one warp per chunk: classify from the approximate start and build m -> m + a[m & 1]
__global__ void k_chunk_fns(const double* __restrict__ q, int64_t n, int64_t B, const double* __restrict__ cstart,
                            const double* __restrict__ tot, int64_t nchunks, ChunkFn* __restrict__ fn) {
  const int lane = threadIdx.x & 31;
  const int64_t k = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (k >= nchunks) return;
  const double c0 = cstart[k], c1 = c0 + tot[k];
  ChunkFn f{0, 0, 0, 0};
  const bool ok = c0 >= 0x1p-1000 && c0 < 0x1p1000 && ilogb(c0) == ilogb(c1);
  if (!ok) {
    if (lane == 0) fn[k] = f;
    return;
  }
  const int e = ilogb(c0);
  const int64_t lo = k * B, hi = min(n, lo + B);
  long long sum = 0;
  int ties = 0;
  for (int64_t i = lo + lane; i < hi; i += 32) {
    long long kk;
    int cls;
    inc_of(q[i], e, kk, cls);
    sum += kk + (cls == 1);
    ties |= cls == 2;
  }
  int big = sum >= (1ll << 57);  // partials stay far from int64 overflow
  if (big) sum = 0;
  for (int o = 16; o; o >>= 1) {
    sum += __shfl_xor_sync(0xffffffffu, sum, o);
    ties |= __shfl_xor_sync(0xffffffffu, ties, o);
    big |= __shfl_xor_sync(0xffffffffu, big, o);
  }
  if (big || sum >= (1ll << 53)) {  // the chunk leaves its binade: walk it element by element
    if (lane == 0) fn[k] = f;
    return;
  }
  if (lane == 0) {
    f.e = e;
    f.simple = 1;
    f.a0 = f.a1 = sum;
    if (ties) {  // rare: the tie rounds to the even running sum, which depends on the start parity
      for (int p = 0; p < 2; ++p) {
        long long tot_inc = 0;
        int par = p;
        for (int64_t i = lo; i < hi; ++i) {
          long long kk;
          int cls;
          inc_of(q[i], e, kk, cls);
          const long long inc = kk + (cls == 1 ? 1 : (cls == 2 ? ((par + kk) & 1) : 0));
          tot_inc += inc;
          par = (int)((par + inc) & 1);
        }
        if (p == 0)
          f.a0 = tot_inc;
        else
          f.a1 = tot_inc;
      }
    }
    fn[k] = f;
  }
}

// one warp: c <- fl(c + q_i) over [lo, hi), all lanes hold the same c
__device__ double warp_seq_add(const double* __restrict__ q, int64_t lo, int64_t hi, double c) {
  const int lane = threadIdx.x & 31;
  for (int64_t b = lo; b < hi; b += 32) {
    const double v = b + lane < hi ? q[b + lane] : 0.0;
    const int cnt = (int)min((int64_t)32, hi - b);
    for (int j = 0; j < cnt; ++j) c = __dadd_rn(c, __shfl_sync(0xffffffffu, v, j));
  }
  return c;
}

// the walk: one warp, chunks in order from the exact start c_in
__global__ void k_cdf_walk(const double* __restrict__ q, int64_t n, int64_t B, const ChunkFn* __restrict__ fn,
                           int64_t nchunks, const double* __restrict__ c_in, double* __restrict__ cend,
                           long long* __restrict__ nslow) {
  const int lane = threadIdx.x & 31;
  double c = *c_in;
  long long slow = 0;
  for (int64_t k0 = 0; k0 < nchunks; k0 += 32) {
    ChunkFn mine{0, 0, 0, 0};
    if (k0 + lane < nchunks) mine = fn[k0 + lane];
    double ends = 0.0;
    const int cnt = (int)min((int64_t)32, nchunks - k0);
    for (int j = 0; j < cnt; ++j) {
      const long long a0 = __shfl_sync(0xffffffffu, mine.a0, j);
      const long long a1 = __shfl_sync(0xffffffffu, mine.a1, j);
      const int e = __shfl_sync(0xffffffffu, mine.e, j);
      const int simple = __shfl_sync(0xffffffffu, mine.simple, j);
      const int64_t k = k0 + j;
      bool done = false;
      if (simple && c >= 0x1p-1000 && ilogb(c) == e) {
        const long long m = (long long)ldexp(c, 52 - e);
        const long long me = m + ((m & 1) ? a1 : a0);
        if (me < (1ll << 53)) {
          c = ldexp((double)me, e - 52);
          done = true;
        }
      }
      if (!done) {
        c = warp_seq_add(q, k * B, min(n, (k + 1) * B), c);
        ++slow;
      }
      if (lane == j) ends = c;
    }
    if (k0 + lane < nchunks) cend[k0 + lane] = ends;
  }
  if (lane == 0) *nslow = slow;
}

// per shot: first chunk whose end cdf exceeds u, then the first element of it
__global__ void k_cdf_search(const double* __restrict__ q, int64_t n, int64_t B, const double* __restrict__ cend,
                             int64_t nchunks, int64_t chunk_base, int64_t my_lo, int64_t my_hi,
                             double c_last, const double* __restrict__ u,
                             int64_t nshots, int64_t index_base, int64_t* __restrict__ out) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nshots; s += (int64_t)gridDim.x * blockDim.x) {
    const double us = u[s];
    int64_t lo = 0, hi = nchunks - 1;  // global chunk ends (all processes)
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (__ddiv_rn(cend[mid], c_last) > us)
        hi = mid;
      else
        lo = mid + 1;
    }
    int64_t res = -1;
    if (lo >= my_lo && lo < my_hi) {  // the chunk is this process's: find the element
      const int64_t kl = lo - chunk_base;
      double c = lo > 0 ? cend[lo - 1] : 0.0;
      const int64_t b = kl * B, e = min(n, b + B);
      res = e - 1;
      for (int64_t i = b; i < e; ++i) {
        c = __dadd_rn(c, q[i]);
        if (__ddiv_rn(c, c_last) > us) {
          res = i;
          break;
        }
      }
      res += index_base;
    }
    out[s] = res;
  }
}

int lut_of(const int32_t* bits, int nbits, DepositLut& dl) {
  if (nbits < 0 || nbits > 48) {
    set_error("deposit lut: %d bits", nbits);
    return SVB_EINVAL;
  }
  dl.nchunks = nbits > 0 ? (nbits + 7) / 8 : 1;
  for (int c = 0; c < dl.nchunks; ++c)
    for (int v = 0; v < 256; ++v) {
      uint64_t j = 0;
      for (int k = 0; k < 8; ++k) {
        const int s = 8 * c + k;
        if (s < nbits && ((v >> k) & 1)) {
          if (bits[s] < 0 || bits[s] >= 64) {
            set_error("deposit lut: bad bit %d", bits[s]);
            return SVB_EINVAL;
          }
          j |= uint64_t(1) << bits[s];
        }
      }
      dl.lut[c * 256 + v] = j;
    }
  return SVB_OK;
}

unsigned grid_for(uint64_t n, int per_sm) {
  uint64_t b = (n + 255) / 256;
  const uint64_t cap = (uint64_t)num_sms() * per_sm;
  if (b > cap) b = cap;
  return b ? (unsigned)b : 1u;
}

}  // namespace
}  // namespace svb

using namespace svb;

extern "C" int64_t svb_cdf_chunk_elems(void) { return int64_t(1) << kChunkLog2; }

extern "C" int svb_probs_numpy(const svb_c128* shard, int D, const int32_t* perm, double* out, void* stream) {
  DepositLut dl;
  int rc = lut_of(perm, D, dl);
  if (rc != SVB_OK) return rc;
  const uint64_t n = uint64_t(1) << D;
  k_probs_numpy<<<grid_for(n, 16), 256, 0, as_stream(stream)>>>(reinterpret_cast<const double2*>(shard), n, dl, out);
  SVB_CHECK_LAUNCH("svb_probs_numpy");
  return SVB_OK;
}

extern "C" int svb_deposit_scatter(const double* src, int64_t n, int nbits, const int32_t* dst_bits, uint64_t or_val,
                                   double* dst, void* stream) {
  if (n <= 0) return SVB_OK;
  DepositLut dl;
  int rc = lut_of(dst_bits, nbits, dl);
  if (rc != SVB_OK) return rc;
  k_deposit_scatter<<<grid_for((uint64_t)n, 16), 256, 0, as_stream(stream)>>>(src, (uint64_t)n, dl, or_val, dst);
  SVB_CHECK_LAUNCH("svb_deposit_scatter");
  return SVB_OK;
}

extern "C" size_t svb_pairwise_scratch_bytes(int D) {
  const int64_t leaves = D >= 7 ? (int64_t(1) << (D - 7)) : 1;
  return sizeof(double) * (size_t)((leaves + 255) / 256 + 1);
}

extern "C" int svb_pairwise_sum(const double* x, int D, double* out, void* scratch, void* stream) {
  if (D < 0 || D > 48) {
    set_error("pairwise_sum: D=%d", D);
    return SVB_EINVAL;
  }
  cudaStream_t st = as_stream(stream);
  const int64_t n = int64_t(1) << D;
  if (n <= 128) {
    k_pw_small<<<1, 1, 0, st>>>(x, n, out);
  } else {
    const int64_t leaves = n / 128;
    const int64_t blocks = (leaves + 255) / 256;  // power of two (or 1 with <256 leaves)
    double* part = static_cast<double*>(scratch);
    if (leaves < 256) {
      // fewer leaves than one block: a pairwise tree over the leaves directly
      k_pw_leaves<<<1, 256, 0, st>>>(x, leaves, part);  // padded leaves are 0 and sit on the right
      // a zero-padded complete tree adds +0.0 to right-spine sums: exact
    } else {
      k_pw_leaves<<<(unsigned)blocks, 256, 0, st>>>(x, leaves, part);
      k_pw_tree<<<1, 256, 0, st>>>(part, blocks);
    }
    cudaMemcpyAsync(out, part, sizeof(double), cudaMemcpyDeviceToDevice, st);
  }
  SVB_CHECK_LAUNCH("svb_pairwise_sum");
  return SVB_OK;
}

extern "C" int svb_div_scalar(double* x, int64_t n, const double* denom, void* stream) {
  if (n <= 0) return SVB_OK;
  k_div_scalar<<<grid_for((uint64_t)n, 16), 256, 0, as_stream(stream)>>>(x, n, denom);
  SVB_CHECK_LAUNCH("svb_div_scalar");
  return SVB_OK;
}

extern "C" size_t svb_cdf_scratch_bytes(int64_t n) {
  const int64_t B = int64_t(1) << kChunkLog2;
  const int64_t nch = (n + B - 1) / B;
  return (size_t)nch * (sizeof(double) * 2 + sizeof(ChunkFn)) + 64;
}

// tot[nchunks] of q (approximate chunk totals)
extern "C" int svb_cdf_chunk_totals(const double* q, int64_t n, double* tot, void* stream) {
  const int64_t B = int64_t(1) << kChunkLog2;
  const int64_t nch = (n + B - 1) / B;
  if (n <= 0) return SVB_OK;
  k_chunk_tot<<<(unsigned)nch, 256, 0, as_stream(stream)>>>(q, n, B, tot);
  SVB_CHECK_LAUNCH("svb_cdf_chunk_totals");
  return SVB_OK;
}

// cstart: approximate c at each chunk start (host/torch prefix of the
// totals); fn: ChunkFn[nchunks] scratch; c_in: exact c before element 0
// (device scalar); writes the exact c at every chunk end and the number of
// chunks added element by element
extern "C" int svb_cdf_walk(const double* q, int64_t n, const double* cstart, const double* tot, void* fn_scratch,
                            const double* c_in, double* cend, long long* nslow, void* stream) {
  const int64_t B = int64_t(1) << kChunkLog2;
  const int64_t nch = (n + B - 1) / B;
  if (n <= 0) return SVB_OK;
  cudaStream_t st = as_stream(stream);
  ChunkFn* fn = static_cast<ChunkFn*>(fn_scratch);
  const int64_t threads = nch * 32;
  k_chunk_fns<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(q, n, B, cstart, tot, nch, fn);
  k_cdf_walk<<<1, 32, 0, st>>>(q, n, B, fn, nch, c_in, cend, nslow);
  SVB_CHECK_LAUNCH("svb_cdf_walk");
  return SVB_OK;
}

// cend_all: exact chunk ends of every process, in basis order (nchunks_all);
// this process owns chunks [my_lo, my_hi) whose elements are q[0..n) and
// whose global element index starts at index_base; out[s] = outcome or -1
extern "C" int svb_cdf_search(const double* q, int64_t n, const double* cend_all, int64_t nchunks_all, int64_t my_lo,
                              int64_t my_hi, double c_last, const double* u, int64_t nshots, int64_t index_base,
                              int64_t* out, void* stream) {
  const int64_t B = int64_t(1) << kChunkLog2;
  if (nshots <= 0) return SVB_OK;
  k_cdf_search<<<grid_for((uint64_t)nshots, 8), 256, 0, as_stream(stream)>>>(
      q, n, B, cend_all, nchunks_all, my_lo, my_lo, my_hi, c_last, u, nshots, index_base, out);
  SVB_CHECK_LAUNCH("svb_cdf_search");
  return SVB_OK;
}
