// Measurement sampling on the device (svpart/executor.py:375-383).
//
// The reference draws rng.choice(2^d, shots, p=|psi|^2 / sum), which numpy
// evaluates as cdf = cumsum(p); cdf /= cdf[-1]; u = rng.random(shots);
// outcome = searchsorted(cdf, u, side="right") over the BASIS order (qubit 0
// most significant).  A process holds a shard of the state in storage order:
// its elements' basis indices share fixed bits (its top rank bits) and run
// over all values of the other D bits.  So:
//   svb_probs_sorted   writes |a|^2 of the shard in basis-sorted shard order
//                      (a bit permutation), ready for an inclusive scan;
//   svb_sample_prefix  gives, for each shot's candidate basis index m, the
//                      shard's share of the CDF at m: the scan value at the
//                      number of shard elements with basis index <= m.
// The host runs a binary search over [0, 2^d) per shot, summing the shares
// of all processes at every step (paper_2509_14098_b200/sampling.py).
#include "common.cuh"

namespace svb {
namespace {

struct SortPerm {
  int nchunks;
  uint64_t lut[5 * 256];  // shard index chunk -> sorted index bits
};

__global__ void k_probs_sorted(const double2* __restrict__ a, uint64_t n, const __grid_constant__ SortPerm sp,
                               double* __restrict__ out) {
  __shared__ uint64_t lut[5 * 256];
  for (int i = threadIdx.x; i < sp.nchunks * 256; i += blockDim.x) lut[i] = sp.lut[i];
  __syncthreads();
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < n;
       t += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t j = 0;
    for (int c = 0; c < sp.nchunks; ++c) j |= lut[c * 256 + ((t >> (8 * c)) & 255)];
    const double2 v = a[t];
    const double m = hypot(v.x, v.y);  // numpy: np.abs(z) ** 2
    out[j] = __dmul_rn(m, m);
  }
}

struct PrefixArgs {
  uint64_t fixed_mask;  // basis bits fixed for this shard
  uint64_t fixed_val;
  int d;
  int nfree_below[64];  // free basis positions strictly below p
};

// number of shard elements whose basis index is <= m
__device__ __forceinline__ uint64_t shard_rank(uint64_t m, const PrefixArgs& a) {
  uint64_t cnt = 0;
  for (int p = a.d - 1; p >= 0; --p) {
    const uint64_t mb = (m >> p) & 1;
    if ((a.fixed_mask >> p) & 1) {
      const uint64_t fb = (a.fixed_val >> p) & 1;
      if (mb > fb) return cnt + (uint64_t(1) << a.nfree_below[p]);
      if (mb < fb) return cnt;
    } else if (mb) {
      cnt += uint64_t(1) << a.nfree_below[p];  // this bit 0: everything below is smaller
    }
  }
  return cnt + 1;  // equal
}

__global__ void k_sample_prefix(const double* __restrict__ cdf, const int64_t* __restrict__ mid, int64_t nshots,
                                const __grid_constant__ PrefixArgs a, double* __restrict__ out) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nshots;
       s += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t c = shard_rank((uint64_t)mid[s], a);
    out[s] = c ? cdf[c - 1] : 0.0;
  }
}

}  // namespace
}  // namespace svb

using namespace svb;

extern "C" int svb_probs_sorted(const svb_c128* shard, int D, const int32_t* perm, double* out, void* stream) {
  if (D < 0 || D > 40) {
    set_error("probs_sorted: D=%d out of range", D);
    return SVB_EINVAL;
  }
  SortPerm sp;
  sp.nchunks = D > 0 ? (D + 7) / 8 : 1;
  uint64_t used = 0;
  for (int s = 0; s < D; ++s) {
    if (perm[s] < 0 || perm[s] >= D || (used >> perm[s] & 1)) {
      set_error("probs_sorted: perm is not a permutation of %d bits", D);
      return SVB_EINVAL;
    }
    used |= uint64_t(1) << perm[s];
  }
  for (int c = 0; c < sp.nchunks; ++c)
    for (int v = 0; v < 256; ++v) {
      uint64_t j = 0;
      for (int k = 0; k < 8; ++k) {
        const int s = 8 * c + k;
        if (s < D && ((v >> k) & 1)) j |= uint64_t(1) << perm[s];
      }
      sp.lut[c * 256 + v] = j;
    }
  const uint64_t n = uint64_t(1) << D;
  uint64_t blocks = (n + 255) / 256;
  if (blocks > (uint64_t)num_sms() * 16) blocks = (uint64_t)num_sms() * 16;
  k_probs_sorted<<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(reinterpret_cast<const double2*>(shard), n,
                                                                   sp, out);
  SVB_CHECK_LAUNCH("svb_probs_sorted");
  return SVB_OK;
}

extern "C" int svb_sample_prefix(const double* cdf, int d, uint64_t fixed_mask, uint64_t fixed_val,
                                 const int64_t* mid, int64_t nshots, double* out, void* stream) {
  if (d < 0 || d > 62 || nshots < 0) {
    set_error("sample_prefix: bad arguments (d=%d)", d);
    return SVB_EINVAL;
  }
  if (nshots == 0) return SVB_OK;
  PrefixArgs a;
  a.fixed_mask = fixed_mask;
  a.fixed_val = fixed_val & fixed_mask;
  a.d = d;
  int below = 0;
  for (int p = 0; p < 64; ++p) {
    a.nfree_below[p] = below;
    if (p < d && !((fixed_mask >> p) & 1)) ++below;
  }
  int64_t blocks = (nshots + 255) / 256;
  if (blocks > num_sms() * 8) blocks = num_sms() * 8;
  k_sample_prefix<<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(cdf, mid, nshots, a, out);
  SVB_CHECK_LAUNCH("svb_sample_prefix");
  return SVB_OK;
}
