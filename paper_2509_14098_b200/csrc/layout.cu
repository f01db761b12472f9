// Layout kernels: qubit remap between co-resident ranks, region pack/unpack
// around the NCCL exchange, and storage<->basis bit permutations.
//
// Reference: Pack/Exchange/Unpack (svpart/executor.py:224-281) with the
// rank-bit helpers (:100-120); gather/scatter via _storage_to_basis
// (:310-343).  All three are pure index permutations: bit-exact by
// construction, HBM-bound.
#include "common.cuh"

namespace svb {
namespace {

struct BitSwap {
  int m;
  int u[16], w[16];
  int rest[SVB_MAX_DEV_BITS];  // bits not involved in any swap, ascending
  int nrest;
};

// Thread per (base, combo): combo enumerates the 2m swapped bits (fastest
// varying, so a warp touches neighbouring addresses when swapped bits are
// low), base enumerates the untouched bits.  The permutation is an
// involution; only combo < partner(combo) moves data.
__global__ void k_bitswap(double2* __restrict__ s, BitSwap bs, uint64_t total) {
  const int cb = 2 * bs.m;
  for (uint64_t gid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; gid < total;
       gid += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t combo = (uint32_t)(gid & ((uint64_t(1) << cb) - 1));
    uint64_t r = gid >> cb;
    uint64_t base = 0;
    for (int i = 0; i < bs.nrest && r; ++i, r >>= 1)
      if (r & 1) base |= uint64_t(1) << bs.rest[i];
    // combo bit 2i -> u[i], bit 2i+1 -> w[i]; partner swaps each pair
    uint32_t partner = 0;
    uint64_t x = base, y = base;
    for (int i = 0; i < bs.m; ++i) {
      const uint32_t bu = (combo >> (2 * i)) & 1, bw = (combo >> (2 * i + 1)) & 1;
      partner |= (bw << (2 * i)) | (bu << (2 * i + 1));
      x |= (uint64_t)bu << bs.u[i] | (uint64_t)bw << bs.w[i];
      y |= (uint64_t)bw << bs.u[i] | (uint64_t)bu << bs.w[i];
    }
    if (combo < partner) {
      const double2 a = s[x], b = s[y];
      s[x] = b;
      s[y] = a;
    }
  }
}

struct Region {
  int L, m;
  uint64_t selmask;  // sel deposited into lbits
  int nchunks;       // 8-bit chunks of the element index
  uint64_t lut[5 * 256];  // deposit of element-index chunks into the free bits
};

__device__ __forceinline__ uint64_t region_index(const uint64_t* lut, int nchunks, int L, int m,
                                                 uint64_t selmask, uint64_t k) {
  // k = row * 2^(L-m) + e  ->  row * 2^L + deposit(e) | selmask
  const int eb = L - m;
  const uint64_t row = k >> eb;
  const uint64_t e = k & ((uint64_t(1) << eb) - 1);
  uint64_t loc = selmask;
  for (int c = 0; c < nchunks; ++c) loc |= lut[c * 256 + ((e >> (8 * c)) & 255)];
  return (row << L) | loc;
}

template <bool PACK>
__global__ void k_region(double2* __restrict__ s, const __grid_constant__ Region r, int64_t off,
                         int64_t count, double2* __restrict__ buf) {
  __shared__ uint64_t lut[5 * 256];
  for (int i = threadIdx.x; i < r.nchunks * 256; i += blockDim.x) lut[i] = r.lut[i];
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t a = region_index(lut, r.nchunks, r.L, r.m, r.selmask, (uint64_t)(off + i));
    if (PACK)
      buf[i] = s[a];
    else
      s[a] = buf[i];
  }
}

// dst[P(f)] = src[f]; P built from 8-bit lookup tables (kernel parameter,
// copied to shared memory: 10 KB, fits the 32 KB parameter space)
struct PermLut {
  uint64_t v[5 * 256];
};

__global__ void k_bitperm(const double2* __restrict__ src, double2* __restrict__ dst, int nbits,
                          const __grid_constant__ PermLut lut_p, uint64_t total) {
  __shared__ uint64_t lut[5 * 256];
  const int nchunks = (nbits + 7) / 8;
  for (int i = threadIdx.x; i < nchunks * 256; i += blockDim.x) lut[i] = lut_p.v[i];
  __syncthreads();
  for (uint64_t f = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; f < total;
       f += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t p = 0;
    for (int c = 0; c < nchunks; ++c) p |= lut[c * 256 + ((f >> (8 * c)) & 255)];
    dst[p] = src[f];
  }
}

int grid_for(uint64_t work, int threads) {
  uint64_t b = (work + threads - 1) / threads;
  const uint64_t cap = (uint64_t)num_sms() * 32;
  if (b > cap) b = cap;
  return b ? (int)b : 1;
}

int make_region(int64_t rows, int L, const int32_t* lbits, int m, uint32_t sel, Region& r) {
  if (m < 0 || m > L || L > 62 || rows <= 0 || L - m > 40) {
    set_error("bad region geometry (m=%d, L=%d)", m, L);
    return SVB_EINVAL;
  }
  r.L = L;
  r.m = m;
  r.selmask = 0;
  uint64_t used = 0;
  for (int i = 0; i < m; ++i) {
    if (lbits[i] < 0 || lbits[i] >= L || (used >> lbits[i] & 1)) {
      set_error("bad region bit %d", lbits[i]);
      return SVB_EINVAL;
    }
    used |= uint64_t(1) << lbits[i];
    // selector bit (m-1-i) <-> lbits[i]  (swap i <-> selector bit m-1-i,
    // executor.py:100-105)
    if ((sel >> (m - 1 - i)) & 1) r.selmask |= uint64_t(1) << lbits[i];
  }
  int free_bits[64], nfree = 0;
  for (int b = 0; b < L; ++b)
    if (!(used >> b & 1)) free_bits[nfree++] = b;
  r.nchunks = (nfree + 7) / 8;
  for (int c = 0; c < r.nchunks; ++c)
    for (int v = 0; v < 256; ++v) {
      uint64_t d = 0;
      for (int j = 0; j < 8; ++j) {
        const int k = 8 * c + j;
        if (k < nfree && ((v >> j) & 1)) d |= uint64_t(1) << free_bits[k];
      }
      r.lut[c * 256 + v] = d;
    }
  return SVB_OK;
}

}  // namespace
}  // namespace svb

using namespace svb;

extern "C" int svb_bitswap(svb_c128* state, int D, const int32_t* u, const int32_t* w, int m,
                           void* stream) {
  if (m < 0 || m > 8 || D > 62) {
    set_error("bitswap: m=%d out of range", m);
    return SVB_ERANGE;
  }
  if (m == 0) return SVB_OK;
  BitSwap bs;
  bs.m = m;
  uint64_t used = 0;
  for (int i = 0; i < m; ++i) {
    if (u[i] < 0 || u[i] >= D || w[i] < 0 || w[i] >= D || u[i] == w[i] || (used >> u[i] & 1) ||
        (used >> w[i] & 1)) {
      set_error("bitswap: bad bit pair (%d, %d)", u[i], w[i]);
      return SVB_EINVAL;
    }
    used |= (uint64_t(1) << u[i]) | (uint64_t(1) << w[i]);
    bs.u[i] = u[i];
    bs.w[i] = w[i];
  }
  bs.nrest = 0;
  for (int b = 0; b < D; ++b)
    if (!(used >> b & 1)) bs.rest[bs.nrest++] = b;
  const uint64_t total = uint64_t(1) << D;  // (2^(D-2m) bases) x (4^m combos)
  k_bitswap<<<grid_for(total, 256), 256, 0, as_stream(stream)>>>(
      reinterpret_cast<double2*>(state), bs, total);
  SVB_CHECK_LAUNCH("svb_bitswap");
  return SVB_OK;
}

extern "C" int svb_pack_region(const svb_c128* state, int64_t rows, int L, const int32_t* lbits,
                               int m, uint32_t sel, int64_t off, int64_t count, svb_c128* out,
                               void* stream) {
  Region r;
  if (int rc = make_region(rows, L, lbits, m, sel, r)) return rc;
  if (off < 0 || count < 0 || off + count > (rows << (L - m))) {
    set_error("pack: range [%lld, +%lld) outside region", (long long)off, (long long)count);
    return SVB_EINVAL;
  }
  if (!count) return SVB_OK;
  k_region<true><<<grid_for(count, 256), 256, 0, as_stream(stream)>>>(
      const_cast<double2*>(reinterpret_cast<const double2*>(state)), r, off, count,
      reinterpret_cast<double2*>(out));
  SVB_CHECK_LAUNCH("svb_pack_region");
  return SVB_OK;
}

extern "C" int svb_unpack_region(svb_c128* state, int64_t rows, int L, const int32_t* lbits, int m,
                                 uint32_t sel, int64_t off, int64_t count, const svb_c128* in,
                                 void* stream) {
  Region r;
  if (int rc = make_region(rows, L, lbits, m, sel, r)) return rc;
  if (off < 0 || count < 0 || off + count > (rows << (L - m))) {
    set_error("unpack: range [%lld, +%lld) outside region", (long long)off, (long long)count);
    return SVB_EINVAL;
  }
  if (!count) return SVB_OK;
  k_region<false><<<grid_for(count, 256), 256, 0, as_stream(stream)>>>(
      reinterpret_cast<double2*>(state), r, off, count,
      const_cast<double2*>(reinterpret_cast<const double2*>(in)));
  SVB_CHECK_LAUNCH("svb_unpack_region");
  return SVB_OK;
}

// perm: host array (bit k of the source index moves to bit perm[k])
extern "C" int svb_bitperm(const svb_c128* src, svb_c128* dst, int nbits, const int32_t* perm,
                           void* stream) {
  if (nbits < 0 || nbits > 40) {
    set_error("bitperm: %d bits out of range", nbits);
    return SVB_ERANGE;
  }
  uint64_t used = 0;
  for (int k = 0; k < nbits; ++k) {
    if (perm[k] < 0 || perm[k] >= nbits || (used >> perm[k] & 1)) {
      set_error("bitperm: not a permutation");
      return SVB_EINVAL;
    }
    used |= uint64_t(1) << perm[k];
  }
  PermLut lut;
  const int nchunks = (nbits + 7) / 8;
  for (int c = 0; c < nchunks; ++c)
    for (int v = 0; v < 256; ++v) {
      uint64_t p = 0;
      for (int j = 0; j < 8; ++j) {
        const int k = 8 * c + j;
        if (k < nbits && ((v >> j) & 1)) p |= uint64_t(1) << perm[k];
      }
      lut.v[c * 256 + v] = p;
    }
  const uint64_t total = uint64_t(1) << nbits;
  k_bitperm<<<grid_for(total, 256), 256, 0, as_stream(stream)>>>(
      reinterpret_cast<const double2*>(src), reinterpret_cast<double2*>(dst), nbits, lut, total);
  SVB_CHECK_LAUNCH("svb_bitperm");
  return SVB_OK;
}
