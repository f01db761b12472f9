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

// ---- tiled bit permutation ---------------------------------------------
// A tile is the set of elements that differ only in the tile bits T: T holds
// the low source bits (coalesced 16-byte loads in runs of 2^a) and the
// source bits that land on the low destination bits (coalesced stores),
// padded with further low source bits up to kTileBits.  A CTA loads a tile
// into shared memory in source order and writes it out in destination
// order; the XOR swizzle keeps both access patterns conflict free.  With
// src == dst the permutation must map every tile onto itself (bit swaps
// whose bits are all tile bits): the swap is then in place.
constexpr int kTileBits = 11;
constexpr int kTileThreads = 256;

struct TilePerm {
  int nt;                        // tile bits
  int nrest;                     // non-tile source bits (tile index), ascending
  int rest[SVB_MAX_DEV_BITS];
  int rest_dst[SVB_MAX_DEV_BITS];  // perm[rest[i]]
  uint64_t ld_lo[64], ld_hi[32];  // load-order index (low 6 / high 5 bits) -> source offset bits
  uint64_t st_lo[64], st_hi[32];  // store-order index -> destination offset bits
  uint16_t jmap_lo[64], jmap_hi[32];  // store-order index -> swizzled smem slot
  uint32_t swz_lo[64], swz_hi[32];    // load-order index -> swizzled smem slot
};

__global__ void __launch_bounds__(kTileThreads) k_tperm(const double2* __restrict__ src, double2* __restrict__ dst,
                                                        const __grid_constant__ TilePerm tp, uint64_t ntiles) {
  extern __shared__ __align__(16) double2 tile[];
  // per-lane table lookups from shared memory (parameter-space reads with
  // lane-varying indices would serialise in the constant cache)
  __shared__ uint64_t ld_lo[64], ld_hi[32], st_lo[64], st_hi[32];
  __shared__ uint32_t sw_lo[64], sw_hi[32], jm_lo[64], jm_hi[32];
  const int lane = threadIdx.x & 31;
  // tile bases: lane l deposits non-tile bit l of the tile index (source and
  // destination position), OR-reduced over the warp
  const int rest_src = lane < tp.nrest ? tp.rest[lane] : 0;
  const int rest_dst = lane < tp.nrest ? tp.rest_dst[lane] : 0;
  if (threadIdx.x < 64) {
    const int v = threadIdx.x;
    ld_lo[v] = tp.ld_lo[v];
    st_lo[v] = tp.st_lo[v];
    sw_lo[v] = tp.swz_lo[v];
    jm_lo[v] = tp.jmap_lo[v];
  }
  if (threadIdx.x < 32) {
    const int v = threadIdx.x;
    ld_hi[v] = tp.ld_hi[v];
    st_hi[v] = tp.st_hi[v];
    sw_hi[v] = tp.swz_hi[v];
    jm_hi[v] = tp.jmap_hi[v];
  }
  __syncthreads();
  const int n = 1 << tp.nt;
  for (uint64_t ti = blockIdx.x; ti < ntiles; ti += gridDim.x) {
    const uint64_t on = lane < tp.nrest ? (ti >> lane) & 1ull : 0ull;
    uint64_t sb = on << rest_src, db = on << rest_dst;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      sb |= __shfl_xor_sync(0xffffffffu, sb, o);
      db |= __shfl_xor_sync(0xffffffffu, db, o);
    }
#pragma unroll 8
    for (int j = threadIdx.x; j < n; j += blockDim.x)
      tile[sw_lo[j & 63] ^ sw_hi[j >> 6]] = src[sb | ld_lo[j & 63] | ld_hi[j >> 6]];
    __syncthreads();
#pragma unroll 8
    for (int k = threadIdx.x; k < n; k += blockDim.x)
      st_stream(dst + (db | st_lo[k & 63] | st_hi[k >> 6]), tile[jm_lo[k & 63] ^ jm_hi[k >> 6]]);
    __syncthreads();
  }
}

// build the tile geometry of permutation perm (source bit k -> perm[k]);
// inplace: the tile must be closed under perm.  Returns false when no tile
// of at most kTileBits bits exists (the caller uses the element kernel).
bool make_tile_perm(int nbits, const int32_t* perm, bool inplace, TilePerm& tp) {
  if (nbits < 1 || nbits > SVB_MAX_DEV_BITS) return false;
  int inv[64];
  for (int k = 0; k < nbits; ++k) inv[perm[k]] = k;
  const int a = nbits < 5 ? nbits : 5;
  bool in_t[64] = {false};
  int cnt = 0;
  auto add = [&](int b) {
    if (!in_t[b]) {
      in_t[b] = true;
      ++cnt;
    }
  };
  for (int b = 0; b < a; ++b) add(b);
  for (int b = 0; b < a; ++b) add(inv[b]);
  if (inplace) {  // every moving bit in the tile, closed under perm: the tile maps onto itself
    for (int b = 0; b < nbits; ++b)
      if (perm[b] != b) add(b);
    bool grew = true;
    while (grew) {
      grew = false;
      for (int b = 0; b < nbits; ++b)
        if (in_t[b] && !in_t[perm[b]]) {
          add(perm[b]);
          grew = true;
        }
    }
    for (int b = 0; b < nbits; ++b)
      if (!in_t[b] && perm[b] != b) return false;  // a moving bit outside the tile
  }
  if (cnt > kTileBits) return false;
  for (int b = 0; b < nbits && cnt < kTileBits; ++b)
    if (!in_t[b] && (!inplace || perm[b] == b)) add(b);
  const int nt = cnt;
  int src_t[kTileBits], dst_t[kTileBits], ns = 0;
  for (int b = 0; b < nbits; ++b)
    if (in_t[b]) src_t[ns++] = b;
  int nd = 0;
  for (int b = 0; b < nbits; ++b)
    if (in_t[inv[b]]) dst_t[nd++] = b;
  tp.nt = nt;
  tp.nrest = 0;
  for (int b = 0; b < nbits; ++b)
    if (!in_t[b]) {
      tp.rest_dst[tp.nrest] = perm[b];
      tp.rest[tp.nrest++] = b;
    }
  if (tp.nrest > 32) return false;  // one warp lane per non-tile bit
  // load-order position of each store-order bit
  int pos_of_src[64];
  for (int i = 0; i < nt; ++i) pos_of_src[src_t[i]] = i;
  int jpos[kTileBits];
  for (int i = 0; i < nt; ++i) jpos[i] = pos_of_src[inv[dst_t[i]]];
  // swizzle: load positions >= 3 that hold the low 3 store bits are folded
  // onto the low slot bits the low 3 store bits do not already occupy
  int fold_from[3], fold_to[3], nf = 0;
  bool low_used[3] = {false, false, false};
  for (int i = 0; i < 3 && i < nt; ++i)
    if (jpos[i] < 3) low_used[jpos[i]] = true;
  int free_low[3], nfl = 0;
  for (int b = 0; b < 3 && b < nt; ++b)
    if (!low_used[b]) free_low[nfl++] = b;
  for (int i = 0; i < 3 && i < nt; ++i)
    if (jpos[i] >= 3) {
      fold_from[nf] = jpos[i];
      fold_to[nf] = free_low[nf];
      ++nf;
    }
  auto swz = [&](uint32_t j) {
    uint32_t x = j;
    for (int f = 0; f < nf; ++f) x ^= ((j >> fold_from[f]) & 1u) << fold_to[f];
    return x;
  };
  // index tables split into the low 6 and high 5 index bits; the swizzle is
  // linear over XOR, so slot(j) = slot(j & 63) ^ slot(j & ~63)
  for (int v = 0; v < 64; ++v) {
    uint64_t llo = 0, slo = 0;
    uint32_t jlo = 0;
    for (int i = 0; i < 6 && i < nt; ++i)
      if ((v >> i) & 1) {
        llo |= uint64_t(1) << src_t[i];
        slo |= uint64_t(1) << dst_t[i];
        jlo |= 1u << jpos[i];
      }
    tp.ld_lo[v] = llo;
    tp.st_lo[v] = slo;
    tp.swz_lo[v] = swz((uint32_t)v);
    tp.jmap_lo[v] = (uint16_t)swz(jlo);
  }
  for (int v = 0; v < 32; ++v) {
    uint64_t lhi = 0, shi = 0;
    uint32_t jhi = 0;
    for (int i = 0; i < 5 && i + 6 < nt; ++i)
      if ((v >> i) & 1) {
        lhi |= uint64_t(1) << src_t[i + 6];
        shi |= uint64_t(1) << dst_t[i + 6];
        jhi |= 1u << jpos[i + 6];
      }
    tp.ld_hi[v] = lhi;
    tp.st_hi[v] = shi;
    tp.swz_hi[v] = swz((uint32_t)v << 6);
    tp.jmap_hi[v] = (uint16_t)swz(jhi);
  }
  return true;
}

int launch_tperm(const double2* src, double2* dst, int nbits, const TilePerm& tp, cudaStream_t st) {
  const uint64_t ntiles = uint64_t(1) << (nbits - tp.nt);
  const size_t smem = sizeof(double2) << tp.nt;
  uint64_t grid = (uint64_t)num_sms() * 6;  // 32 KB tiles: six CTAs per SM
  if (grid > ntiles) grid = ntiles;
  k_tperm<<<(unsigned)grid, kTileThreads, smem, st>>>(src, dst, tp, ntiles);
  SVB_CHECK_LAUNCH("tiled bit permutation");
  return SVB_OK;
}

// dst[t] = src[P(base + t)], t < count (P from 8-bit lookup tables): one
// contiguous chunk of a permuted order, e.g. basis-sorted shard order for
// the chunked gather
__global__ void k_gather_bits(const double2* __restrict__ src, double2* __restrict__ dst, int nbits,
                              const __grid_constant__ PermLut lut_p, uint64_t base, uint64_t count) {
  __shared__ uint64_t lut[5 * 256];
  const int nchunks = (nbits + 7) / 8;
  for (int i = threadIdx.x; i < nchunks * 256; i += blockDim.x) lut[i] = lut_p.v[i];
  __syncthreads();
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < count; t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t f = base + t;
    uint64_t p = 0;
    for (int c = 0; c < nchunks; ++c) p |= lut[c * 256 + ((f >> (8 * c)) & 255)];
    dst[t] = src[p];
  }
}

// state[region dst][k] = state[region src][k]: one region of the swapped
// local bits moved onto another (the local remap after a replicated prefix)
__global__ void k_region_move(double2* __restrict__ s, const __grid_constant__ Region r, uint64_t dst_mask,
                              uint64_t count) {
  __shared__ uint64_t lut[5 * 256];
  for (int i = threadIdx.x; i < r.nchunks * 256; i += blockDim.x) lut[i] = r.lut[i];
  __syncthreads();
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < count; k += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t a = region_index(lut, r.nchunks, r.L, r.m, r.selmask, k);
    const uint64_t b = (a & ~r.selmask) | dst_mask;
    st_stream(s + b, ld_stream(s + a));
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
  {  // tiled in place when the swapped bits and the low bits fit one tile
    int32_t perm[64];
    for (int b = 0; b < D; ++b) perm[b] = b;
    for (int i = 0; i < m; ++i) {
      perm[u[i]] = w[i];
      perm[w[i]] = u[i];
    }
    static thread_local TilePerm tp;  // host-side parameter block (about 13 KB)
    if (D >= kTileBits && make_tile_perm(D, perm, true, tp))
      return launch_tperm(reinterpret_cast<const double2*>(state), reinterpret_cast<double2*>(state), D, tp,
                          as_stream(stream));
  }
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
  {
    static thread_local TilePerm tp;
    if (nbits >= kTileBits && make_tile_perm(nbits, perm, false, tp))
      return launch_tperm(reinterpret_cast<const double2*>(src), reinterpret_cast<double2*>(dst), nbits, tp,
                          as_stream(stream));
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

// dst[t] = src[P(base + t)] for t < count, P(f) = sum_k bit_k(f) << perm[k]
extern "C" int svb_gather_bits(const svb_c128* src, int nbits, const int32_t* perm, uint64_t base, int64_t count,
                               svb_c128* dst, void* stream) {
  if (nbits < 0 || nbits > 40 || count < 0) {
    set_error("gather_bits: bad arguments (nbits=%d)", nbits);
    return SVB_ERANGE;
  }
  uint64_t used = 0;
  for (int k = 0; k < nbits; ++k) {
    if (perm[k] < 0 || perm[k] >= nbits || (used >> perm[k] & 1)) {
      set_error("gather_bits: not a permutation");
      return SVB_EINVAL;
    }
    used |= uint64_t(1) << perm[k];
  }
  if (count == 0) return SVB_OK;
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
  k_gather_bits<<<grid_for((uint64_t)count, 256), 256, 0, as_stream(stream)>>>(
      reinterpret_cast<const double2*>(src), reinterpret_cast<double2*>(dst), nbits, lut, base, (uint64_t)count);
  SVB_CHECK_LAUNCH("svb_gather_bits");
  return SVB_OK;
}

extern "C" int svb_region_move(svb_c128* state, int nbits, const int32_t* lbits, int m, uint32_t src_sel,
                               uint32_t dst_sel, void* stream) {
  Region r;
  if (int rc = make_region(1, nbits, lbits, m, src_sel, r)) return rc;
  if (src_sel == dst_sel) return SVB_OK;
  uint64_t dst_mask = 0;
  for (int i = 0; i < m; ++i)
    if ((dst_sel >> (m - 1 - i)) & 1) dst_mask |= uint64_t(1) << lbits[i];
  const uint64_t count = uint64_t(1) << (nbits - m);
  k_region_move<<<grid_for(count, 256), 256, 0, as_stream(stream)>>>(reinterpret_cast<double2*>(state), r, dst_mask,
                                                                      count);
  SVB_CHECK_LAUNCH("svb_region_move");
  return SVB_OK;
}
