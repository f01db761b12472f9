// Peer-memory remap: the inter-GPU Pack -> Exchange -> Unpack
// (svpart/executor.py:224-281) as ONE in-place kernel over NVLink.
//
// Process w (rank bits alpha at the swapped positions) and peer p = w[e:=v]
// hold the two halves of every exchanged pair: w.region(v)[k] <-> p.region(alpha)[k]
// (DESIGN.md "Remap").  With the peer's state mapped into this process
// (CUDA IPC), each process swaps half of the pairs of every peer: it loads
// its own element and the peer's element, then stores each into the other's
// place -- one NVLink read and one NVLink write per pair, no staging buffer,
// no pack/unpack pass and no NCCL kernels.  The caller orders the launch
// between barriers (both sides' data final before, both done after).
#include <string.h>

#include "common.cuh"

namespace svb {
namespace {

constexpr int kMaxPeers = 8;

struct PeerSwapArgs {
  double2* local;
  double2* peer[kMaxPeers];
  uint64_t sel_local[kMaxPeers];   // region of this process exchanged with peer j
  uint64_t sel_remote[kMaxPeers];  // region of peer j that lands here
  int64_t first[kMaxPeers];        // this process swaps pairs [first, first+count)
  int64_t count[kMaxPeers];
  int L, eb, nchunks;              // eb = L - m (element index bits per row)
  uint64_t lut[5 * 256];           // element index -> free local bits
};

__device__ __forceinline__ uint64_t elem_addr(const uint64_t* lut, int nchunks, int L, int eb,
                                              uint64_t sel, uint64_t k) {
  const uint64_t row = k >> eb;
  const uint64_t e = k & ((uint64_t(1) << eb) - 1);
  uint64_t loc = sel;
  for (int c = 0; c < nchunks; ++c) loc |= lut[c * 256 + ((e >> (8 * c)) & 255)];
  return (row << L) | loc;
}

// grid.y = peer; 4 pairs per thread with all loads issued before the stores
__global__ void __launch_bounds__(1024) k_peer_swap(const __grid_constant__ PeerSwapArgs a) {
  __shared__ uint64_t lut[5 * 256];
  for (int i = threadIdx.x; i < a.nchunks * 256; i += blockDim.x) lut[i] = a.lut[i];
  __syncthreads();
  const int j = blockIdx.y;
  double2* __restrict__ mine = a.local;
  double2* __restrict__ theirs = a.peer[j];
  const int64_t n = a.count[j];
  const int64_t step = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < n; i0 += 4 * step) {
    uint64_t ia[4], ib[4];
    double2 x[4], y[4];
    bool ok[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t i = i0 + u * step;
      ok[u] = i < n;
      const uint64_t k = (uint64_t)(a.first[j] + (ok[u] ? i : 0));
      ia[u] = elem_addr(lut, a.nchunks, a.L, a.eb, a.sel_local[j], k);
      ib[u] = elem_addr(lut, a.nchunks, a.L, a.eb, a.sel_remote[j], k);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (ok[u]) {
        x[u] = mine[ia[u]];
        y[u] = theirs[ib[u]];
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (ok[u]) {
        mine[ia[u]] = y[u];
        theirs[ib[u]] = x[u];
      }
    }
  }
  __threadfence_system();  // peer stores visible before the completion barrier
}

// ---- bulk-copy (TMA engine) swap ------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n.reg .pred P1;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst_smem, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst_smem)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, const void* src_smem, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_u32(src_smem)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// wait until at most n store groups still read shared memory (n < 8)
__device__ __forceinline__ void bulk_wait_read(int n) {
  switch (n) {
    case 0: asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); break;
    case 1: asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); break;
    case 2: asm volatile("cp.async.bulk.wait_group.read 2;" ::: "memory"); break;
    case 3: asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory"); break;
    case 4: asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory"); break;
    case 5: asm volatile("cp.async.bulk.wait_group.read 5;" ::: "memory"); break;
    case 6: asm volatile("cp.async.bulk.wait_group.read 6;" ::: "memory"); break;
    default: asm volatile("cp.async.bulk.wait_group.read 7;" ::: "memory"); break;
  }
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

struct BulkArgs {
  double2* local;
  double2* peer[kMaxPeers];
  uint64_t sel_local[kMaxPeers];
  uint64_t sel_remote[kMaxPeers];
  int64_t first[kMaxPeers];
  int64_t count[kMaxPeers];
  int64_t pfirst[kMaxPeers];  // first absolute piece index per peer
  int64_t pstart[kMaxPeers + 1];  // prefix sum of pieces over peers
  int L, eb, nchunks, npeers;
  int interleave;  // all partners have the same number of pieces
  int piece;   // elements per piece (power of two, divides the contiguous run)
  int stages, ahead;  // ring size; pieces loading ahead (stages - ahead stores may pend)
  uint64_t lut[5 * 256];
};

// One thread per CTA drives the copy engine: piece t is bulk-loaded from both
// sides into stage t % stages, then bulk-stored crosswise; `stages - 2`
// `ahead` pieces load while up to stages - ahead store.
__global__ void __launch_bounds__(32) k_peer_swap_bulk(const __grid_constant__ BulkArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  if (threadIdx.x != 0) return;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
  unsigned char* data = smem + 128;
  const int NS = a.stages;
  const unsigned pbytes = (unsigned)a.piece * 16u;
  for (int s = 0; s < NS; ++s) mbar_init(&bars[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const int64_t total = a.pstart[a.npeers];
  const int64_t n = total > blockIdx.x ? (total - 1 - blockIdx.x) / gridDim.x + 1 : 0;

  struct Piece {
    double2* mine;
    double2* theirs;
    unsigned bytes;
  };
  auto piece_at = [&](int64_t t) -> Piece {
    const int64_t gi = blockIdx.x + t * gridDim.x;
    int j = 0;
    int64_t idx;
    if (a.interleave) {  // round-robin over partners: every link busy all the time
      j = (int)(gi % a.npeers);
      idx = gi / a.npeers;
    } else {
      while (gi >= a.pstart[j + 1]) ++j;
      idx = gi - a.pstart[j];
    }
    const int64_t abs_piece = a.pfirst[j] + idx;
    int64_t k0 = abs_piece * a.piece;
    int64_t k1 = k0 + a.piece;
    if (k0 < a.first[j]) k0 = a.first[j];
    if (k1 > a.first[j] + a.count[j]) k1 = a.first[j] + a.count[j];
    const uint64_t row = (uint64_t)k0 >> a.eb;
    const uint64_t e = (uint64_t)k0 & ((uint64_t(1) << a.eb) - 1);
    uint64_t loc = 0;
    for (int c = 0; c < a.nchunks; ++c) loc |= a.lut[c * 256 + ((e >> (8 * c)) & 255)];
    const uint64_t base = (row << a.L) | loc;
    Piece p;
    p.mine = a.local + (base | a.sel_local[j]);
    p.theirs = a.peer[j] + (base | a.sel_remote[j]);
    p.bytes = (unsigned)(k1 - k0) * 16u;
    return p;
  };
  auto issue_load = [&](int64_t t) {
    const int s = (int)(t % NS);
    const Piece p = piece_at(t);
    unsigned char* A = data + (size_t)s * 2 * pbytes;
    mbar_expect_tx(&bars[s], 2 * p.bytes);
    bulk_load(A, p.mine, p.bytes, &bars[s]);
    bulk_load(A + pbytes, p.theirs, p.bytes, &bars[s]);
  };
  const int ahead = a.ahead;
  for (int64_t t = 0; t < ahead && t < n; ++t) issue_load(t);
  for (int64_t t = 0; t < n; ++t) {
    if (t + ahead < n) {
      // the stage of piece t+ahead was piece t+ahead-NS's: its stores (committed
      // NS-ahead iterations ago) must have read it out
      bulk_wait_read(NS - ahead - 1);
      issue_load(t + ahead);
    }
    const int s = (int)(t % NS);
    mbar_wait(&bars[s], (unsigned)((t / NS) & 1));
    const Piece p = piece_at(t);
    unsigned char* A = data + (size_t)s * 2 * pbytes;
    bulk_store(p.mine, A + pbytes, p.bytes);  // the peer's element lands here
    bulk_store(p.theirs, A, p.bytes);         // ours lands there
    bulk_commit();
  }
  bulk_wait_all();
  __threadfence_system();
}

// plain 16-byte copy; either side may be a mapped peer pointer
__global__ void __launch_bounds__(256) k_copy(double2* __restrict__ dst, const double2* __restrict__ src,
                                              int64_t n) {
  const int64_t step = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < n; i0 += 4 * step) {
    double2 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (i0 + u * step < n) v[u] = src[i0 + u * step];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (i0 + u * step < n) dst[i0 + u * step] = v[u];
  }
  __threadfence_system();
}

}  // namespace
}  // namespace svb

using namespace svb;

extern "C" int svb_dev_alloc(size_t bytes, void** ptr) {
  cudaError_t e = cudaMalloc(ptr, bytes);
  return e == cudaSuccess ? SVB_OK : cuda_status(e, "cudaMalloc");
}

extern "C" int svb_dev_free(void* ptr) {
  cudaError_t e = cudaFree(ptr);
  return e == cudaSuccess ? SVB_OK : cuda_status(e, "cudaFree");
}

extern "C" int svb_ipc_handle(void* ptr, void* handle64) {
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, ptr);
  if (e != cudaSuccess) return cuda_status(e, "cudaIpcGetMemHandle");
  static_assert(sizeof(h) == 64, "IPC handle size");
  memcpy(handle64, &h, sizeof(h));
  return SVB_OK;
}

extern "C" int svb_ipc_open(const void* handle64, void** ptr) {
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, sizeof(h));
  cudaError_t e = cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess);
  return e == cudaSuccess ? SVB_OK : cuda_status(e, "cudaIpcOpenMemHandle");
}

extern "C" int svb_ipc_close(void* ptr) {
  cudaError_t e = cudaIpcCloseMemHandle(ptr);
  return e == cudaSuccess ? SVB_OK : cuda_status(e, "cudaIpcCloseMemHandle");
}

extern "C" int svb_peer_swap_bulk(svb_c128* local, void* const* peers, int npeers, int64_t rows,
                                  int L, const int32_t* lbits, int m, const uint64_t* sel_local_idx,
                                  const uint64_t* sel_remote_idx, const int64_t* first,
                                  const int64_t* count, int grid, int piece_bytes, int stages,
                                  int ahead, void* stream) {
  if (ahead == 0) ahead = stages - 2;
  if (npeers < 1 || npeers > kMaxPeers || m < 1 || m > L || L - m > 40 || rows <= 0 || grid < 1 ||
      stages < 2 || ahead < 1 || ahead >= stages || stages - ahead > 8 || piece_bytes < 16 || (piece_bytes & (piece_bytes - 1)) ||
      128 + (size_t)stages * 2 * piece_bytes > 227 * 1024) {
    set_error("peer_swap_bulk: bad arguments (peers=%d, m=%d, L=%d, grid=%d, piece=%d, stages=%d)",
              npeers, m, L, grid, piece_bytes, stages);
    return SVB_EINVAL;
  }
  BulkArgs a;
  memset(&a, 0, sizeof(a));
  a.local = reinterpret_cast<double2*>(local);
  a.L = L;
  a.eb = L - m;
  a.npeers = npeers;
  a.stages = stages;
  a.ahead = ahead;
  uint64_t used = 0;
  int lowest = L;
  for (int i = 0; i < m; ++i) {
    if (lbits[i] < 0 || lbits[i] >= L || (used >> lbits[i] & 1)) {
      set_error("peer_swap_bulk: bad local bit %d", lbits[i]);
      return SVB_EINVAL;
    }
    used |= uint64_t(1) << lbits[i];
    if (lbits[i] < lowest) lowest = lbits[i];
  }
  // a piece is a contiguous run: at most 2^lowest elements (the free bits below
  // the lowest swapped bit), and never more than piece_bytes
  int64_t piece = int64_t(1) << lowest;
  if (piece > piece_bytes / 16) piece = piece_bytes / 16;
  a.piece = (int)piece;
  a.pstart[0] = 0;
  for (int j = 0; j < npeers; ++j) {
    a.peer[j] = reinterpret_cast<double2*>(peers[j]);
    uint64_t sl = 0, sr = 0;
    for (int i = 0; i < m; ++i) {
      if ((sel_local_idx[j] >> (m - 1 - i)) & 1) sl |= uint64_t(1) << lbits[i];
      if ((sel_remote_idx[j] >> (m - 1 - i)) & 1) sr |= uint64_t(1) << lbits[i];
    }
    a.sel_local[j] = sl;
    a.sel_remote[j] = sr;
    a.first[j] = first[j];
    a.count[j] = count[j];
    const int64_t p0 = first[j] / piece;
    const int64_t p1 = count[j] > 0 ? (first[j] + count[j] - 1) / piece + 1 : p0;
    a.pfirst[j] = p0;
    a.pstart[j + 1] = a.pstart[j] + (p1 - p0);
  }
  int free_bits[64], nfree = 0;
  for (int b = 0; b < L; ++b)
    if (!(used >> b & 1)) free_bits[nfree++] = b;
  a.nchunks = (nfree + 7) / 8;
  for (int c = 0; c < a.nchunks; ++c)
    for (int v = 0; v < 256; ++v) {
      uint64_t d = 0;
      for (int jj = 0; jj < 8; ++jj) {
        const int k = 8 * c + jj;
        if (k < nfree && ((v >> jj) & 1)) d |= uint64_t(1) << free_bits[k];
      }
      a.lut[c * 256 + v] = d;
    }
  if (a.pstart[npeers] == 0) return SVB_OK;
  a.interleave = 1;
  for (int j = 1; j < npeers; ++j)
    if (a.pstart[j + 1] - a.pstart[j] != a.pstart[1]) a.interleave = 0;
  const size_t smem = 128 + (size_t)stages * 2 * piece_bytes;
  cudaError_t e = cudaFuncSetAttribute(k_peer_swap_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return cuda_status(e, "peer_swap_bulk smem");
  e = cudaFuncSetAttribute(k_peer_swap_bulk, cudaFuncAttributePreferredSharedMemoryCarveout,
                           cudaSharedmemCarveoutMaxShared);
  if (e != cudaSuccess) return cuda_status(e, "peer_swap_bulk carveout");
  int64_t g = grid;
  if (g > a.pstart[npeers]) g = a.pstart[npeers];
  k_peer_swap_bulk<<<(unsigned)g, 32, smem, as_stream(stream)>>>(a);
  SVB_CHECK_LAUNCH("svb_peer_swap_bulk");
  return SVB_OK;
}

extern "C" int svb_copy(svb_c128* dst, const svb_c128* src, int64_t n, int grid_limit, void* stream) {
  if (n < 0) {
    set_error("copy: negative length");
    return SVB_EINVAL;
  }
  if (n == 0) return SVB_OK;
  int64_t gx = (n + 4 * 256 - 1) / (4 * 256);
  const int64_t cap = grid_limit > 0 ? grid_limit : (int64_t)num_sms() * 8;
  if (gx > cap) gx = cap;
  k_copy<<<(unsigned)gx, 256, 0, as_stream(stream)>>>(reinterpret_cast<double2*>(dst),
                                                      reinterpret_cast<const double2*>(src), n);
  SVB_CHECK_LAUNCH("svb_copy");
  return SVB_OK;
}

extern "C" int svb_peer_swap(svb_c128* local, void* const* peers, int npeers, int64_t rows, int L,
                             const int32_t* lbits, int m, const uint64_t* sel_local_idx,
                             const uint64_t* sel_remote_idx, const int64_t* first,
                             const int64_t* count, int grid_limit, int block, void* stream) {
  if (block == 0) block = 256;
  if (block < 32 || block > 1024 || block % 32) {
    set_error("peer_swap: block size %d", block);
    return SVB_EINVAL;
  }
  if (npeers < 1 || npeers > kMaxPeers || m < 1 || m > L || L - m > 40 || rows <= 0) {
    set_error("peer_swap: bad geometry (peers=%d, m=%d, L=%d)", npeers, m, L);
    return SVB_EINVAL;
  }
  PeerSwapArgs a;
  a.local = reinterpret_cast<double2*>(local);
  a.L = L;
  a.eb = L - m;
  uint64_t used = 0;
  for (int i = 0; i < m; ++i) {
    if (lbits[i] < 0 || lbits[i] >= L || (used >> lbits[i] & 1)) {
      set_error("peer_swap: bad local bit %d", lbits[i]);
      return SVB_EINVAL;
    }
    used |= uint64_t(1) << lbits[i];
  }
  int64_t maxn = 0;
  for (int j = 0; j < npeers; ++j) {
    a.peer[j] = reinterpret_cast<double2*>(peers[j]);
    // selectors are given as values over lbits (bit m-1-i <-> lbits[i])
    uint64_t sl = 0, sr = 0;
    for (int i = 0; i < m; ++i) {
      if ((sel_local_idx[j] >> (m - 1 - i)) & 1) sl |= uint64_t(1) << lbits[i];
      if ((sel_remote_idx[j] >> (m - 1 - i)) & 1) sr |= uint64_t(1) << lbits[i];
    }
    a.sel_local[j] = sl;
    a.sel_remote[j] = sr;
    a.first[j] = first[j];
    a.count[j] = count[j];
    if (count[j] > maxn) maxn = count[j];
  }
  int free_bits[64], nfree = 0;
  for (int b = 0; b < L; ++b)
    if (!(used >> b & 1)) free_bits[nfree++] = b;
  a.nchunks = (nfree + 7) / 8;
  for (int c = 0; c < a.nchunks; ++c)
    for (int v = 0; v < 256; ++v) {
      uint64_t d = 0;
      for (int jj = 0; jj < 8; ++jj) {
        const int k = 8 * c + jj;
        if (k < nfree && ((v >> jj) & 1)) d |= uint64_t(1) << free_bits[k];
      }
      a.lut[c * 256 + v] = d;
    }
  if (maxn == 0) return SVB_OK;
  int64_t gx = (maxn + 4 * block - 1) / (4 * block);
  const int64_t cap = grid_limit > 0 ? grid_limit : (int64_t)num_sms() * 2048 / block;
  if (gx > cap) gx = cap;
  k_peer_swap<<<dim3((unsigned)gx, (unsigned)npeers), block, 0, as_stream(stream)>>>(a);
  SVB_CHECK_LAUNCH("svb_peer_swap");
  return SVB_OK;
}

// ---- stream-ordered cross-process flags ------------------------------------
// cuStreamWriteValue32 / cuStreamWaitValue32 through the runtime's driver
// entry points (no link against libcuda).  A process signals a peer by
// writing into the peer's flag word (mapped with svb_ipc_open) and waits on
// its own: chunk-level ordering between GPUs with no host round trip.
namespace {
typedef int (*StreamValueFn)(void* stream, unsigned long long addr, unsigned value, unsigned flags);
StreamValueFn g_write = nullptr, g_wait = nullptr;

int stream_value_fns() {
  if (g_write && g_wait) return SVB_OK;
  cudaDriverEntryPointQueryResult q;
  void* fw = nullptr;
  void* fv = nullptr;
  cudaError_t e = cudaGetDriverEntryPoint("cuStreamWriteValue32", &fw, cudaEnableDefault, &q);
  if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fw) {
    set_error("cuStreamWriteValue32 unavailable");
    return SVB_ECUDA;
  }
  e = cudaGetDriverEntryPoint("cuStreamWaitValue32", &fv, cudaEnableDefault, &q);
  if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fv) {
    set_error("cuStreamWaitValue32 unavailable");
    return SVB_ECUDA;
  }
  g_write = reinterpret_cast<StreamValueFn>(fw);
  g_wait = reinterpret_cast<StreamValueFn>(fv);
  return SVB_OK;
}
}  // namespace

extern "C" int svb_stream_write_u32(void* addr, uint32_t value, void* stream) {
  int rc = stream_value_fns();
  if (rc != SVB_OK) return rc;
  const int r = g_write(stream, reinterpret_cast<unsigned long long>(addr), value, 0 /* with barrier */);
  if (r != 0) {
    set_error("cuStreamWriteValue32 failed (%d)", r);
    return SVB_ECUDA;
  }
  return SVB_OK;
}

extern "C" int svb_stream_wait_u32(void* addr, uint32_t value, void* stream) {
  int rc = stream_value_fns();
  if (rc != SVB_OK) return rc;
  const int r = g_wait(stream, reinterpret_cast<unsigned long long>(addr), value, 0 /* GEQ */);
  if (r != 0) {
    set_error("cuStreamWaitValue32 failed (%d)", r);
    return SVB_ECUDA;
  }
  return SVB_OK;
}

extern "C" int svb_stream_create(void** stream) {
  cudaStream_t s;
  cudaError_t e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  if (e != cudaSuccess) return cuda_status(e, "cudaStreamCreateWithFlags");
  *stream = reinterpret_cast<void*>(s);
  return SVB_OK;
}
