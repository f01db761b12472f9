// Fused leaf sweep: one HBM read + one HBM write of the device state per
// sweep, with a whole gate program applied to 2^K-amplitude tiles on chip.
//
// Replaces the per-gate passes of the reference's ApplyFused
// (svpart/executor.py:123-176 -> kernels/_core.pyx:7-106): there every gate
// is a full pass over all ranks' blocks; here a leaf of the partition tree
// (the level-1 "tile", plan.py:78-102) costs one pass.
//
// Execution model:
//   * a CTA owns one tile at a time (persistent over tiles): the K tile bits
//     vary inside the tile, every other device-index bit ("tile bits" F) is
//     fixed per tile;
//   * the tile is staged in shared memory (XOR-swizzled per sweep so every
//     stage mapping is bank-conflict free), each thread holds 16 amplitudes
//     in registers: the 4 "register slots" of the current stage;
//   * ops act on registers; OP_STAGE re-maps which 4 tile bits live in
//     registers (a round trip through shared memory);
//   * diagonal phases are pre-combined on the host and applied as
//     per-thread / per-tile / per-register factors (OP_PH*, pre-phase of
//     OP_U1/OP_H), so a long run of cp gates costs a few complex multiplies.
#include "common.cuh"

namespace svb {
namespace {

constexpr int RB = SVB_REG_BITS;  // register slots per thread
constexpr int NR = 1 << RB;       // amplitudes per thread
#define SVB_MAX_TILE_BITS_SWEEP 12     // double-buffered 2 x 64 KB tiles
constexpr int kMaxCtab = 512;    // per-tile scalar slots

struct SweepArgs {
  svb_sweep_desc d;
  const svb_op* ops;
  const double2* coef;
  const double2* tab;
  const svb_cterm* cterms;
  const int32_t* cofs;  // cterm CSR offsets, nctab+1 entries
  double* norm_out;
  int fbits[SVB_MAX_DEV_BITS];  // non-tile device bits, ascending
  int nf;
};

__device__ __forceinline__ double2 one2() { return make_double2(1.0, 0.0); }

// uniform-address coefficient load that the compiler may not hoist or CSE
// (keeps matrix entries out of the register budget of the amplitudes)
__device__ __forceinline__ double2 ldu(const double2* p) {
  double2 r;
  asm volatile("ld.global.nc.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}

// ---- phase application: depth-first product over register slots ---------
// Leaves are the register amplitudes V with slot A set; the phase of leaf V
// is p * prod_{s != A, bit s of V} c_s with c_s = ph[1+s] when bit s of `nt`
// is set (slots whose factor is exactly 1 are skipped).
template <int A, int S, int V, int MODE>
__device__ __forceinline__ void phase_dfs(double2 (&x)[NR], double2 p, const double2* __restrict__ ph,
                                          int nt) {
  if constexpr (S == RB) {
    if constexpr (MODE == 0) {  // phase only
      x[V] = cmul(x[V], p);
    } else {  // phase, then unscaled H on slot A
      const double2 x1 = cmul(x[V], p);
      const double2 x0 = x[V ^ (1 << A)];
      x[V ^ (1 << A)] = cadd(x0, x1);
      x[V] = csub(x0, x1);
    }
  } else if constexpr (S == A) {
    phase_dfs<A, S + 1, V, MODE>(x, p, ph, nt);
  } else {
    phase_dfs<A, S + 1, V, MODE>(x, p, ph, nt);
    const double2 q = ((nt >> S) & 1) ? cmul(p, __ldg(ph + 1 + S)) : p;
    phase_dfs<A, S + 1, V | (1 << S), MODE>(x, q, ph, nt);
  }
}

template <int A>
__device__ __forceinline__ void apply_h(double2 (&x)[NR], uint32_t cm, uint32_t cv) {
#pragma unroll
  for (int v = 0; v < NR; ++v) {
    if ((v >> A) & 1) continue;
    if ((v & cm) != cv) continue;
    double2 x0 = x[v], x1 = x[v | (1 << A)];
    x[v] = cadd(x0, x1);
    x[v | (1 << A)] = csub(x0, x1);
  }
}

template <int A>
__device__ __forceinline__ void apply_u1(double2 (&x)[NR], uint32_t cm, uint32_t cv, double2 m00, double2 m01,
                                         double2 m10, double2 m11) {
#pragma unroll
  for (int v = 0; v < NR; ++v) {
    if ((v >> A) & 1) continue;
    if ((v & cm) != cv) continue;
    double2 x0 = x[v], x1 = x[v | (1 << A)];
    x[v] = cfma(m01, x1, cmul(m00, x0));
    x[v | (1 << A)] = cfma(m11, x1, cmul(m10, x0));
  }
}

template <int A>
__device__ __forceinline__ void apply_x(double2 (&x)[NR], uint32_t cm, uint32_t cv) {
#pragma unroll
  for (int v = 0; v < NR; ++v) {
    if ((v >> A) & 1) continue;
    if ((v & cm) != cv) continue;
    double2 t = x[v];
    x[v] = x[v | (1 << A)];
    x[v | (1 << A)] = t;
  }
}

// 4x4 on slots (A, B); matrix index bit 1 <-> slot A, bit 0 <-> slot B
template <int A, int B>
__device__ __forceinline__ void apply_u2(double2 (&x)[NR], uint32_t cm, const double2* __restrict__ m) {
  // matrix rows are streamed from L1 (uniform addresses) to keep the
  // register budget for the 16 amplitudes
#pragma unroll
  for (int v = 0; v < NR; ++v) {
    if ((v >> A) & 1) continue;
    if ((v >> B) & 1) continue;
    if ((v & cm) != cm) continue;
    const int i0 = v, i1 = v | (1 << B), i2 = v | (1 << A), i3 = v | (1 << A) | (1 << B);
    const double2 a0 = x[i0], a1 = x[i1], a2 = x[i2], a3 = x[i3];
    double2 y[4];
#pragma unroll
    for (int r = 0; r < 4; ++r)
      y[r] = cfma(ldu(m + 4 * r + 3), a3,
                  cfma(ldu(m + 4 * r + 2), a2, cfma(ldu(m + 4 * r + 1), a1, cmul(ldu(m + 4 * r), a0))));
    x[i0] = y[0];
    x[i1] = y[1];
    x[i2] = y[2];
    x[i3] = y[3];
  }
}

template <int MODE>
__device__ __forceinline__ void phase_dispatch(int a, double2 (&x)[NR], double2 p,
                                               const double2* __restrict__ ph, int nt) {
  switch (a) {
    case 0: phase_dfs<0, 0, 1, MODE>(x, p, ph, nt); break;
    case 1: phase_dfs<1, 0, 2, MODE>(x, p, ph, nt); break;
    case 2: phase_dfs<2, 0, 4, MODE>(x, p, ph, nt); break;
    default: phase_dfs<3, 0, 8, MODE>(x, p, ph, nt); break;
  }
}

__device__ __forceinline__ void cp_async16(double2* smem_dst, const double2* gmem_src) {
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// Issue the asynchronous copy of tile `base` into `buf` (16 elements per
// thread).  Element c = t + NT*it: bits [0, K-4) of c come from t, the rest
// from it; all index maps are linear over GF(2), so the per-thread parts are
// XORed with per-iteration parts.
__device__ __forceinline__ void prefetch_tile(const double2* __restrict__ state, double2* buf,
                                              uint64_t base, const svb_sweep_desc& d, int K, int t) {
  uint64_t ld_dev_t = 0;
  uint32_t ld_s_t = 0;
  for (int k = 0; k < K - RB; ++k) {
    if ((t >> k) & 1) {
      ld_dev_t |= uint64_t(1) << d.tin[k];
      ld_s_t ^= (uint32_t)d.sw[k];
    }
  }
#pragma unroll
  for (int it = 0; it < NR; ++it) {
    uint64_t dev = ld_dev_t;
    uint32_t s = ld_s_t;
#pragma unroll
    for (int q = 0; q < RB; ++q) {
      if ((it >> q) & 1) {
        dev |= uint64_t(1) << d.tin[K - RB + q];
        s ^= (uint32_t)d.sw[K - RB + q];
      }
    }
    cp_async16(buf + s, state + (base | dev));
  }
  cp_async_commit();
}

__device__ __forceinline__ uint64_t tile_origin(int64_t tile_id, const SweepArgs& a) {
  uint64_t base = 0, r = (uint64_t)tile_id;
  for (int i = 0; i < a.nf && r; ++i, r >>= 1)
    if (r & 1) base |= uint64_t(1) << a.fbits[i];
  return base;
}

// Persistent: one CTA per SM, tiles strided by gridDim.x; the next tile is
// copied into the second shared buffer while the current one is computed.
__global__ void __launch_bounds__(1 << (SVB_MAX_TILE_BITS_SWEEP - RB), 1)
    k_sweep(double2* __restrict__ state, const SweepArgs args) {
  extern __shared__ __align__(16) double2 smem[];
  __shared__ double red[32];
  const svb_sweep_desc& d = args.d;
  const int K = d.K;
  const int t = threadIdx.x;
  const int NT = 1 << (K - RB);
  double2* bufs[2] = {smem, smem + (1 << K)};
  double2* ctab = smem + (2 << K);

  double nrm = 0.0;
  const int64_t ntiles = int64_t(1) << (d.D - K);
  const svb_op* ops = args.ops;

  int64_t tile_id = blockIdx.x;
  if (tile_id < ntiles) prefetch_tile(state, bufs[0], tile_origin(tile_id, args), d, K, t);

  for (int iter = 0; tile_id < ntiles; ++iter, tile_id += gridDim.x) {
    double2* tile = bufs[iter & 1];
    const uint64_t base = tile_origin(tile_id, args);
    // per-tile phase slots (products of terms over the fixed bits)
    for (int i = t; i < d.nctab; i += NT) {
      double2 acc = one2();
      for (int q = args.cofs[i]; q < args.cofs[i + 1]; ++q) {
        const svb_cterm ct = args.cterms[q];
        if ((base & ct.mask) == ct.mask) acc = cmul(acc, make_double2(ct.re, ct.im));
      }
      ctab[i] = acc;
    }
    cp_async_wait_all();
    __syncthreads();  // tile data + ctab visible; previous tile fully stored
    {
      const int64_t nxt = tile_id + gridDim.x;
      if (nxt < ntiles) prefetch_tile(state, bufs[(iter + 1) & 1], tile_origin(nxt, args), d, K, t);
    }

    double2 x[NR];
    uint32_t sbase = 0;
    uint32_t soff[RB] = {0, 0, 0, 0};
    uint64_t dev_base = base;
    bool live = false;

    for (int oi = 0; oi < d.op_count; ++oi) {
      const svb_op& op = ops[oi];
      const int kind = op.kind;
      if (kind == SVB_OP_STAGE) {
        if (live) {
#pragma unroll
          for (int v = 0; v < NR; ++v) {
            uint32_t s = sbase;
#pragma unroll
            for (int q = 0; q < RB; ++q)
              if ((v >> q) & 1) s ^= soff[q];
            tile[s] = x[v];
          }
          __syncthreads();
        }
        // register slot q <- q-th lowest bit of rmask; thread bit i <- i-th
        // lowest bit of the complement
        const uint32_t rm = op.rmask;
        {
          uint32_t r = rm;
#pragma unroll
          for (int q = 0; q < RB; ++q) {
            soff[q] = (uint32_t)d.sw[__ffs(r) - 1];
            r &= r - 1;
          }
        }
        sbase = 0;
        dev_base = base;
        for (int k = 0, i = 0; k < K; ++k) {
          if (!((rm >> k) & 1)) {
            if ((t >> i) & 1) {
              sbase ^= (uint32_t)d.sw[k];
              dev_base |= uint64_t(1) << d.tin[k];
            }
            ++i;
          }
        }
#pragma unroll
        for (int v = 0; v < NR; ++v) {
          uint32_t s = sbase;
#pragma unroll
          for (int qq = 0; qq < RB; ++qq)
            if ((v >> qq) & 1) s ^= soff[qq];
          x[v] = tile[s];
        }
        live = true;
        continue;
      }
      if ((dev_base & op.pmask) != op.pval) continue;  // thread-uniform predicate
      const double2* cf = args.coef + op.coef;
      switch (kind) {
        case SVB_OP_H:
        case SVB_OP_U1:
        case SVB_OP_PH: {
          const bool has_phase = (kind == SVB_OP_PH) || (op.flags & SVB_F_PHASE);
          if (has_phase) {
            const double2* ph = (kind == SVB_OP_PH) ? cf : cf + 4;
            double2 p = __ldg(ph);
            if (op.ctab >= 0) p = cmul(p, ctab[op.ctab]);
            if (op.tab >= 0) p = cmul(p, __ldg(args.tab + op.tab + t));
            if (op.tf >= 0) {
              for (int i = 0; i < K - RB; ++i)
                if ((t >> i) & 1) p = cmul(p, ctab[op.tf + i]);
            }
            const int nt = (op.flags >> SVB_F_PREG_SHIFT) & 0xF;
            if (kind == SVB_OP_H && op.rmask == 0) {
              phase_dispatch<1>(op.a, x, p, ph, nt);  // pre-phase fused into H
              break;
            }
            phase_dispatch<0>(op.a, x, p, ph, nt);
            if (kind == SVB_OP_PH) break;
          }
          if (kind == SVB_OP_H) {
            switch (op.a) {
              case 0: apply_h<0>(x, op.rmask, (uint32_t)op.b); break;
              case 1: apply_h<1>(x, op.rmask, (uint32_t)op.b); break;
              case 2: apply_h<2>(x, op.rmask, (uint32_t)op.b); break;
              default: apply_h<3>(x, op.rmask, (uint32_t)op.b); break;
            }
          } else {
            const double2 m00 = __ldg(cf), m01 = __ldg(cf + 1), m10 = __ldg(cf + 2),
                          m11 = __ldg(cf + 3);
            switch (op.a) {
              case 0: apply_u1<0>(x, op.rmask, (uint32_t)op.b, m00, m01, m10, m11); break;
              case 1: apply_u1<1>(x, op.rmask, (uint32_t)op.b, m00, m01, m10, m11); break;
              case 2: apply_u1<2>(x, op.rmask, (uint32_t)op.b, m00, m01, m10, m11); break;
              default: apply_u1<3>(x, op.rmask, (uint32_t)op.b, m00, m01, m10, m11); break;
            }
          }
          break;
        }
        case SVB_OP_X:
          switch (op.a) {
            case 0: apply_x<0>(x, op.rmask, (uint32_t)op.b); break;
            case 1: apply_x<1>(x, op.rmask, (uint32_t)op.b); break;
            case 2: apply_x<2>(x, op.rmask, (uint32_t)op.b); break;
            default: apply_x<3>(x, op.rmask, (uint32_t)op.b); break;
          }
          break;
        case SVB_OP_U2:  // host normalises a < b (matrix permuted accordingly)
          switch (op.a * 4 + op.b) {
            case 1: apply_u2<0, 1>(x, op.rmask, cf); break;
            case 2: apply_u2<0, 2>(x, op.rmask, cf); break;
            case 3: apply_u2<0, 3>(x, op.rmask, cf); break;
            case 6: apply_u2<1, 2>(x, op.rmask, cf); break;
            case 7: apply_u2<1, 3>(x, op.rmask, cf); break;
            case 11: apply_u2<2, 3>(x, op.rmask, cf); break;
            default: break;
          }
          break;
        case SVB_OP_PHALL: {
          double2 p = __ldg(cf);
          if (op.ctab >= 0) p = cmul(p, ctab[op.ctab]);
          if (op.tab >= 0) p = cmul(p, __ldg(args.tab + op.tab + t));
          if (op.tf >= 0) {
            for (int i = 0; i < K - RB; ++i)
              if ((t >> i) & 1) p = cmul(p, ctab[op.tf + i]);
          }
#pragma unroll
          for (int v = 0; v < NR; ++v) x[v] = cmul(x[v], p);
          break;
        }
        case SVB_OP_SCALE: {
          const double2 s = __ldg(cf);
#pragma unroll
          for (int v = 0; v < NR; ++v) x[v] = cmul(x[v], s);
          break;
        }
        default:
          break;
      }
    }

    // spill the last stage, then store in output (store-order) mapping
    if (live) {
#pragma unroll
      for (int v = 0; v < NR; ++v) {
        uint32_t s = sbase;
#pragma unroll
        for (int q = 0; q < RB; ++q)
          if ((v >> q) & 1) s ^= soff[q];
        tile[s] = x[v];
      }
    }
    __syncthreads();
    uint64_t st_dev_t = 0;
    uint32_t st_s_t = 0;
    for (int k = 0; k < K - RB; ++k) {
      if ((t >> k) & 1) {
        st_dev_t |= uint64_t(1) << d.st_dev[k];
        st_s_t ^= (uint32_t)d.st_sw[k];
      }
    }
#pragma unroll
    for (int it = 0; it < NR; ++it) {
      uint32_t s = st_s_t;
      uint64_t dev = st_dev_t;
#pragma unroll
      for (int q = 0; q < RB; ++q) {
        if ((it >> q) & 1) {
          dev |= uint64_t(1) << d.st_dev[K - RB + q];
          s ^= (uint32_t)d.st_sw[K - RB + q];
        }
      }
      const double2 v = tile[s];
      nrm = fma(v.x, v.x, fma(v.y, v.y, nrm));
      st_stream(state + (base | (dev ^ d.st_flip)), v);
    }
  }
  cp_async_wait_all();

  if (args.norm_out != nullptr && d.norm_slot >= 0) {
    // block reduction (works for partial warps when NT < 32)
    const unsigned full = NT >= 32 ? 0xffffffffu : ((1u << NT) - 1u);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
      if (o < NT) nrm += __shfl_xor_sync(full, nrm, o);
    const int lane = t & 31, wid = t >> 5;
    __syncthreads();
    if (lane == 0) red[wid] = nrm;
    __syncthreads();
    if (t == 0) {
      double s = 0.0;
      for (int w = 0; w < (NT + 31) / 32; ++w) s += red[w];
      atomicAdd(args.norm_out + d.norm_slot, s);
    }
  }
}

int launch_sweep(double2* state, const SweepArgs& a, int grid_limit, cudaStream_t st) {
  const int K = a.d.K;
  const size_t smem = sizeof(double2) * ((size_t(2) << K) + (size_t)a.d.nctab);
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(
        k_sweep, cudaFuncAttributeMaxDynamicSharedMemorySize,
        (int)(sizeof(double2) * ((size_t(2) << SVB_MAX_TILE_BITS_SWEEP) + kMaxCtab)));
    if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(k_sweep)");
    attr_set = true;
  }
  const int64_t ntiles = int64_t(1) << (a.d.D - K);
  int64_t grid = num_sms();
  if (grid_limit > 0 && grid > grid_limit) grid = grid_limit;
  if (grid > ntiles) grid = ntiles;
  k_sweep<<<(unsigned)grid, 1 << (K - RB), smem, st>>>(state, a);
  SVB_CHECK_LAUNCH("k_sweep");
  return SVB_OK;
}
}  // namespace
}  // namespace svb

using namespace svb;

extern "C" int svb_run_sweeps(svb_c128* state, int64_t rows, int L, const void* prog,
                              const svb_sweep_desc* desc, int nsweeps, double* norm_out,
                              int grid_limit, void* stream) {
  if (rows <= 0 || (rows & (rows - 1))) {
    set_error("rows must be a power of two, got %lld", (long long)rows);
    return SVB_EINVAL;
  }
  int h = 0;
  while ((int64_t(1) << h) < rows) ++h;
  const char* pb = static_cast<const char*>(prog);
  for (int s = 0; s < nsweeps; ++s) {
    const svb_sweep_desc& d = desc[s];
    if (d.rb != RB || d.K < RB || d.K > SVB_MAX_TILE_BITS_SWEEP || d.D != L + h || d.K > d.D ||
        d.D > SVB_MAX_DEV_BITS) {
      set_error("sweep %d: bad geometry K=%d D=%d (L=%d, rows=%lld)", s, d.K, d.D, L,
                (long long)rows);
      return SVB_EINVAL;
    }
    if (d.nctab > kMaxCtab) {
      set_error("sweep %d: %d per-tile slots exceed 512", s, d.nctab);
      return SVB_ERANGE;
    }
    SweepArgs a;
    a.d = d;
    a.ops = reinterpret_cast<const svb_op*>(pb + d.ops_off) + d.op_begin;
    a.coef = reinterpret_cast<const double2*>(pb + d.coef_off);
    a.tab = reinterpret_cast<const double2*>(pb + d.tab_off);
    a.cterms = reinterpret_cast<const svb_cterm*>(pb + d.cterm_off);
    a.cofs = reinterpret_cast<const int32_t*>(pb + d.cofs_off);
    a.norm_out = norm_out;
    uint64_t tmask = 0;
    for (int k = 0; k < d.K; ++k) {
      if (d.tin[k] < 0 || d.tin[k] >= d.D || (tmask >> d.tin[k] & 1)) {
        set_error("sweep %d: bad tile bit map", s);
        return SVB_EINVAL;
      }
      tmask |= uint64_t(1) << d.tin[k];
    }
    a.nf = 0;
    for (int b = 0; b < d.D; ++b)
      if (!(tmask >> b & 1)) a.fbits[a.nf++] = b;
    int rc = launch_sweep(reinterpret_cast<double2*>(state), a, grid_limit, as_stream(stream));
    if (rc) return rc;
  }
  return SVB_OK;
}
