/*
 * svb200.h -- C ABI of the B200 state-vector executor (libsvb200.so).
 *
 * Plain pointers and sizes only: no torch / Python types cross this line.
 * Every state pointer is DEVICE memory holding complex128 amplitudes
 * (interleaved re, im doubles), laid out exactly like the reference's
 * `blocks` array: row r = rank r's block of 2^L amplitudes, local bit b
 * (0 = most significant) has stride 2^(L-1-b)  (svpart/plan.py:3-8,
 * svpart/kernels/numpy_backend.py:3-4).
 *
 * All calls are asynchronous on the given CUDA stream (a cudaStream_t passed
 * as void*; NULL = legacy default stream) and return SVB_OK or an error
 * code; svb_last_error() gives the message of the last failure on the
 * calling thread.  Nothing here allocates device memory: scratch is passed
 * in by the caller.
 *
 * Which reference interface each entry point replaces is cited per function.
 */
#ifndef SVB200_H
#define SVB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SVB_OK 0
#define SVB_EINVAL 1 /* bad width / shape: the reference raises ValueError   */
#define SVB_ECUDA 2  /* CUDA launch or runtime failure                       */
#define SVB_ERANGE 3 /* size outside what the kernel supports                */

typedef struct svb_c128 {
  double re, im;
} svb_c128;

/* Library identity and last error (thread-local). */
int svb_abi_version(void);
const char* svb_last_error(void);
/* sizeof(svb_op), sizeof(svb_cterm), sizeof(svb_sweep_desc): lets a binding
 * check its struct mirrors against the compiled library. */
void svb_abi_sizes(size_t* op, size_t* cterm, size_t* desc);

/* ------------------------------------------------------------------------
 * 1. Inner kernel plugin: in-place gate application on (ranks, 2^L) blocks.
 *
 * Replaces svpart.kernels._core.apply_gate / apply_diagonal
 * (svpart/kernels/_core.pyx:7-9 and :63-65; dispatcher
 * svpart/kernels/__init__.py:39-60).  `bits` are local bit positions in
 * gate-slot order (0 = MSB of the local index); slot i addresses matrix
 * index bit p-1-i.  `matrix` / `diag` are DEVICE pointers (dim x dim row
 * major / dim entries).  Returns SVB_EINVAL when dim != 2^p, a bit is out
 * of range or repeated, or p exceeds max_width (the reference's compiled
 * core uses max_width = 6, _core.pyx:14-15).
 * ---------------------------------------------------------------------- */
int svb_apply_gate(svb_c128* blocks, int64_t ranks, int64_t n,
                   const svb_c128* matrix, int64_t dim,
                   const int64_t* bits, int p, int max_width, void* stream);

int svb_apply_diagonal(svb_c128* blocks, int64_t ranks, int64_t n,
                       const svb_c128* diag, int64_t dim,
                       const int64_t* bits, int p, int max_width, void* stream);

/* ------------------------------------------------------------------------
 * 2. Fused leaf sweeps: one ApplyFused task (svpart/executor.py:215-222,
 *    _apply_fused :123-176) as one or more HBM sweeps.
 *
 * A sweep reads every amplitude of the device-resident rows once, applies a
 * compiled gate program to 2^K-amplitude tiles in shared memory/registers
 * and writes them back once.  The program (ops, coefficients, per-thread
 * phase tables, per-tile phase terms) is built on the host by
 * paper_2509_14098_b200/program.py and lives in device memory at `prog`.
 * `desc` is a HOST array of `nsweeps` descriptors.  If `norm_out` is not
 * NULL, the sum of |amp|^2 over the state after each sweep is ADDED to
 * norm_out[desc[i].norm_slot] (the reference's drift check,
 * executor.py:220-222).
 * ---------------------------------------------------------------------- */
#define SVB_MAX_TILE_BITS 13
#define SVB_MAX_DEV_BITS 40
#define SVB_REG_BITS 4

typedef struct svb_op {
  int32_t kind;   /* SVB_OP_*                                                */
  int32_t a, b;   /* register slots (0..3)                                   */
  uint32_t rmask; /* STAGE: tile-local register bits; else register ctl mask */
  uint64_t pmask; /* thread-uniform predicate (dev_base & pmask) == pval     */
  uint64_t pval;
  int32_t coef;   /* offset (complex units) into the coefficient pool         */
  int32_t tab;    /* offset of a 2^(K-4)-entry per-thread table, or -1        */
  int32_t ctab;   /* per-tile scalar slot, or -1                              */
  int32_t tf;     /* first of K-4 per-tile per-thread-bit slots, or -1        */
  int32_t flags;  /* SVB_F_*                                                  */
  int32_t pad[3];
} svb_op;

enum {
  SVB_OP_STAGE = 1, /* spill registers to smem, reload with new rmask        */
  SVB_OP_U1 = 2,    /* 2x2 on slot a (+ optional pre-phase)                  */
  SVB_OP_H = 3,     /* unscaled Hadamard on slot a (+ optional pre-phase)    */
  SVB_OP_X = 4,     /* bit flip on slot a                                    */
  SVB_OP_U2 = 5,    /* 4x4 on slots (a, b); a is the matrix MSB              */
  SVB_OP_PH = 6,    /* phase on amplitudes whose slot-a bit is 1             */
  SVB_OP_PHALL = 7, /* thread-uniform phase on all register amplitudes       */
  SVB_OP_SCALE = 8  /* multiply every amplitude by coef[0]                   */
};

enum {
  SVB_F_PHASE = 1,     /* U1/H: apply the pre-phase before the gate          */
  SVB_F_PREG_SHIFT = 4 /* bits 4..7: register slots with a non-unit factor   */
};

typedef struct svb_cterm { /* ctab[dst] *= c  if (tile_base & mask) == mask */
  int32_t dst;
  int32_t pad;
  uint64_t mask;
  double re, im;
} svb_cterm;

typedef struct svb_sweep_desc {
  int32_t K;                            /* tile bits (4..13)                  */
  int32_t D;                            /* device index bits (L + log2 rows)  */
  int32_t tin[SVB_MAX_TILE_BITS];       /* tile bit k -> device bit (load)    */
  int32_t sw[SVB_MAX_TILE_BITS];        /* smem swizzle image of tile bit k   */
  int32_t st_dev[SVB_MAX_TILE_BITS];    /* store-order bit i -> device bit    */
  int32_t st_sw[SVB_MAX_TILE_BITS];     /* store-order bit i -> swizzle image */
  uint64_t st_flip;                     /* device bits inverted at store      */
  int32_t op_begin, op_count;           /* ops [op_begin, op_begin+op_count)  */
  int32_t nctab;                        /* per-tile scalar slots              */
  int32_t norm_slot;                    /* -1: no norm accumulation           */
  int32_t rb;                           /* register bits per thread (2^(K-rb) threads) */
  int32_t groups;                       /* generated kernels: tile groups per CTA
                                           (0/1: one; 2: 2^(K-rb+1) threads) */
  int64_t ops_off, coef_off, tab_off;   /* byte offsets into prog             */
  int64_t cterm_off, cofs_off;          /* per-tile terms + CSR offsets       */
} svb_sweep_desc;

int svb_run_sweeps(svb_c128* state, int64_t rows, int L, const void* prog,
                   const svb_sweep_desc* desc, int nsweeps, double* norm_out,
                   int grid_limit, void* stream);

/* ------------------------------------------------------------------------
 * 3. Qubit remap and layout kernels.
 *
 * svb_bitswap: in-place exchange of device-index bits u[i] <-> w[i]
 *   (index bits counted from the LSB of row*2^L + local).  This is
 *   Pack -> Exchange -> Unpack (executor.py:224-281) when every rank of the
 *   swap group lives on this device.
 * svb_pack_region / svb_unpack_region: copy the sub-block of every row whose
 *   local bits `lbits` (LSB-indexed) read `sel` into / out of a contiguous
 *   buffer, elements [off, off+count) of the region in enumeration order.
 *   Used around the NCCL exchange between devices.
 * svb_bitperm: out-of-place dst[P(f)] = src[f] where bit k of f moves to
 *   bit perm[k]; gather/scatter by _storage_to_basis (executor.py:310-343).
 * ---------------------------------------------------------------------- */
int svb_bitswap(svb_c128* state, int D, const int32_t* u, const int32_t* w,
                int m, void* stream);

int svb_pack_region(const svb_c128* state, int64_t rows, int L,
                    const int32_t* lbits, int m, uint32_t sel, int64_t off,
                    int64_t count, svb_c128* out, void* stream);

int svb_unpack_region(svb_c128* state, int64_t rows, int L,
                      const int32_t* lbits, int m, uint32_t sel, int64_t off,
                      int64_t count, const svb_c128* in, void* stream);

int svb_bitperm(const svb_c128* src, svb_c128* dst, int nbits,
                const int32_t* perm, void* stream);

/* ------------------------------------------------------------------------
 * 4. Reductions (executor.py:220 norm; compare :361-372).
 *
 * svb_norm2: out[0] += sum |x|^2 (out is a device double).
 * svb_compare: out[0] = max |a - phi*b| with phi aligned at argmax |a||b|;
 *   scratch must hold svb_compare_scratch_bytes(n) bytes of device memory.
 * ---------------------------------------------------------------------- */
int svb_norm2(const svb_c128* x, int64_t n, double* out, void* stream);

size_t svb_compare_scratch_bytes(int64_t n);
int svb_compare(const svb_c128* a, const svb_c128* b, int64_t n, double* out,
                void* scratch, void* stream);

/* Distributed compare (one shard per process, executor.py:361-372):
 * svb_shard_argmax: over shard elements i (storage index base + i), the
 *   largest |a_i||b_i|, ties to the smallest basis index, where perm[s] is
 *   the basis bit of storage bit s (nbits bits).  out[0] = weight,
 *   out[1] = basis index (int64 bits), out[2], out[3] = a_k conj(b_k).
 * svb_shard_maxdev: out[0] = max_i |a_i - phi b_i|.
 * Both need svb_shard_scratch_bytes(n) bytes of device scratch. */
size_t svb_shard_scratch_bytes(int64_t n);
int svb_shard_argmax(const svb_c128* a, const svb_c128* b, int64_t n, uint64_t base, int nbits,
                     const int32_t* perm, double* out, void* scratch, void* stream);
int svb_shard_maxdev(const svb_c128* a, const svb_c128* b, int64_t n, double phi_re, double phi_im,
                     double* out, void* scratch, void* stream);

/* Device sampling: section 7 (numpy-identical CDF). */

/* ------------------------------------------------------------------------
 * 5. Run-time specialised sweep kernels (paper_2509_14098_b200/jit.py).
 *
 * svb_jit_compile: NVRTC-compile CUDA source for sm_100a into a cubin
 *   (malloc'd, release with svb_jit_free); `log` receives the compiler log.
 * svb_jit_load: load a cubin and return a launchable kernel handle.
 * svb_jit_launch_sweep: launch a generated sweep kernel on one sweep
 *   descriptor (same program blob and descriptor as svb_run_sweeps).
 * ---------------------------------------------------------------------- */
int svb_jit_compile(const char* src, const char* name, int nopts, const char** opts,
                    void** image, size_t* size, char* log, size_t logcap);
void svb_jit_free(void* image);
int svb_jit_load(const void* image, const char* kernel_name, void** kernel);
int svb_jit_launch_sweep(void* kernel, svb_c128* state, const void* prog,
                         const svb_sweep_desc* desc, double* norm_out, int grid_limit,
                         void* stream);
/* Part launch: only the tiles whose chunk bits (compiled into the kernel)
 * read part_val (device-index bits); part_tid is the same value in
 * tile-index coordinates, ntiles the number of tiles in the part.  Lets a
 * sweep run in parts that overlap a remap on another stream. */
int svb_jit_launch_sweep_part(void* kernel, svb_c128* state, const void* prog,
                              const svb_sweep_desc* desc, double* norm_out, int grid_limit,
                              uint64_t part_val, uint64_t part_tid, int64_t ntiles,
                              void* stream);

/* ------------------------------------------------------------------------
 * 6. Peer-memory remap (paper_2509_14098_b200/comm.py), replacing the
 *    inter-GPU Pack -> Exchange -> Unpack of svpart/executor.py:224-281.
 *
 * svb_dev_alloc / svb_dev_free: plain cudaMalloc'd state storage that can
 *   be shared with the other processes of the job.
 * svb_ipc_handle: the 64-byte CUDA IPC handle of an svb_dev_alloc pointer;
 *   svb_ipc_open maps a peer's handle into this process (svb_ipc_close).
 * svb_peer_swap: in-place pairwise swap with npeers peers.  The m local
 *   bits lbits[0..m) select regions; for peer j, pairs
 *   k in [first[j], first[j]+count[j]) of local region sel_local[j] and the
 *   peer's region sel_remote[j] (selector bit m-1-i <-> lbits[i]) are
 *   exchanged.  k enumerates rows (outer) then the free local bits in
 *   ascending order, like svb_pack_region.  The two processes of a pair
 *   must split the k range between them and order the launch between
 *   cross-process barriers.  grid_limit caps the CTAs per peer (0: fill the
 *   GPU), block is the CTA size (0: 256); a small grid of 1024-thread CTAs
 *   leaves the other SMs to sweeps running concurrently.
 * ---------------------------------------------------------------------- */
int svb_dev_alloc(size_t bytes, void** ptr);
int svb_dev_free(void* ptr);
int svb_ipc_handle(void* ptr, void* handle64);
int svb_ipc_open(const void* handle64, void** ptr);
int svb_ipc_close(void* ptr);
/* svb_peer_swap_bulk: the same swap driven by the bulk-copy (TMA) engine:
 *   `grid` persistent CTAs of one warp, each a ring of `stages` shared-memory
 *   stages of 2 x piece_bytes (power of two), `ahead` of them loading
 *   (0: stages - 2) while the rest store; leaves the other SMs' compute
 *   free, so a remap can run beside the sweeps. */
int svb_peer_swap_bulk(svb_c128* local, void* const* peers, int npeers, int64_t rows, int L,
                       const int32_t* lbits, int m, const uint64_t* sel_local,
                       const uint64_t* sel_remote, const int64_t* first, const int64_t* count,
                       int grid, int piece_bytes, int stages, int ahead, void* stream);
/* Stream-ordered 32-bit flags (cuStreamWriteValue32 / cuStreamWaitValue32):
 *   write `value` to addr (own or a mapped peer's device memory) after all
 *   earlier work of the stream; or hold the stream until *addr >= value. */
int svb_stream_write_u32(void* addr, uint32_t value, void* stream);
int svb_stream_wait_u32(void* addr, uint32_t value, void* stream);
/* svb_stream_create: a non-blocking CUDA stream on the current device for
 *   one purpose (uploads, downloads, overlapped remap chunks); never freed.
 *   Dedicated handles never alias each other or torch's pooled streams. */
int svb_stream_create(void** stream);
/* ------------------------------------------------------------------------
 * 7. numpy-identical sampling (paper_2509_14098_b200/sampling.py), replacing
 *    svpart/executor.py:375-383 (probs = |psi|^2 / sum; rng.choice(p=probs)).
 *
 * svb_probs_numpy: |a|^2 of a shard with numpy's complex absolute value,
 *   written in basis-sorted shard order (perm: storage bit -> sorted bit).
 * svb_deposit_scatter: dst[deposit(i, dst_bits) | or_val] = src[i].
 * svb_pairwise_sum: numpy's pairwise sum of 2^D doubles into *out.
 * svb_div_scalar: x[i] /= *denom (device scalar).
 * svb_cdf_chunk_totals / svb_cdf_walk: the exact sequential cumsum of n
 *   doubles at every chunk end (svb_cdf_chunk_elems() elements per chunk),
 *   from the exact start *c_in; cstart holds approximate chunk starts.
 * svb_cdf_search: per shot the first element whose fl(c / c_last) exceeds
 *   u (numpy searchsorted side="right"), over the chunk ends of all
 *   processes; out[s] = global index, or -1 if another process owns it.
 * ---------------------------------------------------------------------- */
int64_t svb_cdf_chunk_elems(void);
int svb_probs_numpy(const svb_c128* shard, int D, const int32_t* perm, double* out, void* stream);
int svb_deposit_scatter(const double* src, int64_t n, int nbits, const int32_t* dst_bits, uint64_t or_val,
                        double* dst, void* stream);
size_t svb_pairwise_scratch_bytes(int D);
int svb_pairwise_sum(const double* x, int D, double* out, void* scratch, void* stream);
int svb_div_scalar(double* x, int64_t n, const double* denom, void* stream);
size_t svb_cdf_scratch_bytes(int64_t n);
int svb_cdf_chunk_totals(const double* q, int64_t n, double* tot, void* stream);
int svb_cdf_walk(const double* q, int64_t n, const double* cstart, const double* tot, void* fn_scratch,
                 const double* c_in, double* cend, long long* nslow, void* stream);
int svb_cdf_search(const double* q, int64_t n, const double* cend_all, int64_t nchunks_all, int64_t my_lo,
                   int64_t my_hi, double c_last, const double* u, int64_t nshots, int64_t index_base,
                   int64_t* out, void* stream);
/* svb_region_move: in place, region dst_sel of the m local bits lbits
 *   (selector bit m-1-i <-> lbits[i], like svb_pack_region) takes the
 *   amplitudes of region src_sel: the remap after a replicated sparse prefix
 *   (program.localize_applies), which moves no data between GPUs. */
int svb_region_move(svb_c128* state, int nbits, const int32_t* lbits, int m, uint32_t src_sel, uint32_t dst_sel,
                    void* stream);
/* svb_gather_bits: dst[t] = src[P(base + t)], t < count, with
 *   P(f) = sum_k bit_k(f) << perm[k] (one chunk of a permuted order: the
 *   chunked gather of a sharded state, svpart/executor.py:310-326). */
int svb_gather_bits(const svb_c128* src, int nbits, const int32_t* perm, uint64_t base, int64_t count,
                    svb_c128* dst, void* stream);
/* svb_copy: n-amplitude SM copy; either pointer may be a mapped peer's. */
int svb_copy(svb_c128* dst, const svb_c128* src, int64_t n, int grid_limit, void* stream);
int svb_peer_swap(svb_c128* local, void* const* peers, int npeers, int64_t rows, int L,
                  const int32_t* lbits, int m, const uint64_t* sel_local,
                  const uint64_t* sel_remote, const int64_t* first, const int64_t* count,
                  int grid_limit, int block, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SVB200_H */
