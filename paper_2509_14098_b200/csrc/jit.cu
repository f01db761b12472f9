// Runtime specialisation of sweep kernels.
//
// The host compiler (program.py) turns each sweep into a short op list; for
// large states jit.py renders that list as straight-line CUDA (compile-time
// register slots, literal coefficients, precomputed index bases) and this
// file compiles it with NVRTC for sm_100a, loads the cubin with the runtime's
// library API and launches it.  This is the paper's code-generation path
// (a kernel per partition) done at run time on the B200 host.
//
// NVRTC is opened with dlopen on first use so the library still loads on
// hosts without it (the build container checks symbol exports only).
#include <dlfcn.h>
#include <stdlib.h>
#include <string.h>

#include "common.cuh"

namespace svb {
namespace {

typedef int nvrtcResult_;
typedef struct _nvrtcProgram* nvrtcProgram_;
struct Nvrtc {
  nvrtcResult_ (*create)(nvrtcProgram_*, const char*, const char*, int, const char* const*,
                         const char* const*);
  nvrtcResult_ (*compile)(nvrtcProgram_, int, const char* const*);
  nvrtcResult_ (*cubin_size)(nvrtcProgram_, size_t*);
  nvrtcResult_ (*cubin)(nvrtcProgram_, char*);
  nvrtcResult_ (*log_size)(nvrtcProgram_, size_t*);
  nvrtcResult_ (*log)(nvrtcProgram_, char*);
  nvrtcResult_ (*destroy)(nvrtcProgram_*);
  const char* (*errstr)(nvrtcResult_);
  bool ok = false;
};

Nvrtc& nvrtc() {
  static Nvrtc n;
  static bool tried = false;
  if (tried) return n;
  tried = true;
  const char* names[] = {"libnvrtc.so.12", "libnvrtc.so", "/usr/local/cuda/lib64/libnvrtc.so.12"};
  void* h = nullptr;
  for (const char* nm : names)
    if ((h = dlopen(nm, RTLD_NOW | RTLD_LOCAL))) break;
  if (!h) return n;
#define SVB_SYM(f, s) n.f = reinterpret_cast<decltype(n.f)>(dlsym(h, s))
  SVB_SYM(create, "nvrtcCreateProgram");
  SVB_SYM(compile, "nvrtcCompileProgram");
  SVB_SYM(cubin_size, "nvrtcGetCUBINSize");
  SVB_SYM(cubin, "nvrtcGetCUBIN");
  SVB_SYM(log_size, "nvrtcGetProgramLogSize");
  SVB_SYM(log, "nvrtcGetProgramLog");
  SVB_SYM(destroy, "nvrtcDestroyProgram");
  SVB_SYM(errstr, "nvrtcGetErrorString");
#undef SVB_SYM
  n.ok = n.create && n.compile && n.cubin_size && n.cubin && n.log_size && n.log && n.destroy;
  return n;
}

}  // namespace
}  // namespace svb

using namespace svb;

extern "C" int svb_jit_compile(const char* src, const char* name, int nopts, const char** opts,
                               void** image, size_t* size, char* log, size_t logcap) {
  Nvrtc& nv = nvrtc();
  if (!nv.ok) {
    set_error("NVRTC not available (dlopen libnvrtc.so.12 failed)");
    return SVB_ECUDA;
  }
  nvrtcProgram_ prog = nullptr;
  if (nv.create(&prog, src, name, 0, nullptr, nullptr) != 0) {
    set_error("nvrtcCreateProgram failed");
    return SVB_ECUDA;
  }
  const int rc = nv.compile(prog, nopts, opts);
  if (log && logcap) {
    size_t ls = 0;
    nv.log_size(prog, &ls);
    char* buf = static_cast<char*>(malloc(ls + 1));
    nv.log(prog, buf);
    buf[ls] = 0;
    strncpy(log, buf, logcap - 1);
    log[logcap - 1] = 0;
    free(buf);
  }
  if (rc != 0) {
    set_error("NVRTC compile of %s failed: %s", name, nv.errstr ? nv.errstr(rc) : "?");
    nv.destroy(&prog);
    return SVB_EINVAL;
  }
  size_t n = 0;
  nv.cubin_size(prog, &n);
  void* out = malloc(n);
  nv.cubin(prog, static_cast<char*>(out));
  nv.destroy(&prog);
  *image = out;
  *size = n;
  return SVB_OK;
}

extern "C" void svb_jit_free(void* image) { free(image); }

extern "C" int svb_jit_load(const void* image, const char* kernel_name, void** kernel) {
  cudaLibrary_t lib;
  cudaError_t e = cudaLibraryLoadData(&lib, image, nullptr, nullptr, 0, nullptr, nullptr, 0);
  if (e != cudaSuccess) return cuda_status(e, "cudaLibraryLoadData");
  cudaKernel_t k;
  e = cudaLibraryGetKernel(&k, lib, kernel_name);
  if (e != cudaSuccess) return cuda_status(e, "cudaLibraryGetKernel");
  e = cudaFuncSetAttribute(reinterpret_cast<const void*>(k),
                           cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(jit)");
  // keep every SM at the full shared-memory carveout so a remap kernel can
  // share the SM with a running sweep (csrc/peer.cu)
  e = cudaFuncSetAttribute(reinterpret_cast<const void*>(k),
                           cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(jit carveout)");
  *kernel = reinterpret_cast<void*>(k);
  return SVB_OK;
}

// Launch a generated sweep kernel: one CTA per SM (persistent), 2^(K-rb)
// threads, three rotating tile buffers plus per-tile slots of dynamic
// shared memory.  A "part" launch covers only the tiles whose chunk bits
// (compiled into the kernel) read part_val; ntiles counts those tiles and
// part_tid is part_val in tile-index coordinates (per-tile slot tables).
extern "C" int svb_jit_launch_sweep_part(void* kernel, svb_c128* state, const void* prog,
                                         const svb_sweep_desc* desc, double* norm_out,
                                         int grid_limit, uint64_t part_val, uint64_t part_tid,
                                         int64_t ntiles, void* stream) {
  const svb_sweep_desc& d = *desc;
  const char* pb = static_cast<const char*>(prog);
  const double2* tab = reinterpret_cast<const double2*>(pb + d.tab_off);
  const svb_cterm* ct = reinterpret_cast<const svb_cterm*>(pb + d.cterm_off);
  const int32_t* cofs = reinterpret_cast<const int32_t*>(pb + d.cofs_off);
  double2* st = reinterpret_cast<double2*>(state);
  double* nrm = (norm_out && d.norm_slot >= 0) ? norm_out + d.norm_slot : nullptr;
  long long nt = ntiles;
  void* args[] = {&st, &tab, &ct, &cofs, &nrm, &part_val, &part_tid, &nt};
  int64_t grid = num_sms();
  if (grid_limit > 0 && grid > grid_limit) grid = grid_limit;
  if (grid > ntiles) grid = ntiles;
  if (grid <= 0) return SVB_OK;
  // 3 tile buffers + per-tile slots double-buffered by tile parity
  const size_t smem = sizeof(double2) * ((size_t(3) << d.K) + 2 * (size_t)(d.nctab > 0 ? d.nctab : 1));
  if (smem > 220 * 1024) {
    set_error("jit sweep: %zu bytes of shared memory exceed the 220 KB budget", smem);
    return SVB_ERANGE;
  }
  const unsigned groups = d.groups > 1 ? (unsigned)d.groups : 1u;
  cudaError_t e = cudaLaunchKernel(reinterpret_cast<const void*>(kernel), dim3((unsigned)grid),
                                   dim3(groups << (d.K - d.rb)), args, smem, as_stream(stream));
  if (e != cudaSuccess) return cuda_status(e, "jit sweep launch");
  return SVB_OK;
}

extern "C" int svb_jit_launch_sweep(void* kernel, svb_c128* state, const void* prog,
                                    const svb_sweep_desc* desc, double* norm_out, int grid_limit,
                                    void* stream) {
  return svb_jit_launch_sweep_part(kernel, state, prog, desc, norm_out, grid_limit, 0, 0,
                                   int64_t(1) << (desc->D - desc->K), stream);
}
