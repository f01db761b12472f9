// Device helpers for NVRTC-generated sweep kernels (see jit.py).  Self
// contained: NVRTC compiles it without the CUDA runtime headers.
#pragma once

typedef unsigned long long u64;
typedef unsigned int u32;

struct svb_cterm {
  int dst;
  int pad;
  u64 mask;
  double re, im;
};

#define SVB_F __device__ __forceinline__

SVB_F double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// a * (cr + i ci) with literal parts
SVB_F double2 cmulc(double2 a, double cr, double ci) {
  return make_double2(fma(a.x, cr, -a.y * ci), fma(a.x, ci, a.y * cr));
}
SVB_F double2 cmulr(double2 a, double cr) { return make_double2(a.x * cr, a.y * cr); }
// acc + a * (cr + i ci)
SVB_F double2 cfmac(double2 a, double cr, double ci, double2 acc) {
  return make_double2(fma(a.x, cr, fma(-a.y, ci, acc.x)), fma(a.x, ci, fma(a.y, cr, acc.y)));
}
// acc + a * cr and acc + a * (i ci): real or imaginary literals (rx, ry, sqrt-X
// blocks) need two FMAs, not four
SVB_F double2 cfmar(double2 a, double cr, double2 acc) { return make_double2(fma(a.x, cr, acc.x), fma(a.y, cr, acc.y)); }
SVB_F double2 cfmai(double2 a, double ci, double2 acc) { return make_double2(fma(-a.y, ci, acc.x), fma(a.x, ci, acc.y)); }
SVB_F double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
SVB_F double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }

SVB_F void cp_async16(double2* smem_dst, const double2* gmem_src) {
  const u32 sa = (u32)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem_src) : "memory");
}
// zero-fill forms (src-size 0 reads no global memory; the address stays valid)
SVB_F void cp_async16_zero(double2* smem_dst, const double2* any_gmem) {
  const u32 sa = (u32)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, 0;" ::"r"(sa), "l"(any_gmem) : "memory");
}
SVB_F void cp_async16_pred(double2* smem_dst, const double2* gmem_src, bool live, const double2* any_gmem) {
  const u32 sa = (u32)__cvta_generic_to_shared(smem_dst);
  const u32 n = live ? 16u : 0u;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(live ? gmem_src : any_gmem), "r"(n)
               : "memory");
}
SVB_F void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
SVB_F void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
SVB_F void st_stream(double2* p, double2 v) {
  asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
}

// ---- two tile groups per CTA (jit.kernel_source_2g) ------------------------
// mbarriers track the cp.async loads of each tile buffer: every thread of the
// loading group arrives (noinc) once its prior cp.asyncs have landed, so the
// barrier's count is the group size and the consuming group waits on the
// phase parity of the buffer's use.
SVB_F u32 smem_addr(const void* p) { return (u32)__cvta_generic_to_shared(p); }
SVB_F void mbar_init(unsigned long long* bar, u32 count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
SVB_F void mbar_init_fence() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
SVB_F void cp_async_mbar_arrive(unsigned long long* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_addr(bar)) : "memory");
}
SVB_F void mbar_wait_parity(unsigned long long* bar, u32 parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
// named barrier of one tile group (id 0 is __syncthreads)
SVB_F void bar_group(u32 id, u32 nthreads) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory"); }
