/*
 * sv_oracle.c -- CPU restatement of the reference's compiled gate kernels.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker (and the
 * "port" CPU baseline of bench.py); nothing in paper_2509_14098_b200/ links,
 * loads or calls it.
 *
 * Restates svpart/kernels/_core.pyx (the only native code of the
 * reference):
 *   apply_gate      _core.pyx:7-60   in-place y = U x over every 2^p-amp
 *                                    group of every rank row
 *   apply_diagonal  _core.pyx:63-106 in-place x *= diag[t]
 * Conventions (_core.pyx:22-38): `bits` are local positions, 0 = MSB of the
 * local index, given in gate-slot order; slot i addresses matrix index bit
 * p-1-i; group bases come from inserting zeros at the ascending LSB
 * positions.  The arithmetic (complex multiply-add in slot order, row by
 * row) follows the reference loop so results agree to float rounding.
 *
 * Unlike the reference (single thread, _core.pyx:46), the group loop can be
 * spread over OpenMP threads (`nthreads`); results do not depend on it.
 */
#include <complex.h>
#include <stdint.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef double complex cplx;

static int log2_len(int64_t n) {
  int L = 0;
  while (((int64_t)1 << L) < n) ++L;
  return L;
}

/* zero-insertion order and per-slot strides (_core.pyx:22-38) */
static void geometry(const int64_t* bits, int p, int L, int64_t* ibit, int64_t* ins, int64_t* offs) {
  for (int i = 0; i < p; ++i) {
    ibit[i] = L - 1 - bits[i];
    ins[i] = ibit[i];
  }
  for (int i = 1; i < p; ++i)
    for (int j = i; j > 0 && ins[j] < ins[j - 1]; --j) {
      int64_t t = ins[j];
      ins[j] = ins[j - 1];
      ins[j - 1] = t;
    }
  for (int t = 0; t < (1 << p); ++t) {
    offs[t] = 0;
    for (int i = 0; i < p; ++i)
      if ((t >> (p - 1 - i)) & 1) offs[t] += (int64_t)1 << ibit[i];
  }
}

static inline int64_t base_of(int64_t k, const int64_t* ins, int p) {
  for (int i = 0; i < p; ++i) {
    int64_t low = ((int64_t)1 << ins[i]) - 1;
    k = ((k & ~low) << 1) | (k & low);
  }
  return k;
}

/* returns 0 on success, 1 on a width/shape error (the reference's ValueError) */
int orc_apply_gate(cplx* blocks, int64_t ranks, int64_t n, const cplx* matrix, int64_t dim,
                   const int64_t* bits, int p, int nthreads) {
  if (p > 6 || dim != ((int64_t)1 << p)) return 1;
  const int L = log2_len(n);
  int64_t ibit[6], ins[6], offs[64];
  geometry(bits, p, L, ibit, ins, offs);
  const int D = 1 << p;
  const int64_t groups = n >> p;
  const int64_t total = ranks * groups;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(static) if (nthreads > 1)
#endif
  for (int64_t w = 0; w < total; ++w) {
    const int64_t r = w / groups, k = w - r * groups;
    cplx* row = blocks + r * n;
    const int64_t base = base_of(k, ins, p);
    cplx xs[64], ys[64];
    for (int t = 0; t < D; ++t) xs[t] = row[base + offs[t]];
    for (int t = 0; t < D; ++t) {
      cplx acc = 0;
      for (int j = 0; j < D; ++j) acc = acc + matrix[t * D + j] * xs[j];
      ys[t] = acc;
    }
    for (int t = 0; t < D; ++t) row[base + offs[t]] = ys[t];
  }
  return 0;
}

int orc_apply_diagonal(cplx* blocks, int64_t ranks, int64_t n, const cplx* diag, int64_t dim,
                       const int64_t* bits, int p, int nthreads) {
  if (p > 6 || dim != ((int64_t)1 << p)) return 1;
  const int L = log2_len(n);
  int64_t ibit[6], ins[6], offs[64];
  geometry(bits, p, L, ibit, ins, offs);
  const int D = 1 << p;
  const int64_t groups = n >> p;
  const int64_t total = ranks * groups;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(static) if (nthreads > 1)
#endif
  for (int64_t w = 0; w < total; ++w) {
    const int64_t r = w / groups, k = w - r * groups;
    cplx* row = blocks + r * n;
    const int64_t base = base_of(k, ins, p);
    for (int t = 0; t < D; ++t) row[base + offs[t]] = row[base + offs[t]] * diag[t];
  }
  return 0;
}
