// FP64 tensor-core (DMMA m8n8k4) block product used by K3: one warp's share
// of y = A x for an (8*MT)-row, (8*NT)-RHS tile over a K range.  Shared by
// ds_solve.cu and tools/product_micro.cu.
#pragma once
#include "ds_common.cuh"

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// ---- cp.async staging helpers (K3m-T transforms, K2b trailing updates)
__device__ __forceinline__ uint32_t smem_addr(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
// 16-byte async copy; src_bytes = 0 zero-fills the destination
__device__ __forceinline__ void cp16(void *dst, const void *src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_addr(dst)), "l"(src),
               "r"(src_bytes)
               : "memory");
}
// the same with a shared-memory byte address
__device__ __forceinline__ void cp16s(uint32_t dst, const void *src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(src_bytes)
               : "memory");
}
// DMMA without `volatile`: the scheduler may move it across the cp.async
// issue of the same loop iteration (its operands are registers only)
__device__ __forceinline__ void dmma_nv(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// One warp's share of y = A x for an (8*MT)-row, (8*NT)-RHS tile over
// k-steps [kb, ke) of 4 columns: complex product as four real m8n8k4 DMMAs
// (re*re - im*im, re*im + im*re).  Fragments of step kq+1 are loaded into
// registers before the DMMAs of step kq issue, hiding shared-memory latency.
// X2 (the middle block's second input) is added while loading.
template <int MT, int NT, bool HX2>
__device__ __forceinline__ void mma_product(const cplx *__restrict__ A, int lda,
                                            const cplx *__restrict__ X, const cplx *__restrict__ X2,
                                            int rg, int m, int kb, int ke, int g, int tg,
                                            double (&cr)[2][2][2], double (&ci)[2][2][2]) {
  if (kb >= ke) return;
  cplx a[MT], b[NT], an[MT], bn[NT];
  auto load = [&](int kq, cplx(&aa)[MT], cplx(&bb)[NT]) {
    const int kk = kq * 4 + tg;
    const bool kin = kk < m;
    const int kc = kin ? kk : 0;  // clamped address, value zeroed below
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      cplx v = X[kc * rg + nt * 8 + g];
      if (HX2) v = cadd(v, X2[kc * rg + nt * 8 + g]);
      bb[nt] = kin ? v : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      cplx v = A[(mt * 8 + g) * lda + kc];
      aa[mt] = kin ? v : make_double2(0.0, 0.0);
    }
  };
  load(kb, a, b);
#ifndef K3_4M
  // 3M complex product: P1 = Ar Br, P2 = Ai Bi, P3 = (Ar + Ai)(Br + Bi);
  // Re = P1 - P2, Im = P3 - P1 - P2 (3 DMMAs per tile and k-step instead
  // of 4; normwise error of the same order).  The k-loop is
  // unrolled by two with alternating fragment registers (a/b <-> an/bn), so
  // the prefetch of step k+1 never has to be copied (a copy would wait for
  // the shared-memory load it was meant to hide).
  double p1[MT][NT][2] = {}, p2[MT][NT][2] = {}, p3[MT][NT][2] = {};
  auto step = [&](const cplx(&aa)[MT], const cplx(&bb)[NT]) {
    double bs[NT];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) bs[nt] = bb[nt].x + bb[nt].y;
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      const double as = aa[mt].x + aa[mt].y;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        dmma(p1[mt][nt], aa[mt].x, bb[nt].x);
        dmma(p2[mt][nt], aa[mt].y, bb[nt].y);
        dmma(p3[mt][nt], as, bs[nt]);
      }
    }
  };
#ifdef K3_PF2
  // prefetch distance 2: three fragment buffers in rotation
  cplx a2[MT], b2[NT];
  if (kb + 1 < ke) load(kb + 1, an, bn);
  int kq = kb;
  for (; kq + 2 < ke; kq += 3) {
    load(kq + 2, a2, b2);
    step(a, b);
    if (kq + 3 < ke) load(kq + 3, a, b);
    step(an, bn);
    if (kq + 4 < ke) load(kq + 4, an, bn);
    step(a2, b2);
  }
  if (kq < ke) step(a, b);
  if (kq + 1 < ke) step(an, bn);
#else
  int kq = kb;
  for (; kq + 1 < ke; kq += 2) {
    load(kq + 1, an, bn);
    step(a, b);
    if (kq + 2 < ke) load(kq + 2, a, b);
    step(an, bn);
  }
  if (kq < ke) step(a, b);
#endif
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        cr[mt][nt][e] = p1[mt][nt][e] - p2[mt][nt][e];
        ci[mt][nt][e] = p3[mt][nt][e] - p1[mt][nt][e] - p2[mt][nt][e];
      }
#else
  for (int kq = kb; kq < ke; ++kq) {
    if (kq + 1 < ke) load(kq + 1, an, bn);
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        dmma(cr[mt][nt], a[mt].x, b[nt].x);
        dmma(ci[mt][nt], a[mt].x, b[nt].y);
      }
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        dmma(cr[mt][nt], -a[mt].y, b[nt].y);
        dmma(ci[mt][nt], a[mt].y, b[nt].x);
      }
    }
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) a[mt] = an[mt];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) b[nt] = bn[nt];
  }
#endif
}

