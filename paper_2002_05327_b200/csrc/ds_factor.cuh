// Shared pieces of the block-tridiagonal factorization (on-chip and blocked
// paths): the per-chain job description and the entries of the diagonal
// blocks D_k of a window operator in block layout.
#pragma once
#include "ds_common.cuh"

struct FactJob {
  OpDev op;
  FactDev f;
  cplx *sinv;
  int half;  // 0 top chain, 1 bottom chain, 2 middle block
};


// D_k[i][c] of the block layout (i, c in-slab indices)
__device__ __forceinline__ cplx d_entry(const FactJob &J, int k, int i, int c) {
  const OpDev &o = J.op;
  const FactDev &f = J.f;
  int ba = f.block_axis;
  if (f.other[1] < 0) {  // 2D: one in-slab axis
    int oa = f.other[0];
    if (c == i) {
      int coord[3] = {0, 0, 0};
      coord[ba] = k;
      coord[oa] = i;
      double k2;
      if (o.kappa2_kind == 0) k2 = o.kappa2[0];
      else if (o.kappa2_kind == 1) k2 = o.kappa2[coord[o.kappa2_axis]];
      else k2 = o.kappa2[(int64_t)coord[0] * o.shape[1] + coord[1]];
      cplx acc = make_double2(k2, 0.0);
      for (int a = 0; a < 2; ++a) {
        cplx lo = o.c_lo[a][coord[a]], hi = o.c_hi[a][coord[a]];
        acc.x += -(lo.x + hi.x);
        acc.y += -(lo.y + hi.y);
      }
      return acc;
    }
    if (c == i - 1) return o.c_lo[oa][i];
    if (c == i + 1) return o.c_hi[oa][i];
    return make_double2(0.0, 0.0);
  }
  // 3D: in-slab index i = i0 * n1 + i1 over axes other[0], other[1]
  int o0 = f.other[0], o1 = f.other[1];
  int n1 = f.win_shape[o1];
  int i0 = i / n1, i1 = i % n1;
  if (c == i) {
    int coord[3];
    coord[ba] = k;
    coord[o0] = i0;
    coord[o1] = i1;
    double k2;
    if (o.kappa2_kind == 0) k2 = o.kappa2[0];
    else if (o.kappa2_kind == 1) k2 = o.kappa2[coord[o.kappa2_axis]];
    else k2 = o.kappa2[((int64_t)coord[0] * o.shape[1] + coord[1]) * o.shape[2] + coord[2]];
    cplx acc = make_double2(k2, 0.0);
    for (int a = 0; a < 3; ++a) {
      cplx lo = o.c_lo[a][coord[a]], hi = o.c_hi[a][coord[a]];
      acc.x += -(lo.x + hi.x);
      acc.y += -(lo.y + hi.y);
    }
    return acc;
  }
  if (c == i - 1 && i1 > 0) return o.c_lo[o1][i1];
  if (c == i + 1 && i1 < n1 - 1) return o.c_hi[o1][i1];
  if (c == i - n1) return o.c_lo[o0][i0];
  if (c == i + n1) return o.c_hi[o0][i0];
  return make_double2(0.0, 0.0);
}


// blocked (GEMM-based) factorization of the jobs whose slab is too large for
// the on-chip Gauss-Jordan path (3D windows); chains of `half` 0/1, then 2
int ds_blocked_factor(ds_ctx *ctx, const FactJob *jobs, int njobs, const cplx *const *l_host,
                      const cplx *const *u_host, int *status_dev);
