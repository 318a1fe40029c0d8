// K3g: staged block substitution for large slabs (3D windows, m ~ 460-4225).
//
// Same twisted schedule as K3 (ds_solve.cu), but a stage of a 3D window is a
// full-GPU amount of work (the block inverse is m^2 complex = 3.4-92 MB), so
// every stage is one launch over all (visit, half) items active at that
// stage; the launch boundary is the chain dependency.  Each CTA owns a
// 64-row tile of one item's block inverse and streams it from HBM once,
// against the block vector vin (<= 8 right-hand sides per grid.z chunk),
// which every CTA forms on the fly from b and the previous stage's output:
//   top fwd  vin = b_k - l_k y_{k-1}    bottom fwd vin = b_k - u_k z_{k+1}
//   middle   vin = b_t - l_t y_{t-1} - u_t z_{t+1}
//   top bwd  vin = x_{k+1}              bottom bwd vin = x_{k-1}
// Roofline: HBM, 16 m^2 B per (item, stage, RHS chunk of 8).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "ds_common.cuh"
#include "ds_mma.cuh"

#define ST_THREADS 256
#define ST_ROWS 32   // rows of the block inverse per CTA
#define ST_KL 8      // K lanes per row (lanes 8i..8i+7 share a row)
#define ST_KC 128    // vin rows per shared-memory chunk (x2 buffers)
#define ST_RC 8      // right-hand sides per grid.z chunk

struct StageItem {
  const FactDev *f;  // device pointer (block layout / factor base)
  const cplx *rhs;
  cplx *x;
  int m, nb, k, kind, half;  // kind 0 fwd, 1 middle, 2 bwd
  cplx la, lb;               // vin coefficients (see above)
  int ka, kb;                // blocks feeding vin (-1 = none)
  int has_b;                 // vin includes b_k
  cplx ecoef;                // bwd epilogue: x_k = aux - ecoef * acc
};

// vin of every item of a stage, formed once: [item][m][nrhs] (global scratch)
__global__ void k_stage_vin(const StageItem *__restrict__ items, int nrhs, cplx *vin_all,
                            size_t vin_stride) {
  const StageItem &I = items[blockIdx.y];
  const int m = I.m;
  const size_t ldx = nrhs;
  cplx *vout = vin_all + blockIdx.y * vin_stride;
  const int64_t total = (int64_t)m * nrhs;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const size_t j = e / nrhs, col = e % nrhs;
    cplx v;
    if (I.kind == 2) {
      v = I.x[((size_t)I.ka * m + j) * ldx + col];  // x_{k+-1}
    } else {
      v = I.has_b ? I.rhs[((size_t)I.k * m + j) * ldx + col] : make_double2(0.0, 0.0);
      if (I.ka >= 0) v = csub(v, cmul(I.la, I.x[((size_t)I.ka * m + j) * ldx + col]));
      if (I.kb >= 0) v = csub(v, cmul(I.lb, I.x[((size_t)I.kb * m + j) * ldx + col]));
    }
    vout[e] = v;
  }
}

__device__ __forceinline__ void st_cp_async16(void *dst, const void *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(
                   (unsigned)__cvta_generic_to_shared(dst)),
               "l"(src)
               : "memory");
}

__global__ void __launch_bounds__(ST_THREADS, 3)
    k_stage_gemv(const StageItem *__restrict__ items, int nrhs, const cplx *vin_all,
                 size_t vin_stride) {
  const StageItem &I = items[blockIdx.y];
  const int m = I.m;
  const int r0 = blockIdx.x * ST_ROWS;
  if (r0 >= m) return;
  const int c0 = blockIdx.z * ST_RC;
  const int rcc = min(ST_RC, nrhs - c0);
  if (rcc <= 0) return;
  const int t = threadIdx.x;
  const int row = r0 + t / ST_KL, kq = t % ST_KL;
  const bool rvalid = row < m;
  const size_t ldx = nrhs;
  const cplx *A = I.f->sinv + ((size_t)I.k * m) * m;
  const cplx *vg = vin_all + blockIdx.y * vin_stride;
  // rows padded to ST_RC+1: the 8 K-lanes of a warp read 8 different rows,
  // a 128-B row stride would put them all on the same 4 banks
  __shared__ __align__(16) cplx vin[2][ST_KC][ST_RC + 1];
  cplx acc[ST_RC];
#pragma unroll
  for (int c = 0; c < ST_RC; ++c) acc[c] = make_double2(0.0, 0.0);
  auto prefetch = [&](int chunk) {  // vin rows [chunk*KC, ...) -> buffer chunk&1
    const int j0 = chunk * ST_KC, jn = min(ST_KC, m - j0);
    cplx(*dst)[ST_RC + 1] = vin[chunk & 1];
    for (int e = t; e < jn * ST_RC; e += ST_THREADS) {
      const int jj = e / ST_RC, c = e % ST_RC;
      if (c < rcc) st_cp_async16(&dst[jj][c], vg + (size_t)(j0 + jj) * ldx + c0 + c);
      else dst[jj][c] = make_double2(0.0, 0.0);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  const int nchunk = (m + ST_KC - 1) / ST_KC;
  prefetch(0);
  for (int ch = 0; ch < nchunk; ++ch) {
    const int j0 = ch * ST_KC, jn = min(ST_KC, m - j0);
    if (ch + 1 < nchunk) {
      prefetch(ch + 1);
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    }
    __syncthreads();
    cplx(*V)[ST_RC + 1] = vin[ch & 1];
    if (rvalid) {
      // 8 independent 16-B factor loads in flight per thread, then the FMAs
      const cplx *a = A + (size_t)row * m + j0;
      int jj = kq;
      for (; jj + 7 * ST_KL < jn; jj += 8 * ST_KL) {
        cplx av[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) av[u] = __ldcs(a + jj + u * ST_KL);
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
          for (int c = 0; c < ST_RC; ++c) cfma(acc[c], av[u], V[jj + u * ST_KL][c]);
      }
      for (; jj < jn; jj += ST_KL) {
        const cplx av = __ldcs(a + jj);
#pragma unroll
        for (int c = 0; c < ST_RC; ++c) cfma(acc[c], av, V[jj][c]);
      }
    }
    __syncthreads();  // buffer ch&1 is refilled two chunks later
  }
#pragma unroll
  for (int c = 0; c < ST_RC; ++c)
#pragma unroll
    for (int off = 1; off < ST_KL; off <<= 1) {
      acc[c].x += __shfl_xor_sync(0xffffffffu, acc[c].x, off);
      acc[c].y += __shfl_xor_sync(0xffffffffu, acc[c].y, off);
    }
  if (rvalid && kq == 0) {
#pragma unroll
    for (int c = 0; c < ST_RC; ++c) {
      if (c >= rcc) break;
      const size_t off = ((size_t)I.k * m + row) * ldx + c0 + c;
      if (I.kind == 2) {
        cplx aux = I.x[off];  // y_k / z_k from the forward pass
        I.x[off] = csub(aux, cmul(I.ecoef, acc[c]));
      } else {
        I.x[off] = acc[c];
      }
    }
  }
}

// K3g on the FP64 tensor cores.  ncu on config 4 showed k_stage_gemv bound
// by L1/shared-memory throughput (92% L1TEX, shared wavefronts 74% of peak,
// DRAM 35%): every streamed factor element was multiplied with 8 RHS values
// read from shared memory.  Here each warp owns an 8-row x 8-RHS tile over the
// whole K: the factor rows are streamed from HBM as DMMA A fragments (8 loads
// in flight per thread), the block vector is read from shared memory once per
// k-step as the B fragment, and the complex product uses 3 real m8n8k4 DMMAs.
#define SM_WARPS 8
#define SM_KC 128  // vin rows per shared-memory chunk (x2 buffers)
#ifndef SM_DEPTH
#define SM_DEPTH 8  // factor k-steps loaded per batch (loads in flight per thread)
#endif
#ifndef SM_MINB
#define SM_MINB 3  // measured best (config 4: 10.0 vs 9.8 RHS/s at 2, 8.3 with 16-deep)
#endif
__global__ void __launch_bounds__(32 * SM_WARPS, SM_MINB)
    k_stage_gemv_mma(const StageItem *__restrict__ items, int nrhs, const cplx *vin_all,
                     size_t vin_stride) {
  const StageItem &I = items[blockIdx.y];
  const int m = I.m;
  const int r0 = blockIdx.x * (8 * SM_WARPS);
  if (r0 >= m) return;
  const int c0 = blockIdx.z * ST_RC;
  const int rcc = min(ST_RC, nrhs - c0);
  if (rcc <= 0) return;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31, g = lane >> 2, tg = lane & 3;
  const int row = r0 + warp * 8 + g;  // A-fragment row of this lane
  const bool rvalid = row < m;
  const size_t ldx = nrhs;
  const cplx *A = I.f->sinv + ((size_t)I.k * m) * m + (size_t)(rvalid ? row : 0) * m;
  const cplx *vg = vin_all + blockIdx.y * vin_stride;
  __shared__ __align__(16) cplx vin[2][SM_KC][ST_RC];
  double p1[2] = {0.0, 0.0}, p2[2] = {0.0, 0.0}, p3[2] = {0.0, 0.0};
  auto prefetch = [&](int chunk) {
    const int j0 = chunk * SM_KC, jn = min(SM_KC, m - j0);
    cplx(*dst)[ST_RC] = vin[chunk & 1];
    for (int e = t; e < SM_KC * ST_RC; e += 32 * SM_WARPS) {
      const int jj = e / ST_RC, c = e % ST_RC;
      if (jj < jn && c < rcc) st_cp_async16(&dst[jj][c], vg + (size_t)(j0 + jj) * ldx + c0 + c);
      else dst[jj][c] = make_double2(0.0, 0.0);  // K tail and RHS tail read as zero
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  const int nchunk = (m + SM_KC - 1) / SM_KC;
  prefetch(0);
  for (int ch = 0; ch < nchunk; ++ch) {
    const int j0 = ch * SM_KC, jn = min(SM_KC, m - j0);
    if (ch + 1 < nchunk) {
      prefetch(ch + 1);
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    }
    __syncthreads();
    cplx(*V)[ST_RC] = vin[ch & 1];
    const int nks = (jn + 3) >> 2;
    for (int kg = 0; kg < nks; kg += SM_DEPTH) {
      cplx a[SM_DEPTH];
#pragma unroll
      for (int u = 0; u < SM_DEPTH; ++u) {  // SM_DEPTH independent factor loads in flight
        const int kk = (kg + u) * 4 + tg;
        a[u] = (rvalid && kg + u < nks && kk < jn) ? __ldcs(A + j0 + kk) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < SM_DEPTH; ++u) {
        if (kg + u >= nks) break;
        const cplx b = V[(kg + u) * 4 + tg][g];
        const double as = a[u].x + a[u].y, bs = b.x + b.y;
        dmma(p1, a[u].x, b.x);
        dmma(p2, a[u].y, b.y);
        dmma(p3, as, bs);
      }
    }
    __syncthreads();  // buffer ch&1 is refilled two chunks later
  }
  // C fragment: row r0 + 8 warp + g, columns 2 tg, 2 tg + 1 of the chunk
  const int orow = r0 + warp * 8 + g;
  if (orow < m) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int c = 2 * tg + e;
      if (c >= rcc) continue;
      const cplx acc = make_double2(p1[e] - p2[e], p3[e] - p1[e] - p2[e]);
      const size_t off = ((size_t)I.k * m + orow) * ldx + c0 + c;
      if (I.kind == 2) {
        cplx aux = I.x[off];  // y_k / z_k from the forward pass
        I.x[off] = csub(aux, cmul(I.ecoef, acc));
      } else {
        I.x[off] = acc;
      }
    }
  }
}


// host: the twisted schedule of one visit
static bool stage_item(const FactDev &f, int s, int half, StageItem &I) {
  const int nb = f.nb, tw = f.twist, nt = tw, nbt = nb - 1 - tw;
  const int F = std::max(nt, nbt);
  int k = -1, kind = 0;
  if (s < F) {
    if (half == 0 && s >= F - nt) k = s - (F - nt);
    if (half == 1 && s >= F - nbt) k = nb - 1 - (s - (F - nbt));
    kind = 0;
  } else if (s == F) {
    if (half == 0) k = tw;
    kind = 1;
  } else {
    int j = s - F - 1;
    if (half == 0 && j < nt) k = tw - 1 - j;
    if (half == 1 && j < nbt) k = tw + 1 + j;
    kind = 2;
  }
  if (k < 0) return false;
  I.k = k;
  I.kind = kind;
  I.half = half;
  I.m = f.m;
  I.nb = nb;
  I.ka = I.kb = -1;
  I.has_b = 0;
  return true;
}

int ds_launch_solve_staged(ds_ctx *ctx, const SolveVisit *visits_host, const FactDev *facts_host,
                           const cplx *const *l_host, const cplx *const *u_host, int nvisit,
                           int nrhs, void *items_dev, size_t items_cap) {
  if (nvisit < 1) return DS_OK;
  int S = 0;
  for (int v = 0; v < nvisit; ++v) {
    const FactDev &f = facts_host[v];
    S = std::max(S, 2 * std::max(f.twist, f.nb - 1 - f.twist) + 1);
  }
  std::vector<StageItem> items;
  StageItem *ditems = (StageItem *)items_dev;
  // all stages' items are uploaded once (launch s reads its own range)
  std::vector<int> off(S + 1, 0);
  for (int s = 0; s < S; ++s) {
    off[s] = (int)items.size();
    for (int v = 0; v < nvisit; ++v) {
      const FactDev &f = facts_host[v];
      const int Fv = std::max(f.twist, f.nb - 1 - f.twist);
      if (s >= 2 * Fv + 1) continue;
      for (int half = 0; half < 2; ++half) {
        StageItem I;
        memset(&I, 0, sizeof(I));
        if (!stage_item(f, s, half, I)) continue;
        I.f = visits_host[v].f;
        I.rhs = visits_host[v].rhs;
        I.x = visits_host[v].x;
        const int k = I.k, tw = f.twist, nb = f.nb;
        const cplx lk = l_host[v][k], uk = u_host[v][k];
        if (I.kind == 0) {
          I.has_b = 1;
          if (half == 0 && k > 0) { I.ka = k - 1; I.la = lk; }
          if (half == 1 && k < nb - 1) { I.ka = k + 1; I.la = uk; }
        } else if (I.kind == 1) {
          I.has_b = 1;
          if (tw > 0) { I.ka = tw - 1; I.la = lk; }
          if (tw < nb - 1) { I.kb = tw + 1; I.lb = uk; }
        } else {
          I.ka = half == 0 ? k + 1 : k - 1;
          I.ecoef = half == 0 ? uk : lk;
        }
        items.push_back(I);
      }
    }
  }
  off[S] = (int)items.size();

  DS_CUDA(cudaMemcpyAsync(ditems, items.data(), items.size() * sizeof(StageItem),
                          cudaMemcpyHostToDevice, ctx->stream));
  int mmax = 0;
  for (int v = 0; v < nvisit; ++v) mmax = std::max(mmax, facts_host[v].m);
  const int nchunks = (nrhs + ST_RC - 1) / ST_RC;
  // vin scratch follows the item table in the workspace
  const size_t item_bytes = ((items.size() * sizeof(StageItem) + 255) / 256) * 256;
  const size_t vin_stride = (size_t)mmax * nrhs;
  int maxn = 0;
  for (int s = 0; s < S; ++s) maxn = std::max(maxn, off[s + 1] - off[s]);
  if (item_bytes + (size_t)maxn * vin_stride * sizeof(cplx) > items_cap)
    return ds_fail(DS_ECONFIG, "staged solve: workspace too small");
  cplx *vin_all = (cplx *)((char *)items_dev + item_bytes);
  for (int s = 0; s < S; ++s) {
    int n = off[s + 1] - off[s];
    if (!n) continue;
    int vb = (int)std::min<int64_t>(256, ((int64_t)mmax * nrhs + 255) / 256);
    k_stage_vin<<<dim3(vb, n), 256, 0, ctx->stream>>>(ditems + off[s], nrhs, vin_all, vin_stride);
    if (ctx->opt.k3g_mma) {
      dim3 grid((mmax + 8 * SM_WARPS - 1) / (8 * SM_WARPS), n, nchunks);
      k_stage_gemv_mma<<<grid, 32 * SM_WARPS, 0, ctx->stream>>>(ditems + off[s], nrhs, vin_all,
                                                                vin_stride);
    } else {
      dim3 grid((mmax + ST_ROWS - 1) / ST_ROWS, n, nchunks);
      k_stage_gemv<<<grid, ST_THREADS, 0, ctx->stream>>>(ditems + off[s], nrhs, vin_all, vin_stride);
    }
    ctx->launches += 2;
  }
  DS_CHECK_LAUNCH();
  // the host item vector must outlive the async copy
  DS_CUDA(cudaStreamSynchronize(ctx->stream));
  return DS_OK;
}

size_t ds_stage_items_bytes(int nvisit, int max_nb, int max_m, int nrhs) {
  size_t items = sizeof(StageItem) * (size_t)nvisit * 2 * (2 * max_nb + 2);
  items = ((items + 255) / 256) * 256;
  return items + (size_t)nvisit * 2 * max_m * nrhs * sizeof(cplx);
}

// ------------------------------------------------------------------------
// Small slabs (2D windows, m <= DS_LARGE_SLAB): one fused kernel per stage,
// launched with programmatic dependent launch.  Before griddepcontrol.wait a
// CTA only prefetches its rows of the block inverse (read-only, independent
// of the chain), so the next stage's prologue overlaps the current stage.
template <int RC>
__global__ void __launch_bounds__(ST_THREADS)
    k_stage_small(const StageItem *__restrict__ items, int nrhs, int rt) {
  const StageItem &I = items[blockIdx.y];
  const int m = I.m;
  const int r0 = blockIdx.x * rt;
  const int c0 = blockIdx.z * RC;
  const int t = threadIdx.x;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cplx *At = (cplx *)smem_raw;        // [rt][m]
  cplx *vin = At + (size_t)rt * m;    // [m][RC+1]
  const bool active = r0 < m && c0 < nrhs;
  const int nr = active ? min(rt, m - r0) : 0;
  if (active) {
    const cplx *src = I.f->sinv + ((size_t)I.k * m + r0) * m;
    for (int e = t; e < nr * m; e += ST_THREADS) st_cp_async16(At + e, src + e);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  }
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  if (!active) return;
  const int rcc = min(RC, nrhs - c0);
  const size_t ldx = nrhs;
  // form vin with every global load of a thread in flight at once (the loads
  // are L2 round trips on the critical path of the chain)
  constexpr int VPT = 12;  // m * RC <= 12 * ST_THREADS for m <= DS_LARGE_SLAB
  {
    cplx b[VPT], xa[VPT], xb[VPT];
#pragma unroll
    for (int u = 0; u < VPT; ++u) {
      const int e = t + u * ST_THREADS;
      const int j = e / RC, c = e % RC;
      const bool ok = e < m * RC && c < rcc;
      const size_t col = c0 + c;
      b[u] = xa[u] = xb[u] = make_double2(0.0, 0.0);
      if (ok) {
        if (I.has_b) b[u] = I.rhs[((size_t)I.k * m + j) * ldx + col];
        if (I.ka >= 0) xa[u] = I.x[((size_t)I.ka * m + j) * ldx + col];
        if (I.kb >= 0) xb[u] = I.x[((size_t)I.kb * m + j) * ldx + col];
      }
    }
#pragma unroll
    for (int u = 0; u < VPT; ++u) {
      const int e = t + u * ST_THREADS;
      if (e >= m * RC) break;
      const int j = e / RC, c = e % RC;
      cplx v = xa[u];  // bwd: x_{k+-1}
      if (I.kind != 2) v = csub(csub(b[u], cmul(I.la, xa[u])), cmul(I.lb, xb[u]));
      vin[j * (RC + 1) + c] = v;
    }
  }
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  __syncthreads();
  // outputs (row, c) of this tile; KS lanes split K for each output
  const int nout = rt * RC;
  int KS = ST_THREADS / nout;
  KS = KS >= 32 ? 32 : (KS >= 16 ? 16 : (KS >= 8 ? 8 : (KS >= 4 ? 4 : (KS >= 2 ? 2 : 1))));
  for (int base = 0; base < nout; base += ST_THREADS / KS) {
    const int o = base + t / KS, ks = t % KS;
    const bool valid = o < nout;
    const int row = valid ? o / RC : 0, c = valid ? o % RC : 0;
    cplx a0 = make_double2(0.0, 0.0), a1 = a0;
    if (valid && row < nr) {
      const cplx *a = At + (size_t)row * m;
      int j = ks;
      for (; j + KS < m; j += 2 * KS) {
        cfma(a0, a[j], vin[j * (RC + 1) + c]);
        cfma(a1, a[j + KS], vin[(j + KS) * (RC + 1) + c]);
      }
      if (j < m) cfma(a0, a[j], vin[j * (RC + 1) + c]);
    }
    cplx acc = cadd(a0, a1);
    for (int off = 1; off < KS; off <<= 1) {
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, off);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, off);
    }
    if (valid && row < nr && ks == 0 && c < rcc) {
      const size_t off = ((size_t)I.k * m + r0 + row) * ldx + c0 + c;
      if (I.kind == 2) {
        const cplx aux = I.x[off];
        I.x[off] = csub(aux, cmul(I.ecoef, acc));
      } else {
        I.x[off] = acc;
      }
    }
  }
}

// ------------------------------------------------------------------------
// Stage programs: every stage item of every step, built once per plan.
struct StageProgram {
  StageItem *items = nullptr;           // device
  std::vector<std::vector<int>> off;    // [step][stage + 1] offsets into items
  std::vector<int> base;                // [step] first item of the step
  int max_m = 0;
  bool small = true;
  cplx *vin = nullptr;                  // large path scratch
  size_t vin_elems = 0;
  int max_items_stage = 0;
};

StageProgram *ds_stage_program_create(const std::vector<std::vector<SolveVisit>> &step_visits,
                                      const std::vector<std::vector<FactDev>> &step_facts,
                                      const std::vector<std::vector<const cplx *>> &step_l,
                                      const std::vector<std::vector<const cplx *>> &step_u,
                                      int nrhs_max, std::string *err) {
  StageProgram *P = new StageProgram();
  std::vector<StageItem> all;
  for (size_t q = 0; q < step_visits.size(); ++q) {
    const auto &vs = step_visits[q];
    const auto &fs = step_facts[q];
    P->base.push_back((int)all.size());
    int S = 0;
    for (auto &f : fs) {
      S = std::max(S, 2 * std::max(f.twist, f.nb - 1 - f.twist) + 1);
      P->max_m = std::max(P->max_m, f.m);
    }
    std::vector<int> off(S + 1, 0);
    for (int s = 0; s < S; ++s) {
      off[s] = (int)all.size();
      for (size_t v = 0; v < vs.size(); ++v) {
        const FactDev &f = fs[v];
        const int Fv = std::max(f.twist, f.nb - 1 - f.twist);
        if (s >= 2 * Fv + 1) continue;
        for (int half = 0; half < 2; ++half) {
          StageItem I;
          memset(&I, 0, sizeof(I));
          if (!stage_item(f, s, half, I)) continue;
          I.f = vs[v].f;
          I.rhs = vs[v].rhs;
          I.x = vs[v].x;
          const int k = I.k, tw = f.twist, nb = f.nb;
          const cplx lk = step_l[q][v][k], uk = step_u[q][v][k];
          if (I.kind == 0) {
            I.has_b = 1;
            if (half == 0 && k > 0) { I.ka = k - 1; I.la = lk; }
            if (half == 1 && k < nb - 1) { I.ka = k + 1; I.la = uk; }
          } else if (I.kind == 1) {
            I.has_b = 1;
            if (tw > 0) { I.ka = tw - 1; I.la = lk; }
            if (tw < nb - 1) { I.kb = tw + 1; I.lb = uk; }
          } else {
            I.ka = half == 0 ? k + 1 : k - 1;
            I.ecoef = half == 0 ? uk : lk;
          }
          all.push_back(I);
        }
      }
      P->max_items_stage = std::max(P->max_items_stage, (int)all.size() - off[s]);
    }
    off[S] = (int)all.size();
    for (auto &o : off) o -= P->base.back();
    P->off.push_back(off);
  }
  P->small = P->max_m <= DS_LARGE_SLAB;
  if (cudaMalloc(&P->items, std::max<size_t>(1, all.size()) * sizeof(StageItem)) != cudaSuccess) {
    *err = "stage program: out of device memory";
    delete P;
    return nullptr;
  }
  cudaMemcpy(P->items, all.data(), all.size() * sizeof(StageItem), cudaMemcpyHostToDevice);
  if (!P->small) {
    P->vin_elems = (size_t)P->max_items_stage * P->max_m * nrhs_max;
    if (cudaMalloc(&P->vin, std::max<size_t>(1, P->vin_elems) * sizeof(cplx)) != cudaSuccess) {
      cudaFree(P->items);
      *err = "stage program: out of device memory (vin scratch)";
      delete P;
      return nullptr;
    }
  }
  return P;
}

void ds_stage_program_destroy(StageProgram *P) {
  if (!P) return;
  cudaFree(P->items);
  cudaFree(P->vin);
  delete P;
}

static int small_rows(const ds_ctx *ctx) {
  // rows per CTA (option "stage_rows", default 16): every CTA re-forms the
  // whole block vector from L2, so fewer, fatter tiles are cheaper
  return ctx->opt.stage_rows > 0 ? ctx->opt.stage_rows : 16;
}

template <int RC>
static int launch_small(ds_ctx *ctx, const StageItem *items, int n, int nrhs, int m) {
  const int nchunk = (nrhs + RC - 1) / RC;
  const int rt = small_rows(ctx);
  size_t smem = ((size_t)rt * m + (size_t)m * (RC + 1)) * sizeof(cplx);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_stage_small<RC>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3((m + rt - 1) / rt, n, nchunk);
  cfg.blockDim = dim3(ST_THREADS, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  DS_CUDA(cudaLaunchKernelEx(&cfg, k_stage_small<RC>, items, nrhs, rt));
  ctx->launches++;
  return DS_OK;
}

int ds_stage_program_launch_step(ds_ctx *ctx, StageProgram *P, int step, int nrhs) {
  const auto &off = P->off[step];
  const StageItem *base = P->items + P->base[step];
  const int S = (int)off.size() - 1;
  const int m = P->max_m;
  for (int s = 0; s < S; ++s) {
    const int n = off[s + 1] - off[s];
    if (!n) continue;
    const StageItem *it = base + off[s];
    int rc;
    if (P->small) {
      if (nrhs >= 16) rc = launch_small<16>(ctx, it, n, nrhs, m);
      else if (nrhs >= 8) rc = launch_small<8>(ctx, it, n, nrhs, m);
      else if (nrhs >= 4) rc = launch_small<4>(ctx, it, n, nrhs, m);
      else if (nrhs >= 2) rc = launch_small<2>(ctx, it, n, nrhs, m);
      else rc = launch_small<1>(ctx, it, n, nrhs, m);
      if (rc) return rc;
    } else {
      const size_t vin_stride = (size_t)m * nrhs;
      if ((size_t)n * vin_stride > P->vin_elems)
        return ds_fail(DS_ECONFIG, "stage program: vin scratch too small");
      int vb = (int)std::min<int64_t>(256, ((int64_t)m * nrhs + 255) / 256);
      k_stage_vin<<<dim3(vb, n), 256, 0, ctx->stream>>>(it, nrhs, P->vin, vin_stride);
      if (ctx->opt.k3g_mma) {
        dim3 grid((m + 8 * SM_WARPS - 1) / (8 * SM_WARPS), n, (nrhs + ST_RC - 1) / ST_RC);
        k_stage_gemv_mma<<<grid, 32 * SM_WARPS, 0, ctx->stream>>>(it, nrhs, P->vin, vin_stride);
      } else {
        dim3 grid((m + ST_ROWS - 1) / ST_ROWS, n, (nrhs + ST_RC - 1) / ST_RC);
        k_stage_gemv<<<grid, ST_THREADS, 0, ctx->stream>>>(it, nrhs, P->vin, vin_stride);
      }
      ctx->launches += 2;
    }
  }
  DS_CHECK_LAUNCH();
  return DS_OK;
}
