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
#include <cstring>
#include <vector>

#include "ds_common.cuh"

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
    dim3 grid((mmax + ST_ROWS - 1) / ST_ROWS, n, nchunks);
    k_stage_gemv<<<grid, ST_THREADS, 0, ctx->stream>>>(ditems + off[s], nrhs, vin_all, vin_stride);
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
