// K3: batched block forward/back substitution — one launch per
// anti-diagonal step, one thread-block cluster per (subdomain visit, RHS
// chunk).  Replaces Factorization.solve (diagsweep/subdomain.py:77-106,
// :127-133) as called at ddm.py:259.
//
//   forward  y_k = S_k^{-1} (b_k - l_k y_{k-1})          k = 0 .. n_b-1
//   backward x_k = y_k - u_k S_k^{-1} x_{k+1}            k = n_b-2 .. 0
//
// The C CTAs of a cluster split the m rows of every S_k^{-1}; each CTA
// streams its row slice of the next block into shared memory with
// cp.async while it multiplies the current one (the factor stream does not
// depend on the substitution chain), and the cluster exchanges the
// finished block vector through L2 with one cluster barrier (release /
// acquire) per stage.  Arithmetic: 16*n_b*m^2 flop per (visit, RHS) in FP64
// FMA; the factor bytes 2*n_b*m^2*16 are read once per visit for all RHS
// of the chunk.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>

#include "ds_common.cuh"

namespace cg = cooperative_groups;

#define SOLVE_THREADS 256
#define SOLVE_MAX_RC 32

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__global__ void __launch_bounds__(SOLVE_THREADS, 1)
    k_block_solve(const SolveVisit *__restrict__ visits, int nrhs, int rc, int rows_max) {
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int C = (int)cluster.num_blocks();
  const SolveVisit V = visits[blockIdx.y];
  const FactDev f = *V.f;
  const int m = f.m, nb = f.nb;
  const int chunk0 = blockIdx.z * rc;
  const int rcc = min(rc, nrhs - chunk0);
  const int t = threadIdx.x;

  // skip visits whose right-hand sides are all exactly zero (ddm.py:256-258)
  if (V.nz) {
    int any = 0;
    for (int r = 0; r < rcc; ++r) any |= V.nz[chunk0 + r];
    if (!any) return;  // uniform across the cluster
  }

  const int rows_per = (m + C - 1) / C;
  const int r0 = rank * rows_per;
  const int nr = max(0, min(rows_per, m - r0));

  extern __shared__ __align__(16) unsigned char smem_raw[];
  cplx *vec = (cplx *)smem_raw;                     // [m][rc]
  cplx *fac = vec + (size_t)m * rc;                 // [2][rows_max][m]
  cplx *red = fac + 2 * (size_t)rows_max * m;       // [SOLVE_THREADS]

  const int nout = nr * rcc;
  int nslice = 1;
  if (nout > 0 && nout < SOLVE_THREADS) nslice = min(16, SOLVE_THREADS / nout);
  const int ks = (m + nslice - 1) / nslice;

  const int S = 2 * nb - 1;
  auto tile_of = [&](int s) { return s < nb ? s : 2 * nb - 2 - s; };
  auto prefetch = [&](int s) {
    int k = tile_of(s);
    const cplx *src = f.sinv + ((size_t)k * m + r0) * m;
    cplx *dstb = fac + (size_t)(s & 1) * rows_max * m;
    int n = nr * m;
    for (int e = t; e < n; e += SOLVE_THREADS) cp_async16(dstb + e, src + e);
  };

  prefetch(0);
  cp_async_commit();
  for (int s = 0; s < S; ++s) {
    const int k = tile_of(s);
    const bool fwd = s < nb;
    if (s + 1 < S) prefetch(s + 1);
    cp_async_commit();
    // ---- assemble the block vector
    if (fwd) {
      const cplx lk = k > 0 ? f.lcoef[k] : make_double2(0.0, 0.0);
      for (int e = t; e < m * rcc; e += SOLVE_THREADS) {
        int j = e / rcc, c = e % rcc;
        size_t off = ((size_t)k * m + j) * nrhs + chunk0 + c;
        cplx b = V.rhs[off];
        if (k > 0) b = csub(b, cmul(lk, __ldcg(V.x + off - (size_t)m * nrhs)));
        vec[j * rc + c] = b;
      }
    } else {
      for (int e = t; e < m * rcc; e += SOLVE_THREADS) {
        int j = e / rcc, c = e % rcc;
        vec[j * rc + c] = __ldcg(V.x + ((size_t)(k + 1) * m + j) * nrhs + chunk0 + c);
      }
    }
    cp_async_wait<1>();
    __syncthreads();
    // ---- rows [r0, r0+nr) of S_k^{-1} times vec
    const cplx *A = fac + (size_t)(s & 1) * rows_max * m;
    if (nout > 0) {
      if (nslice > 1) {
        int o = t % nout, sl = t / nout;
        cplx acc = make_double2(0.0, 0.0);
        if (sl < nslice) {
          int row = o / rcc, c = o % rcc;
          int j0 = sl * ks, j1 = min(m, j0 + ks);
          const cplx *a = A + (size_t)row * m;
          for (int j = j0; j < j1; ++j) cfma(acc, a[j], vec[j * rc + c]);
        }
        red[t] = acc;
        __syncthreads();
        if (t < nout) {
          cplx sum = red[t];
          for (int q = 1; q < nslice; ++q) sum = cadd(sum, red[q * nout + t]);
          int row = t / rcc, c = t % rcc;
          size_t off = ((size_t)k * m + r0 + row) * nrhs + chunk0 + c;
          if (fwd) {
            V.x[off] = sum;
          } else {
            cplx y = __ldcg(V.x + off);
            V.x[off] = csub(y, cmul(f.ucoef[k], sum));
          }
        }
      } else {
        for (int o = t; o < nout; o += SOLVE_THREADS) {
          int row = o / rcc, c = o % rcc;
          const cplx *a = A + (size_t)row * m;
          cplx acc = make_double2(0.0, 0.0);
          for (int j = 0; j < m; ++j) cfma(acc, a[j], vec[j * rc + c]);
          size_t off = ((size_t)k * m + r0 + row) * nrhs + chunk0 + c;
          if (fwd) {
            V.x[off] = acc;
          } else {
            cplx y = __ldcg(V.x + off);
            V.x[off] = csub(y, cmul(f.ucoef[k], acc));
          }
        }
      }
    }
    cluster.sync();  // release my rows of y_k / x_k, acquire the peers'
  }
  cp_async_wait<0>();
}

static size_t solve_smem(int max_m, int rc, int C) {
  int rows_max = (max_m + C - 1) / C;
  return ((size_t)max_m * rc + 2 * (size_t)rows_max * max_m + SOLVE_THREADS) * sizeof(cplx);
}

// Largest cluster (16 non-portable, then 8, 4) that the occupancy API
// accepts for this shared-memory footprint.
static int pick_cluster(int max_m, int rc, size_t *smem_out) {
  static int cached_key_m = -1, cached_key_rc = -1, cached_C = 0;
  static size_t cached_smem = 0;
  if (max_m == cached_key_m && rc == cached_key_rc) {
    *smem_out = cached_smem;
    return cached_C;
  }
  cudaFuncSetAttribute(k_block_solve, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int C : {16, 8, 4}) {
    size_t smem = solve_smem(max_m, rc, C);
    if (smem > 232448) continue;
    if (cudaFuncSetAttribute(k_block_solve, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess) {
      cudaGetLastError();
      continue;
    }
    cudaLaunchConfig_t cfg;
    memset(&cfg, 0, sizeof(cfg));
    cfg.gridDim = dim3(C, 1, 1);
    cfg.blockDim = dim3(SOLVE_THREADS, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int nclusters = 0;
    if (cudaOccupancyMaxActiveClusters(&nclusters, k_block_solve, &cfg) == cudaSuccess &&
        nclusters > 0) {
      cached_key_m = max_m;
      cached_key_rc = rc;
      cached_C = C;
      cached_smem = smem;
      *smem_out = smem;
      return C;
    }
    cudaGetLastError();
  }
  return 0;
}

int ds_launch_solve_table(ds_ctx *ctx, const void *visits_dev, int nvisit, int nrhs,
                          int max_m) {
  if (nvisit < 1) return DS_OK;
  int rc = std::min(nrhs, SOLVE_MAX_RC);
  int nchunks = (nrhs + rc - 1) / rc;
  size_t smem = 0;
  int C = pick_cluster(max_m, rc, &smem);
  if (!C) return ds_fail(DS_ECONFIG, "block solve: no feasible cluster configuration");
  DS_CUDA(cudaFuncSetAttribute(k_block_solve, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem));
  int rows_max = (max_m + C - 1) / C;
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3(C, nvisit, nchunks);
  cfg.blockDim = dim3(SOLVE_THREADS, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  DS_CUDA(cudaLaunchKernelEx(&cfg, k_block_solve, (const SolveVisit *)visits_dev, nrhs, rc,
                             rows_max));
  ctx->launches++;
  return DS_OK;
}
