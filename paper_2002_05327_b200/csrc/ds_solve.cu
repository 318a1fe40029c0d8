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


// ------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;\n" ::"r"(
                   smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// TMA bulk copy global -> this CTA's shared memory, completing on `bar`
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes,
                                         uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// bulk copy of this CTA's shared memory into peer `rank`'s shared memory at
// the same offset as `dst_local`, completing on the peer's copy of `bar`
__device__ __forceinline__ void bulk_s2peer(void *dst_local, const void *src, uint32_t bytes,
                                            uint64_t *bar_local, uint32_t rank) {
  uint32_t rdst, rbar;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(rdst) : "r"(smem_u32(dst_local)), "r"(rank));
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(rbar) : "r"(smem_u32(bar_local)), "r"(rank));
  asm volatile(
      "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, "
      "[%3];\n" ::"r"(rdst),
      "r"(smem_u32(src)), "r"(bytes), "r"(rbar)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}

#define FAC_STAGES 3

// Cluster rank q owns rows [q*rows_per, q*rows_per + nr) of every S_k^{-1}.
// Stage s (s < n_b: forward block k = s; else backward block 2n_b-2-s):
//   wait vec[s&1] (filled by all peers' bulk pushes) and the factor tile,
//   acc = S_k^{-1}[rows, :] * vec          (2x2 register micro-tiles, K split)
//   forward : y_k = acc, next = b_{k+1} - l_{k+1} y_k   (or y_k at the turn)
//   backward: x_k = y_k - u_k acc, next = x_k
//   push `next` rows to every peer's vec[(s+1)&1].
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
    if (!any) return;  // uniform across the cluster (before any barrier)
  }

  const int rows_per = (m + C - 1) / C;
  const int r0 = rank * rows_per;
  const int nr = max(0, min(rows_per, m - r0));

  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t *vbar = (uint64_t *)smem_raw;                 // [2]
  uint64_t *fbar = vbar + 2;                             // [FAC_STAGES]
  cplx *vec = (cplx *)(smem_raw + 128);                  // [2][m*rcc + 2]
  const int vstride = m * rc + 2;
  cplx *stg = vec + 2 * vstride;                         // [2][rows_max*rc]
  cplx *fac = stg + 2 * rows_max * rc;                   // [FAC_STAGES][rows_max*m + 2]
  const int fstride = rows_max * m + 2;
  cplx *red = fac + FAC_STAGES * fstride;                // [16 * rows_max * rc]

  const int S = 2 * nb - 1;
  auto tile_of = [&](int s) { return s < nb ? s : 2 * nb - 2 - s; };
  const uint32_t vec_bytes = (uint32_t)(m * rcc * sizeof(cplx));
  const uint32_t push_bytes = (uint32_t)(nr * rcc * sizeof(cplx));
  const uint32_t fac_bytes = (uint32_t)(nr * m * sizeof(cplx));
  const size_t ldx = nrhs;  // row stride of the global block vectors

  if (t == 0) {
    mbar_init(&vbar[0], 1);
    mbar_init(&vbar[1], 1);
    for (int i = 0; i < FAC_STAGES; ++i) mbar_init(&fbar[i], 1);
    fence_mbar_init();
  }
  cluster.sync();  // every peer's barriers are initialised before any push
  if (t == 0) {
    mbar_expect_tx(&vbar[0], vec_bytes);
    if (S > 1) mbar_expect_tx(&vbar[1], vec_bytes);
    for (int i = 0; i < FAC_STAGES - 1 && i < S; ++i) {
      mbar_expect_tx(&fbar[i], fac_bytes);
      if (fac_bytes)
        bulk_g2s(fac + i * fstride, f.sinv + ((size_t)tile_of(i) * m + r0) * m, fac_bytes, &fbar[i]);
    }
  }
  // prologue: push my rows of b_0
  for (int e = t; e < nr * rcc; e += SOLVE_THREADS) {
    int row = e / rcc, c = e % rcc;
    stg[e] = V.rhs[(size_t)(r0 + row) * ldx + chunk0 + c];
  }
  fence_proxy_async();
  __syncthreads();
  if (t == 0 && push_bytes)
    for (int q = 0; q < C; ++q) bulk_s2peer(vec + r0 * rcc, stg, push_bytes, &vbar[0], q);

  // compute decomposition: 2x2 (row, rhs) micro-tiles, K split into slices
  const int TR = (nr + 1) / 2, TC = (rcc + 1) / 2;
  const int ntile = TR * TC;
  int nslice = ntile > 0 ? SOLVE_THREADS / ntile : 1;
  nslice = max(1, min(16, nslice));
  const int ks = (m + nslice - 1) / nslice;
  const int nout = nr * rcc;

  for (int s = 0; s < S; ++s) {
    const int k = tile_of(s);
    const bool fwd = s < nb;
    const int b = s & 1;
    // refill the factor ring (slot consumed at stage s-1)
    if (t == 0 && s + FAC_STAGES - 1 < S) {
      int sn = s + FAC_STAGES - 1, slot = sn % FAC_STAGES;
      mbar_expect_tx(&fbar[slot], fac_bytes);
      if (fac_bytes)
        bulk_g2s(fac + slot * fstride, f.sinv + ((size_t)tile_of(sn) * m + r0) * m, fac_bytes,
                 &fbar[slot]);
    }
    // epilogue operands (independent of the chain): issue the loads early
    cplx aux = make_double2(0.0, 0.0);
    int orow = t / max(rcc, 1), oc = t % max(rcc, 1);
    if (t < nout) {
      if (fwd && k + 1 < nb)
        aux = V.rhs[((size_t)(k + 1) * m + r0 + orow) * ldx + chunk0 + oc];
      else if (!fwd)
        aux = __ldcg(V.x + ((size_t)k * m + r0 + orow) * ldx + chunk0 + oc);
    }
    mbar_wait(&vbar[b], (s >> 1) & 1);
    mbar_wait(&fbar[s % FAC_STAGES], (s / FAC_STAGES) & 1);
    const cplx *A = fac + (s % FAC_STAGES) * fstride;
    const cplx *X = vec + b * vstride;
    for (int tile = ntile ? t % ntile : 0, sl = ntile ? t / ntile : nslice;
         sl < nslice && tile < ntile; tile += SOLVE_THREADS) {
      const int tr = tile / TC, tc = tile % TC;
      const int row = 2 * tr, c = 2 * tc;
      const int j0 = (ntile > SOLVE_THREADS) ? 0 : sl * ks;
      const int j1 = (ntile > SOLVE_THREADS) ? m : min(m, j0 + ks);
      cplx a00 = make_double2(0.0, 0.0), a01 = a00, a10 = a00, a11 = a00;
      const cplx *ar0 = A + (size_t)row * m;
      const cplx *ar1 = ar0 + m;
#pragma unroll 4
      for (int j = j0; j < j1; ++j) {
        cplx x0 = X[j * rcc + c], x1 = X[j * rcc + c + 1];
        cplx f0 = ar0[j], f1 = ar1[j];
        cfma(a00, f0, x0);
        cfma(a01, f0, x1);
        cfma(a10, f1, x0);
        cfma(a11, f1, x1);
      }
      cplx *rp = red + (size_t)((ntile > SOLVE_THREADS) ? 0 : sl) * rows_max * rc;
      rp[row * rcc + c] = a00;
      if (c + 1 < rcc) rp[row * rcc + c + 1] = a01;
      if (row + 1 < nr) {
        rp[(row + 1) * rcc + c] = a10;
        if (c + 1 < rcc) rp[(row + 1) * rcc + c + 1] = a11;
      }
      if (ntile <= SOLVE_THREADS) break;
    }
    __syncthreads();
    // next-stage block vector rows + outputs
    if (t < nout) {
      cplx acc = red[t];
      if (ntile <= SOLVE_THREADS)
        for (int q = 1; q < nslice; ++q) acc = cadd(acc, red[(size_t)q * rows_max * rc + t]);
      size_t off = ((size_t)k * m + r0 + orow) * ldx + chunk0 + oc;
      cplx nxt;
      if (fwd) {
        V.x[off] = acc;  // y_k
        nxt = (k + 1 < nb) ? csub(aux, cmul(f.lcoef[k + 1], acc)) : acc;
      } else {
        cplx xk = csub(aux, cmul(f.ucoef[k], acc));
        V.x[off] = xk;
        nxt = xk;
      }
      stg[((s + 1) & 1) * rows_max * rc + t] = nxt;
    }
    if (t == 0 && s + 2 < S) mbar_expect_tx(&vbar[b], vec_bytes);  // phase for stage s+2
    fence_proxy_async();
    __syncthreads();
    if (t == 0 && s + 1 < S && push_bytes) {
      cplx *src = stg + ((s + 1) & 1) * rows_max * rc;
      cplx *dst = vec + ((s + 1) & 1) * vstride + r0 * rcc;
      for (int q = 0; q < C; ++q) bulk_s2peer(dst, src, push_bytes, &vbar[(s + 1) & 1], q);
    }
  }
  cluster.sync();  // no CTA leaves while peers may still push into it
}

static int solve_rows_max(int max_m, int C) {
  int r = (max_m + C - 1) / C;
  return r + (r & 1);  // even: 2-row micro-tiles may read one padding row
}

static size_t solve_smem(int max_m, int rc, int C) {
  size_t rows_max = solve_rows_max(max_m, C);
  size_t elems = 2 * ((size_t)max_m * rc + 2) + 2 * rows_max * rc +
                 FAC_STAGES * (rows_max * max_m + 2) + 16 * rows_max * rc;
  return 128 + elems * sizeof(cplx);
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
  int rows_max = solve_rows_max(max_m, C);
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
