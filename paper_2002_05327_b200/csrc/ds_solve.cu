// K3: batched block forward/back substitution of the block-LU factors --
// one launch per step of the launch schedule, one thread-block cluster per
// (subdomain visit, RHS chunk).  Replaces Factorization.solve
// (diagsweep/subdomain.py:77-106, :127-133) as called at ddm.py:259.
//
// Twisted substitution (see ds_factor.cu): with t = twist, the top chain
// runs y_k = S_k^{-1} (b_k - l_k y_{k-1}) for k < t, the bottom chain the
// mirror image for k > t, the middle block joins both, and the backward
// sweeps x_k = y_k - (u_k or l_k) S_k^{-1} x_{k+-1} run outwards: a chain of
// ~n_b + 1 dependent stages instead of 2 n_b - 1.  Per stage every CTA of
// the cluster multiplies its row slice of the two next block inverses
// (streamed from HBM by TMA into a 2-deep shared-memory ring) with the
// exchanged block vectors on the FP64 tensor cores (DMMA m8n8k4, 3M complex
// product, ds_mma.cuh), applies the chain update and multicasts its rows of
// the next vector to every CTA of the cluster (cp.async.bulk multicast,
// completing on one mbarrier per stage parity).  Arithmetic 16 n_b m^2 flop
// per (visit, RHS); the factor bytes n_b m^2 16 are read once per RHS chunk.
// DESIGN.md §4 "K3" has the version history (v1-v7 measured slower and
// removed; tools/ holds their microbenchmarks).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <tuple>
#include <vector>

#include "ds_common.cuh"
#include "ds_mma.cuh"

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
__device__ __forceinline__ bool mbar_try(uint64_t *bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Bounded spin: a protocol error traps (a CUDA error on the host) instead of
// hanging the GPU.  ~2^22 polls of a suspending try_wait is seconds.
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  for (uint32_t i = 0; !mbar_try(bar, parity); ++i)
    if (i > (1u << 22)) __trap();
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

#ifndef FAC_STAGES
#define FAC_STAGES 2
#endif

#ifdef DS_SOLVE_TRACE5
// v5 phase trace: thread 0 of cluster rank 0 of the first (visit, chunk) of
// every launch appends [stage][phase] clock64 stamps (tools/trace_solve5.py)
__device__ long long g_tr5[64][16][160][12];
__device__ int g_tr5_n;
#define TRACE5(i)                                        \
  if (tr5 >= 0 && t == 0 && s < 160) g_tr5[tr5][rank & 15][s][(i)] = clock64();
#else
#define TRACE5(i)
#endif

// multicast TMA: global -> the same shared offset of every CTA in `mask`,
// completing on each receiver's mbarrier at the same offset
__device__ __forceinline__ void bulk_g2s_multicast(void *dst, const void *src, uint32_t bytes,
                                                   uint64_t *bar, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster "
      "[%0], [%1], %2, [%3], %4;\n" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;\n" ::: "memory");
}

// K3 v8: v5's schedule (fused halves, 256 threads, TMA issue spread over
// warps 0/4 (multicasts) and 2/6 (factor tiles)) with v6's loop-invariant
// addressing and the row-tile count MT as a template parameter (1 for
// 16-CTA clusters, 2 for 8-CTA ones), so only the (NT, X2) product variants
// are inlined: fewer registers, no spills, no per-stage integer division.
#ifdef K3_TILE_CPASYNC
// factor tiles by per-thread cp.async (LDGSTS) instead of TMA bulk copies:
// leaves the SM's TMA unit to the exchange multicasts; each thread's copies
// arrive on the tile mbarrier (count = threads) when they complete
__device__ __forceinline__ void cp_async16(void *dst, const void *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_arrive(uint64_t *bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
#endif

template <int MT, int NW>
__global__ void __launch_bounds__(64 * NW, 1)
    k_block_solve8(const SolveVisit *__restrict__ visits, int nrhs, int rc, int rows_max) {
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int C = (int)cluster.num_blocks();
  // grid (cluster rank, RHS chunk, visit): the block scheduler dispatches
  // y fastest after x, so the chunks of one visit are co-resident and stream
  // the visit's factor tiles through L2 together instead of once each
  const SolveVisit V = visits[blockIdx.z];
  const FactDev f = *V.f;
  const int m = f.m, nb = f.nb, tw = f.twist;
  const int chunk0 = blockIdx.y * rc;
  const int rg = min(rc, nrhs - chunk0);
  const int t = threadIdx.x;
  constexpr int HT = 32 * NW, NT_ = 2 * HT;  // threads per half / per CTA
  const int hh = t / HT, tl = t % HT;
  if (V.nz) {
    int any = 0;
    for (int r = 0; r < rg; ++r) any |= V.nz[chunk0 + r];
    if (!any) return;
  }
  const int rows_per = (m + C - 1) / C;
  const int r0 = rank * rows_per;
  const int nr = max(0, min(rows_per, m - r0));
  const int nt = tw, nbt = nb - 1 - tw, F = max(nt, nbt), S = 2 * F + 1;
  const size_t ldx = nrhs;
  const uint16_t mask = (uint16_t)((1u << C) - 1);
  constexpr int NSL = NW;  // K-slices = warps per half

  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t *vbar = (uint64_t *)smem_raw;   // [2 parity]
  uint64_t *fbar = vbar + 2;               // [2 halves][FAC_STAGES]
  cplx *vec = (cplx *)(smem_raw + 256);    // [2 halves][2 parity][vstride]
  const int vstride = m * rc + 2;
  cplx *fac = vec + 4 * vstride;           // [2 halves][FAC_STAGES][fstride]
  const int fstride = ((rows_max + 7) & ~7) * m + 2;
  cplx *red = fac + 2 * FAC_STAGES * fstride;  // [2 halves][NSL][rows_max*rc]
  const int rstride = rows_max * rc;
  auto VEC = [&](int h, int p) { return vec + (h * 2 + p) * vstride; };
  cplx *xg = V.xg + (size_t)blockIdx.y * 4 * m * rc;
  auto XG = [&](int h, int p) { return xg + ((size_t)h * 2 + p) * m * rg; };

  auto block_of = [&](int h, int st, int &kind) -> int {
    kind = st < F ? 0 : (st == F ? 1 : 2);
    if (h == 0) {
      if (st < F) return st >= F - nt ? st - (F - nt) : -1;
      if (st == F) return tw;
      int j = st - F - 1;
      return j < nt ? tw - 1 - j : -1;
    }
    if (st < F) return st >= F - nbt ? nb - 1 - (st - (F - nbt)) : -1;
    if (st == F) return -1;
    int j = st - F - 1;
    return j < nbt ? tw + 1 + j : -1;
  };
  auto fseq = [&](int h, int st) {
    if (h == 0) return st - (F - nt);
    return st < F ? st - (F - nbt) : st - (F - nbt) - 1;
  };
  auto deliveries = [&](int st) {
    if (st < 0 || st >= S) return 0;
    int kind, n = 0;
    if (block_of(0, st, kind) >= 0) ++n;
    if (block_of(1, st, kind) >= 0 && st != F + 1) ++n;
    if (st == F && nbt > 0) ++n;
    return n;
  };
  const uint32_t vec_bytes = (uint32_t)(m * rg * sizeof(cplx));
  const uint32_t fac_bytes = (uint32_t)(nr * m * sizeof(cplx));
  const uint32_t push_bytes = (uint32_t)(nr * rg * sizeof(cplx));
  auto load_tile = [&](int h, int st) {
    int kind, k = block_of(h, st, kind);
    if (k < 0) return;
    const int q = fseq(h, st), slot = q % FAC_STAGES;
    uint64_t *bar = &fbar[h * FAC_STAGES + slot];
#ifdef K3_TILE_CPASYNC
    // all threads: 16-byte pieces, then an arrival when they complete
    const char *src = (const char *)(f.sinv + ((size_t)k * m + r0) * m);
    char *dst = (char *)(fac + (h * FAC_STAGES + slot) * fstride);
    for (uint32_t b = (uint32_t)t * 16; b < fac_bytes; b += 16 * NT_) cp_async16(dst + b, src + b);
    cp_async_arrive(bar);
#else
    mbar_expect_tx(bar, fac_bytes);
    if (fac_bytes)
      bulk_g2s(fac + (h * FAC_STAGES + slot) * fstride, f.sinv + ((size_t)k * m + r0) * m, fac_bytes, bar);
#endif
  };
  auto push = [&](int h, int p) {
    if (push_bytes)
      bulk_g2s_multicast(VEC(h, p) + r0 * rg, XG(h, p) + r0 * rg, push_bytes, &vbar[p], mask);
  };
  constexpr int TILE_T[2] = {64, HT + 64};  // factor-tile issuers (warp 2 of each half)

#ifdef DS_SOLVE_TRACE5
  int tr5 = -1;
  if (t == 0 && blockIdx.y == 0 && blockIdx.z == 0) {
    tr5 = *(volatile int *)&g_tr5_n;
    if (tr5 >= 64) tr5 = -1;
  }
#endif
  if (t == 0) {
    mbar_init(&vbar[0], 1);
    mbar_init(&vbar[1], 1);
#ifdef K3_TILE_CPASYNC
    for (int i = 0; i < 2 * FAC_STAGES; ++i) mbar_init(&fbar[i], NT_);
#else
    for (int i = 0; i < 2 * FAC_STAGES; ++i) mbar_init(&fbar[i], 1);
#endif
    fence_mbar_init();
  }
  cluster.sync();
#ifdef DS_SOLVE_TRACE5
  if (t == 0 && rank == 0 && blockIdx.y == 0 && blockIdx.z == 0) atomicAdd(&g_tr5_n, 1);
#endif
  if (t == 0) {
    mbar_expect_tx(&vbar[0], deliveries(0) * vec_bytes);
    if (S > 1) mbar_expect_tx(&vbar[1], deliveries(1) * vec_bytes);
  }
  for (int st = 0; st < FAC_STAGES - 1 && st < S; ++st) {
#ifdef K3_TILE_CPASYNC
    load_tile(0, st);
    load_tile(1, st);
#else
    if (t == TILE_T[0]) load_tile(0, st);
    if (t == TILE_T[1]) load_tile(1, st);
#endif
  }
  for (int h = 0; h < 2; ++h) {
    if (h == 1 && nbt == 0) break;
    const int st0 = h == 0 ? F - nt : F - nbt;
    const int k0 = h == 0 ? 0 : nb - 1;
    for (int e = t; e < nr * rg; e += NT_) {
      int row = e / rg, c = e % rg;
      XG(h, st0 & 1)[(r0 + row) * rg + c] = V.rhs[((size_t)k0 * m + r0 + row) * ldx + chunk0 + c];
    }
  }
  fence_proxy_async_global();
  __syncthreads();
  if (t == 0) push(0, (F - nt) & 1);
  if (t == HT && nbt > 0) push(1, (F - nbt) & 1);

  // ---- loop invariants: my (up to 2) outputs of my half
  const int nout = nr * rg;
  const size_t blk = (size_t)m * ldx;
  constexpr int NU = NW >= 8 ? 1 : 2;  // outputs per thread (<= 256 per half)
  int xoff[NU];
  size_t goff[NU];
  bool has[NU];
#pragma unroll
  for (int u = 0; u < NU; ++u) {
    const int o = tl + u * HT;
    has[u] = o < nout;
    const int orow = has[u] ? o / rg : 0, oc = has[u] ? o % rg : 0;
    xoff[u] = (r0 + orow) * rg + oc;
    goff[u] = (size_t)(r0 + orow) * ldx + chunk0 + oc;
  }
  const int warp = tl >> 5, lane = t & 31, g = lane >> 2, tg = lane & 3;
  const int nk = (m + 3) >> 2, kb = (warp * nk) / NW, ke = ((warp + 1) * nk) / NW;
  const int NT = (rg + 7) >> 3;
  cplx *rp = red + ((size_t)hh * NSL + warp) * rstride;
  const cplx *rq = red + (size_t)hh * NSL * rstride;
  uint32_t vph = 0;

  for (int s = 0; s < S; ++s) {
    const int p = s & 1;
    TRACE5(0);
    if (s + FAC_STAGES - 1 < S) {
#ifdef K3_TILE_CPASYNC
      load_tile(0, s + FAC_STAGES - 1);
      load_tile(1, s + FAC_STAGES - 1);
#else
      if (t == TILE_T[0]) load_tile(0, s + FAC_STAGES - 1);
      if (t == TILE_T[1]) load_tile(1, s + FAC_STAGES - 1);
#endif
    }
    TRACE5(8);
    int kind, k = block_of(hh, s, kind);
    const bool act = k >= 0;
    cplx aux[NU];
#pragma unroll
    for (int u = 0; u < NU; ++u) aux[u] = make_double2(0.0, 0.0);
    cplx coef = make_double2(0.0, 0.0);
    if (act) {
      if (kind == 0) {
        coef = hh == 0 ? f.lcoef[k + 1] : f.ucoef[k - 1];
        const int kn = hh == 0 ? k + 1 : k - 1;
        if (hh == 0 || kn > tw) {
          const cplx *src = V.rhs + (size_t)kn * blk;
#pragma unroll
          for (int u = 0; u < NU; ++u)
            if (has[u]) aux[u] = src[goff[u]];
        }
      } else if (kind == 2) {
        coef = hh == 0 ? f.ucoef[k] : f.lcoef[k];
        const cplx *src = V.x + (size_t)k * blk;
#pragma unroll
        for (int u = 0; u < NU; ++u)
          if (has[u]) aux[u] = __ldcg(src + goff[u]);
      }
    }
    TRACE5(9);
    const int q = act ? fseq(hh, s) : 0;
    if (act) mbar_wait(&fbar[hh * FAC_STAGES + q % FAC_STAGES], (q / FAC_STAGES) & 1);
    TRACE5(1);
    mbar_wait(&vbar[p], (vph >> p) & 1);
    if (t == 0 && s + 2 < S) mbar_expect_tx(&vbar[p], deliveries(s + 2) * vec_bytes);
    vph ^= 1u << p;
    TRACE5(2);
    if (act) {
      const cplx *A = fac + (hh * FAC_STAGES + q % FAC_STAGES) * fstride;
      const cplx *X = VEC((hh == 1 && s == F + 1) ? 0 : hh, p);
      const cplx *X2 = (kind == 1 && nbt > 0) ? VEC(1, p) : nullptr;
      double cr[2][2][2] = {}, ci[2][2][2] = {};
#ifdef K3_NO_COMPUTE
      if (false)
#endif
      {
        const int sel = (NT > 1 ? 2 : 0) + (X2 ? 1 : 0);
#define K3_PRODUCT(nt_, x2_) mma_product<MT, nt_, x2_>(A, m, X, X2, rg, m, kb, ke, g, tg, cr, ci)
        switch (sel) {
          case 0: K3_PRODUCT(1, false); break;
          case 1: K3_PRODUCT(1, true); break;
          case 2: K3_PRODUCT(2, false); break;
          default: K3_PRODUCT(2, true); break;
        }
#undef K3_PRODUCT
      }
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int ntt = 0; ntt < 2; ++ntt)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int row = mt * 8 + g, col = ntt * 8 + 2 * tg + e;
            if (ntt < NT && row < nr && col < rg)
              rp[row * rg + col] = make_double2(cr[mt][ntt][e], ci[mt][ntt][e]);
          }
    }
    TRACE5(3);
    __syncthreads();
    TRACE5(4);
    const bool last = s + 1 >= S;
    cplx outv[NU];
    if (act) {
      cplx *xgo = XG(hh, p ^ 1);
#pragma unroll
      for (int u = 0; u < NU; ++u) {
        if (!has[u]) continue;
        const int o = tl + u * HT;
        cplx acc = rq[o];  // K-slices in a fixed order (deterministic)
#pragma unroll
        for (int q2 = 1; q2 < NSL; ++q2) acc = cadd(acc, rq[o + q2 * rstride]);
        cplx out, nxt;
        if (kind == 0) {
          out = acc;
          nxt = csub(aux[u], cmul(coef, acc));
        } else if (kind == 1) {
          out = acc;
          nxt = acc;
        } else {
          out = csub(aux[u], cmul(coef, acc));
          nxt = out;
        }
        outv[u] = out;
        if (!last) xgo[xoff[u]] = nxt;
      }
    }
    TRACE5(5);
    fence_proxy_async_global();
    __syncthreads();
    TRACE5(6);
    if (tl == 0 && !last) {
      int kd;
      if (hh == 0 && block_of(0, s, kd) >= 0 && block_of(0, s + 1, kd) >= 0) push(0, p ^ 1);
      if (hh == 1 && block_of(1, s, kd) >= 0 && (block_of(1, s + 1, kd) >= 0 || s + 1 == F))
        push(1, p ^ 1);
    }
    if (act) {
      cplx *dst = V.x + (size_t)k * blk;
#pragma unroll
      for (int u = 0; u < NU; ++u)
        if (has[u]) dst[goff[u]] = outv[u];
    }
    TRACE5(7);
  }
  cluster.sync();
}

static size_t solve8_smem(int m, int rc, int C, int nw = 4) {
  int r = (m + C - 1) / C;
  size_t rows_max = r + (r & 1);
  size_t rows_alloc = (rows_max + 7) & ~(size_t)7;
  size_t elems = 4 * ((size_t)m * rc + 2) + 2 * FAC_STAGES * (rows_alloc * m + 2) + 2 * (size_t)nw * rows_max * rc;
  // floor: one CTA per SM (the chain is latency bound: two CTAs sharing an
  // SM would serialise their stages; the wave count assumes one per SM)
  return std::max<size_t>(256 + elems * sizeof(cplx), (size_t)118 * 1024);
}

static int solve_rows_max(int max_m, int C) {
  int r = (max_m + C - 1) / C;
  return r + (r & 1);  // even: 2-row micro-tiles may read one padding row
}


// Co-resident clusters of C CTAs for this footprint (7 x 16 on a 148-SM B200).
static int solve_max_clusters(const void *fn, int threads, int C, size_t smem) {
  static std::vector<std::tuple<const void *, int, int, size_t, int>> memo;
  for (auto &e : memo)
    if (std::get<0>(e) == fn && std::get<1>(e) == threads && std::get<2>(e) == C &&
        std::get<3>(e) == smem)
      return std::get<4>(e);
  cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3(C, 1, 1);
  cfg.blockDim = dim3(threads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, fn, &cfg) != cudaSuccess || n < 0) {
    cudaGetLastError();
    n = 0;
  }
  memo.emplace_back(fn, threads, C, smem, n);
  return n;
}
// Choose the (cluster size, RHS chunk) that runs a step of nvisit visits in
// the fewest waves of co-resident clusters, then the smallest cluster, then
// the least arithmetic per CTA and stage (rows per CTA x chunk width).
template <typename SmemFn>
static bool pick_cluster_chunk(const ds_ctx *ctx, const void *fn, int threads, int nvisit, int nrhs,
                               int max_m, bool mma, SmemFn smem_of, int *Cout, int *rcout,
                               long *waves_out) {
  const int rc_min = std::max(1, ctx->opt.k3_rc_min);
  const int rc_max = std::max(1, ctx->opt.k3_rc_max);
  const int c_only = ctx->opt.k3_cluster;
  int bestC = 0, bestRc = 0;
  long best_waves = 0, best_work = 0, best_waste = 0;
  // cluster sizes need not be powers of two: a 131-row slab (config 3) fits
  // 9 CTAs of 16 rows, two clusters per GPC, where 16-CTA clusters (10
  // rows, 6 of them padding) fit one per GPC -- 7 co-resident on 148 SMs
  for (int C : {16, 12, 10, 9, 8}) {
    if (c_only && C != c_only) continue;
    const int rows = solve_rows_max(max_m, C);
    for (int rc = std::min(nrhs, rc_max); rc >= 1; rc = rc > 1 ? (rc + 1) / 2 : 0) {
      if (rc < std::min(rc_min, nrhs) && bestC) break;
      if (rows * rc > 256 || (mma && rows > 16)) continue;
      size_t smem = smem_of(rc, C);
      if (smem > 232448) continue;
      int maxcl = solve_max_clusters(fn, threads, C, smem);
      if (maxcl < 1) continue;
      long ncl = (long)nvisit * ((nrhs + rc - 1) / rc);
      long waves = (ncl + maxcl - 1) / maxcl;
      long work = waves * (long)rows * rc;
      // DMMA tile padding: rows and RHS are computed in 8 x 8 tiles
      long waste = (long)((rows + 7) / 8 * 8) * ((rc + 7) / 8 * 8) - (long)rows * rc;
      // ties (same waves and work per CTA): less padding, then the smaller
      // cluster -- config 2 measured 8 CTAs x (16 rows, 8 RHS) faster than
      // 16 CTAs x (8 rows, 16 RHS): half as many CTAs in every exchange
      // same waves: the smaller cluster (config 3: with two RHS groups on
      // two streams, launches that pick 16-CTA clusters for less work per
      // CTA fragment the GPCs under the other group's 9-CTA clusters --
      // 125 RHS/s against 151 with 9-CTA clusters throughout)
      bool better = !bestC || waves < best_waves || (waves == best_waves && C < bestC) ||
                    (waves == best_waves && C == bestC && work < best_work);
      if (!better && waves == best_waves && C == bestC && work == best_work)
        better = waste < best_waste;
      if (better) {
        bestC = C;
        bestRc = rc;
        best_waves = waves;
        best_work = work;
        best_waste = waste;
      }
      if (rc == 1) break;
    }
  }
  *Cout = bestC;
  *rcout = bestRc;
  *waves_out = best_waves;
  return bestC != 0;
}

static int launch_v8(ds_ctx *ctx, const void *visits_dev, int nvisit, int nrhs, int max_m) {
  // warps per half: 4 (256 threads) or 8 (512 threads, more latency hiding
  // for the lockstep DMMA product, 128 registers)
  const int nw = ctx->opt.k3_warps >= 8 ? 8 : 4;
  const int threads = 64 * nw;
  const void *fn16 = nw == 8 ? (const void *)k_block_solve8<1, 8> : (const void *)k_block_solve8<1, 4>;
  int C, rc;
  long waves;
  if (!pick_cluster_chunk(ctx, fn16, threads, nvisit, nrhs, max_m, true,
                          [&](int r, int c) { return solve8_smem(max_m, r, c, nw); }, &C, &rc, &waves))
    return ds_fail(DS_ECONFIG, "block solve v8: no feasible cluster configuration");
  const int rows = solve_rows_max(max_m, C);
  const void *fn = rows > 8 ? (nw == 8 ? (const void *)k_block_solve8<2, 8> : (const void *)k_block_solve8<2, 4>)
                            : fn16;
  const size_t smem = solve8_smem(max_m, rc, C, nw);
  cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  DS_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3(C, (nrhs + rc - 1) / rc, nvisit);
  cfg.blockDim = dim3(threads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const SolveVisit *vt = (const SolveVisit *)visits_dev;
  const int rmax = solve_rows_max(max_m, C);
  if (nw == 8) {
    if (rows > 8)
      DS_CUDA(cudaLaunchKernelEx(&cfg, k_block_solve8<2, 8>, vt, nrhs, rc, rmax));
    else
      DS_CUDA(cudaLaunchKernelEx(&cfg, k_block_solve8<1, 8>, vt, nrhs, rc, rmax));
  } else {
    if (rows > 8)
      DS_CUDA(cudaLaunchKernelEx(&cfg, k_block_solve8<2, 4>, vt, nrhs, rc, rmax));
    else
      DS_CUDA(cudaLaunchKernelEx(&cfg, k_block_solve8<1, 4>, vt, nrhs, rc, rmax));
  }
  ctx->launches++;
  return DS_OK;
}

int ds_launch_solve_table(ds_ctx *ctx, const void *visits_dev, int nvisit, int nrhs,
                          int max_m) {
  if (nvisit < 1) return DS_OK;
  return launch_v8(ctx, visits_dev, nvisit, nrhs, max_m);
}

#ifdef DS_SOLVE_TRACE5
extern "C" DS_API int ds_debug_solve_trace5(long long *out, int *count) {
  DS_CUDA(cudaDeviceSynchronize());
  DS_CUDA(cudaMemcpyFromSymbol(out, g_tr5, sizeof(long long) * 64 * 16 * 160 * 12));
  DS_CUDA(cudaMemcpyFromSymbol(count, g_tr5_n, sizeof(int)));
  return DS_OK;
}
extern "C" DS_API int ds_debug_solve_trace5_reset() {
  int z = 0;
  DS_CUDA(cudaMemcpyToSymbol(g_tr5_n, &z, sizeof(int)));
  return DS_OK;
}
#endif
