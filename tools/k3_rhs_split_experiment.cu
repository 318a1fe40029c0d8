// EXPERIMENT (not built): K3 v4, RHS-split block substitution with multicast
// factor panels.  Correct (passes the GPU parity suite) but slower than the
// row-split K3 in csrc/ds_solve.cu: the multicast ring is latency-bound
// ("K3 design history").

// K3: batched block substitution of the twisted block-tridiagonal LU (see
// ds_factor.cu) — one launch per anti-diagonal step, one thread-block
// cluster per (subdomain visit, RHS chunk).  Replaces Factorization.solve
// (diagsweep/subdomain.py:77-106, :127-133) as called at ddm.py:259.
//
// With twist t (top blocks 0..t-1, middle t, bottom t+1..n_b-1):
//   top fwd    y_k = S_k^{-1} (b_k - l_k y_{k-1})             k = 0..t-1
//   bottom fwd z_k = T_k^{-1} (b_k - u_k z_{k+1})             k = n_b-1..t+1
//   middle     x_t = M_t^{-1} (b_t - l_t y_{t-1} - u_t z_{t+1})
//   top bwd    x_k = y_k - u_k S_k^{-1} x_{k+1}               k = t-1..0
//   bottom bwd x_k = z_k - l_k T_k^{-1} x_{k-1}               k = t+1..n_b-1
//
// Decomposition (measured): each CTA owns a pack of rg
// right-hand sides and computes ALL m rows of every block product, so a
// substitution chain never leaves the CTA.  The cluster exists only to
// share the factor stream: per half, one issuer CTA multicasts row panels
// of the block inverses (TMA, global -> every CTA of the half) into a
// shared-memory ring guarded by full/empty mbarriers, so each panel is read
// from L2 once per cluster.  The top and bottom CTAs of a pack exchange
// vectors only at the middle block (two bulk shared::cluster copies).
// Arithmetic: 16 n_b m^2 flop per (visit, RHS), FP64 FMA; factor bytes
// 2 n_b m^2 16 per visit and RHS chunk.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
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
__device__ __forceinline__ bool mbar_try(uint64_t *bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
#ifdef DS_MBAR_TRYWAIT
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
#else
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
#endif
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
    if (i > (1u << 30)) __trap();
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

#define NS 3        // panel ring depth
#define PR 32       // rows per factor panel
#define RGMAX 8     // max right-hand sides per CTA

#ifdef DS_SOLVE_TRACE
// clock64 per (rank, item): 0 item start, 1 first panel landed,
// 2 panels done, 3 epilogue done, 4 summed panel-wait cycles
__device__ long long g_solve_trace[16][1024][6];
#define TRACE(i, v)                                                              \
  if (t == 0 && blockIdx.y == 0 && blockIdx.z == 0 && rank < 16 && it < 1024)   \
    g_solve_trace[rank][it][i] = (v);
#else
#define TRACE(i, v)
#endif

__device__ __forceinline__ void bulk_g2s_multicast(void *dst, const void *src, uint32_t bytes,
                                                   uint64_t *bar, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster "
      "[%0], [%1], %2, [%3], %4;\n" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void mbar_remote_arrive(uint64_t *bar_local, uint32_t rank) {
  uint32_t rbar;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(rbar) : "r"(smem_u32(bar_local)), "r"(rank));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(rbar) : "memory");
}
__device__ __forceinline__ void cp_async16(void *dst, const void *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;\n" ::: "memory");
}

struct SolveGeom {
  int m, nb, tw, nt, nbt;
};

// block / kind of item i of half h (kind 0 fwd, 1 middle, 2 bwd)
__device__ __forceinline__ int item_block(const SolveGeom &g, int h, int i, int &kind) {
  if (h == 0) {
    if (i < g.nt) { kind = 0; return i; }
    if (i == g.nt) { kind = 1; return g.tw; }
    kind = 2;
    return g.tw - 1 - (i - g.nt - 1);
  }
  if (i < g.nbt) { kind = 0; return g.nb - 1 - i; }
  kind = 2;
  return g.tw + 1 + (i - g.nbt);
}

template <int RG>
__global__ void __launch_bounds__(SOLVE_THREADS, 1)
    k_block_solve(const SolveVisit *__restrict__ visits, int nrhs, int npc) {
  constexpr int rg = RG;
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const SolveVisit V = visits[blockIdx.y];
  const FactDev f = *V.f;
  SolveGeom G;
  G.m = f.m;
  G.nb = f.nb;
  G.tw = f.twist;
  G.nt = G.tw;
  G.nbt = G.nb - 1 - G.tw;
  const int m = G.m;
  const int t = threadIdx.x;
  const int h = rank / npc, pk = rank % npc;
  const int chunk0 = blockIdx.z * npc * rg;
  const int c0 = chunk0 + pk * rg;
  const int rgc = max(0, min(rg, nrhs - c0));
  const size_t ldx = nrhs;

  if (V.nz) {  // skip visits whose right-hand sides are all exactly zero
    int any = 0;
    for (int r = chunk0; r < min(nrhs, chunk0 + npc * rg); ++r) any |= V.nz[r];
    if (!any) return;  // uniform across the cluster (before any barrier)
  }
  const int nitems = h == 0 ? 2 * G.nt + 1 : 2 * G.nbt;
  const int np = (m + PR - 1) / PR;  // panels per block
  const int issuer = h * npc;
  const uint16_t hmask = (uint16_t)(((1u << npc) - 1) << (h * npc));

  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t *full = (uint64_t *)smem_raw;  // [NS]
  uint64_t *empty = full + NS;            // [NS]   (issuer only)
  uint64_t *xbar = empty + NS;            // [2]: 0 bottom part -> top, 1 x_t -> bottom
  cplx *ring = (cplx *)(smem_raw + 128);  // [NS][PR*m]
  cplx *vin = ring + NS * PR * m;         // [m*rg] current input vector
  cplx *ybuf = vin + m * rg;              // [m*rg] block product
  cplx *abuf = ybuf + m * rg;             // [m*rg] epilogue operand
  cplx *xch = abuf + m * rg;              // [m*rg] middle exchange landing buffer
  cplx *sbuf = xch + m * rg;              // [m*rg] middle exchange source (sent once)

  auto panel_rows = [&](int j) { return min(PR, m - j * PR); };
  auto issue_panel = [&](int q) {  // issuer thread 0: panel q of this half
    int kind, k = item_block(G, h, q / np, kind);
    int j = q % np, slot = q % NS;
    uint32_t bytes = (uint32_t)(panel_rows(j) * m * sizeof(cplx));
    bulk_g2s_multicast(ring + slot * PR * m, f.sinv + ((size_t)k * m + j * PR) * m, bytes,
                       &full[slot], hmask);
  };
  auto arm_full = [&](int q) {  // every CTA's thread 0: expect panel q
    int j = q % np;
    mbar_expect_tx(&full[q % NS], (uint32_t)(panel_rows(j) * m * sizeof(cplx)));
  };

  if (t == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], npc);
    }
    mbar_init(&xbar[0], 1);
    mbar_init(&xbar[1], 1);
    fence_mbar_init();
  }
  cluster.sync();  // every barrier of the cluster exists before any traffic
  const int nq = nitems * np;
  if (t == 0 && nitems > 0) {
    for (int q = 0; q < NS && q < nq; ++q) arm_full(q);
    if (h == 0 && G.nbt > 0) mbar_expect_tx(&xbar[0], (uint32_t)(m * rg * sizeof(cplx)));
    if (h == 1) mbar_expect_tx(&xbar[1], (uint32_t)(m * rg * sizeof(cplx)));
  }
  cluster.sync();  // all receivers armed before the first multicast lands
  if (t == 0 && rank == issuer && nitems > 0)
    for (int q = 0; q < NS && q < nq; ++q) issue_panel(q);

  // initial input: b_0 (top) or b_{n_b-1} (bottom) for my right-hand sides
  if (nitems > 0) {
    const int k0 = h == 0 ? 0 : G.nb - 1;
    for (int e = t; e < m * rg; e += SOLVE_THREADS) {
      int row = e / rg, c = e % rg;
      vin[c * m + row] = c < rgc ? V.rhs[((size_t)k0 * m + row) * ldx + c0 + c] : make_double2(0.0, 0.0);
    }
  }
  __syncthreads();

  // compute mapping: thread = (panel row t>>3, K slice t&7); each thread
  // keeps all RG columns of its row in registers, so a factor element is
  // loaded once and used RG times and the vector loads broadcast across the
  // four rows a warp covers
  const int prow_t = t >> 3, ksl = t & 7;
  int q = 0;                      // panel sequence number
  for (int it = 0; it < nitems; ++it) {
    int kind, k = item_block(G, h, it, kind);
    TRACE(0, clock64());
    long long wsum = 0;
    // epilogue operand, streamed in while the block product runs
    const cplx *asrc = nullptr;
    if (kind == 0) {
      int kn = h == 0 ? k + 1 : k - 1;
      if (h == 0 || kn > G.tw) asrc = V.rhs + (size_t)kn * m * ldx;
    } else if (kind == 2) {
      asrc = V.x + (size_t)k * m * ldx;
    }
    if (asrc && rgc == rg && (ldx * sizeof(cplx)) % 16 == 0) {
      for (int e = t; e < m * rg; e += SOLVE_THREADS)
        cp_async16(abuf + e, asrc + (size_t)(e / rg) * ldx + c0 + (e % rg));
    } else {
      for (int e = t; e < m * rg; e += SOLVE_THREADS) {
        int row = e / rg, c = e % rg;
        abuf[e] = (asrc && c < rgc) ? __ldcg(asrc + (size_t)row * ldx + c0 + c) : make_double2(0.0, 0.0);
      }
    }
    if (kind == 1 && G.nbt > 0) {  // middle: add the bottom chain's part
      mbar_wait(&xbar[0], 0);
      for (int e = t; e < m * rg; e += SOLVE_THREADS) vin[e] = cadd(vin[e], xch[e]);  // both [c][m]
      __syncthreads();
    }
    if (h == 1 && it == G.nbt) {  // bottom's first backward block uses x_t
      mbar_wait(&xbar[1], 0);
      for (int e = t; e < m * rg; e += SOLVE_THREADS) vin[e] = xch[e];
      __syncthreads();
    }
    // ---- ybuf = (block inverse) * vin, panel by panel
    for (int j = 0; j < np; ++j, ++q) {
      const int slot = q % NS;
      long long w0 = clock64();
      mbar_wait(&full[slot], (q / NS) & 1);
      wsum += clock64() - w0;
      if (j == 0) TRACE(1, clock64());
      const cplx *A = ring + slot * PR * m;
      const int prow = panel_rows(j);
      {
        cplx acc[2][RG];
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
          for (int c = 0; c < RG; ++c) acc[u][c] = make_double2(0.0, 0.0);
        if (prow_t < prow) {
          const cplx *a = A + prow_t * m;
          int kk = ksl;
          for (; kk + 8 < m; kk += 16) {
            const cplx a0 = a[kk], a1 = a[kk + 8];
#pragma unroll
            for (int c = 0; c < RG; ++c) {
              cfma(acc[0][c], a0, vin[c * m + kk]);
              cfma(acc[1][c], a1, vin[c * m + kk + 8]);
            }
          }
          if (kk < m) {
            const cplx a0 = a[kk];
#pragma unroll
            for (int c = 0; c < RG; ++c) cfma(acc[0][c], a0, vin[c * m + kk]);
          }
        }
#pragma unroll
        for (int c = 0; c < RG; ++c) {
          cplx v = cadd(acc[0][c], acc[1][c]);
#pragma unroll
          for (int off = 1; off < 8; off <<= 1) {
            v.x += __shfl_xor_sync(0xffffffffu, v.x, off);
            v.y += __shfl_xor_sync(0xffffffffu, v.y, off);
          }
          if (ksl == 0 && prow_t < prow) ybuf[(j * PR + prow_t) * rg + c] = v;
        }
      }
      __syncthreads();  // every thread is done with this slot
      if (t == 0) {
        if (q + NS < nq) arm_full(q + NS);
        mbar_remote_arrive(&empty[slot], issuer);
        if (rank == issuer && q + NS < nq) {
          mbar_wait(&empty[slot], (q / NS) & 1);  // all consumers released it
          issue_panel(q + NS);
        }
      }
    }
    TRACE(2, clock64());
    TRACE(4, wsum);
    cp_async_wait_all();
    __syncthreads();
    // ---- epilogue: outputs and the next input vector
    const bool last = it + 1 == nitems;
    const bool send_mid = (h == 1 && kind == 0 && it == G.nbt - 1);  // bottom part -> top
    const bool send_xt = (h == 0 && kind == 1 && G.nbt > 0);          // x_t -> bottom
    for (int e = t; e < m * rgc; e += SOLVE_THREADS) {
      const int row = e / rgc, c = e % rgc, idx = row * rg + c;
      const cplx y = ybuf[idx];
      const size_t off = ((size_t)k * m + row) * ldx + c0 + c;
      cplx out, nxt;
      if (kind == 0) {
        out = y;  // y_k (top) / z_k (bottom)
        nxt = h == 0 ? csub(abuf[idx], cmul(f.lcoef[k + 1], y)) : csub(abuf[idx], cmul(f.ucoef[k - 1], y));
      } else if (kind == 1) {
        out = y;  // x_t
        nxt = y;
      } else {
        out = csub(abuf[idx], cmul(h == 0 ? f.ucoef[k] : f.lcoef[k], y));
        nxt = out;
      }
      V.x[off] = out;
      if (!last) vin[c * m + row] = nxt;
      if (send_mid || send_xt) sbuf[c * m + row] = nxt;
    }
    if (send_mid || send_xt) {
      fence_proxy_async();
      __syncthreads();
      if (t == 0) {
        // partner: same pack in the other half; lands in its xch buffer
        uint32_t partner = (uint32_t)((1 - h) * npc + pk);
        bulk_s2peer(xch, sbuf, (uint32_t)(m * rg * sizeof(cplx)), &xbar[send_mid ? 0 : 1], partner);
      }
    }
    __syncthreads();
    TRACE(3, clock64());
  }
  cluster.sync();  // no CTA leaves while multicasts into it may be in flight
}

static int env_int(const char *name, int dflt) {
  const char *v = getenv(name);
  return v && *v ? atoi(v) : dflt;
}

static size_t solve_smem(int m, int rg) {
  return 128 + ((size_t)NS * PR * m + 5 * (size_t)m * rg) * sizeof(cplx);
}

int ds_launch_solve_table(ds_ctx *ctx, const void *visits_dev, int nvisit, int nrhs,
                          int max_m) {
  if (nvisit < 1) return DS_OK;
  // right-hand sides per CTA: enough that 2 * ceil(nrhs/rg) * nvisit CTAs
  // fit on the GPU at one CTA per SM (one wave), capped at RGMAX
  int rg = env_int("DS_SOLVE_RG", 0);
  if (rg <= 0) {
    rg = (2 * nrhs * nvisit + ctx->num_sms - 1) / ctx->num_sms;
    rg = std::max(1, std::min(RGMAX, rg));
  }
  rg = std::min(rg, nrhs);
  rg = rg <= 1 ? 1 : (rg <= 2 ? 2 : (rg <= 4 ? 4 : 8));  // template instances
  int packs = (nrhs + rg - 1) / rg;
  int npc = std::min(env_int("DS_SOLVE_NPC", 8), packs);  // packs per cluster (2*npc CTAs)
  int nchunks = (packs + npc - 1) / npc;
  int C = 2 * npc;
  size_t smem = solve_smem(max_m, rg);
  if (smem > 232448) return ds_fail(DS_ECONFIG, "block solve: slab too large for the panel ring");
  void (*kern)(const SolveVisit *, int, int) =
      rg == 1 ? k_block_solve<1> : rg == 2 ? k_block_solve<2> : rg == 4 ? k_block_solve<4> : k_block_solve<8>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  DS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
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
  DS_CUDA(cudaLaunchKernelEx(&cfg, kern, (const SolveVisit *)visits_dev, nrhs, npc));
  ctx->launches++;
  return DS_OK;
}

#ifdef DS_SOLVE_TRACE
extern "C" DS_API int ds_debug_solve_trace(long long *out) {
  DS_CUDA(cudaMemcpyFromSymbol(out, g_solve_trace, sizeof(long long) * 16 * 1024 * 6));
  return DS_OK;
}
#endif
