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
#define GMAX 4

#ifdef DS_SOLVE_TRACE
__device__ long long g_solve_trace[2][1024][6];
// slot 0: stage start; 1/2/3: top chain after wait / compute / epilogue;
// 4/5: bottom chain after wait / epilogue
// slots: 0 stage start; top 1 after vec wait, 2 after compute, 3 after epilogue;
// bottom 4 after vec wait, 5 after epilogue; 6/7 after the top/bottom factor wait
#define TRACE(i)                                                                   \
  if (t == 0 && blockIdx.y == 0 && blockIdx.z == 0 && rank < 16 && s < 1024 &&    \
      ((i) == 0 || h == 0 || (i) != 2))                                             \
    g_solve_trace[rank][s][(i) == 0 ? 0 : (h == 0 ? (i) : ((i) == 1 ? 4 : 5))] = clock64();
#else
#define TRACE(i)
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

// Twisted block substitution (see ds_factor.cu).  t = twist, nt = t top
// blocks, nbt = n_b-1-t bottom blocks, F = max(nt, nbt); stages 0..2F:
//   forward  top    k = s-(F-nt)        for s in [F-nt, F-1]
//            bottom k = n_b-1-(s-(F-nbt)) for s in [F-nbt, F-1]
//   middle   k = t at s = F, input (b_t - l_t y_{t-1}) + (-u_t z_{t+1})
//   backward top    k = t-1-(s-F-1),  bottom k = t+1+(s-F-1)
// Every (half, RHS group) is an independent chain; within a stage the CTA
// walks its chains so one chain's all-gather (rows -> global -> multicast
// TMA into every CTA's shared vector, completing on an mbarrier) overlaps
// the other chains' compute.
__global__ void __launch_bounds__(SOLVE_THREADS, 1)
    k_block_solve(const SolveVisit *__restrict__ visits, int nrhs, int rc, int G, int rows_max) {
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int C = (int)cluster.num_blocks();
  const SolveVisit V = visits[blockIdx.y];
  const FactDev f = *V.f;
  const int m = f.m, nb = f.nb, tw = f.twist;
  const int chunk0 = blockIdx.z * rc;
  const int rcc = min(rc, nrhs - chunk0);
  const int t = threadIdx.x;
  int s = 0;  // stage (also used by TRACE)

  if (V.nz) {  // skip visits whose right-hand sides are all exactly zero
    int any = 0;
    for (int r = 0; r < rcc; ++r) any |= V.nz[chunk0 + r];
    if (!any) return;  // uniform across the cluster (before any barrier)
  }
  const int Gc = (rcc % G == 0) ? G : 1;  // groups must split the chunk evenly
  const int rg = rcc / Gc;                // RHS per group
  const int rows_per = (m + C - 1) / C;
  const int r0 = rank * rows_per;
  const int nr = max(0, min(rows_per, m - r0));
  const int nt = tw, nbt = nb - 1 - tw, F = max(nt, nbt), S = 2 * F + 1;
  const size_t ldx = nrhs;
  const uint16_t mask = (uint16_t)((1u << C) - 1);

  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t *vbar = (uint64_t *)smem_raw;          // [2 halves][GMAX][2]
  uint64_t *fbar = vbar + 4 * GMAX;               // [2 halves][FAC_STAGES]
  cplx *vec = (cplx *)(smem_raw + 256);           // [2][Gc][2][vstride]
  const int vstride = m * rg + 2;
  cplx *fac = vec + 4 * Gc * vstride;             // [2][FAC_STAGES][fstride]
  const int fstride = rows_max * m + 2;
  cplx *red = fac + 2 * FAC_STAGES * fstride;     // [16][rows_max * rg]
  auto VEC = [&](int h, int g, int p) { return vec + ((h * Gc + g) * 2 + p) * vstride; };
  auto VBAR = [&](int h, int g, int p) { return &vbar[(h * GMAX + g) * 2 + p]; };
  // global exchange scratch of this cluster: [2][GMAX][2][m * rg]
  cplx *xg = V.xg + (size_t)blockIdx.z * 4 * m * rc;
  auto XG = [&](int h, int g, int p) { return xg + ((size_t)(h * Gc + g) * 2 + p) * m * rg; };

  // block processed by half h at stage s (-1: idle).  kind 0 fwd, 1 mid, 2 bwd
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
  // factor-ring sequence index of (half, stage)
  auto fseq = [&](int h, int st) {
    if (h == 0) return st - (F - nt);
    return st < F ? st - (F - nbt) : st - (F - nbt) - 1;
  };
  const uint32_t fac_bytes = (uint32_t)(nr * m * sizeof(cplx));
  const uint32_t vec_bytes = (uint32_t)(m * rg * sizeof(cplx));
  const uint32_t push_bytes = (uint32_t)(nr * rg * sizeof(cplx));
  auto load_tile = [&](int h, int st) {  // thread 0 only
    int kind, k = block_of(h, st, kind);
    if (k < 0) return;
    int q = fseq(h, st), slot = q % FAC_STAGES;
    uint64_t *bar = &fbar[h * FAC_STAGES + slot];
    mbar_expect_tx(bar, fac_bytes);
    if (fac_bytes)
      bulk_g2s(fac + (h * FAC_STAGES + slot) * fstride, f.sinv + ((size_t)k * m + r0) * m, fac_bytes, bar);
  };
  // push my rows of the next-stage vector (already in global) to every CTA
  auto push = [&](int h, int g, int p) {  // thread 0 only, after the fence + barrier
    if (push_bytes)
      bulk_g2s_multicast(VEC(h, g, p) + r0 * rg, XG(h, g, p) + r0 * rg, push_bytes, VBAR(h, g, p), mask);
  };

  if (t == 0) {
    for (int i = 0; i < 4 * GMAX; ++i) mbar_init(&vbar[i], 1);
    for (int i = 0; i < 2 * FAC_STAGES; ++i) mbar_init(&fbar[i], 1);
    fence_mbar_init();
  }
  cluster.sync();  // peers' barriers initialised before any multicast
  // vector-buffer phase counters (uniform across threads)
  int vph[2][GMAX][2];
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int g = 0; g < GMAX; ++g) vph[h][g][0] = vph[h][g][1] = 0;
  if (t == 0) {
    for (int h = 0; h < 2; ++h)
      for (int g = 0; g < Gc; ++g) {
        mbar_expect_tx(VBAR(h, g, 0), vec_bytes);
        mbar_expect_tx(VBAR(h, g, 1), vec_bytes);
      }
    for (int st = 0; st < FAC_STAGES - 1 && st < S; ++st) {  // ring prologue
      load_tile(0, st);
      load_tile(1, st);
    }
  }
  // prologue: b_0 for the top chain (stage F-nt), b_{n_b-1} for the bottom
  // chain (stage F-nbt); written to the exchange scratch then multicast
  for (int h = 0; h < 2; ++h) {
    if (h == 1 && nbt == 0) break;
    const int st0 = h == 0 ? F - nt : F - nbt;
    const int k0 = h == 0 ? 0 : nb - 1;
    for (int g = 0; g < Gc; ++g)
      for (int e = t; e < nr * rg; e += SOLVE_THREADS) {
        int row = e / rg, c = e % rg;
        XG(h, g, st0 & 1)[(r0 + row) * rg + c] =
            V.rhs[((size_t)k0 * m + r0 + row) * ldx + chunk0 + g * rg + c];
      }
  }
  fence_proxy_async_global();
  __syncthreads();
  if (t == 0) {
    for (int g = 0; g < Gc; ++g) push(0, g, (F - nt) & 1);
    if (nbt > 0)
      for (int g = 0; g < Gc; ++g) push(1, g, (F - nbt) & 1);
  }

  const int TR = (nr + 1) / 2, TC = (rg + 1) / 2;
  const int ntile = TR * TC;
  int nslice = ntile > 0 ? SOLVE_THREADS / ntile : 1;
  nslice = max(1, min(16, nslice));
  const int ks = (m + nslice - 1) / nslice;
  const int nout = nr * rg;
  const int orow = t / max(rg, 1), oc = t % max(rg, 1);

  for (s = 0; s < S; ++s) {
    const int p = s & 1;
    { const int h = 0; (void)h; TRACE(0); }
    // refill the factor rings FAC_STAGES-1 stages ahead (slot freed at s-1)
    if (t < 32 && s + FAC_STAGES - 1 < S) {
      load_tile(0, s + FAC_STAGES - 1);
      load_tile(1, s + FAC_STAGES - 1);
    }
    int kindh[2], kh[2];
    kh[0] = block_of(0, s, kindh[0]);
    kh[1] = block_of(1, s, kindh[1]);
    // epilogue operands, loaded early (independent of the chain)
    cplx aux[2][GMAX];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int g = 0; g < GMAX; ++g) {
        aux[h][g] = make_double2(0.0, 0.0);
        if (g >= Gc || kh[h] < 0 || t >= nout) continue;
        const int k = kh[h];
        const int col = chunk0 + g * rg + oc;
        if (kindh[h] == 0) {
          int kn = h == 0 ? k + 1 : k - 1;  // next block of this chain
          bool has_b = h == 0 ? true : (kn > tw);
          if (has_b) aux[h][g] = V.rhs[((size_t)kn * m + r0 + orow) * ldx + col];
        } else if (kindh[h] == 2) {
          aux[h][g] = __ldcg(V.x + ((size_t)k * m + r0 + orow) * ldx + col);
        }
      }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (kh[h] < 0) continue;
      const int k = kh[h], kind = kindh[h];
      const int q = fseq(h, s);
      mbar_wait(&fbar[h * FAC_STAGES + q % FAC_STAGES], (q / FAC_STAGES) & 1);
#ifdef DS_SOLVE_TRACE
      if (t == 0 && blockIdx.y == 0 && blockIdx.z == 0 && rank < 16 && s < 1024)
        g_solve_trace[rank][s][6 + h] = clock64();
#endif
      const cplx *A = fac + (h * FAC_STAGES + q % FAC_STAGES) * fstride;
#pragma unroll
      for (int g = 0; g < GMAX; ++g) {
        if (g >= Gc) break;
        // wait for this chain's input vector (the bottom chain's first
        // backward stage reads x_t from the top chain's buffer)
        const int hb = (h == 1 && s == F + 1) ? 0 : h;
        mbar_wait(VBAR(hb, g, p), vph[hb][g][p] & 1);
        const cplx *X = VEC(hb, g, p);
        const cplx *X2 = nullptr;
        if (kind == 1 && nbt > 0) {  // middle: add the bottom chain's part
          mbar_wait(VBAR(1, g, p), vph[1][g][p] & 1);
          X2 = VEC(1, g, p);
        }
        TRACE(1);
        // ---- rows [r0, r0+nr) of the block inverse times the vector
        for (int tile = ntile ? t % ntile : 0, sl = ntile ? t / ntile : nslice;
             sl < nslice && tile < ntile; tile += SOLVE_THREADS) {
          const int tr = tile / TC, tc = tile % TC;
          const int row = 2 * tr, c = 2 * tc;
          const int j0 = (ntile > SOLVE_THREADS) ? 0 : sl * ks;
          const int j1 = (ntile > SOLVE_THREADS) ? m : min(m, j0 + ks);
          cplx a00 = make_double2(0.0, 0.0), a01 = a00, a10 = a00, a11 = a00;
          const cplx *ar0 = A + (size_t)row * m;
          const cplx *ar1 = ar0 + m;
#ifdef K3_NO_COMPUTE
          if (true) {
          } else
#endif
          if (X2) {
            for (int j = j0; j < j1; ++j) {
              cplx x0 = cadd(X[j * rg + c], X2[j * rg + c]);
              cplx x1 = cadd(X[j * rg + c + 1], X2[j * rg + c + 1]);
              cplx f0 = ar0[j], f1 = ar1[j];
              cfma(a00, f0, x0); cfma(a01, f0, x1); cfma(a10, f1, x0); cfma(a11, f1, x1);
            }
          } else {
#pragma unroll 4
            for (int j = j0; j < j1; ++j) {
              cplx x0 = X[j * rg + c], x1 = X[j * rg + c + 1];
              cplx f0 = ar0[j], f1 = ar1[j];
              cfma(a00, f0, x0); cfma(a01, f0, x1); cfma(a10, f1, x0); cfma(a11, f1, x1);
            }
          }
          cplx *rp = red + (size_t)((ntile > SOLVE_THREADS) ? 0 : sl) * rows_max * rg;
          rp[row * rg + c] = a00;
          if (c + 1 < rg) rp[row * rg + c + 1] = a01;
          if (row + 1 < nr) {
            rp[(row + 1) * rg + c] = a10;
            if (c + 1 < rg) rp[(row + 1) * rg + c + 1] = a11;
          }
          if (ntile <= SOLVE_THREADS) break;
        }
        __syncthreads();
        TRACE(2);
        // the input phase(s) of this chain are consumed: re-arm for reuse.
        // x_t (stage F+1) feeds both halves: its last consumer re-arms.
        const bool shared_xt = (s == F + 1) && nbt > 0;
        const bool consume = !(shared_xt && h == 0);
        if (t == 0) {
          if (consume) mbar_expect_tx(VBAR(hb, g, p), vec_bytes);
          if (X2) mbar_expect_tx(VBAR(1, g, p), vec_bytes);
        }
        if (consume) vph[hb][g][p]++;
        if (X2) vph[1][g][p]++;
        // ---- epilogue: next-stage vector rows first (they gate the peers),
        // the y/x outputs after the push so the proxy fence only waits for
        // the exchange rows
        const bool last = s + 1 >= S;
        cplx out = make_double2(0.0, 0.0);
        size_t off = 0;
        if (t < nout) {
          cplx acc = red[t];
          if (ntile <= SOLVE_THREADS)
            for (int q2 = 1; q2 < nslice; ++q2) acc = cadd(acc, red[(size_t)q2 * rows_max * rg + t]);
          off = ((size_t)k * m + r0 + orow) * ldx + chunk0 + g * rg + oc;
          cplx nxt;
          if (kind == 0) {
            out = acc;  // y_k (top) / z_k (bottom)
            if (h == 0) nxt = csub(aux[h][g], cmul(f.lcoef[k + 1], acc));
            else nxt = csub(aux[h][g], cmul(f.ucoef[k - 1], acc));
          } else if (kind == 1) {
            out = acc;  // x_t
            nxt = acc;
          } else {
            out = csub(aux[h][g], cmul(h == 0 ? f.ucoef[k] : f.lcoef[k], acc));
            nxt = out;
          }
          if (!last) XG(h == 1 && kind == 1 ? 0 : h, g, p ^ 1)[(r0 + orow) * rg + oc] = nxt;
        }
        fence_proxy_async_global();
        __syncthreads();
        if (t == 0 && !last) push(h, g, p ^ 1);
        if (t < nout) V.x[off] = out;
        TRACE(3);
      }
    }
  }
  cluster.sync();  // no CTA leaves while multicasts into it may be in flight
}

// K3 v5: the two half-chains fused into one pass per stage.  The ablation
// in DESIGN.md shows the per-stage cost is dominated by fixed overheads
// (barrier waits, two __syncthreads, reduction, proxy fence, push issue), so
// both halves now share them: threads 0-127 compute the top block, 128-255
// the bottom block, one mbarrier per stage parity collects both halves'
// rows (expected bytes = halves delivering to that stage), and both halves'
// rows are multicast back-to-back.
// factor-tile row pitch: lda % 8 == 4 puts consecutive rows in opposite
// halves of the 128-byte bank window, so the 8-row DMMA A fragments (and the
// 2-row DFMA micro-tiles) load without bank conflicts for any m
__host__ __device__ __forceinline__ int solve_lda(int m) { return m + (12 - m % 8) % 8; }

template <bool MMA>
__global__ void __launch_bounds__(SOLVE_THREADS, 1)
    k_block_solve5(const SolveVisit *__restrict__ visits, int nrhs, int rc, int rows_max, int nsl_max,
                   int lda_pad) {
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int C = (int)cluster.num_blocks();
  const SolveVisit V = visits[blockIdx.y];
  const FactDev f = *V.f;
  const int m = f.m, nb = f.nb, tw = f.twist;
  const int chunk0 = blockIdx.z * rc;
  const int rg = min(rc, nrhs - chunk0);
  const int t = threadIdx.x;
  const int hh = t >> 7, tl = t & 127;  // my half, my lane within the half
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

  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t *vbar = (uint64_t *)smem_raw;  // [2 parity]
  uint64_t *fbar = vbar + 2;              // [2 halves][FAC_STAGES]
  cplx *vec = (cplx *)(smem_raw + 256);   // [2 halves][2 parity][vstride]
  const int vstride = m * rc + 2;
  cplx *fac = vec + 4 * vstride;          // [2 halves][FAC_STAGES][fstride]
  const int lda = lda_pad ? solve_lda(m) : m;
  const int fstride = ((rows_max + 7) & ~7) * lda + 2;
  cplx *red = fac + 2 * FAC_STAGES * fstride;  // [2 halves][nsl_max slices][rows_max*rc]
  const int rstride = rows_max * rc;
  auto VEC = [&](int h, int p) { return vec + (h * 2 + p) * vstride; };
  cplx *xg = V.xg + (size_t)blockIdx.z * 4 * m * rc;
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
  // halves delivering input vectors to stage st (one m x rg vector each)
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
  // TMA issue blocks the issuing thread for ~150-400 cycles
  // (tools/issue_latency_micro.cu), so the per-stage copies are issued by
  // different warps: top/bottom multicast by warps 0/4, top/bottom factor
  // tiles by warps 2/6 -- each fits in its warp's slack before the exchange
  const int tile_thread[2] = {64, 192};
  auto load_tile = [&](int h, int st) {  // thread tile_thread[h] (or warp 0 for per-row copies)
    int kind, k = block_of(h, st, kind);
    if (k < 0) return;
    int q = fseq(h, st), slot = q % FAC_STAGES;
    uint64_t *bar = &fbar[h * FAC_STAGES + slot];
    if (lda == m) {  // rows already conflict-free: one copy of the slice
      if (t == tile_thread[h]) {
        mbar_expect_tx(bar, fac_bytes);
        if (fac_bytes)
          bulk_g2s(fac + (h * FAC_STAGES + slot) * fstride, f.sinv + ((size_t)k * m + r0) * m,
                   fac_bytes, bar);
      }
      return;
    }
    if (t == 0) mbar_expect_tx(bar, fac_bytes);
    __syncwarp();
    for (int r = t; r < nr; r += 32)
      bulk_g2s(fac + (h * FAC_STAGES + slot) * fstride + r * lda,
               f.sinv + ((size_t)k * m + r0 + r) * m, (uint32_t)(m * sizeof(cplx)), bar);
  };
  auto push = [&](int h, int p) {  // thread 0, after the fence + barrier
    if (push_bytes)
      bulk_g2s_multicast(VEC(h, p) + r0 * rg, XG(h, p) + r0 * rg, push_bytes, &vbar[p], mask);
  };

#ifdef DS_SOLVE_TRACE5
  // every rank of cluster (0,0) traces; the launch index is the count of
  // rank-0 CTAs seen before (rank 0 bumps it after the kernel's first sync)
  int tr5 = -1;
  if (t == 0 && blockIdx.y == 0 && blockIdx.z == 0) {
    tr5 = *(volatile int *)&g_tr5_n;
    if (tr5 >= 64) tr5 = -1;
  }
#endif
  if (t == 0) {
    mbar_init(&vbar[0], 1);
    mbar_init(&vbar[1], 1);
    for (int i = 0; i < 2 * FAC_STAGES; ++i) mbar_init(&fbar[i], 1);
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
    if (lda == m || t < 32) {
      load_tile(0, st);
      load_tile(1, st);
    }
  }
  // prologue: b_0 (top, stage F-nt) and b_{n_b-1} (bottom, stage F-nbt)
  for (int h = 0; h < 2; ++h) {
    if (h == 1 && nbt == 0) break;
    const int st0 = h == 0 ? F - nt : F - nbt;
    const int k0 = h == 0 ? 0 : nb - 1;
    for (int e = t; e < nr * rg; e += SOLVE_THREADS) {
      int row = e / rg, c = e % rg;
      XG(h, st0 & 1)[(r0 + row) * rg + c] = V.rhs[((size_t)k0 * m + r0 + row) * ldx + chunk0 + c];
    }
  }
  fence_proxy_async_global();
  __syncthreads();
  if (t == 0) {
    push(0, (F - nt) & 1);
    if (nbt > 0) push(1, (F - nbt) & 1);
  }

  // per half: 2x2 (row, rhs) micro-tiles, K split over 128 / ntile slices
  const int TR = (nr + 1) / 2, TC = (rg + 1) / 2;
  const int ntile = TR * TC;
  int nslice = ntile > 0 ? 128 / ntile : 1;
  nslice = MMA ? 4 : max(1, min(nsl_max, nslice));
  const int ks = (m + nslice - 1) / nslice;
  const int nout = nr * rg;  // outputs per half (<= 2 * 128)
  uint32_t vph = 0;  // bit p: phase of vbar[p] (a register, not a local array)

  for (int s = 0; s < S; ++s) {
    const int p = s & 1;
    TRACE5(0);
#ifndef K3_NO_FACSTREAM
    if (s + FAC_STAGES - 1 < S) {
      if (lda == m) {
        if (t == tile_thread[0]) load_tile(0, s + FAC_STAGES - 1);
        if (t == tile_thread[1]) load_tile(1, s + FAC_STAGES - 1);
      } else if (t < 32) {
        load_tile(0, s + FAC_STAGES - 1);
        load_tile(1, s + FAC_STAGES - 1);
      }
    }
#endif
    TRACE5(8);
    int kind, k = block_of(hh, s, kind);
    const bool act = k >= 0;
    // epilogue operands (independent of the chain), up to 2 outputs / thread
    cplx aux[2] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0)};
    cplx coef = make_double2(0.0, 0.0);  // chain coefficient, off the critical path
    if (act) {
      if (kind == 0) coef = hh == 0 ? f.lcoef[k + 1] : f.ucoef[k - 1];
      else if (kind == 2) coef = hh == 0 ? f.ucoef[k] : f.lcoef[k];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int o = tl + u * 128;
        if (o >= nout) break;
        const int orow = o / rg, oc = o % rg;
        const size_t col = chunk0 + oc;
        if (kind == 0) {
          const int kn = hh == 0 ? k + 1 : k - 1;
          if (hh == 0 || kn > tw) aux[u] = V.rhs[((size_t)kn * m + r0 + orow) * ldx + col];
        } else if (kind == 2) {
          aux[u] = __ldcg(V.x + ((size_t)k * m + r0 + orow) * ldx + col);
        }
      }
    }
    TRACE5(9);
    // factor tile first (streamed a stage ahead, normally complete), then
    // the exchanged vectors; the exchange barrier is re-armed for stage s+2
    // at once (its next phase needs this CTA's push of stage s+1, which
    // follows every thread's pass through this wait)
    const int q = act ? fseq(hh, s) : 0;
#ifndef K3_NO_FACSTREAM
    if (act) mbar_wait(&fbar[hh * FAC_STAGES + q % FAC_STAGES], (q / FAC_STAGES) & 1);
#endif
    TRACE5(1);
#ifndef K3_NO_WAIT
    mbar_wait(&vbar[p], (vph >> p) & 1);
#endif
    if (t == 0 && s + 2 < S) mbar_expect_tx(&vbar[p], deliveries(s + 2) * vec_bytes);
    vph ^= 1u << p;
    TRACE5(2);
    if (act) {
      const cplx *A = fac + (hh * FAC_STAGES + q % FAC_STAGES) * fstride;
      // input vector: own half; bottom at F+1 reads x_t (top buffer);
      // the middle block adds the bottom chain's part
      const cplx *X = VEC((hh == 1 && s == F + 1) ? 0 : hh, p);
      const cplx *X2 = (kind == 1 && nbt > 0) ? VEC(1, p) : nullptr;
      if constexpr (MMA) {
        // FP64 tensor cores: per warp all (8-row, 8-RHS) tiles of this
        // half over a quarter of K; complex product as 4 real m8n8k4 DMMAs
        const int warp = tl >> 5, lane = t & 31, g = lane >> 2, tg = lane & 3;
        const int nk = (m + 3) >> 2, kb = (warp * nk) >> 2, ke = ((warp + 1) * nk) >> 2;
        const int MT = (nr + 7) >> 3, NT = (rg + 7) >> 3;
        double cr[2][2][2] = {}, ci[2][2][2] = {};
#ifdef K3_NO_COMPUTE
        if (false)
#endif
        {
          const int sel = (MT > 1 ? 4 : 0) + (NT > 1 ? 2 : 0) + (X2 ? 1 : 0);
#define K3_PRODUCT(mt_, nt_, x2_) \
  mma_product<mt_, nt_, x2_>(A, lda, X, X2, rg, m, kb, ke, g, tg, cr, ci)
          switch (sel) {
            case 0: K3_PRODUCT(1, 1, false); break;
            case 1: K3_PRODUCT(1, 1, true); break;
            case 2: K3_PRODUCT(1, 2, false); break;
            case 3: K3_PRODUCT(1, 2, true); break;
            case 4: K3_PRODUCT(2, 1, false); break;
            case 5: K3_PRODUCT(2, 1, true); break;
            case 6: K3_PRODUCT(2, 2, false); break;
            default: K3_PRODUCT(2, 2, true); break;
          }
#undef K3_PRODUCT
        }
        cplx *rp = red + ((size_t)hh * nsl_max + warp) * rstride;
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int nt = 0; nt < 2; ++nt)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int row = mt * 8 + g, col = nt * 8 + 2 * tg + e;
              if (mt < MT && nt < NT && row < nr && col < rg)
                rp[row * rg + col] = make_double2(cr[mt][nt][e], ci[mt][nt][e]);
            }
      } else {
      const int tile = ntile ? tl % ntile : 0, sl = ntile ? tl / ntile : nslice;
      if (sl < nslice && tile < ntile) {
        const int tr = tile / TC, tc = tile % TC;
        const int row = 2 * tr, c = 2 * tc;
        const int j0 = sl * ks, j1 = min(m, j0 + ks);
        cplx a00 = make_double2(0.0, 0.0), a01 = a00, a10 = a00, a11 = a00;
        const cplx *ar0 = A + (size_t)row * lda;
        const cplx *ar1 = ar0 + lda;
#ifdef K3_NO_COMPUTE
        if (true) {
        } else
#endif
        if (X2) {
          for (int j = j0; j < j1; ++j) {
            cplx x0 = cadd(X[j * rg + c], X2[j * rg + c]);
            cplx x1 = cadd(X[j * rg + c + 1], X2[j * rg + c + 1]);
            cplx f0 = ar0[j], f1 = ar1[j];
            cfma(a00, f0, x0); cfma(a01, f0, x1); cfma(a10, f1, x0); cfma(a11, f1, x1);
          }
        } else {
#pragma unroll 4
          for (int j = j0; j < j1; ++j) {
            cplx x0 = X[j * rg + c], x1 = X[j * rg + c + 1];
            cplx f0 = ar0[j], f1 = ar1[j];
            cfma(a00, f0, x0); cfma(a01, f0, x1); cfma(a10, f1, x0); cfma(a11, f1, x1);
          }
        }
        cplx *rp = red + ((size_t)hh * nsl_max + sl) * rstride;
        rp[row * rg + c] = a00;
        if (c + 1 < rg) rp[row * rg + c + 1] = a01;
        if (row + 1 < nr) {
          rp[(row + 1) * rg + c] = a10;
          if (c + 1 < rg) rp[(row + 1) * rg + c + 1] = a11;
        }
      }
      }
    }
    TRACE5(3);
    __syncthreads();
    TRACE5(4);
    // epilogue: next-stage rows to the exchange scratch, outputs kept
    const bool last = s + 1 >= S;
    cplx outv[2];
    size_t offs[2] = {0, 0};
    if (act) {
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int o = tl + u * 128;
        if (o >= nout) break;
        const int orow = o / rg, oc = o % rg;
        const cplx *rq = red + (size_t)hh * nsl_max * rstride + o;
        cplx acc = rq[0];
        if constexpr (MMA) {  // 4 K-slices (warps); same summation order
          const cplx r1 = rq[rstride], r2 = rq[2 * rstride], r3 = rq[3 * rstride];
          acc = cadd(cadd(cadd(acc, r1), r2), r3);
        } else {
          for (int q2 = 1; q2 < nslice; ++q2) acc = cadd(acc, rq[(size_t)q2 * rstride]);
        }
        offs[u] = ((size_t)k * m + r0 + orow) * ldx + chunk0 + oc;
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
        if (!last) XG(hh, p ^ 1)[(r0 + orow) * rg + oc] = nxt;
      }
    }
    TRACE5(5);
#ifndef K3_NO_FENCE
    fence_proxy_async_global();  // (v5)
#endif
    __syncthreads();
    TRACE5(6);
    if ((t & 127) == 0 && !last) {
      // exactly the deliveries counted for stage s+1 (see deliveries());
      // thread 0 issues the top half's multicast, thread 128 the bottom's
      int kd;
      if (hh == 0 && block_of(0, s, kd) >= 0 && block_of(0, s + 1, kd) >= 0) push(0, p ^ 1);
      if (hh == 1 && block_of(1, s, kd) >= 0 && (block_of(1, s + 1, kd) >= 0 || s + 1 == F))
        push(1, p ^ 1);
    }
    if (act) {
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int o = tl + u * 128;
        if (o >= nout) break;
        V.x[offs[u]] = outv[u];
      }
    }
    TRACE5(7);
  }
  cluster.sync();
}

// K3 v6: v5 with warp specialisation and loop-invariant addressing.
// The per-stage trace of v5 (tools/trace_solve5.py) showed ~2400 of ~4700
// cycles per stage spent in scalar work on the critical path: thread 0
// issuing the factor-tile bulk copies (the issue blocks while the TMA unit
// is busy) and every thread recomputing output coordinates and 64-bit
// addresses.  Here a ninth (producer) warp streams the factor tiles through
// full/empty mbarrier pairs up to FAC_STAGES tiles ahead, the 8 compute warps
// synchronise on named barrier 1 only, and all per-thread offsets are
// computed once before the stage loop.  Arithmetic, exchange protocol and
// results are those of v5.
#define SOLVE6_THREADS 288
#define SOLVE6_COMPUTE 256

__device__ __forceinline__ void bar_compute() {
  asm volatile("bar.sync 1, %0;\n" ::"n"(SOLVE6_COMPUTE) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

__global__ void __launch_bounds__(SOLVE6_THREADS, 1)
    k_block_solve6(const SolveVisit *__restrict__ visits, int nrhs, int rc, int rows_max) {
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int C = (int)cluster.num_blocks();
  const SolveVisit V = visits[blockIdx.y];
  const FactDev f = *V.f;
  const int m = f.m, nb = f.nb, tw = f.twist;
  const int chunk0 = blockIdx.z * rc;
  const int rg = min(rc, nrhs - chunk0);
  const int t = threadIdx.x;
  const bool producer = t >= SOLVE6_COMPUTE;
  const int hh = (t >> 7) & 1, tl = t & 127;  // compute threads: half, lane in half
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
  constexpr int NSL = 4;  // K-slices = warps per half

  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t *vbar = (uint64_t *)smem_raw;   // [2 parity]
  uint64_t *full = vbar + 2;               // [2 halves][FAC_STAGES]
  uint64_t *empty = full + 2 * FAC_STAGES; // [2 halves][FAC_STAGES]
  cplx *vec = (cplx *)(smem_raw + 256);    // [2 halves][2 parity][vstride]
  const int vstride = m * rc + 2;
  cplx *fac = vec + 4 * vstride;           // [2 halves][FAC_STAGES][fstride]
  const int fstride = ((rows_max + 7) & ~7) * m + 2;
  cplx *red = fac + 2 * FAC_STAGES * fstride;  // [2 halves][NSL][rows_max*rc]
  const int rstride = rows_max * rc;
  auto VEC = [&](int h, int p) { return vec + (h * 2 + p) * vstride; };
  cplx *xg = V.xg + (size_t)blockIdx.z * 4 * m * rc;
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
  auto push = [&](int h, int p) {
    if (push_bytes)
      bulk_g2s_multicast(VEC(h, p) + r0 * rg, XG(h, p) + r0 * rg, push_bytes, &vbar[p], mask);
  };

#ifdef DS_SOLVE_TRACE5
  // every rank of cluster (0,0) traces; the launch index is the count of
  // rank-0 CTAs seen before (rank 0 bumps it after the kernel's first sync)
  int tr5 = -1;
  if (t == 0 && blockIdx.y == 0 && blockIdx.z == 0) {
    tr5 = *(volatile int *)&g_tr5_n;
    if (tr5 >= 64) tr5 = -1;
  }
#endif
  if (t == 0) {
    mbar_init(&vbar[0], 1);
    mbar_init(&vbar[1], 1);
    for (int i = 0; i < 2 * FAC_STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    fence_mbar_init();
  }
  cluster.sync();
#ifdef DS_SOLVE_TRACE5
  if (t == 0 && rank == 0 && blockIdx.y == 0 && blockIdx.z == 0) atomicAdd(&g_tr5_n, 1);
#endif

  if (producer) {
    // ---- factor-tile stream: tiles in stage order, FAC_STAGES ahead
    if (t == SOLVE6_COMPUTE) {
      int kind;
      for (int st = 0; st < S; ++st) {
        for (int h = 0; h < 2; ++h) {
          const int k = block_of(h, st, kind);
          if (k < 0) continue;
          const int q = fseq(h, st), slot = q % FAC_STAGES;
          if (q >= FAC_STAGES) mbar_wait(&empty[h * FAC_STAGES + slot], ((q / FAC_STAGES) - 1) & 1);
          mbar_expect_tx(&full[h * FAC_STAGES + slot], fac_bytes);
          if (fac_bytes)
            bulk_g2s(fac + (h * FAC_STAGES + slot) * fstride, f.sinv + ((size_t)k * m + r0) * m,
                     fac_bytes, &full[h * FAC_STAGES + slot]);
        }
      }
    }
  } else {
    if (t == 0) {
      mbar_expect_tx(&vbar[0], deliveries(0) * vec_bytes);
      if (S > 1) mbar_expect_tx(&vbar[1], deliveries(1) * vec_bytes);
    }
    // prologue: b_0 (top, stage F-nt) and b_{n_b-1} (bottom, stage F-nbt)
    for (int h = 0; h < 2; ++h) {
      if (h == 1 && nbt == 0) break;
      const int st0 = h == 0 ? F - nt : F - nbt;
      const int k0 = h == 0 ? 0 : nb - 1;
      for (int e = t; e < nr * rg; e += SOLVE6_COMPUTE) {
        int row = e / rg, c = e % rg;
        XG(h, st0 & 1)[(r0 + row) * rg + c] = V.rhs[((size_t)k0 * m + r0 + row) * ldx + chunk0 + c];
      }
    }
    fence_proxy_async_global();
    bar_compute();
    if (t == 0) {
      push(0, (F - nt) & 1);
      if (nbt > 0) push(1, (F - nbt) & 1);
    }

    // ---- loop invariants: my (up to 2) outputs of my half
    const int nout = nr * rg;
    const size_t blk = (size_t)m * ldx;  // one block of the [nb][m][nrhs] layout
    int xoff[2];                          // exchange scratch offset (row-major m x rg)
    size_t goff[2];                       // offset of (row, col) in a block of V.rhs / V.x
    bool has[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int o = tl + u * 128;
      has[u] = o < nout;
      const int orow = has[u] ? o / rg : 0, oc = has[u] ? o % rg : 0;
      xoff[u] = (r0 + orow) * rg + oc;
      goff[u] = (size_t)(r0 + orow) * ldx + chunk0 + oc;
    }
    const int warp = tl >> 5, lane = t & 31, g = lane >> 2, tg = lane & 3;
    const int nk = (m + 3) >> 2, kb = (warp * nk) >> 2, ke = ((warp + 1) * nk) >> 2;
    const int MT = (nr + 7) >> 3, NT = (rg + 7) >> 3;
    const int sel = (MT > 1 ? 4 : 0) + (NT > 1 ? 2 : 0);
    cplx *rp = red + ((size_t)hh * NSL + warp) * rstride;
    const cplx *rq = red + (size_t)hh * NSL * rstride;
    uint32_t vph = 0;

    for (int s = 0; s < S; ++s) {
      const int p = s & 1;
      TRACE5(0);
      int kind, k = block_of(hh, s, kind);
      const bool act = k >= 0;
      // epilogue operands (independent of the chain)
      cplx aux[2] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0)};
      cplx coef = make_double2(0.0, 0.0);
      if (act) {
        if (kind == 0) {
          coef = hh == 0 ? f.lcoef[k + 1] : f.ucoef[k - 1];
          const int kn = hh == 0 ? k + 1 : k - 1;
          if (hh == 0 || kn > tw) {
            const cplx *src = V.rhs + (size_t)kn * blk;
#pragma unroll
            for (int u = 0; u < 2; ++u)
              if (has[u]) aux[u] = src[goff[u]];
          }
        } else if (kind == 2) {
          coef = hh == 0 ? f.ucoef[k] : f.lcoef[k];
          const cplx *src = V.x + (size_t)k * blk;
#pragma unroll
          for (int u = 0; u < 2; ++u)
            if (has[u]) aux[u] = __ldcg(src + goff[u]);
        }
      }
      TRACE5(8);
      const int q = act ? fseq(hh, s) : 0;
      if (act) mbar_wait(&full[hh * FAC_STAGES + q % FAC_STAGES], (q / FAC_STAGES) & 1);
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
#define K3_PRODUCT(mt_, nt_, x2_) \
  mma_product<mt_, nt_, x2_>(A, m, X, X2, rg, m, kb, ke, g, tg, cr, ci)
          switch (sel + (X2 ? 1 : 0)) {
            case 0: K3_PRODUCT(1, 1, false); break;
            case 1: K3_PRODUCT(1, 1, true); break;
            case 2: K3_PRODUCT(1, 2, false); break;
            case 3: K3_PRODUCT(1, 2, true); break;
            case 4: K3_PRODUCT(2, 1, false); break;
            case 5: K3_PRODUCT(2, 1, true); break;
            case 6: K3_PRODUCT(2, 2, false); break;
            default: K3_PRODUCT(2, 2, true); break;
          }
#undef K3_PRODUCT
        }
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int ntt = 0; ntt < 2; ++ntt)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int row = mt * 8 + g, col = ntt * 8 + 2 * tg + e;
              if (mt < MT && ntt < NT && row < nr && col < rg)
                rp[row * rg + col] = make_double2(cr[mt][ntt][e], ci[mt][ntt][e]);
            }
      }
      TRACE5(3);
      bar_compute();
      TRACE5(4);
      // the factor tiles of this stage are consumed: hand the slots back
      if (t == 0) {
        int kd;
        for (int h = 0; h < 2; ++h)
          if (block_of(h, s, kd) >= 0) mbar_arrive(&empty[h * FAC_STAGES + fseq(h, s) % FAC_STAGES]);
      }
      // epilogue: split-K sum (fixed order), chain update, exchange rows
      const bool last = s + 1 >= S;
      cplx outv[2];
      if (act) {
        cplx *xgo = XG(hh, p ^ 1);
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          if (!has[u]) continue;
          const int o = tl + u * 128;
          const cplx r1 = rq[o + rstride], r2 = rq[o + 2 * rstride], r3 = rq[o + 3 * rstride];
          const cplx acc = cadd(cadd(cadd(rq[o], r1), r2), r3);
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
      bar_compute();
      TRACE5(6);
      if (tl == 0 && !last) {
        // exactly the deliveries counted for stage s+1 (see deliveries());
        // thread 0 issues the top half's multicast, thread 128 the bottom's
        int kd;
        if (hh == 0 && block_of(0, s, kd) >= 0 && block_of(0, s + 1, kd) >= 0) push(0, p ^ 1);
        if (hh == 1 && block_of(1, s, kd) >= 0 && (block_of(1, s + 1, kd) >= 0 || s + 1 == F))
          push(1, p ^ 1);
      }
      if (act) {
        cplx *dst = V.x + (size_t)k * blk;
#pragma unroll
        for (int u = 0; u < 2; ++u)
          if (has[u]) dst[goff[u]] = outv[u];
      }
      TRACE5(7);
    }
  }
  cluster.sync();  // no CTA leaves while multicasts into it may be in flight
}

// K3 v7: the two twisted half-chains staggered by half a stage.
// The v5 stage is  exchange (~2000 cycles: rows -> L2 -> multicast, plus the
// factor-tile stream sharing the SM's ingress) -> product -> epilogue, all
// in series (tools/exchange_load_micro.cu, tools/trace_solve5.py).  The top
// and bottom chains are independent until the middle block, so here all 8
// warps compute one chain's block product while the other chain's exchange
// is in flight: half-steps alternate top(s), bottom(s), top(s+1), ...
// Exchange barriers are per (input buffer, parity); x_t is multicast into
// both buffers so every buffer has exactly one reader per stage, and a peer
// can only refill a buffer after this CTA's reader has passed its barrier
// (the refill needs this CTA's push, which follows that reader).
// Warps: n-tile = warp / KS, K-slice = warp % KS with KS = 8 / NT.
__global__ void __launch_bounds__(SOLVE_THREADS, 1)
    k_block_solve7(const SolveVisit *__restrict__ visits, int nrhs, int rc, int rows_max) {
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int C = (int)cluster.num_blocks();
  const SolveVisit V = visits[blockIdx.y];
  const FactDev f = *V.f;
  const int m = f.m, nb = f.nb, tw = f.twist;
  const int chunk0 = blockIdx.z * rc;
  const int rg = min(rc, nrhs - chunk0);
  const int t = threadIdx.x;
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

  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t *vbar = (uint64_t *)smem_raw;  // [2 buffers][2 parity]
  uint64_t *fbar = vbar + 4;              // [2 halves][FAC_STAGES]
  cplx *vec = (cplx *)(smem_raw + 256);   // [2 buffers][2 parity][vstride]
  const int vstride = m * rc + 2;
  cplx *fac = vec + 4 * vstride;          // [2 halves][FAC_STAGES][fstride]
  const int fstride = ((rows_max + 7) & ~7) * m + 2;
  cplx *red = fac + 2 * FAC_STAGES * fstride;  // [KS][rows_max * rc]
  const int rstride = rows_max * rc;
  auto VEC = [&](int b, int p) { return vec + (b * 2 + p) * vstride; };
  cplx *xg = V.xg + (size_t)blockIdx.z * 4 * m * rc;
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
  // q-th tile of half h <-> stage
  auto fseq = [&](int h, int st) {
    if (h == 0) return st - (F - nt);
    return st < F ? st - (F - nbt) : st - (F - nbt) - 1;
  };
  auto tile_stage = [&](int h, int q) {
    if (h == 0) return q + (F - nt);
    return q < nbt ? q + (F - nbt) : q + (F - nbt) + 1;
  };
  const int ntiles[2] = {2 * nt + 1, 2 * nbt};
  // vectors delivered into buffer b for stage st (0 or 1)
  auto deliv = [&](int b, int st) -> int {
    if (st < 0 || st >= S) return 0;
    if (b == 0) return st >= F - nt && st <= F + nt;
    return nbt > 0 && st >= F - nbt && st <= F + nbt;
  };
  const uint32_t vec_bytes = (uint32_t)(m * rg * sizeof(cplx));
  const uint32_t fac_bytes = (uint32_t)(nr * m * sizeof(cplx));
  const uint32_t push_bytes = (uint32_t)(nr * rg * sizeof(cplx));
  auto load_tile = [&](int h, int q) {  // thread 0
    if (q >= ntiles[h]) return;
    int kind, k = block_of(h, tile_stage(h, q), kind);
    const int slot = q % FAC_STAGES;
    uint64_t *bar = &fbar[h * FAC_STAGES + slot];
    mbar_expect_tx(bar, fac_bytes);
    if (fac_bytes)
      bulk_g2s(fac + (h * FAC_STAGES + slot) * fstride, f.sinv + ((size_t)k * m + r0) * m, fac_bytes, bar);
  };
  auto push = [&](int b, int h, int p) {  // rows of XG(h, p) -> buffer (b, p) of every CTA
    if (push_bytes)
      bulk_g2s_multicast(VEC(b, p) + r0 * rg, XG(h, p) + r0 * rg, push_bytes, &vbar[b * 2 + p], mask);
  };

#ifdef DS_SOLVE_TRACE5
  int tr5 = -1;
  if (t == 0 && blockIdx.y == 0 && blockIdx.z == 0) {
    tr5 = *(volatile int *)&g_tr5_n;
    if (tr5 >= 64) tr5 = -1;
  }
#endif
  if (t == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(&vbar[i], 1);
    for (int i = 0; i < 2 * FAC_STAGES; ++i) mbar_init(&fbar[i], 1);
    fence_mbar_init();
  }
  cluster.sync();
#ifdef DS_SOLVE_TRACE5
  if (t == 0 && rank == 0 && blockIdx.y == 0 && blockIdx.z == 0) atomicAdd(&g_tr5_n, 1);
#endif
  if (t == 0) {
    for (int b = 0; b < 2; ++b)
      for (int st = 0; st < 2 && st < S; ++st) mbar_expect_tx(&vbar[b * 2 + st], deliv(b, st) * vec_bytes);
    for (int q = 0; q < FAC_STAGES - 1; ++q) {
      load_tile(0, q);
      load_tile(1, q);
    }
  }
  // prologue: b_0 (top, stage F-nt) and b_{n_b-1} (bottom, stage F-nbt)
  for (int h = 0; h < 2; ++h) {
    if (h == 1 && nbt == 0) break;
    const int st0 = h == 0 ? F - nt : F - nbt;
    const int k0 = h == 0 ? 0 : nb - 1;
    for (int e = t; e < nr * rg; e += SOLVE_THREADS) {
      int row = e / rg, c = e % rg;
      XG(h, st0 & 1)[(r0 + row) * rg + c] = V.rhs[((size_t)k0 * m + r0 + row) * ldx + chunk0 + c];
    }
  }
  fence_proxy_async_global();
  __syncthreads();
  if (t == 0) {
    push(0, 0, (F - nt) & 1);
    if (nbt > 0) push(1, 1, (F - nbt) & 1);
  }

  // ---- loop invariants
  const int nout = nr * rg;
  const bool has = t < nout;
  const int orow = has ? t / rg : 0, oc = has ? t % rg : 0;
  const int xoff = (r0 + orow) * rg + oc;
  const size_t goff = (size_t)(r0 + orow) * ldx + chunk0 + oc;
  const size_t blk = (size_t)m * ldx;
  const int warp = t >> 5, lane = t & 31, g = lane >> 2, tg = lane & 3;
  const int MT = (nr + 7) >> 3, NT = (rg + 7) >> 3;
  const int KS = NT > 1 ? 4 : 8;
  const int ntw = warp / KS, ksl = warp % KS;
  const int nk = (m + 3) >> 2, kb = (ksl * nk) / KS, ke = ((ksl + 1) * nk) / KS;
  cplx *rp = red + (size_t)ksl * rstride;

  for (int s = 0; s < S; ++s) {
    const int p = s & 1;
    const uint32_t par = (s >> 1) & 1;
    for (int h = 0; h < 2; ++h) {
      TRACE5(h ? 4 : 0);
      int kind, k = block_of(h, s, kind);
      const bool act = k >= 0;
      // next factor tile of this half, a stage ahead, issued before this
      // half-step's waits so the TMA unit has finished it before the
      // half-step's multicast is issued (a multicast queued behind an HBM
      // load would carry the load's latency into the exchange)
      if (t == 64 + 128 * h && act) load_tile(h, fseq(h, s) + FAC_STAGES - 1);
      cplx aux = make_double2(0.0, 0.0), coef = make_double2(0.0, 0.0);
      if (act && has) {
        if (kind == 0) {
          coef = h == 0 ? f.lcoef[k + 1] : f.ucoef[k - 1];
          const int kn = h == 0 ? k + 1 : k - 1;
          if (h == 0 || kn > tw) aux = V.rhs[(size_t)kn * blk + goff];
        } else if (kind == 2) {
          coef = h == 0 ? f.ucoef[k] : f.lcoef[k];
          aux = __ldcg(V.x + (size_t)k * blk + goff);
        }
      }
      const int q = act ? fseq(h, s) : 0;
      const bool x2 = h == 0 && kind == 1 && nbt > 0;
      if (act) {
        mbar_wait(&fbar[h * FAC_STAGES + q % FAC_STAGES], (q / FAC_STAGES) & 1);
        mbar_wait(&vbar[h * 2 + p], par);
        if (x2) mbar_wait(&vbar[2 + p], par);
      }
      TRACE5(h ? 5 : 1);
      if (act) {
        const cplx *A = fac + (h * FAC_STAGES + q % FAC_STAGES) * fstride;
        const cplx *X = VEC(h, p) + ntw * 8;
        const cplx *X2 = x2 ? VEC(1, p) + ntw * 8 : nullptr;
        double cr[2][2][2] = {}, ci[2][2][2] = {};
        if (ntw < NT) {
#ifdef K3_NO_COMPUTE
          if (false)
#endif
          {
            const int sel = (MT > 1 ? 2 : 0) + (X2 ? 1 : 0);
#define K3_PRODUCT(mt_, x2_) mma_product<mt_, 1, x2_>(A, m, X, X2, rg, m, kb, ke, g, tg, cr, ci)
            switch (sel) {
              case 0: K3_PRODUCT(1, false); break;
              case 1: K3_PRODUCT(1, true); break;
              case 2: K3_PRODUCT(2, false); break;
              default: K3_PRODUCT(2, true); break;
            }
#undef K3_PRODUCT
          }
#pragma unroll
          for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int row = mt * 8 + g, col = ntw * 8 + 2 * tg + e;
              if (mt < MT && row < nr && col < rg)
                rp[row * rg + col] = make_double2(cr[mt][0][e], ci[mt][0][e]);
            }
        }
      }
      TRACE5(h ? 6 : 2);
      __syncthreads();
      // buffer (h, p) has no other reader at stage s: re-arm it for s+2
      if (t == 0 && s + 2 < S) mbar_expect_tx(&vbar[h * 2 + p], deliv(h, s + 2) * vec_bytes);
      const bool last = s + 1 >= S;
      cplx out = make_double2(0.0, 0.0);
      if (act && has) {
        cplx acc = red[t];
        for (int q2 = 1; q2 < KS; ++q2) acc = cadd(acc, red[(size_t)q2 * rstride + t]);
        cplx nxt;
        if (kind == 0) {
          out = acc;
          nxt = csub(aux, cmul(coef, acc));
        } else if (kind == 1) {
          out = acc;
          nxt = acc;
        } else {
          out = csub(aux, cmul(coef, acc));
          nxt = out;
        }
        if (!last) XG(h, p ^ 1)[xoff] = nxt;
      }
      fence_proxy_async_global();
      __syncthreads();
      TRACE5(h ? 7 : 3);
      if (t == 0) {
        if (act && !last) {
          int kd;
          if (h == 0) {
            if (block_of(0, s + 1, kd) >= 0) push(0, 0, p ^ 1);
            if (kind == 1 && nbt > 0) push(1, 0, p ^ 1);  // x_t for the bottom chain
          } else if (block_of(1, s + 1, kd) >= 0 || s + 1 == F) {
            push(1, 1, p ^ 1);
          }
        }
      }
      if (act && has) V.x[(size_t)k * blk + goff] = out;
    }
  }
  cluster.sync();  // no CTA leaves while multicasts into it may be in flight
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
  const SolveVisit V = visits[blockIdx.y];
  const FactDev f = *V.f;
  const int m = f.m, nb = f.nb, tw = f.twist;
  const int chunk0 = blockIdx.z * rc;
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
  cplx *xg = V.xg + (size_t)blockIdx.z * 4 * m * rc;
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
  // floor: one CTA per SM (DS_K3_SMEM_FLOOR=0 lets two small CTAs share an SM)
  static const size_t floor_b = [] {
    const char *v = getenv("DS_K3_SMEM_FLOOR");
    return v && *v ? (size_t)atol(v) : (size_t)118 * 1024;
  }();
  return std::max<size_t>(256 + elems * sizeof(cplx), floor_b);
}

static size_t solve7_smem(int m, int rc, int C) {
  int r = (m + C - 1) / C;
  size_t rows_max = r + (r & 1);
  size_t rows_alloc = (rows_max + 7) & ~(size_t)7;
  size_t elems = 4 * ((size_t)m * rc + 2) + 2 * FAC_STAGES * (rows_alloc * m + 2) + 8 * rows_max * rc;
  return std::max<size_t>(256 + elems * sizeof(cplx), 118 * 1024);
}

static int solve_rows_max(int max_m, int C) {
  int r = (max_m + C - 1) / C;
  return r + (r & 1);  // even: 2-row micro-tiles may read one padding row
}

static size_t solve_smem(int max_m, int rc, int C, int G) {
  size_t rows_max = solve_rows_max(max_m, C);
  size_t rg = (rc + G - 1) / G;
  size_t elems = 4 * G * ((size_t)max_m * rg + 2) + 2 * FAC_STAGES * (rows_max * max_m + 2) +
                 16 * rows_max * rg;
  return 256 + elems * sizeof(cplx);
}

static int env_int(const char *name, int dflt) {
  const char *v = getenv(name);
  return v && *v ? atoi(v) : dflt;
}

// Largest cluster (16 non-portable, then 8, 4) that the occupancy API
// accepts for this shared-memory footprint; RHS chunk rc and groups G.
struct SolveCfg {
  int C, rc, G, rows_max;
  size_t smem;
};

static bool try_cfg(int max_m, int rc, int G, int C, SolveCfg *out) {
  size_t smem = solve_smem(max_m, rc, C, G);
  if (smem > 232448) return false;
  if (cudaFuncSetAttribute(k_block_solve, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem) != cudaSuccess) {
    cudaGetLastError();
    return false;
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
  if (cudaOccupancyMaxActiveClusters(&nclusters, k_block_solve, &cfg) != cudaSuccess ||
      nclusters < 1) {
    cudaGetLastError();
    return false;
  }
  *out = SolveCfg{C, rc, G, solve_rows_max(max_m, C), smem};
  return true;
}

static int pick_cfg(int max_m, int nrhs, SolveCfg *out) {
  static int key_m = -1, key_r = -1;
  static SolveCfg cached;
  if (max_m == key_m && nrhs == key_r) {
    *out = cached;
    return 1;
  }
  cudaFuncSetAttribute(k_block_solve, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  const int Cwant = env_int("DS_SOLVE_CLUSTER", 16);
  const int Gwant = env_int("DS_SOLVE_GROUPS", 1);
  for (int rc = std::min(nrhs, env_int("DS_SOLVE_RC", 32)); rc >= 1; rc = (rc + 1) / 2) {
    for (int C : {16, 8, 4}) {
      if (C > Cwant) continue;
      int G = Gwant;
      while (G > 1 && (rc % G != 0 || G > GMAX)) G /= 2;
      if (try_cfg(max_m, rc, G, C, out)) {
        key_m = max_m;
        key_r = nrhs;
        cached = *out;
        return 1;
      }
    }
    if (rc == 1) break;
  }
  return 0;
}

// split-K slices per half: 8 for full chunks, up to 16 when the chunk is
// narrow (fewer outputs per half leave more threads for the K split)
static int solve5_nsl(int m, int rc, int C, bool mma) {
  if (mma) return 4;  // one K-slice per warp of a half
  int rstride = solve_rows_max(m, C) * rc;
  return std::max(8, std::min(16, 1024 / std::max(1, rstride)));
}

// Dynamic shared memory of one CTA.  At least 118 KB, so a CTA always owns
// its SM: the chain is latency bound, and two CTAs sharing an SM would
// serialise their stages (the wave count below assumes one CTA per SM).
static size_t solve5_smem(int m, int rc, int C, bool mma) {
  size_t rows_max = solve_rows_max(m, C);
  size_t rows_alloc = (rows_max + 7) & ~(size_t)7;
  size_t elems = 4 * ((size_t)m * rc + 2) + 2 * FAC_STAGES * (rows_alloc * solve_lda(m) + 2) +
                 2 * (size_t)solve5_nsl(m, rc, C, mma) * rows_max * rc;
  return std::max<size_t>(256 + elems * sizeof(cplx), 118 * 1024);
}

typedef void (*Solve5Fn)(const SolveVisit *, int, int, int, int, int);

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
static int solve5_max_clusters(Solve5Fn fn, int C, size_t smem) {
  return solve_max_clusters((const void *)fn, SOLVE_THREADS, C, smem);
}

// Choose the (cluster size, RHS chunk) that runs a step of nvisit visits in
// the fewest waves of co-resident clusters, then with the least arithmetic
// per CTA and stage (rows per CTA x chunk width); larger clusters on ties.
template <typename SmemFn>
static bool pick_cluster_chunk(const void *fn, int threads, int nvisit, int nrhs, int max_m,
                               bool mma, SmemFn smem_of, int *Cout, int *rcout, long *waves_out) {
  static const int rc_min = std::max(1, env_int("DS_K3_RCMIN", 4));
  static const int rc_max = std::max(1, env_int("DS_K3_RCMAX", 16));
  static const int c_only = env_int("DS_K3_CLUSTER", 0);
  int bestC = 0, bestRc = 0;
  long best_waves = 0, best_work = 0, best_waste = 0;
  for (int C : {16, 8}) {
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
      bool better = !bestC || waves < best_waves || (waves == best_waves && work < best_work);
      if (!better && waves == best_waves && work == best_work)
        better = waste < best_waste || (waste == best_waste && C < bestC);
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

static size_t solve6_smem(int m, int rc, int C) {
  size_t rows_max = solve_rows_max(m, C);
  size_t rows_alloc = (rows_max + 7) & ~(size_t)7;
  size_t elems = 4 * ((size_t)m * rc + 2) + 2 * FAC_STAGES * (rows_alloc * m + 2) +
                 2 * 4 * rows_max * rc;
  return std::max<size_t>(256 + elems * sizeof(cplx), 118 * 1024);
}

static int launch_v7(ds_ctx *ctx, const void *visits_dev, int nvisit, int nrhs, int max_m) {
  const void *fn = (const void *)k_block_solve7;
  int C, rc;
  long waves;
  if (!pick_cluster_chunk(fn, SOLVE_THREADS, nvisit, nrhs, max_m, true,
                          [&](int r, int c) { return solve7_smem(max_m, r, c); }, &C, &rc, &waves))
    return ds_fail(DS_ECONFIG, "block solve v7: no feasible cluster configuration");
  const size_t smem = solve7_smem(max_m, rc, C);
  if (env_int("DS_K3_DEBUG", 0))
    fprintf(stderr, "K3 v7: nvisit %d nrhs %d m %d -> C %d rc %d waves %ld smem %zu\n", nvisit,
            nrhs, max_m, C, rc, waves, smem);
  DS_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3(C, nvisit, (nrhs + rc - 1) / rc);
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
  DS_CUDA(cudaLaunchKernelEx(&cfg, k_block_solve7, (const SolveVisit *)visits_dev, nrhs, rc,
                             solve_rows_max(max_m, C)));
  ctx->launches++;
  return DS_OK;
}

static int launch_v8(ds_ctx *ctx, const void *visits_dev, int nvisit, int nrhs, int max_m) {
  // warps per half: 4 (256 threads) or 8 (512 threads, more latency hiding
  // for the lockstep DMMA product, 128 registers)
  static const int nw = env_int("DS_K3_NW", 4) >= 8 ? 8 : 4;
  const int threads = 64 * nw;
  const void *fn16 = nw == 8 ? (const void *)k_block_solve8<1, 8> : (const void *)k_block_solve8<1, 4>;
  int C, rc;
  long waves;
  if (!pick_cluster_chunk(fn16, threads, nvisit, nrhs, max_m, true,
                          [&](int r, int c) { return solve8_smem(max_m, r, c, nw); }, &C, &rc, &waves))
    return ds_fail(DS_ECONFIG, "block solve v8: no feasible cluster configuration");
  const int rows = solve_rows_max(max_m, C);
  const void *fn = rows > 8 ? (nw == 8 ? (const void *)k_block_solve8<2, 8> : (const void *)k_block_solve8<2, 4>)
                            : fn16;
  const size_t smem = solve8_smem(max_m, rc, C, nw);
  if (env_int("DS_K3_DEBUG", 0))
    fprintf(stderr, "K3 v8: nvisit %d nrhs %d m %d -> C %d rc %d waves %ld smem %zu nw %d\n", nvisit,
            nrhs, max_m, C, rc, waves, smem, nw);
  cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  DS_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3(C, nvisit, (nrhs + rc - 1) / rc);
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

static int launch_v6(ds_ctx *ctx, const void *visits_dev, int nvisit, int nrhs, int max_m) {
  const void *fn = (const void *)k_block_solve6;
  int C, rc;
  long waves;
  if (!pick_cluster_chunk(fn, SOLVE6_THREADS, nvisit, nrhs, max_m, true,
                          [&](int r, int c) { return solve6_smem(max_m, r, c); }, &C, &rc, &waves))
    return ds_fail(DS_ECONFIG, "block solve v6: no feasible cluster configuration");
  const size_t smem = solve6_smem(max_m, rc, C);
  if (env_int("DS_K3_DEBUG", 0))
    fprintf(stderr, "K3 v6: nvisit %d nrhs %d m %d -> C %d rc %d waves %ld smem %zu\n", nvisit,
            nrhs, max_m, C, rc, waves, smem);
  DS_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3(C, nvisit, (nrhs + rc - 1) / rc);
  cfg.blockDim = dim3(SOLVE6_THREADS, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  DS_CUDA(cudaLaunchKernelEx(&cfg, k_block_solve6, (const SolveVisit *)visits_dev, nrhs, rc,
                             solve_rows_max(max_m, C)));
  ctx->launches++;
  return DS_OK;
}

static int launch_v5(ds_ctx *ctx, const void *visits_dev, int nvisit, int nrhs, int max_m) {
  static const bool mma = env_int("DS_K3_MMA", 1) != 0;
  static const int rc_min = std::max(1, env_int("DS_K3_RCMIN", 4));
  static const int rc_max = std::max(1, env_int("DS_K3_RCMAX", 16));
  static const int c_only = env_int("DS_K3_CLUSTER", 0);
  static const int lda_pad = env_int("DS_K3_LDA_PAD", 0);
  Solve5Fn fn = mma ? k_block_solve5<true> : k_block_solve5<false>;
  // The step is latency bound (one cluster per (visit, RHS chunk), ~n_b
  // dependent stages each).  Choose the (cluster size, chunk) that runs the
  // step in the fewest waves of co-resident clusters, then with the least
  // arithmetic per CTA and stage (rows per CTA x chunk width).
  int bestC = 0, bestRc = 0;
  long best_waves = 0, best_work = 0, best_waste = 0;
  for (int C : {16, 8}) {
    if (c_only && C != c_only) continue;
    const int rows = solve_rows_max(max_m, C);
    for (int rc = std::min(nrhs, rc_max); rc >= 1; rc = rc > 1 ? (rc + 1) / 2 : 0) {
      if (rc < std::min(rc_min, nrhs) && bestC) break;
      if (rows * rc > 256 || (mma && rows > 16)) continue;
      size_t smem = solve5_smem(max_m, rc, C, mma);
      if (smem > 232448) continue;
      int maxcl = solve5_max_clusters(fn, C, smem);
      if (maxcl < 1) continue;
      long ncl = (long)nvisit * ((nrhs + rc - 1) / rc);
      long waves = (ncl + maxcl - 1) / maxcl;
      long work = waves * (long)rows * rc;
      // DMMA tile padding: rows and RHS are computed in 8 x 8 tiles
      long waste = (long)((rows + 7) / 8 * 8) * ((rc + 7) / 8 * 8) - (long)rows * rc;
      // ties (same waves and work per CTA): less padding, then the smaller
      // cluster -- config 2 measured 8 CTAs x (16 rows, 8 RHS) faster than
      // 16 CTAs x (8 rows, 16 RHS): half as many CTAs in every exchange
      bool better = !bestC || waves < best_waves || (waves == best_waves && work < best_work);
      if (!better && waves == best_waves && work == best_work)
        better = waste < best_waste || (waste == best_waste && C < bestC);
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
  if (!bestC) return ds_fail(DS_ECONFIG, "block solve v5: no feasible cluster configuration");
  const int C = bestC, rc = bestRc;
  const size_t smem = solve5_smem(max_m, rc, C, mma);
  if (env_int("DS_K3_DEBUG", 0))
    fprintf(stderr, "K3 v5: nvisit %d nrhs %d m %d -> C %d rc %d waves %ld maxcl %d smem %zu\n", nvisit,
            nrhs, max_m, C, rc, best_waves, solve5_max_clusters(fn, C, smem), smem);
  DS_CUDA(cudaFuncSetAttribute((const void *)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3(C, nvisit, (nrhs + rc - 1) / rc);
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
  DS_CUDA(cudaLaunchKernelEx(&cfg, fn, (const SolveVisit *)visits_dev, nrhs, rc,
                             solve_rows_max(max_m, C), solve5_nsl(max_m, rc, C, mma), lda_pad));
  ctx->launches++;
  return DS_OK;
}

int ds_launch_solve_table(ds_ctx *ctx, const void *visits_dev, int nvisit, int nrhs,
                          int max_m) {
  if (nvisit < 1) return DS_OK;
  {
    const char *v = getenv("DS_K3");
    const std::string k3 = v ? v : "v8";
    if (k3 == "v8") return launch_v8(ctx, visits_dev, nvisit, nrhs, max_m);
    if (k3 == "v7") return launch_v7(ctx, visits_dev, nvisit, nrhs, max_m);
    if (k3 == "v6") return launch_v6(ctx, visits_dev, nvisit, nrhs, max_m);
    if (k3 == "v5") return launch_v5(ctx, visits_dev, nvisit, nrhs, max_m);
  }
  SolveCfg sc;
  if (!pick_cfg(max_m, nrhs, &sc))
    return ds_fail(DS_ECONFIG, "block solve: no feasible cluster configuration");
  DS_CUDA(cudaFuncSetAttribute(k_block_solve, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)sc.smem));
  int nchunks = (nrhs + sc.rc - 1) / sc.rc;
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3(sc.C, nvisit, nchunks);
  cfg.blockDim = dim3(SOLVE_THREADS, 1, 1);
  cfg.dynamicSmemBytes = sc.smem;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = sc.C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  DS_CUDA(cudaLaunchKernelEx(&cfg, k_block_solve, (const SolveVisit *)visits_dev, nrhs, sc.rc,
                             sc.G, sc.rows_max));
  ctx->launches++;
  return DS_OK;
}

#ifdef DS_SOLVE_TRACE
extern "C" DS_API int ds_debug_solve_trace(long long *out) {
  DS_CUDA(cudaMemcpyFromSymbol(out, g_solve_trace, sizeof(long long) * 2 * 1024 * 6));
  return DS_OK;
}
#endif

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
