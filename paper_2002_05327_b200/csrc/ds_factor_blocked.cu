// K2b: blocked factorization for large slabs (3D windows, m ~ 460-4225).
//
// Same twisted block LU as the on-chip path (ds_factor.cu): every chain
// (operator, half) walks its blocks; at each step the Schur complement
//     S = D_k - c1 * S_prev1^{-1} - c2 * S_prev2^{-1}
// is formed directly in the block's factor slot and inverted in place by a
// right-looking blocked Gauss-Jordan with partial pivoting.  Columns go in
// macro-panels of MW = 128 (4 sub-panels of BW = 32):
//   1. per sub-panel: one thread-block cluster per matrix keeps the m x BW
//      panel in distributed shared memory and runs the BW pivot steps
//      (cluster-wide argmax, row interchange through DSMEM, elimination);
//      its row interchanges go to every other column; its rank-BW update
//      A += P'_s T_s is applied to the macro-panel's columns only
//      (P'_s = sub-panel with I subtracted on the pivot rows, T_s = the
//      pivot rows, zero on the sub-panel) -- the macro-panel then holds the
//      pivot columns of the composite elimination E = E_3 .. E_0;
//   2. one rank-MW update of every column outside the macro-panel,
//      A += (E - I)[:, pivots] A[pivot rows, :]   (8 m^2 MW flop, a plain
//      complex GEMM: k_zgemm_acc below, every matrix of the step in one
//      launch) -- a quarter of the full-matrix passes of rank-32 updates and
//      a K = 128 product instead of K = 32 (config 5: 1.68 s per window at
//      MW = 32).  Until round 2 the updates were cublasZgemm3m calls, one
//      per matrix: six config-5 windows 8.08 s one by one / 4.23 s batched
//      with cuBLAS, 5.70 / 3.71 s with k_zgemm_acc (14.1 / 23.6 TFLOP/s).
// Column interchanges are undone at the end.  All chains of a step are
// batched (one panel / swap / copy launch per step for every matrix).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "ds_common.cuh"
#include "ds_factor.cuh"
#include "ds_mma.cuh"

namespace cg = cooperative_groups;

#define BW 32
#define MW 128  // macro-panel: columns per full-matrix update
#define PANEL_THREADS 512
static_assert(PANEL_THREADS == 16 * BW, "panel kernel: one candidate-row element per thread, 16-CTA clusters at most");

struct BlkTask {   // one matrix being inverted at the current chain step
  FactJob J;       // operator, layout, factor base
  int k;           // block index
  cplx co1, co2;   // Schur coefficients (0 if absent)
  int p1, p2;      // previous blocks (-1 if absent)
  cplx *A;         // the m x m matrix (factor slot k)
  int *piv;        // [m] pivot rows
  cplx *T;         // [MW][m]  pivot rows outside the panel
  cplx *P;         // [m][MW]  panel with I subtracted on pivot rows
};

// S = D_k - co1 * A[p1] - co2 * A[p2]   (whole m x m, row-major)
__global__ void k_form_schur(const BlkTask *__restrict__ tasks) {
  const BlkTask &X = tasks[blockIdx.y];
  const int m = X.J.f.m;
  const cplx *s1 = X.p1 >= 0 ? X.J.sinv + (size_t)X.p1 * m * m : nullptr;
  const cplx *s2 = X.p2 >= 0 ? X.J.sinv + (size_t)X.p2 * m * m : nullptr;
  const int64_t total = (int64_t)m * m;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int i = (int)(e / m), c = (int)(e % m);
    cplx v = d_entry(X.J, X.k, i, c);
    if (s1) v = csub(v, cmul(X.co1, s1[e]));
    if (s2) v = csub(v, cmul(X.co2, s2[e]));
    X.A[e] = v;
  }
}

// Panel Gauss-Jordan on columns [p, p+BW) of every task's matrix.  Cluster
// rank q holds rows [q*rpc, q*rpc + rpc) of the panel in shared memory.
// One cluster barrier per pivot step: every CTA publishes its local argmax
// (value, row index and a copy of that row) and, if it owns it, a copy of
// row j, in a buffer of parity jj & 1; after the barrier every CTA reduces
// the C candidates and reads the two rows it needs from the publishers.  A
// buffer of parity b is rewritten two steps later, after the next barrier,
// which every reader of step jj passes only when done reading.  (The
// original form -- candidates, pivot, row fetch and elimination separated
// by three cluster barriers and a serial candidate loop -- took 263 us per
// 32-column panel at m = 2793, 58% of the config-5 factorization.)
// Pivot choice (largest |.|_1, lowest row on ties) and arithmetic unchanged.
__global__ void __launch_bounds__(PANEL_THREADS, 1)
    k_panel_gj(const BlkTask *__restrict__ tasks, int p, int rpc_max, int *status) {
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank(), C = (int)cluster.num_blocks();
  const BlkTask &X = tasks[blockIdx.y];
  const int m = X.J.f.m;
  if (p >= m) return;  // uniform for the cluster
  const int bw = min(BW, m - p);
  const int rpc = (m + C - 1) / C;
  const int r0 = rank * rpc, r1 = min(m, r0 + rpc);
  const int t = threadIdx.x, lane = t & 31;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cplx *pan = (cplx *)smem_raw;            // [rpc_max][BW]
  cplx *rowj = pan + (size_t)rpc_max * BW; // [BW]
  cplx *rowp = rowj + BW;                  // [BW]
  __shared__ cplx pub_row[2][BW];          // my candidate row, per parity
  __shared__ cplx pub_rowj[2][BW];         // row j (if mine), per parity
  __shared__ double pub_v[2];
  __shared__ int pub_i[2];
  __shared__ double red_v[PANEL_THREADS / 32];
  __shared__ int red_i[PANEL_THREADS / 32];
  __shared__ int s_piv, s_win;
  __shared__ double s_best;
  __shared__ cplx cand[16][BW];            // every CTA's candidate row of this step

  for (int e = t; e < (r1 - r0) * BW; e += PANEL_THREADS) {
    int r = e / BW, c = e % BW;
    pan[e] = c < bw ? X.A[(size_t)(r0 + r) * m + p + c] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  for (int jj = 0; jj < bw; ++jj) {
    const int j = p + jj, b = jj & 1;
    // (a) local argmax of |A[r][j]|_1 over my rows r >= j
    double best = -1.0;
    int bi = m;
    for (int r = max(r0, j) + t; r < r1; r += PANEL_THREADS) {
      double v = cabs1(pan[(r - r0) * BW + jj]);
      if (v > best || (v == best && r < bi)) { best = v; bi = r; }
    }
    for (int off = 16; off > 0; off >>= 1) {
      double ov = __shfl_down_sync(0xffffffffu, best, off);
      int oi = __shfl_down_sync(0xffffffffu, bi, off);
      if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
    }
    if (lane == 0) { red_v[t >> 5] = best; red_i[t >> 5] = bi; }
    __syncthreads();
    if (t < 32) {
      double bv = lane < PANEL_THREADS / 32 ? red_v[lane] : -1.0;
      int bidx = lane < PANEL_THREADS / 32 ? red_i[lane] : m;
      for (int off = 16; off > 0; off >>= 1) {
        double ov = __shfl_down_sync(0xffffffffu, bv, off);
        int oi = __shfl_down_sync(0xffffffffu, bidx, off);
        if (ov > bv || (ov == bv && oi < bidx)) { bv = ov; bidx = oi; }
      }
      bidx = __shfl_sync(0xffffffffu, bidx, 0);
      if (lane == 0) { pub_v[b] = bv; pub_i[b] = bidx; }
      // (a2) publish the candidate row and, if mine, row j
      pub_row[b][lane] = (bidx < m && lane < BW) ? pan[(bidx - r0) * BW + lane] : make_double2(0.0, 0.0);
      if (j >= r0 && j < r1) pub_rowj[b][lane] = pan[(j - r0) * BW + lane];
    }
    cluster.sync();
    // (b) + (c) in one remote round trip: every candidate row (C x BW
    // values, one per thread) and row j (its owner is known) are fetched
    // while warp 0 reduces the C candidates; the winner's row is then picked
    // from the local copy
    {
      const int q = t / BW, c = t % BW;  // PANEL_THREADS = 16 x BW: one element per thread
      if (q < C) cand[q][c] = *cluster.map_shared_rank(&pub_row[b][c], q);
    }
    if (t >= PANEL_THREADS - BW) {  // (the last warp: its candidate fetch above is one more load)
      const int c = t - (PANEL_THREADS - BW);
      rowj[c] = *cluster.map_shared_rank(&pub_rowj[b][c], j / rpc);
    }
    if (t < 32) {
      double v = -1.0;
      int i = m, q = C;
      if (lane < C) {
        v = *cluster.map_shared_rank(&pub_v[b], lane);
        i = *cluster.map_shared_rank(&pub_i[b], lane);
        q = lane;
      }
      for (int off = 16; off > 0; off >>= 1) {
        double ov = __shfl_down_sync(0xffffffffu, v, off);
        int oi = __shfl_down_sync(0xffffffffu, i, off);
        int oq = __shfl_down_sync(0xffffffffu, q, off);
        if (ov > v || (ov == v && oi < i)) { v = ov; i = oi; q = oq; }
      }
      if (lane == 0) {
        s_piv = i;
        s_best = v;
        s_win = q < C ? q : 0;
      }
    }
    __syncthreads();
    if (t < BW) rowp[t] = cand[s_win][t];
    __syncthreads();
    const int pv = min(s_piv, m - 1);
    if (t == 0) {
      if (rank == 0) X.piv[j] = s_piv;
      if (!(s_best > 0.0) || s_piv >= m) atomicExch(status, 1);
    }
    // (d) eliminate: new row j = old row pv scaled; other rows updated.  A
    // thread's elements share one column (PANEL_THREADS % BW == 0), so the
    // scaled pivot-row entry is formed once per step
    const cplx pivot = rowp[jj];
    const cplx inv = cinv(pivot);
    {
      const int c = t % BW;
      const cplx rpc_c = rowp[c], rjc = rowj[c], rjj = rowj[jj];
      const cplx rs = cmul(rpc_c, inv);  // rowp[c] / pivot
      if (c < bw)
        for (int e = t; e < (r1 - r0) * BW; e += PANEL_THREADS) {
          const int r = r0 + e / BW;
          cplx nv;
          if (r == j) {
            nv = c == jj ? inv : rs;
          } else {
            const cplx fr = r == pv ? rjj : pan[(r - r0) * BW + jj];
            if (c == jj) nv = cmul(make_double2(-fr.x, -fr.y), inv);
            else nv = csub(r == pv ? rjc : pan[e], cmul(fr, rs));
          }
          pan[e] = nv;
        }
    }
    __syncthreads();
  }
  for (int e = t; e < (r1 - r0) * BW; e += PANEL_THREADS) {
    int r = e / BW, c = e % BW;
    if (c < bw) X.A[(size_t)(r0 + r) * m + p + c] = pan[e];
  }
  cluster.sync();  // no CTA leaves while another may still read its buffers
}

// apply the panel's row interchanges to the columns outside the panel
__global__ void k_row_swaps(const BlkTask *__restrict__ tasks, int p) {
  const BlkTask &X = tasks[blockIdx.y];
  const int m = X.J.f.m;
  if (p >= m) return;
  const int bw = min(BW, m - p);
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < m; c += gridDim.x * blockDim.x) {
    if (c >= p && c < p + bw) continue;
    for (int jj = 0; jj < bw; ++jj) {
      const int j = p + jj, pv = X.piv[j];
      if (pv == j) continue;
      cplx a = X.A[(size_t)j * m + c], b = X.A[(size_t)pv * m + c];
      X.A[(size_t)j * m + c] = b;
      X.A[(size_t)pv * m + c] = a;
    }
  }
}

// T = pivot rows [p, p+w) outside the panel (zero on the panel columns);
// P' = panel columns [p, p+w) with I subtracted on the pivot rows; w <= W,
// the buffers' row pitch / column count (BW for a sub-panel, MW for a
// macro-panel)
__global__ void k_panel_operands(const BlkTask *__restrict__ tasks, int p, int width, int W) {
  const BlkTask &X = tasks[blockIdx.y];
  const int m = X.J.f.m;
  if (p >= m) return;
  const int bw = min(width, m - p);
  const int64_t nT = (int64_t)W * m, nP = (int64_t)m * W;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nT + nP;
       e += (int64_t)gridDim.x * blockDim.x) {
    if (e < nT) {
      int tr = (int)(e / m), c = (int)(e % m);
      cplx v = make_double2(0.0, 0.0);
      if (tr < bw && !(c >= p && c < p + bw)) v = X.A[(size_t)(p + tr) * m + c];
      X.T[e] = v;
    } else {
      int64_t f = e - nT;
      int r = (int)(f / W), tc = (int)(f % W);
      cplx v = make_double2(0.0, 0.0);
      if (tc < bw) {
        v = X.A[(size_t)r * m + p + tc];
        if (r == p + tc) v.x -= 1.0;
      }
      X.P[f] = v;
    }
  }
}

// K2b trailing update on the FP64 tensor cores, every matrix of the step in
// one launch:  A[r][c0 + c] += sum_kk P[r][kk] T[kk][c0 + c]   (r < m,
// c < nc, kk < K; A, T row-major with pitch m, P with pitch ldp).  The tile
// kernel of the modal transforms (ds_modal.cu, K3m-T): 32 x 32 per CTA,
// 4 warps of 16 x 16, K chunks of 8 through a 4-stage cp.async ring, DMMA
// m8n8k4, 3M complex product (6 real flop per complex multiply-add, the
// imaginary part formed by subtraction -- the factorization residuals stay
// <= 1e-10, tests/test_gpu_pool.py).
// mode 0: a sub-panel's rank-BW update of its macro-panel's columns
// (c0 = p0, nc = min(MW, m - p0), skipped when the macro-panel is the
// sub-panel); mode 1: the macro-panel's rank-MW update of every column.
#define ZG_TM 32
#define ZG_TN 32
#define ZG_TK 8
#define ZG_NS 4
__global__ void __launch_bounds__(128, 4)
    k_zgemm_acc(const BlkTask *__restrict__ tasks, int p, int c0, int ncmax, int K, int ldp, int mode) {
  constexpr int TM = ZG_TM, TN = ZG_TN, TK = ZG_TK, NS = ZG_NS, NTH = 128, MT = 2;
  constexpr int AP = TK + 4, BP = TN + 2;
  constexpr int A_STEP = NTH / TK, A_N = TM / A_STEP, B_STEP = NTH / TN, B_N = TK / B_STEP;
  constexpr uint32_t A_BUF = TM * AP * sizeof(cplx), B_BUF = TK * BP * sizeof(cplx);
  __shared__ __align__(16) cplx smem[NS * (TM * AP + TK * BP)];
  const BlkTask &X = tasks[blockIdx.z];
  const int m = X.J.f.m;
  if (p >= m) return;
  const int nc = min(ncmax, m - c0);
  if (mode == 0 ? nc <= min(BW, m - p) : min(MW, m - p) >= m) return;
  const int row0 = blockIdx.y * TM, col0 = blockIdx.x * TN;
  if (row0 >= m || col0 >= nc) return;
  const int t = threadIdx.x;
  const int a_col = t % TK, a_row = t / TK, b_col = t % TN, b_row = t / TN;
  const cplx *srcA[A_N];
  bool okA[A_N];
#pragma unroll
  for (int q = 0; q < A_N; ++q) {
    const int gr = row0 + a_row + q * A_STEP;
    okA[q] = gr < m;
    srcA[q] = X.P + (okA[q] ? (size_t)gr * ldp + a_col : 0);
  }
  const bool bok = col0 + b_col < nc;
  const cplx *srcB = X.T + (bok ? (size_t)b_row * m + c0 + col0 + b_col : 0);
  const uint32_t dstA = smem_addr(smem + a_row * AP + a_col);
  const uint32_t dstB = smem_addr(smem + NS * TM * AP + b_row * BP + b_col);
  auto stage = [&](int kc, int buf, bool on) {
    const int k0 = kc * TK;
#pragma unroll
    for (int q = 0; q < A_N; ++q) {
      const bool ok = on && okA[q] && k0 + a_col < K;
      cp16s(dstA + buf * A_BUF + q * (A_STEP * AP * (uint32_t)sizeof(cplx)), srcA[q] + (ok ? k0 : 0),
            ok ? 16 : 0);
    }
#pragma unroll
    for (int q = 0; q < B_N; ++q) {
      const int r = q * B_STEP;
      const bool ok = on && bok && k0 + b_row + r < K;
      cp16s(dstB + buf * B_BUF + r * (BP * (uint32_t)sizeof(cplx)), srcB + (ok ? (size_t)(k0 + r) * m : 0),
            ok ? 16 : 0);
    }
    cp_commit();
  };
  const int warp = t >> 5, lane = t & 31, g = lane >> 2, tg = lane & 3;
  const int wr = warp % 2, wc = warp / 2;
  const int nk = (K + TK - 1) / TK;
#pragma unroll
  for (int i = 0; i < NS - 1; ++i) stage(i, i, i < nk);
  const cplx *fragA = smem + (wr * 8 * MT + g) * AP + tg;
  const cplx *fragB = smem + NS * TM * AP + tg * BP + wc * 16 + g;
  double p1[MT][2][2] = {}, p2[MT][2][2] = {}, p3[MT][2][2] = {};
  for (int it = 0; it < nk; ++it) {
    const int buf = it % NS;
    cp_wait<NS - 2>();
    __syncthreads();
    const cplx *As = fragA + buf * (TM * AP), *Bs = fragB + buf * (TK * BP);
    cplx a[TK / 4][MT], b[TK / 4][2];
#pragma unroll
    for (int k4 = 0; k4 < TK / 4; ++k4) {
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) a[k4][mt] = As[mt * 8 * AP + k4 * 4];
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) b[k4][nt] = Bs[k4 * 4 * BP + nt * 8];
    }
    stage(it + NS - 1, (it + NS - 1) % NS, it + NS - 1 < nk);
#pragma unroll
    for (int k4 = 0; k4 < TK / 4; ++k4) {
      double bs[2] = {b[k4][0].x + b[k4][0].y, b[k4][1].x + b[k4][1].y};
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const double as = a[k4][mt].x + a[k4][mt].y;
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          dmma_nv(p1[mt][nt], a[k4][mt].x, b[k4][nt].x);
          dmma_nv(p2[mt][nt], a[k4][mt].y, b[k4][nt].y);
          dmma_nv(p3[mt][nt], as, bs[nt]);
        }
      }
    }
  }
  cp_wait<0>();
  // A += product: Re = P1 - P2, Im = P3 - P1 - P2
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
    const int gr = row0 + wr * 8 * MT + mt * 8 + g;
    if (gr >= m) continue;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      const int cc = col0 + wc * 16 + nt * 8 + 2 * tg;  // two adjacent columns
      cplx *dst = X.A + (size_t)gr * m + c0 + cc;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        if (cc + e >= nc) continue;
        const cplx o = dst[e];
        dst[e] = make_double2(o.x + (p1[mt][nt][e] - p2[mt][nt][e]),
                              o.y + (p3[mt][nt][e] - p1[mt][nt][e] - p2[mt][nt][e]));
      }
    }
  }
}

// undo the column interchanges: A[r][c] <- A[r][src[c]] (one CTA per row)
__global__ void k_col_unpermute(const BlkTask *__restrict__ tasks, int *srcbuf, int mmax) {
  const BlkTask &X = tasks[blockIdx.y];
  const int m = X.J.f.m;
  int *src = srcbuf + (size_t)blockIdx.y * mmax;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cplx *row = (cplx *)smem_raw;
  for (int r = blockIdx.x; r < m; r += gridDim.x) {
    for (int c = threadIdx.x; c < m; c += blockDim.x) row[c] = X.A[(size_t)r * m + c];
    __syncthreads();
    for (int c = threadIdx.x; c < m; c += blockDim.x) X.A[(size_t)r * m + c] = row[src[c]];
    __syncthreads();
  }
}

__global__ void k_src_map(const BlkTask *__restrict__ tasks, int *srcbuf, int mmax) {
  const BlkTask &X = tasks[blockIdx.x];
  const int m = X.J.f.m;
  int *src = srcbuf + (size_t)blockIdx.x * mmax;
  if (threadIdx.x != 0) return;
  for (int c = 0; c < m; ++c) src[c] = c;
  for (int j = m - 1; j >= 0; --j) {
    int a = src[j];
    src[j] = src[X.piv[j]];
    src[X.piv[j]] = a;
  }
}

static int launch_cluster(const void *kern, dim3 grid, int C, size_t smem, cudaStream_t st,
                          void **args) {
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = grid;
  cfg.blockDim = dim3(PANEL_THREADS, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  DS_CUDA(cudaLaunchKernelExC(&cfg, kern, args));
  return DS_OK;
}

// panel cluster size and shared memory for slabs up to mmax rows; sets the
// kernels' dynamic shared-memory limits (callers do this once for the
// largest slab before any group starts: the limits are per function, not
// per stream)
static int panel_setup(int mmax, int &PC, size_t &panel_smem) {
  // enough CTAs that the panel rows fit in shared memory (16 CTAs of 512
  // threads from m = 1024 up: a pivot step's elimination is rows/CTA x 32
  // complex updates; 8 x 256 took 242 us per panel at m = 2793)
  PC = mmax >= 1024 ? 16 : 4;
  while (PC < 16 && ((size_t)((mmax + PC - 1) / PC) * BW + 2 * BW) * sizeof(cplx) > 200 * 1024) PC *= 2;
  const int rpc_max = (mmax + PC - 1) / PC;
  panel_smem = ((size_t)rpc_max * BW + 2 * BW) * sizeof(cplx);
  if (panel_smem > 220 * 1024) return ds_fail(DS_ECONFIG, "blocked factorization: slab too large");
  return DS_OK;
}
static int panel_attributes(int mmax) {
  int PC;
  size_t smem;
  if (int rc = panel_setup(mmax, PC, smem)) return rc;
  DS_CUDA(cudaFuncSetAttribute(k_panel_gj, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  DS_CUDA(cudaFuncSetAttribute(k_panel_gj, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  DS_CUDA(cudaFuncSetAttribute(k_col_unpermute, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)(mmax * sizeof(cplx))));
  return DS_OK;
}

// one group of matrices on stream st (host-synchronous: returns with the
// stream drained); `launches` counts the kernels issued
static int blocked_factor_group(ds_ctx *ctx, cudaStream_t st, const FactJob *jobs, int njobs,
                                const cplx *const *lh, const cplx *const *uh, int *status,
                                int64_t &launches) {
  if (njobs == 0) return DS_OK;
  int mmax = 0;
  for (int i = 0; i < njobs; ++i) mmax = std::max(mmax, jobs[i].f.m);
  int PC;
  size_t panel_smem;
  if (int rc0 = panel_setup(mmax, PC, panel_smem)) return rc0;
  const int rpc_max = (mmax + PC - 1) / PC;
  // per-chain workspaces (pivots, T, P', unpermute map)
  std::vector<void *> ws;
  auto alloc = [&](size_t bytes) -> void * {
    void *p = nullptr;
    if (cudaMalloc(&p, bytes) != cudaSuccess) return nullptr;
    ws.push_back(p);
    return p;
  };
  const int nchains = 2 * njobs;
  int *piv = (int *)alloc(sizeof(int) * (size_t)nchains * mmax);
  int *srcb = (int *)alloc(sizeof(int) * (size_t)nchains * mmax);
  cplx *Tb = (cplx *)alloc(sizeof(cplx) * (size_t)nchains * MW * mmax);
  cplx *Pb = (cplx *)alloc(sizeof(cplx) * (size_t)nchains * MW * mmax);
  BlkTask *dtasks = (BlkTask *)alloc(sizeof(BlkTask) * nchains);
  auto cleanup = [&]() {
    for (void *p : ws) cudaFree(p);
  };
  if (!piv || !srcb || !Tb || !Pb || !dtasks) {
    cleanup();
    return ds_fail(DS_ECUDA, "blocked factorization: out of device memory for workspaces");
  }
  int rc = DS_OK;
  // phases: 0 = chains (top and bottom halves together), 1 = middle blocks
  for (int phase = 0; phase < 2 && rc == DS_OK; ++phase) {
    int maxsteps = 0;
    for (int i = 0; i < njobs; ++i) {
      const FactDev &f = jobs[i].f;
      maxsteps = std::max(maxsteps, phase == 0 ? std::max(f.twist, f.nb - 1 - f.twist) : 1);
    }
    for (int step = 0; step < maxsteps && rc == DS_OK; ++step) {
      std::vector<BlkTask> tasks;
      std::vector<int> task_job;
      for (int i = 0; i < njobs; ++i) {
        const FactJob &J = jobs[i];
        const FactDev &f = J.f;
        const int ba = f.block_axis, nb = f.nb, tw = f.twist;
        for (int half = (phase == 0 ? 0 : 2); half <= (phase == 0 ? 1 : 2); ++half) {
          int nsteps = half == 0 ? tw : (half == 1 ? nb - 1 - tw : 1);
          if (step >= nsteps) continue;
          BlkTask X;
          memset(&X, 0, sizeof(X));
          X.J = J;
          X.k = half == 0 ? step : (half == 1 ? nb - 1 - step : tw);
          X.p1 = X.p2 = -1;
          const int k = X.k;
          if ((half == 0 || half == 2) && k > 0) X.p1 = k - 1;
          if ((half == 1 || half == 2) && k < nb - 1) X.p2 = k + 1;
          // coefficients from the host copies held by the job's operator view
          X.A = J.sinv + (size_t)k * f.m * f.m;
          size_t slot = tasks.size();
          X.piv = piv + slot * mmax;
          X.T = Tb + slot * MW * mmax;
          X.P = Pb + slot * MW * mmax;
          (void)ba;
          tasks.push_back(X);
          task_job.push_back(i);
        }
      }
      if (tasks.empty()) continue;
      // Schur coefficients from the host copies of the block-axis couplings
      for (size_t ti = 0; ti < tasks.size(); ++ti) {
        BlkTask &X = tasks[ti];
        const cplx *hl = lh[task_job[ti]], *hu = uh[task_job[ti]];
        const int k = X.k;
        if (X.p1 >= 0) X.co1 = cmul(hl[k], hu[k - 1]);  // l_k u_{k-1}
        if (X.p2 >= 0) X.co2 = cmul(hu[k], hl[k + 1]);  // u_k l_{k+1}
      }
      const int nt = (int)tasks.size();
      DS_CUDA(cudaMemcpyAsync(dtasks, tasks.data(), sizeof(BlkTask) * nt, cudaMemcpyHostToDevice, st));
      int mstep = 0;
      for (auto &X : tasks) mstep = std::max(mstep, X.J.f.m);
      k_form_schur<<<dim3(std::max(1, std::min(1024, (int)((int64_t)mstep * mstep / 256 / 4))), nt), 256, 0, st>>>(dtasks);
      launches++;
      for (int p0 = 0; p0 < mstep && rc == DS_OK; p0 += MW) {
        for (int p = p0; p < std::min(p0 + MW, mstep) && rc == DS_OK; p += BW) {
          void *args[] = {(void *)&dtasks, (void *)&p, (void *)&rpc_max, (void *)&status};
          rc = launch_cluster((const void *)k_panel_gj, dim3(PC, nt, 1), PC, panel_smem, st, args);
          if (rc) break;
          k_row_swaps<<<dim3((mstep + 255) / 256, nt), 256, 0, st>>>(dtasks, p);
          int width = BW, W = BW;
          k_panel_operands<<<dim3(std::max(1, (2 * W * mstep + 255) / 256), nt), 256, 0, st>>>(
              dtasks, p, width, W);
          launches += 3;
          // the sub-panel's update, restricted to the macro-panel's columns
          {
            const int ncm = std::min(MW, mstep - p0);
            k_zgemm_acc<<<dim3((ncm + ZG_TN - 1) / ZG_TN, (mstep + ZG_TM - 1) / ZG_TM, nt), 128, 0, st>>>(
                dtasks, p, p0, MW, BW, BW, 0);
            launches++;
          }
          DS_CHECK_LAUNCH();
        }
        if (rc) break;
        // rank-MW update of every column outside the macro-panel
        k_panel_operands<<<dim3(std::max(1, (2 * MW * mstep + 255) / 256), nt), 256, 0, st>>>(
            dtasks, p0, MW, MW);
        launches++;
        k_zgemm_acc<<<dim3((mstep + ZG_TN - 1) / ZG_TN, (mstep + ZG_TM - 1) / ZG_TM, nt), 128, 0, st>>>(
            dtasks, p0, 0, mstep, MW, MW, 1);
        launches++;
        DS_CHECK_LAUNCH();
      }
      if (rc) break;
      k_src_map<<<nt, 32, 0, st>>>(dtasks, srcb, mmax);
      k_col_unpermute<<<dim3(std::min(mstep, 512), nt), 256, mmax * sizeof(cplx), st>>>(dtasks, srcb, mmax);
      launches += 2;
      DS_CHECK_LAUNCH();
      DS_CUDA(cudaStreamSynchronize(st));  // tasks vector reused next step
    }
  }
  cudaStreamSynchronize(st);
  cleanup();
  return rc;
}

// Batches of two or more windows run as up to "k2b_groups" groups, each on
// its own stream and driven by its own host thread: a group's panel kernels
// (one 16-CTA cluster per matrix) leave most SMs idle, and the other groups'
// trailing-update GEMMs fill them ("k2b_groups" = 1: one group).
int ds_blocked_factor(ds_ctx *ctx, const FactJob *jobs, int njobs, const cplx *const *lh,
                      const cplx *const *uh, int *status) {
  if (njobs == 0) return DS_OK;
  int mall = 0;
  for (int i = 0; i < njobs; ++i) mall = std::max(mall, jobs[i].f.m);
  if (int rc0 = panel_attributes(mall)) return rc0;
  const int G = std::max(1, std::min(ctx->opt.k2b_groups, njobs));
  if (G == 1) {
    int64_t l0 = 0;
    const int rc = blocked_factor_group(ctx, ctx->stream, jobs, njobs, lh, uh, status, l0);
    ctx->launches += l0;
    return rc;
  }
  struct Group {
    std::vector<FactJob> jobs;
    std::vector<const cplx *> l, u;
    cudaStream_t st = nullptr;
    int rc = DS_OK;
    int64_t launches = 0;
    std::string err;
  };
  std::vector<Group> gs(G);
  // largest first, dealt in snake order: even work per group
  std::vector<int> order(njobs);
  for (int i = 0; i < njobs; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) {
    return (double)jobs[x].f.nb * jobs[x].f.m * jobs[x].f.m > (double)jobs[y].f.nb * jobs[y].f.m * jobs[y].f.m;
  });
  for (int q = 0; q < njobs; ++q) {
    const int r = q % (2 * G), g = r < G ? r : 2 * G - 1 - r, i = order[q];
    gs[g].jobs.push_back(jobs[i]);
    gs[g].l.push_back(lh[i]);
    gs[g].u.push_back(uh[i]);
  }
  cudaEvent_t ev;
  DS_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  DS_CUDA(cudaEventRecord(ev, ctx->stream));  // every group after the caller's prior work
  gs[0].st = ctx->stream;
  for (int g = 1; g < G; ++g) {
    DS_CUDA(cudaStreamCreateWithFlags(&gs[g].st, cudaStreamNonBlocking));
    DS_CUDA(cudaStreamWaitEvent(gs[g].st, ev, 0));
  }
  auto run = [&](Group &gr) {
    gr.rc = blocked_factor_group(ctx, gr.st, gr.jobs.data(), (int)gr.jobs.size(), gr.l.data(), gr.u.data(),
                                 status, gr.launches);
    if (gr.rc) gr.err = ds_last_error();
  };
  std::vector<std::thread> th;
  for (int g = 1; g < G; ++g)
    th.emplace_back([&, g]() {
      cudaSetDevice(ctx->device);
      run(gs[g]);
    });
  run(gs[0]);
  for (auto &t : th) t.join();
  cudaEventDestroy(ev);
  for (int g = 1; g < G; ++g) cudaStreamDestroy(gs[g].st);
  for (auto &gr : gs) ctx->launches += gr.launches;
  for (auto &gr : gs)
    if (gr.rc) return ds_fail(gr.rc, gr.err);
  return DS_OK;
}
