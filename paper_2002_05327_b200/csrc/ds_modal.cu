// K2m / K3m: modal factorization and solve of separable subdomain operators.
//
// Replaces SeparableFactorization (diagsweep/subdomain.py:43-96) for
// operators whose kappa^2 is constant or varies along one axis
// (pml.py 'const' / 'axis'): the window operator is the Kronecker sum of
// per-axis 1D tridiagonals T_a (pml.py:95-102 couplings) plus kappa^2.  The
// reference triangularizes the 1D matrices (Schur) and solves a triangular
// Sylvester equation (ztrsyl), an inherently sequential recurrence.  Here
// the in-slab axes (all axes but the block axis of the block layout) are
// diagonalised instead, T_a = V_a diag(lambda_a) W_a, W_a = V_a^{-1}, so
// with g in block layout [n_b][m][R]:
//
//   1. ghat_k = (W_0 (x) W_1) g_k        for every block k   (batched GEMMs)
//   2. per in-slab mode j: the scalar tridiagonal system along the block
//      axis  l_k y_{k-1} + (d_k + mu_j) y_k + u_k y_{k+1} = ghat_k,
//      mu_j = sum_a lambda_a(j_a), d_k = -(c_lo + c_hi)_ba[k] + kappa^2,
//      by its LU (mode-wise pivots precomputed at factorization time)
//   3. x_k = (V_0 (x) V_1) y_k                                (batched GEMMs)
//
// The flop count of 1 + 3 in 2D equals the block-LU substitution's
// (16 n_b m^2 per RHS) but there is no chain of dependent block products:
// the transforms are plain batched GEMMs over every (visit, block, RHS) of a
// launch on the FP64 tensor cores, and the only recurrence is the cheap
// mode-wise one (O(n_b m) per RHS).  In 3D the in-slab transform factors
// per axis (two small GEMMs per direction), 16 n_b m (n_0 + n_1) flop per
// RHS instead of 16 n_b m^2.  The mode-wise LU has the stability of the
// block LU without block pivoting (its Schur complements are
// V diag(piv_k) W); accuracy vs the reference is ~1e-12.
//
// The eigen-decompositions of the 1D matrices (n_a <= a few hundred) come
// from the host (ds_modal_desc); the device builds the pivots.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "ds_common.cuh"
#include "ds_mma.cuh"

#define RMAX_MODAL 256

// ------------------------------------------------------------ pivots (K2m)
struct PivJob {
  FactDev f;
  OpDev op;
  const cplx *lam[2];
  cplx *mul, *inv;
};

// one thread per (operator, mode j): LU of the block-axis tridiagonal
// shifted by mu_j (no pivoting, as the block LU of ds_factor.cu)
__global__ void k_modal_pivots(const PivJob *__restrict__ jobs, int *status) {
  const PivJob &J = jobs[blockIdx.y];
  const FactDev &f = J.f;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= f.m) return;
  cplx mu = J.lam[0][f.naxes == 1 ? j : j / f.nax[1]];
  if (f.naxes == 2) mu = cadd(mu, J.lam[1][j % f.nax[1]]);
  const int ba = f.block_axis;
  const OpDev &o = J.op;
  cplx prev = make_double2(1.0, 0.0);
  bool bad = false;
  for (int k = 0; k < f.nb; ++k) {
    const cplx lo = o.c_lo[ba][k], hi = o.c_hi[ba][k];
    cplx d = make_double2(-(lo.x + hi.x), -(lo.y + hi.y));
    if (o.kappa2_kind == 0) d.x += o.kappa2[0];
    else if (o.kappa2_kind == 1 && o.kappa2_axis == ba) d.x += o.kappa2[k];
    cplx piv = cadd(d, mu);
    cplx mul = make_double2(0.0, 0.0);
    if (k > 0) {
      mul = cmul(lo, cinv(prev));  // l_k / piv_{k-1}
      piv = csub(piv, cmul(mul, o.c_hi[ba][k - 1]));
    }
    if (!(isfinite(piv.x) && isfinite(piv.y)) || (piv.x == 0.0 && piv.y == 0.0)) bad = true;
    J.mul[(size_t)k * f.m + j] = mul;
    J.inv[(size_t)k * f.m + j] = cinv(piv);
    prev = piv;
  }
  if (bad) atomicExch(status, 1);
}

// ------------------------------------------------------- pass geometry
// forward passes p < naxes transform along in-slab axis a = naxes-1-p with
// W_a; inverse passes p >= naxes along a = p - naxes with V_a.  A pass is
// out[b][j][c] = sum_i A[j][i] in[b][i][c] over `outer` batches of n x ncols
// row-major matrices (n = n_a, ncols = prod_{b>a} n_b * R).
struct PassGeo {
  const cplx *A;
  const cplx *in;
  cplx *out;
  int n, ncols, outer;  // ncols = inner * nrhs: row stride of a batch matrix
  int inner;            // inner in-slab extent (3D pass along axis 0), else 1
};

__host__ __device__ inline PassGeo pass_geo(const FactDev &f, const ModalJob &J, int pass,
                                            int nrhs) {
  PassGeo G;
  const int na = f.naxes;
  const bool fwd = pass < na;
  const int a = fwd ? na - 1 - pass : pass - na;  // na <= 2: selects, no local arrays
  G.n = a == 0 ? f.nax[0] : f.nax[1];
  const int inner = (a == 0 && na == 2) ? f.nax[1] : 1;
  G.outer = f.nb * (a == 1 ? f.nax[0] : 1);
  G.ncols = inner * nrhs;
  G.inner = inner;
  G.A = fwd ? (a == 0 ? f.mW[0] : f.mW[1]) : (a == 0 ? f.mV[0] : f.mV[1]);
  auto buf = [&](int i) { return (i & 1) ? J.s1 : J.s0; };
  if (fwd) {
    G.in = pass == 0 ? J.rhs : buf(pass - 1);
    G.out = buf(pass);
  } else {
    const int q = pass - na;
    G.in = buf(na - 1 + q);
    G.out = q == na - 1 ? J.x : buf(na + q);
  }
  return G;
}

__device__ __forceinline__ bool job_any(const ModalJob &J, int nrhs) {
  if (!J.nz) return true;
  int any = 0;
  for (int r = 0; r < nrhs; ++r) any |= J.nz[r];
  return any != 0;
}

// Active (nonzero) RHS columns of a visit, in order, into shared memory:
// the reference skips exact-zero solves (ddm.py:256-258); here the
// transforms and recurrences also skip the exact-zero RHS columns of
// visits with some nonzero RHS (config 2: 42% of the (visit, RHS) pairs are
// nonzero, 87% of the visits).  Returns the count; call from all threads.
__device__ __forceinline__ int active_rhs(const int *nz, int nrhs, int *act) {
  if (threadIdx.x < 32) {
    int base = 0;
    for (int r0 = 0; r0 < nrhs; r0 += 32) {
      const int r = r0 + (int)threadIdx.x;
      const bool on = r < nrhs && (!nz || nz[r]);
      const unsigned mk = __ballot_sync(0xffffffffu, on);
      if (on) act[base + __popc(mk & ((1u << threadIdx.x) - 1))] = r;
      base += __popc(mk);
    }
    if (threadIdx.x == 0) act[RMAX_MODAL] = base;
  }
  __syncthreads();
  return act[RMAX_MODAL];
}

// compact column c (outer x inner x active) -> element offset of row 0
__device__ __forceinline__ int64_t col_offset(const PassGeo &G, int c, int A, const int *act,
                                              int nrhs) {
  if (A == nrhs) {  // every RHS active: the plain batched layout
    const int b = c / G.ncols;
    return (int64_t)b * G.n * G.ncols + (c - b * G.ncols);
  }
  const int ia = G.inner * A;
  const int b = c / ia, rem = c - b * ia;
  const int ii = rem / A, a = rem - ii * A;
  return (int64_t)b * G.n * G.ncols + (int64_t)ii * nrhs + act[a];
}

// ---------------------------------------------------- transforms (K3m-T)
// One CTA computes a TM x TN tile of one pass of one visit: A tile (TM x TK)
// and B tile (TK x TN) double-buffered through shared memory by cp.async,
// each warp an (8 MT) x 16 sub-tile with DMMA m8n8k4 and the 3M complex
// product (as K3, ds_mma.cuh).  Row pitches: A % 8 == 4, B % 8 == 2 complex
// (conflict-free fragment loads).
// The tile body: rows [row0, row0 + TM) x columns [col0, col0 + colw),
// colw <= TN (columns past colw are zero-filled and not stored).
// NS-stage cp.async ring: chunk kc lives in buffer kc % NS; NS - 1 chunks
// are in flight while one is multiplied (NS = 2: double buffering).
// The K-chunks visited: sparse -- the set bits of kmask in ascending order
// (the others hold exact zeros of B: skipping them leaves every sum's value
// unchanged); dense -- chunks 0 .. nkc-1.
template <int MT, int WR, int WC, int TK, int NS = 2>
__device__ __forceinline__ void gemm_accum(const PassGeo &G, int row0, int col0, int colw, bool sparse,
                                           uint32_t kmask, int nkc, cplx *smem_mg, const int *act,
                                           int A, int nrhs, double (&p1)[MT][2][2],
                                           double (&p2)[MT][2][2], double (&p3)[MT][2][2]) {
  constexpr int NTH = 32 * WR * WC, TM = 8 * MT * WR, TN = 16 * WC;
  constexpr int AP = TK + 4, BP = TN + 2;
  static_assert(NTH % TK == 0 && NTH % TN == 0, "tile/thread mapping");
  constexpr int A_STEP = NTH / TK, A_N = TM / A_STEP;
  constexpr int B_STEP = NTH / TN, B_N = TK / B_STEP;
  static_assert(TM % A_STEP == 0 && TK % B_STEP == 0, "staging maps cover the tiles exactly");
  constexpr uint32_t A_BUF = TM * AP * sizeof(cplx), B_BUF = TK * BP * sizeof(cplx);
  const int n = G.n;
  const int t = threadIdx.x;
  // staging maps: A -- fixed column t % TK, rows t / TK + q * A_STEP;
  // B -- fixed column t % TN, rows t / TN + q * B_STEP.  Everything that
  // does not depend on the chunk is hoisted: per-thread source pointers at
  // chunk 0, shared-memory byte addresses in ring buffer 0, and the row /
  // column validity bits; a chunk then costs one multiply-add per copy.
  const int a_col = t % TK, a_row = t / TK;
  const int b_col = t % TN, b_row = t / TN;
  const bool bcol_ok = b_col < colw;
  const cplx *srcA[A_N];
  bool okA[A_N];
#pragma unroll
  for (int q = 0; q < A_N; ++q) {
    const int gr = row0 + a_row + q * A_STEP;
    okA[q] = gr < n;
    srcA[q] = G.A + (okA[q] ? (int64_t)gr * n + a_col : 0);
  }
  const cplx *srcB = G.in + (bcol_ok ? col_offset(G, col0 + b_col, A, act, nrhs) + (int64_t)b_row * G.ncols : 0);
  const int ncols = G.ncols;
  const uint32_t dstA = smem_addr(smem_mg + a_row * AP + a_col);
  const uint32_t dstB = smem_addr(smem_mg + NS * TM * AP + b_row * BP + b_col);
  // stage chunk kc into ring buffer buf; on == false issues zero-filling
  // copies from a valid address (the loop below stays branch-free, so the
  // copies and their address arithmetic interleave with the DMMAs)
  auto stage = [&](int kc, int buf, bool on) {
    const int k0 = kc * TK;
#pragma unroll
    for (int q = 0; q < A_N; ++q) {
      const bool ok = on && okA[q] && k0 + a_col < n;
      cp16s(dstA + buf * A_BUF + q * (A_STEP * AP * (uint32_t)sizeof(cplx)), srcA[q] + (ok ? k0 : 0),
            ok ? 16 : 0);
    }
#pragma unroll
    for (int q = 0; q < B_N; ++q) {
      const int r = q * B_STEP;  // row offset from b_row
      const bool ok = on && bcol_ok && k0 + b_row + r < n;
      cp16s(dstB + buf * B_BUF + r * (BP * (uint32_t)sizeof(cplx)),
            srcB + (ok ? (int64_t)(k0 + r) * ncols : 0), ok ? 16 : 0);
    }
    cp_commit();
  };
  const int warp = t >> 5, lane = t & 31, g = lane >> 2, tg = lane & 3;
  const int wr = warp % WR, wc = warp / WR;
  const int nk = sparse ? __popc(kmask) : nkc;
  uint32_t rem = kmask;
  int seq = 0;
  auto next_chunk = [&]() -> int {  // the next chunk to stage (branch-free)
    const int ks = __ffs(rem) - 1;
    rem &= rem - 1;
    const int kd = seq++;
    return sparse ? ks : kd;
  };
  // prologue: the first NS-1 chunks (empty commit groups keep the group count)
#pragma unroll
  for (int i = 0; i < NS - 1; ++i) stage(next_chunk(), i, i < nk);
  const cplx *fragA = smem_mg + (wr * 8 * MT + g) * AP + tg;
  const cplx *fragB = smem_mg + NS * TM * AP + tg * BP + wc * 16 + g;
  for (int it = 0; it < nk; ++it) {
    const int buf = it % NS;
    cp_wait<NS - 2>();  // chunk it landed (this thread's copies)
    __syncthreads();    // ... and every thread's; buffer (it - 1) % NS is free
    // the chunk's fragments first, then the next copies, then the products
    // (free to move up between the copies' address arithmetic)
    const cplx *As = fragA + buf * (TM * AP), *Bs = fragB + buf * (TK * BP);
    constexpr int NK4 = TK / 4;
    cplx a[NK4][MT], b[NK4][2];
#pragma unroll
    for (int k4 = 0; k4 < NK4; ++k4) {
      const int kk = k4 * 4;
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) a[k4][mt] = As[mt * 8 * AP + kk];
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) b[k4][nt] = Bs[kk * BP + nt * 8];
    }
    stage(next_chunk(), (it + NS - 1) % NS, it + NS - 1 < nk);
#pragma unroll
    for (int k4 = 0; k4 < NK4; ++k4) {
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
  __syncthreads();  // the CTA's next tile restages the ring
}

// Store a finished tile: Re = P1 - P2, Im = P3 - P1 - P2 (3M complex product).
template <int MT, int WR, int WC>
__device__ __forceinline__ void gemm_store(const PassGeo &G, int row0, int col0, int colw,
                                           const int *act, int A, int nrhs,
                                           const double (&p1)[MT][2][2], const double (&p2)[MT][2][2],
                                           const double (&p3)[MT][2][2]) {
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31, g = lane >> 2, tg = lane & 3;
  const int wr = warp % WR, wc = warp / WR;
  if (wc * 16 >= colw) return;
  int64_t coff[2][2];  // the thread's 4 output columns (row 0 offsets)
#pragma unroll
  for (int nt = 0; nt < 2; ++nt)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int cc = wc * 16 + nt * 8 + 2 * tg + e;
      coff[nt][e] = cc < colw ? col_offset(G, col0 + cc, A, act, nrhs) : -1;
    }
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
    const int gr = row0 + wr * 8 * MT + mt * 8 + g;
    if (gr >= G.n) continue;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        if (coff[nt][e] < 0) continue;
        const int64_t off = coff[nt][e] + (int64_t)gr * G.ncols;
        G.out[off] = make_double2(p1[mt][nt][e] - p2[mt][nt][e],
                                  p3[mt][nt][e] - p1[mt][nt][e] - p2[mt][nt][e]);
      }
  }
}

template <int MT, int WR, int WC, int TK, int NS = 2>
__device__ __forceinline__ void gemm_tile(const PassGeo &G, int row0, int col0, int colw, bool sparse,
                                          uint32_t kmask, cplx *smem_mg, const int *act, int A,
                                          int nrhs) {
  double p1[MT][2][2] = {}, p2[MT][2][2] = {}, p3[MT][2][2] = {};
  const int nkc = (G.n + TK - 1) / TK;
  gemm_accum<MT, WR, WC, TK, NS>(G, row0, col0, colw, sparse, kmask, nkc, smem_mg, act, A, nrhs, p1,
                                 p2, p3);
  gemm_store<MT, WR, WC>(G, row0, col0, colw, act, A, nrhs, p1, p2, p3);
}

// One tile per CTA on a 1D grid over the launch's non-empty tiles: the
// tiles of visit 0 (column tile fastest, then row tile), then visit 1, ..
// Which tiles exist depends on the data (the exact-zero RHS columns of each
// visit are compacted away), so the host sizes the grid for all RHS active
// and every CTA derives the compact tile table from the K6 flags; CTAs past
// the last tile exit.  They carry the highest block indices, so they are
// dispatched after every working CTA -- with a (column, row, visit) grid the
// exiting CTAs of each visit sat between the working ones of the next and
// held their CTA slots (about 55% of config 2's grid) for a prologue each.
// Before the dependency wait the CTA stages the static pass geometry of all
// visits of the launch in shared memory, one visit per thread.
// kskip: the first forward pass visits only the K-chunks that K6 marked
// nonzero in any of the tile's input rows (J.km; payload-only visits: ~70%
// of the chunks are exact zeros -- the payload bands are thin strips of the
// window), which shortens the tile's latency chain, not just its arithmetic.
#define MG_MAXJ 32  // visits per kernel launch (the host splits longer lists)
struct TileJob {
  PassGeo G;
  const int *nz;
  const uint32_t *km;
  int ny;  // row tiles
};

// Active RHS of the launch's visits from the K6 flags: warp w takes visits
// w, w + nw, ..; cnt[v] = active count, mask[v][..] = the ballot words.
// Call from all threads; the caller synchronizes afterwards.
// fin(v, count) runs on lane 0 (derived per-visit quantities).
template <typename JobT, typename Fin>
__device__ __forceinline__ void count_active(const JobT *job, int njob, int nrhs, int nw, int *cnt,
                                             uint32_t (*mask)[RMAX_MODAL / 32], Fin fin) {
  const int lane = threadIdx.x & 31;
  if ((int)(threadIdx.x >> 5) >= nw) return;  // a trailing partial warp sits out
  for (int v = threadIdx.x >> 5; v < njob; v += nw) {
    const int *nz = job[v].nz;
    int c = 0;
    for (int r0 = 0; r0 < nrhs; r0 += 32) {
      const int r = r0 + lane;
      const uint32_t mk = __ballot_sync(0xffffffffu, r < nrhs && (!nz || nz[r]));
      if (lane == 0) mask[v][r0 >> 5] = mk;
      c += __popc(mk);
    }
    if (lane == 0) {
      cnt[v] = c;
      fin(v, c);
    }
  }
}
// the ordered list of a visit's active RHS from its ballot words (no global
// reads); call from all threads, synchronizes
__device__ __forceinline__ void active_list(const uint32_t *mask, int nrhs, int *act) {
  for (int r = threadIdx.x; r < nrhs; r += blockDim.x) {
    const uint32_t mk = mask[r >> 5];
    if ((mk >> (r & 31)) & 1u) {
      int pos = __popc(mk & ((1u << (r & 31)) - 1));
      for (int w = 0; w < (r >> 5); ++w) pos += __popc(mask[w]);
      act[pos] = r;
    }
  }
  __syncthreads();
}

// COMPACT (2D): the 1D grid described above.  Otherwise (3D: nearly every
// RHS is active and the passes are short, so the table costs more than the
// exiting CTAs) the grid is (column tiles, row tiles, visits).
// early: the K6 flags were final before the previous kernel of the stream
// started (inverse passes), so they are read before the dependency wait.
template <int MT, int WR, int WC, int TK = 16, int MINB = 1, int NS = 2, bool COMPACT = true>
__global__ void __launch_bounds__(32 * WR * WC, MINB)
    k_modal_gemm(const ModalJob *__restrict__ jobs, int njob, int pass, int nrhs, int kskip, int early,
                 unsigned long long *work) {
  constexpr int TM = 8 * MT * WR, TN = 16 * WC, NW = WR * WC;
  static_assert(TK == 8, "K6 chunk masks are in units of 8");
  extern __shared__ __align__(16) cplx smem_mg[];
  __shared__ int act[RMAX_MODAL + 1];
  __shared__ uint32_t s_kmask;
  PassGeo G;
  const uint32_t *km;
  int row0, col0, A;
  if (COMPACT) {
    __shared__ TileJob s_job[MG_MAXJ];
    __shared__ int s_cnt[MG_MAXJ], s_nx[MG_MAXJ], s_nt[MG_MAXJ];
    __shared__ uint32_t s_mask[MG_MAXJ][RMAX_MODAL / 32];
    const int t = threadIdx.x;
    if (t < njob) {  // static tables only
      const ModalJob J = jobs[t];
      const FactDev f = *J.f;
      TileJob tj;
      tj.G = pass_geo(f, J, pass, nrhs);
      tj.nz = J.nz;
      tj.km = J.km;
      tj.ny = (tj.G.n + TM - 1) / TM;
      s_job[t] = tj;
    }
    if (!early) pdl_wait();
    __syncthreads();
    count_active(s_job, njob, nrhs, NW, s_cnt, s_mask, [&](int v, int c) {
      const PassGeo &Gv = s_job[v].G;  // column tiles and tiles of visit v
      s_nx[v] = (Gv.outer * Gv.inner * c + TN - 1) / TN;
      s_nt[v] = s_nx[v] * s_job[v].ny;
    });
    __syncthreads();
    int L = blockIdx.x, v = 0;
    for (; v < njob; ++v) {
      const int nt = s_nt[v];
      if (L < nt) break;
      L -= nt;
    }
    if (v == njob) return;
    const int nx = s_nx[v];
    G = s_job[v].G;
    km = s_job[v].km;
    row0 = (L / nx) * TM;
    col0 = (L - (L / nx) * nx) * TN;
    A = s_cnt[v];
    active_list(s_mask[v], nrhs, act);
    if (early) pdl_wait();
  } else {
    const ModalJob J = jobs[blockIdx.z];
    const FactDev f = *J.f;
    G = pass_geo(f, J, pass, nrhs);
    km = J.km;
    row0 = blockIdx.y * TM;
    col0 = blockIdx.x * TN;
    if (row0 >= G.n || col0 >= G.outer * G.ncols) return;
    pdl_wait();
    A = active_rhs(J.nz, nrhs, act);
    if (col0 >= G.outer * G.inner * A) return;
  }
  const int total = G.outer * G.inner * A;  // compact columns
  const int colw = min(TN, total - col0);
  // pass 0 has inner == 1: compact column c is (input row c / A, RHS)
  const bool sparse = kskip && pass == 0 && km != nullptr && G.inner == 1;
  if (sparse) {
    if (threadIdx.x < 32) {
      const int b0 = col0 / A, b1 = (col0 + colw - 1) / A;
      uint32_t mk = 0;
      for (int b = b0 + (int)threadIdx.x; b <= b1; b += 32) mk |= km[b];
      mk = __reduce_or_sync(0xffffffffu, mk);
      if (threadIdx.x == 0) s_kmask = mk;
    }
    __syncthreads();
  }
  if (work && threadIdx.x == 0) {  // executed complex multiply-adds of this tile (ds_ctx_work)
    int kx = G.n;
    if (sparse) {
      const int last = (G.n - 1) / TK;  // the last chunk may be partial
      kx = __popc(s_kmask) * TK - (((s_kmask >> last) & 1u) ? (last + 1) * TK - G.n : 0);
    }
    atomicAdd(work, (unsigned long long)min(TM, G.n - row0) * colw * kx);
  }
  gemm_tile<MT, WR, WC, TK, NS>(G, row0, col0, colw, sparse, sparse ? s_kmask : 0u, smem_mg, act, A,
                                nrhs);
}

// ------------------------------------------- mode-wise recurrences (K3m-R)
// One thread per (visit, mode j, RHS r): forward elimination and back
// substitution along the block axis, in place on the transformed buffer.
// Loads of a chunk of MR blocks are issued before its dependent arithmetic.
#define MR 8
__global__ void __launch_bounds__(256) k_modal_thomas(const ModalJob *__restrict__ jobs, int nrhs) {
  const ModalJob J = jobs[blockIdx.y];
  const FactDev &f = *J.f;
  const int m = f.m, nb = f.nb;
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= m * nrhs) return;
  const int j = q / nrhs, r = q % nrhs;
  if (J.nz && !J.nz[r]) return;  // exact-zero RHS: never read downstream
  cplx *p = ((f.naxes - 1) & 1 ? J.s1 : J.s0) + q;
  const size_t st = (size_t)m * nrhs;
  const cplx *mul = f.mmul + j, *inv = f.minv + j;
  const cplx *uc = f.ucoef;
  cplx prev = make_double2(0.0, 0.0);
  for (int k0 = 0; k0 < nb; k0 += MR) {
    cplx gv[MR], mv[MR];
#pragma unroll
    for (int i = 0; i < MR; ++i) {
      const int k = k0 + i;
      if (k < nb) {
        gv[i] = p[k * st];
        mv[i] = mul[(size_t)k * m];
      }
    }
#pragma unroll
    for (int i = 0; i < MR; ++i) {
      const int k = k0 + i;
      if (k < nb) {
        prev = k == 0 ? gv[i] : csub(gv[i], cmul(mv[i], prev));
        p[k * st] = prev;
      }
    }
  }
  cplx y = make_double2(0.0, 0.0);
  for (int k1 = nb - 1; k1 >= 0; k1 -= MR) {
    cplx gv[MR], iv[MR], uv[MR];
#pragma unroll
    for (int i = 0; i < MR; ++i) {
      const int k = k1 - i;
      if (k >= 0) {
        gv[i] = k == nb - 1 ? prev : p[k * st];
        iv[i] = inv[(size_t)k * m];
        uv[i] = uc[k];
      }
    }
#pragma unroll
    for (int i = 0; i < MR; ++i) {
      const int k = k1 - i;
      if (k >= 0) {
        y = k == nb - 1 ? cmul(gv[i], iv[i]) : cmul(csub(gv[i], cmul(uv[i], y)), iv[i]);
        p[k * st] = y;
      }
    }
  }
}

// K3m-R v2: one half-warp block per 16 consecutive (mode, RHS) columns of a visit.  The
// whole column block (n_b rows of 256 contiguous bytes) is staged into
// shared memory with one cp.async per (row, lane), all in flight at once --
// the v1 kernel above was bound by memory-level parallelism (ncu, config 2:
// 66 us per launch, 58 SMs with 8 outstanding loads per thread) -- then the
// recurrences run out of shared memory and the block is written back
// coalesced.  Arithmetic and order are v1's.
#define TQ 16
// mode columns a TQ-column block can touch
__host__ __device__ inline int thomas_modes(int nrhs) { return (TQ - 1) / nrhs + 2 < TQ ? (TQ - 1) / nrhs + 2 : TQ; }
__global__ void __launch_bounds__(TQ) k_modal_thomas2(const ModalJob *__restrict__ jobs, int nrhs) {
  extern __shared__ __align__(16) cplx smem_th[];
  const ModalJob J = jobs[blockIdx.y];
  const FactDev &f = *J.f;
  const int m = f.m, nb = f.nb;
  const int q0 = blockIdx.x * TQ, t = threadIdx.x, q = q0 + t;
  if (q0 >= m * nrhs) return;
  pdl_wait();
  if (!job_any(J, nrhs)) return;
  const bool live = q < m * nrhs;
  const int JM = thomas_modes(nrhs), j0 = q0 / nrhs;
  const int nj = min(JM, m - j0);
  cplx *sg = smem_th;                  // [nb][TQ] the columns
  cplx *sm = sg + (size_t)nb * TQ;     // [nb][JM] multipliers
  cplx *si = sm + (size_t)nb * JM;     // [nb][JM] inverse pivots
  cplx *su = si + (size_t)nb * JM;     // [nb] block-axis couplings u_k
  cplx *T = ((f.naxes - 1) & 1 ? J.s1 : J.s0);
  const size_t st = (size_t)m * nrhs;
  for (int k = 0; k < nb; ++k)
    cp16(sg + k * TQ + t, T + (live ? k * st + q : 0), live ? 16 : 0);
  for (int e = t; e < nb * nj; e += TQ) {
    const int k = e / nj, jj = e % nj;
    cp16(sm + k * JM + jj, f.mmul + (size_t)k * m + j0 + jj, 16);
    cp16(si + k * JM + jj, f.minv + (size_t)k * m + j0 + jj, 16);
  }
  for (int k = t; k < nb; k += TQ) cp16(su + k, f.ucoef + k, 16);
  cp_commit();
  cp_wait<0>();
  __syncthreads();
  if (!live) return;
  const int j = q / nrhs, r = q % nrhs, jj = j - j0;
  if (J.nz && !J.nz[r]) return;  // exact-zero RHS: never read downstream
  cplx *p = sg + t;
  cplx prev = make_double2(0.0, 0.0);
  for (int k0 = 0; k0 < nb; k0 += MR) {
    cplx gv[MR], mv[MR];
#pragma unroll
    for (int i = 0; i < MR; ++i) {
      const int k = k0 + i;
      if (k < nb) {
        gv[i] = p[k * TQ];
        mv[i] = sm[k * JM + jj];
      }
    }
#pragma unroll
    for (int i = 0; i < MR; ++i) {
      const int k = k0 + i;
      if (k < nb) {
        prev = k == 0 ? gv[i] : csub(gv[i], cmul(mv[i], prev));
        p[k * TQ] = prev;
      }
    }
  }
  cplx y = make_double2(0.0, 0.0);
  for (int k1 = nb - 1; k1 >= 0; k1 -= MR) {
    cplx gv[MR], iv[MR], uv[MR];
#pragma unroll
    for (int i = 0; i < MR; ++i) {
      const int k = k1 - i;
      if (k >= 0) {
        gv[i] = p[k * TQ];
        iv[i] = si[k * JM + jj];
        uv[i] = su[k];
      }
    }
#pragma unroll
    for (int i = 0; i < MR; ++i) {
      const int k = k1 - i;
      if (k >= 0) {
        y = k == nb - 1 ? cmul(gv[i], iv[i]) : cmul(csub(gv[i], cmul(uv[i], y)), iv[i]);
        T[k * st + q] = y;
      }
    }
  }
}

// K3m-R v3 (default): segmented recurrences.  v2 above was a single-warp
// latency chain (ncu: ~39k cycles per block for 2 x 115 dependent complex
// steps plus issue-bound copy loops, IPC 0.5).  Both sweeps are first-order
// linear recurrences z_k = b_k + a_k z_{k-1} (forward: a_k = -mul_k,
// b_k = ghat_k; backward, downwards: a_k = -inv_k u_k, b_k = inv_k g'_k),
// so each is split into NSEG segments of L blocks: warp s runs segment s
// for 32 consecutive (mode, RHS) columns from a zero carry while tracking
// the segment's partial products, warp 0 chains the segment carries
// (NSEG steps), and every warp adds partial product x carry.  Critical path
// L + NSEG + 1 steps instead of n_b; forward values stay in registers for
// the backward sweep; loads are 512-byte coalesced rows.
struct RecJob {
  const int *nz;
  cplx *T;
  const cplx *mmul, *minv, *ucoef;
  int m, nb;
};
// 1D grid over the launch's non-empty column blocks (the compact tile table
// of k_modal_gemm): the K6 flags were final two kernels ago, so the table is
// built before the dependency wait and the blocks past the last one exit
// without holding an SM (one 512-thread block per SM).
// CW columns per block (32, or 16: half the threads, two blocks per SM).
template <int L, int CW>
__global__ void __launch_bounds__(16 * CW, 32 / CW) k_modal_thomas3(const ModalJob *__restrict__ jobs,
                                                                    int njob, int nrhs) {
  __shared__ cplx sP[16][CW], sZ[16][CW], sC[16][CW];
  __shared__ int actl[RMAX_MODAL + 1];
  __shared__ RecJob s_job[MG_MAXJ];
  __shared__ int s_cnt[MG_MAXJ], s_nblk[MG_MAXJ];
  __shared__ uint32_t s_mask[MG_MAXJ][RMAX_MODAL / 32];
  const int lane = threadIdx.x % CW, seg = threadIdx.x / CW;
  if ((int)threadIdx.x < njob) {
    const ModalJob J = jobs[threadIdx.x];
    const FactDev &f = *J.f;
    RecJob r;
    r.nz = J.nz;
    r.T = ((f.naxes - 1) & 1 ? J.s1 : J.s0);
    r.mmul = f.mmul;
    r.minv = f.minv;
    r.ucoef = f.ucoef;
    r.m = f.m;
    r.nb = f.nb;
    s_job[threadIdx.x] = r;
  }
  __syncthreads();
  count_active(s_job, njob, nrhs, (int)blockDim.x >> 5, s_cnt, s_mask,
               [&](int v, int c) { s_nblk[v] = (s_job[v].m * c + CW - 1) / CW; });
  __syncthreads();
  int blk = blockIdx.x, v = 0;
  for (; v < njob; ++v) {
    const int nblk = s_nblk[v];
    if (blk < nblk) break;
    blk -= nblk;
  }
  if (v == njob) return;
  const RecJob f = s_job[v];
  const int m = f.m, nb = f.nb, A = s_cnt[v];
  const int nseg = (nb + L - 1) / L;
  active_list(s_mask[v], nrhs, actl);  // compact (mode, active RHS) columns
  const int qc = blk * CW + lane;
  const bool live = qc < m * A;
  const int qcc = live ? qc : 0;
  const int j = qcc / A;
  const int q = j * nrhs + actl[qcc - j * A];  // full-layout column of this thread
  const int qq = q;
  cplx *T = f.T;
  const size_t st = (size_t)m * nrhs;
  const int k0 = seg * L;
  const bool act = seg < nseg;
  // loads of the segment: data, multipliers, inverse pivots, couplings
  cplx g[L], mu[L], iv[L], uc[L];
#pragma unroll
  for (int i = 0; i < L; ++i) {  // factor data: in flight across the dependency wait
    const int k = k0 + i;
    mu[i] = act && k < nb ? f.mmul[(size_t)k * m + j] : make_double2(0.0, 0.0);
  }
  pdl_wait();
#pragma unroll
  for (int i = 0; i < L; ++i) {
    const int k = k0 + i;
    g[i] = act && k < nb ? T[k * st + qq] : make_double2(0.0, 0.0);
  }
  // ---- forward: z_k = g_k - mul_k z_{k-1}  (mul_0 = 0)
  cplx P[L];
  {
    cplx z = make_double2(0.0, 0.0), pp = make_double2(1.0, 0.0);
#pragma unroll
    for (int i = 0; i < L; ++i) {
      const cplx a = make_double2(-mu[i].x, -mu[i].y);
      z = cadd(g[i], cmul(a, z));
      pp = cmul(a, pp);
      g[i] = z;
      P[i] = pp;
    }
    if (act) {
      sP[seg][lane] = pp;
      sZ[seg][lane] = z;
    }
  }
  // backward-sweep operands, in flight across the carry chain
#pragma unroll
  for (int i = 0; i < L; ++i) {
    const int k = k0 + i;
    const bool in = act && k < nb;
    iv[i] = in ? f.minv[(size_t)k * m + j] : make_double2(0.0, 0.0);
    uc[i] = in ? f.ucoef[k] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  if (seg == 0) {  // carries into every segment
    cplx c = make_double2(0.0, 0.0);
    for (int s2 = 0; s2 < nseg; ++s2) {
      sC[s2][lane] = c;
      c = cadd(sZ[s2][lane], cmul(sP[s2][lane], c));
    }
  }
  __syncthreads();
  if (act) {
    const cplx c = sC[seg][lane];
#pragma unroll
    for (int i = 0; i < L; ++i) g[i] = cadd(g[i], cmul(P[i], c));  // g'_k
  }
  __syncthreads();
  // ---- backward (k descending): y_k = inv_k g'_k - inv_k u_k y_{k+1}
  {
    cplx z = make_double2(0.0, 0.0), pp = make_double2(1.0, 0.0);
#pragma unroll
    for (int i = L - 1; i >= 0; --i) {
      const int k = k0 + i;
      const bool last = k >= nb - 1;  // k = nb-1 starts the chain (a = 0); k >= nb: padding
      const cplx b = cmul(iv[i], g[i]);
      const cplx iu = cmul(iv[i], uc[i]);
      const cplx a = last ? make_double2(0.0, 0.0) : make_double2(-iu.x, -iu.y);
      z = cadd(b, cmul(a, z));
      pp = cmul(a, pp);
      g[i] = z;
      P[i] = pp;
    }
    if (act) {
      sP[seg][lane] = pp;
      sZ[seg][lane] = z;
    }
  }
  __syncthreads();
  if (seg == 0) {
    cplx c = make_double2(0.0, 0.0);
    for (int s2 = nseg - 1; s2 >= 0; --s2) {
      sC[s2][lane] = c;
      c = cadd(sZ[s2][lane], cmul(sP[s2][lane], c));
    }
  }
  __syncthreads();
  if (!act || !live) return;
  const cplx c = sC[seg][lane];
#pragma unroll
  for (int i = 0; i < L; ++i) {
    const int k = k0 + i;
    if (k < nb) T[k * st + q] = cadd(g[i], cmul(P[i], c));
  }
}

// ------------------------------------------------------------- launcher
template <int MT, int WR, int WC, int TK = 16, int MINB = 1, int NS = 2, bool COMPACT = true>
static int launch_gemm(ds_ctx *ctx, const ModalJob *jobs_dev, const FactDev *facts, int njob,
                       int pass, int nrhs) {
  constexpr int TM = 8 * MT * WR, TN = 16 * WC;
  const size_t smem = sizeof(cplx) * NS * (TM * (TK + 4) + TK * (TN + 2));
  auto kern = k_modal_gemm<MT, WR, WC, TK, MINB, NS, COMPACT>;
  static bool attr_set = false;
  if (!attr_set) {
    DS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr_set = true;
  }
  unsigned long long *work = ctx->opt.count_work ? ctx->work : nullptr;
  const int early = pass >= facts[0].naxes;  // inverse passes: the K6 flags are long final
  ModalJob dummy;
  memset(&dummy, 0, sizeof(dummy));
  if constexpr (!COMPACT) {
    int gx = 1, gy = 1;
    for (int i = 0; i < njob; ++i) {
      const PassGeo G = pass_geo(facts[i], dummy, pass, nrhs);
      gx = std::max(gx, (G.outer * G.ncols + TN - 1) / TN);
      gy = std::max(gy, (G.n + TM - 1) / TM);
    }
    DS_CUDA(launch_pdl(kern, dim3(gx, gy, njob), dim3(32 * WR * WC), smem, ctx->stream, jobs_dev,
                       njob, pass, nrhs, ctx->opt.kskip, 0, work));
    ctx->launches++;
    DS_CHECK_LAUNCH();
    return DS_OK;
  } else {
  for (int j0 = 0; j0 < njob; j0 += MG_MAXJ) {  // at most MG_MAXJ visits per kernel launch
    const int nj = std::min(MG_MAXJ, njob - j0);
    int tiles = 0;  // every RHS active: the upper bound of the compact tile count
    for (int i = j0; i < j0 + nj; ++i) {
      const PassGeo G = pass_geo(facts[i], dummy, pass, nrhs);
      tiles += ((G.outer * G.ncols + TN - 1) / TN) * ((G.n + TM - 1) / TM);
    }
    DS_CUDA(launch_pdl(kern, dim3(std::max(1, tiles)), dim3(32 * WR * WC), smem, ctx->stream,
                       jobs_dev + j0, nj, pass, nrhs, ctx->opt.kskip, early, work));
    ctx->launches++;
    DS_CHECK_LAUNCH();
  }
  return DS_OK;
  }
}

// phase 0: forward transforms, 1: mode-wise recurrences, 2: inverse
// transforms, -1: all three
int ds_launch_modal_phase(ds_ctx *ctx, const ModalJob *jobs_dev, const FactDev *facts, int njob,
                          int nrhs, int phase) {
  if (njob <= 0) return DS_OK;
  const int na = facts[0].naxes;
  for (int i = 1; i < njob; ++i)
    if (facts[i].naxes != na) return ds_fail(DS_ECONFIG, "modal solve: mixed dimensions in one launch");
  // transform tile (measured best of 28 shapes / pipelines on configs 2 and
  // 4): 32 x 32 per CTA, 2 x 2 warps of 16 x 16, K chunks of
  // 8 through a 4-stage cp.async ring, 4 CTAs per SM
  auto launch_pass = [&](int pass) -> int {
    if (na == 2) return launch_gemm<2, 2, 2, 8, 4, 4, false>(ctx, jobs_dev, facts, njob, pass, nrhs);
    return launch_gemm<2, 2, 2, 8, 4, 4, true>(ctx, jobs_dev, facts, njob, pass, nrhs);
  };
  if (phase == 0 || phase == -1)
    for (int p = 0; p < na; ++p)
      if (int rc = launch_pass(p)) return rc;
  if (phase == 1 || phase == -1) {
    int mmax = 1, nbmax = 1;
    for (int i = 0; i < njob; ++i) {
      mmax = std::max(mmax, facts[i].m);
      nbmax = std::max(nbmax, facts[i].nb);
    }
    const size_t tsm = sizeof(cplx) * (size_t)nbmax * (TQ + 2 * thomas_modes(nrhs) + 1);
    static int th_attr = 0;
    if (nbmax > 64 && nbmax <= 16 * 16) {  // segmented recurrences (long chains, 2D)
      const int L = nbmax <= 64 ? 4 : (nbmax <= 128 ? 8 : 16);
      const int nseg = (nbmax + L - 1) / L;
      const int cw = ctx->opt.r3_cols == 16 ? 16 : 32;
      for (int j0 = 0; j0 < njob; j0 += MG_MAXJ) {
        const int nj = std::min(MG_MAXJ, njob - j0);
        int blocks = 0;  // every RHS active: the upper bound of the compact block count
        for (int i = j0; i < j0 + nj; ++i) blocks += (facts[i].m * nrhs + cw - 1) / cw;
        const dim3 grid(std::max(1, blocks)), block(cw * nseg);
#define R3_LAUNCH(L_, CW_) \
  DS_CUDA(launch_pdl(k_modal_thomas3<L_, CW_>, grid, block, 0, ctx->stream, jobs_dev + j0, nj, nrhs))
        if (cw == 16) {
          if (L == 4) R3_LAUNCH(4, 16);
          else if (L == 8) R3_LAUNCH(8, 16);
          else R3_LAUNCH(16, 16);
        } else {
          if (L == 4) R3_LAUNCH(4, 32);
          else if (L == 8) R3_LAUNCH(8, 32);
          else R3_LAUNCH(16, 32);
        }
#undef R3_LAUNCH
        if (j0 > 0) ctx->launches++;
      }
    } else if (tsm <= 200 * 1024) {  // short chains (3D): the staged v2 streams better
      if ((int)tsm > th_attr) {
        DS_CUDA(cudaFuncSetAttribute(k_modal_thomas2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsm));
        th_attr = (int)tsm;
      }
      DS_CUDA(launch_pdl(k_modal_thomas2, dim3((mmax * nrhs + TQ - 1) / TQ, njob), dim3(TQ), tsm,
                         ctx->stream, jobs_dev, nrhs));
    } else {
      // chains too long to stage (n_b > 256 and no shared-memory fit): v1
      k_modal_thomas<<<dim3((mmax * nrhs + 255) / 256, njob), 256, 0, ctx->stream>>>(jobs_dev, nrhs);
    }
    ctx->launches++;
    DS_CHECK_LAUNCH();
  }
  if (phase == 2 || phase == -1)
    for (int p = na; p < 2 * na; ++p)
      if (int rc = launch_pass(p)) return rc;
  return DS_OK;
}

int ds_launch_modal(ds_ctx *ctx, const ModalJob *jobs_dev, const FactDev *facts, int njob,
                    int nrhs) {
  return ds_launch_modal_phase(ctx, jobs_dev, facts, njob, nrhs, -1);
}

// --------------------------------------------------------- factorization
extern "C" int ds_fact_create_modal(ds_ctx *ctx, ds_op *const *ops, int32_t n,
                                    const ds_modal_desc *descs, ds_fact **out) {
  if (!ctx || !ops || n < 1 || !descs || !out)
    return ds_fail(DS_ECONFIG, "ds_fact_create_modal: bad argument");
  ds_fact *F = new ds_fact();
  auto fail = [&](int code) {
    for (void *p : F->allocations) cudaFree(p);
    delete F;
    return code;
  };
  std::vector<PivJob> jobs(n);
  int mmax = 1;
  for (int i = 0; i < n; ++i) {
    if (!ops[i]) return fail(ds_fail(DS_ECONFIG, "ds_fact_create_modal: null operator"));
    const OpDev &o = ops[i]->dev;
    const ds_modal_desc &D = descs[i];
    FactDev f;
    memset(&f, 0, sizeof(f));
    ds_fill_layout(o, f);
    if (o.kappa2_kind == 2)
      return fail(ds_fail(DS_ECONFIG, "modal factorization: kappa^2 is not tensor-structured"));
    if (D.block_axis != f.block_axis || D.naxes != o.dim - 1)
      return fail(ds_fail(DS_ECONFIG, "modal factorization: block axis / axis count mismatch"));
    f.kind = 1;
    f.naxes = o.dim - 1;
    size_t elems = 2 * (size_t)f.nb + 2 * (size_t)f.nb * f.m;
    for (int a = 0; a < f.naxes; ++a) {
      f.nax[a] = o.shape[f.other[a]];
      if (!D.v[a] || !D.vinv[a] || !D.lambda[a])
        return fail(ds_fail(DS_ECONFIG, "modal factorization: missing eigen-decomposition"));
      elems += 2 * (size_t)f.nax[a] * f.nax[a] + f.nax[a];
    }
    void *mem = nullptr;
    if (cudaMalloc(&mem, elems * sizeof(cplx)) != cudaSuccess)
      return fail(ds_fail(DS_ECUDA, "ds_fact_create_modal: out of device memory"));
    F->allocations.push_back(mem);
    cplx *p = (cplx *)mem;
    cplx *lc = p, *uc = lc + f.nb;
    p = uc + f.nb;
    DS_CUDA(cudaMemcpy(lc, o.c_lo[f.block_axis], f.nb * sizeof(cplx), cudaMemcpyDeviceToDevice));
    DS_CUDA(cudaMemcpy(uc, o.c_hi[f.block_axis], f.nb * sizeof(cplx), cudaMemcpyDeviceToDevice));
    f.lcoef = lc;
    f.ucoef = uc;
    PivJob &J = jobs[i];
    memset(&J, 0, sizeof(J));
    for (int a = 0; a < f.naxes; ++a) {
      const size_t na2 = (size_t)f.nax[a] * f.nax[a];
      cplx *W = p, *V = W + na2, *L = V + na2;
      p = L + f.nax[a];
      DS_CUDA(cudaMemcpy(W, D.vinv[a], na2 * sizeof(cplx), cudaMemcpyHostToDevice));
      DS_CUDA(cudaMemcpy(V, D.v[a], na2 * sizeof(cplx), cudaMemcpyHostToDevice));
      DS_CUDA(cudaMemcpy(L, D.lambda[a], f.nax[a] * sizeof(cplx), cudaMemcpyHostToDevice));
      f.mW[a] = W;
      f.mV[a] = V;
      J.lam[a] = L;
    }
    J.mul = p;
    J.inv = p + (size_t)f.nb * f.m;
    f.mmul = J.mul;
    f.minv = J.inv;
    J.f = f;
    J.op = o;
    mmax = std::max(mmax, f.m);
    F->facts.push_back(f);
    F->h_l.push_back(ops[i]->h_clo[f.block_axis]);
    F->h_u.push_back(ops[i]->h_chi[f.block_axis]);
    F->bytes.push_back((int64_t)(elems * sizeof(cplx)));
    F->bytes_total += (int64_t)(elems * sizeof(cplx));
  }
  PivJob *djobs = nullptr;
  int *dstatus = nullptr;
  if (cudaMalloc(&djobs, sizeof(PivJob) * n) != cudaSuccess || cudaMalloc(&dstatus, sizeof(int)) != cudaSuccess)
    return fail(ds_fail(DS_ECUDA, "ds_fact_create_modal: out of device memory"));
  cudaMemcpy(djobs, jobs.data(), sizeof(PivJob) * n, cudaMemcpyHostToDevice);
  cudaMemset(dstatus, 0, sizeof(int));
  k_modal_pivots<<<dim3((mmax + 127) / 128, n), 128, 0, ctx->stream>>>(djobs, dstatus);
  ctx->launches++;
  int status = 0;
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
  if (e == cudaSuccess) e = cudaMemcpy(&status, dstatus, sizeof(int), cudaMemcpyDeviceToHost);
  cudaFree(djobs);
  cudaFree(dstatus);
  if (e != cudaSuccess) return fail(ds_fail(DS_ECUDA, std::string("modal pivots: ") + cudaGetErrorString(e)));
  if (status) return fail(ds_fail(DS_ESOLVER, "modal factorization: zero or non-finite pivot"));
  *out = F;
  return DS_OK;
}

extern "C" int ds_fact_kind(const ds_fact *F, int32_t i) {
  if (!F || i < 0 || i >= (int)F->facts.size()) return ds_fail(DS_ECONFIG, "ds_fact_kind: bad index");
  return F->facts[i].kind;
}
