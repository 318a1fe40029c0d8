// K2: block-tridiagonal factorization of subdomain operators (2D windows).
//
// Replaces SeparableFactorization / SparseLuFactorization
// (diagsweep/subdomain.py:43-133).  The window is cut into n_b slabs along
// its longest axis (block axis); the operator is block tridiagonal with
// diagonal blocks D_k (the in-slab stencil plus kappa^2 and the block-axis
// diagonal) and scalar off-diagonal blocks l_k I, u_k I (c_lo/c_hi of the
// block axis, pml.py:95-102).  Block LU:
//     S_0 = D_0,   S_k = D_k - (l_k u_{k-1}) S_{k-1}^{-1},
// and every S_k^{-1} is stored densely (complex128) so the substitution is
// pure GEMV/GEMM work (K3).
//
// Twisted ("burn at both ends") variant: with t = n_b/2 the top chain
// builds S_0..S_{t-1} as above while an independent bottom chain builds
//     T_{n_b-1} = D_{n_b-1},  T_k = D_k - (u_k l_{k+1}) T_{k+1}^{-1},
// and the middle block M_t = D_t - (l_t u_{t-1}) S_{t-1}^{-1}
//                                - (u_t l_{t+1}) T_{t+1}^{-1}
// closes the system.  Halving the chain length halves the latency of both
// the factorization and every substitution (K3).
//
// One thread-block cluster per (operator, half) walks its chain; each CTA
// owns a column slice of S_k in shared memory and the cluster inverts it by
// Gauss-Jordan elimination with partial pivoting (pivot column broadcast
// through distributed shared memory, one cluster barrier per pivot).  The
// explicit inverse keeps the backward error at ~1e-15 for these operators
// (cond(S_k) ~ 1e2), measured against the reference's Schur/Sylvester
// solver in DESIGN.md.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "ds_common.cuh"
#include "ds_factor.cuh"

namespace cg = cooperative_groups;

#define GJ_THREADS 512

// old - a * b with four fused multiply-adds (the rank-1 update's only
// arithmetic; cmul + csub would issue 6 FP64 instructions)
__device__ __forceinline__ cplx cfms(cplx old, cplx a, cplx b) {
  cplx r;
  r.x = fma(a.y, b.y, fma(-a.x, b.x, old.x));
  r.y = fma(-a.y, b.x, fma(-a.x, b.y, old.y));
  return r;
}
static const size_t kSmemLimit = 232448;  // 227 KB opt-in per CTA on sm_100

__global__ void __launch_bounds__(GJ_THREADS, 1)
    k_factor_gj(const FactJob *__restrict__ jobs, int mcper_max, int *status) {
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int C = (int)cluster.num_blocks();
  const FactJob &J = jobs[blockIdx.y];
  const int m = J.f.m, nb = J.f.nb, tw = J.f.twist;
  const int nsteps = J.half == 0 ? tw : (J.half == 1 ? nb - 1 - tw : 1);
  const int mcper = (m + C - 1) / C;
  const int c0 = rank * mcper;
  const int c1 = min(m, c0 + mcper);
  const int mc = max(0, c1 - c0);
  const int t = threadIdx.x, T = blockDim.x;

  extern __shared__ __align__(16) unsigned char smem_raw[];
  cplx *S = (cplx *)smem_raw;               // [m][mcper_max]
  cplx *colj = S + (size_t)m * mcper_max;   // [2][m]
  cplx *prow = colj + 2 * m;                // [mcper_max]
  cplx *rowj_old = prow + mcper_max;        // [mcper_max]
  int *piv = (int *)(rowj_old + mcper_max); // [m]
  int *dst = piv + m;                       // [m]
  __shared__ double red_v[GJ_THREADS / 32];
  __shared__ int red_i[GJ_THREADS / 32];
  __shared__ int s_bad;
  if (t == 0) s_bad = 0;

  const int ld = mcper_max;
  const int ba = J.f.block_axis;
  // fixed 2D thread mapping over my m x mc slice: thread t owns column
  // cc = t % mc and rows i0, i0 + istep, ... (no per-element division; the
  // pivot row entries of its column stay in registers for a whole pivot)
  const int cc_t = mc > 0 ? t % mc : 0;
  const int i0_t = mc > 0 ? t / mc : m;
  const int istep = mc > 0 ? T / mc : 1;
  const bool col_thread = mc > 0 && t < istep * mc;
  for (int step = 0; step < nsteps; ++step) {
    // ---- Schur complement of block k (my columns):
    //   top    S_k = D_k - (l_k u_{k-1}) S_{k-1}^{-1}
    //   bottom T_k = D_k - (u_k l_{k+1}) T_{k+1}^{-1}
    //   middle M_t = D_t - (l_t u_{t-1}) S_{t-1}^{-1} - (u_t l_{t+1}) T_{t+1}^{-1}
    const int k = J.half == 0 ? step : (J.half == 1 ? nb - 1 - step : tw);
    cplx co1 = make_double2(0.0, 0.0), co2 = co1;
    const cplx *p1 = nullptr, *p2 = nullptr;
    if ((J.half == 0 || J.half == 2) && k > 0) {
      co1 = cmul(J.op.c_lo[ba][k], J.op.c_hi[ba][k - 1]);
      p1 = J.sinv + (size_t)(k - 1) * m * m;
    }
    if ((J.half == 1 || J.half == 2) && k < nb - 1) {
      co2 = cmul(J.op.c_hi[ba][k], J.op.c_lo[ba][k + 1]);
      p2 = J.sinv + (size_t)(k + 1) * m * m;
    }
    if (col_thread) {
      const int cc = cc_t, c = c0 + cc;
      for (int i = i0_t; i < m; i += istep) {
        cplx v = d_entry(J, k, i, c);
        if (p1) v = csub(v, cmul(co1, __ldcg(p1 + (size_t)i * m + c)));
        if (p2) v = csub(v, cmul(co2, __ldcg(p2 + (size_t)i * m + c)));
        S[i * ld + cc] = v;
      }
    }
    cluster.sync();
    // ---- Gauss-Jordan inversion with partial pivoting
    for (int j = 0; j < m; ++j) {
      const int owner = j / mcper;
      cplx *cj = colj + (j & 1) * m;
      if (rank == owner) {
        const int jj = j - c0;
        double best = -1.0;
        int bi = m;
        for (int i = j + t; i < m; i += T) {
          double v = cabs1(S[i * ld + jj]);
          if (v > best || (v == best && i < bi)) { best = v; bi = i; }
        }
        for (int off = 16; off > 0; off >>= 1) {
          double ov = __shfl_down_sync(0xffffffffu, best, off);
          int oi = __shfl_down_sync(0xffffffffu, bi, off);
          if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
        }
        if ((t & 31) == 0) { red_v[t >> 5] = best; red_i[t >> 5] = bi; }
        __syncthreads();
        if (t == 0) {
          double bv = red_v[0];
          int bidx = red_i[0];
          for (int w = 1; w < T / 32; ++w)
            if (red_v[w] > bv || (red_v[w] == bv && red_i[w] < bidx)) { bv = red_v[w]; bidx = red_i[w]; }
          red_i[0] = bidx;
        }
        __syncthreads();
        const int p = red_i[0];
        for (int q = 0; q < C; ++q) {
          cplx *rc = cluster.map_shared_rank(cj, q);
          int *rp = cluster.map_shared_rank(piv, q);
          for (int i = t; i < m; i += T) rc[i] = S[i * ld + jj];
          if (t == 0) rp[j] = p;
        }
      }
      if (C == 1)
        __syncthreads();
      else
        cluster.sync();
      const int p = piv[j];
      const cplx pivot = cj[p];
      if (t == 0 && !(cabs1(pivot) > 0.0 && isfinite(pivot.x) && isfinite(pivot.y))) s_bad = 1;
      const cplx inv = cinv(pivot);
      for (int cc = t; cc < mc; cc += T) {
        prow[cc] = cmul(S[p * ld + cc], inv);
        rowj_old[cc] = S[j * ld + cc];
      }
      __syncthreads();
      if (col_thread) {
        const int cc = cc_t, c = c0 + cc;
        const cplx pr = prow[cc], ro = rowj_old[cc];
        if (c == j) {
          for (int i = i0_t; i < m; i += istep) {
            const cplx fi = cj[i == j ? p : (i == p ? j : i)];
            S[i * ld + cc] = (i == j) ? inv : cmul(make_double2(-fi.x, -fi.y), inv);
          }
        } else {
          // rows: i == j takes the scaled pivot row, i == p the old row j,
          // every other row S_i -= f_i * prow (branch-free selects)
#pragma unroll 4
          for (int i = i0_t; i < m; i += istep) {
            const cplx fi = cj[i == p ? j : i];
            cplx old = S[i * ld + cc];
            old = (i == p) ? ro : old;
            const cplx nv = cfms(old, fi, pr);
            S[i * ld + cc] = (i == j) ? pr : nv;
          }
        }
      }
      __syncthreads();
    }
    // ---- undo the column interchanges while storing S_k^{-1}
    if (t == 0) {
      for (int c = 0; c < m; ++c) dst[c] = c;  // dst used as src first
      for (int j = m - 1; j >= 0; --j) {
        int a = dst[j];
        dst[j] = dst[piv[j]];
        dst[piv[j]] = a;
      }
      // invert: src[c] -> dst[src[c]] = c ; reuse colj buffer (int view)
      int *tmp = (int *)(colj);
      for (int c = 0; c < m; ++c) tmp[dst[c]] = c;
      for (int c = 0; c < m; ++c) dst[c] = tmp[c];
    }
    __syncthreads();
    cplx *out = J.sinv + (size_t)k * m * m;
    if (col_thread) {
      const int cc = cc_t, dc = dst[c0 + cc];
      for (int i = i0_t; i < m; i += istep) out[(size_t)i * m + dc] = S[i * ld + cc];
    }
    cluster.sync();
  }
  if (t == 0 && s_bad) atomicExch(status, 1);
}

static int choose_cluster(int m, int *mcper_out, size_t *smem_out) {
  for (int C = 1; C <= 8; C *= 2) {
    int mcper = (m + C - 1) / C;
    size_t smem = (size_t)m * mcper * sizeof(cplx) + 2 * (size_t)m * sizeof(cplx) +
                  2 * (size_t)mcper * sizeof(cplx) + 2 * (size_t)m * sizeof(int);
    if (smem <= kSmemLimit - 4096) {
      *mcper_out = mcper;
      *smem_out = smem;
      return C;
    }
  }
  return 0;
}

void ds_fill_layout(const OpDev &o, FactDev &f) {
  int ba = 0;
  for (int a = 1; a < o.dim; ++a)
    if (o.shape[a] > o.shape[ba]) ba = a;
  f.block_axis = ba;
  f.nb = o.shape[ba];
  f.twist = f.nb / 2;
  f.m = 1;
  f.other[0] = f.other[1] = -1;
  int n = 0;
  for (int a = 0; a < o.dim; ++a) {
    f.win_shape[a] = o.shape[a];
    if (a == ba) continue;
    f.other[n++] = a;
    f.m *= o.shape[a];
  }
  for (int a = o.dim; a < 3; ++a) f.win_shape[a] = 1;
}

extern "C" int ds_fact_create(ds_ctx *ctx, ds_op *const *ops, int32_t n_in, ds_fact **out) {
  int n = n_in;
  if (!ctx || !ops || n < 1 || !out) return ds_fail(DS_ECONFIG, "ds_fact_create: bad argument");
  ds_fact *F = new ds_fact();
  std::vector<FactJob> jobs(n);
  int maxm = 0;
  for (int i = 0; i < n; ++i) {
    if (!ops[i]) {
      delete F;
      return ds_fail(DS_ECONFIG, "ds_fact_create: null operator");
    }
    const OpDev &o = ops[i]->dev;
    FactDev f;
    memset(&f, 0, sizeof(f));
    ds_fill_layout(o, f);
    size_t bytes = (size_t)f.nb * f.m * f.m * sizeof(cplx) + 2 * (size_t)f.nb * sizeof(cplx);
    void *mem = nullptr;
    if (cudaMalloc(&mem, bytes) != cudaSuccess) {
      for (void *p : F->allocations) cudaFree(p);
      delete F;
      return ds_fail(DS_ECUDA, "ds_fact_create: out of device memory for factors");
    }
    F->allocations.push_back(mem);
    cplx *sinv = (cplx *)mem;
    cplx *lc = sinv + (size_t)f.nb * f.m * f.m;
    cplx *uc = lc + f.nb;
    cudaMemcpy(lc, o.c_lo[f.block_axis], f.nb * sizeof(cplx), cudaMemcpyDeviceToDevice);
    cudaMemcpy(uc, o.c_hi[f.block_axis], f.nb * sizeof(cplx), cudaMemcpyDeviceToDevice);
    f.sinv = sinv;
    f.lcoef = lc;
    f.ucoef = uc;
    F->facts.push_back(f);
    F->h_l.push_back(ops[i]->h_clo[f.block_axis]);
    F->h_u.push_back(ops[i]->h_chi[f.block_axis]);
    F->bytes.push_back((int64_t)bytes);
    F->bytes_total += bytes;
    jobs[i].op = o;
    jobs[i].f = f;
    jobs[i].sinv = sinv;
    maxm = std::max(maxm, f.m);
  }
  (void)maxm;
  // small slabs (2D windows): on-chip Gauss-Jordan chains; large (3D): blocked
  std::vector<FactJob> small, large;
  std::vector<const cplx *> large_l, large_u;
  for (int i = 0; i < n; ++i) {
    if (jobs[i].f.m <= DS_LARGE_SLAB) {
      small.push_back(jobs[i]);
    } else {
      large.push_back(jobs[i]);
      large_l.push_back(F->h_l[i].data());
      large_u.push_back(F->h_u[i].data());
    }
  }
  int status = 0;
  if (!large.empty()) {
    int *dst = nullptr;
    DS_CUDA(cudaMalloc(&dst, sizeof(int)));
    DS_CUDA(cudaMemset(dst, 0, sizeof(int)));
    int rc = ds_blocked_factor(ctx, large.data(), (int)large.size(), large_l.data(),
                               large_u.data(), dst);
    if (rc) {
      cudaFree(dst);
      for (void *p : F->allocations) cudaFree(p);
      delete F;
      return rc;
    }
    DS_CUDA(cudaMemcpy(&status, dst, sizeof(int), cudaMemcpyDeviceToHost));
    cudaFree(dst);
    if (status) {
      for (void *p : F->allocations) cudaFree(p);
      delete F;
      return ds_fail(DS_ESOLVER, "blocked LU: zero or non-finite pivot in a Schur complement");
    }
  }
  if (small.empty()) {
    *out = F;
    return DS_OK;
  }
  int smaxm = 0;
  for (auto &j : small) smaxm = std::max(smaxm, j.f.m);
  int mcper = 0;
  size_t smem = 0;
  int C = choose_cluster(smaxm, &mcper, &smem);
  if (C == 0) {
    for (void *p : F->allocations) cudaFree(p);
    delete F;
    return ds_fail(DS_ECONFIG, "ds_fact_create: no on-chip configuration for m=" +
                                   std::to_string(smaxm));
  }
  n = (int)small.size();
  jobs = small;
  // jobs: [top chains | bottom chains] then [middle blocks]
  std::vector<FactJob> chain_jobs, mid_jobs;
  for (int i = 0; i < n; ++i) {
    FactJob a = jobs[i];
    a.half = 0;
    chain_jobs.push_back(a);
  }
  for (int i = 0; i < n; ++i) {
    FactJob a = jobs[i];
    a.half = 1;
    chain_jobs.push_back(a);
  }
  for (int i = 0; i < n; ++i) {
    FactJob a = jobs[i];
    a.half = 2;
    mid_jobs.push_back(a);
  }
  FactJob *djobs = nullptr;
  int *dstatus = nullptr;
  DS_CUDA(cudaMalloc(&djobs, 3 * n * sizeof(FactJob)));
  DS_CUDA(cudaMalloc(&dstatus, sizeof(int)));
  DS_CUDA(cudaMemcpy(djobs, chain_jobs.data(), 2 * n * sizeof(FactJob), cudaMemcpyHostToDevice));
  DS_CUDA(cudaMemcpy(djobs + 2 * n, mid_jobs.data(), n * sizeof(FactJob), cudaMemcpyHostToDevice));
  DS_CUDA(cudaMemset(dstatus, 0, sizeof(int)));
  DS_CUDA(cudaFuncSetAttribute(k_factor_gj, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem));
  for (int launch = 0; launch < 2; ++launch) {
    cudaLaunchConfig_t cfg;
    memset(&cfg, 0, sizeof(cfg));
    cfg.gridDim = dim3(C, launch == 0 ? 2 * n : n, 1);
    cfg.blockDim = dim3(GJ_THREADS, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = ctx->stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    DS_CUDA(cudaLaunchKernelEx(&cfg, k_factor_gj, (const FactJob *)(djobs + (launch ? 2 * n : 0)),
                               mcper, dstatus));
    ctx->launches++;
  }
  DS_CUDA(cudaStreamSynchronize(ctx->stream));
  DS_CUDA(cudaMemcpy(&status, dstatus, sizeof(int), cudaMemcpyDeviceToHost));
  cudaFree(djobs);
  cudaFree(dstatus);
  if (status) {
    for (void *p : F->allocations) cudaFree(p);
    delete F;
    return ds_fail(DS_ESOLVER, "block LU: zero or non-finite pivot in a Schur complement");
  }
  *out = F;
  return DS_OK;
}

// ------------------------------------------------------------ factor pool
// Out-of-core factorization (config 5: 64 raster windows need 638 GB of dense
// block inverses, HBM holds ~10 windows' worth): ds_fact_create_pool lays
// out every operator and allocates `nslots` factor slots of the largest
// operator's size; ds_fact_pool_load factors operator i into a slot (the
// blocked K2b path, same arithmetic as ds_fact_create), evicting the slot's
// previous operator.  A sweep plan built with a per-visit slot table
// (ds_plan_desc.visit_slot) reads each visit's factors from its slot; the
// host loads the slots a launch needs before issuing it.
extern "C" int ds_fact_create_pool(ds_ctx *ctx, ds_op *const *ops, int32_t n, int32_t nslots,
                                   ds_fact **out) {
  if (!ctx || !ops || n < 1 || nslots < 1 || !out)
    return ds_fail(DS_ECONFIG, "ds_fact_create_pool: bad argument");
  ds_fact *F = new ds_fact();
  F->pool = true;
  auto fail = [&](int code, const std::string &msg) {
    for (void *p : F->allocations) cudaFree(p);
    delete F;
    return ds_fail(code, msg);
  };
  size_t slot = 0;
  for (int i = 0; i < n; ++i) {
    if (!ops[i]) return fail(DS_ECONFIG, "ds_fact_create_pool: null operator");
    const OpDev &o = ops[i]->dev;
    FactDev f;
    memset(&f, 0, sizeof(f));
    ds_fill_layout(o, f);
    void *mem = nullptr;
    if (cudaMalloc(&mem, 2 * (size_t)f.nb * sizeof(cplx)) != cudaSuccess)
      return fail(DS_ECUDA, "ds_fact_create_pool: out of device memory");
    F->allocations.push_back(mem);
    cplx *lc = (cplx *)mem, *uc = lc + f.nb;
    cudaMemcpy(lc, o.c_lo[f.block_axis], f.nb * sizeof(cplx), cudaMemcpyDeviceToDevice);
    cudaMemcpy(uc, o.c_hi[f.block_axis], f.nb * sizeof(cplx), cudaMemcpyDeviceToDevice);
    f.sinv = nullptr;
    f.lcoef = lc;
    f.ucoef = uc;
    const size_t bytes = (size_t)f.nb * f.m * f.m * sizeof(cplx);
    slot = std::max(slot, bytes);
    F->facts.push_back(f);
    F->h_l.push_back(ops[i]->h_clo[f.block_axis]);
    F->h_u.push_back(ops[i]->h_chi[f.block_axis]);
    F->bytes.push_back((int64_t)(bytes + 2 * (size_t)f.nb * sizeof(cplx)));
    F->ops.push_back(ops[i]);
  }
  F->slot_bytes = slot;
  for (int c = 0; c < nslots; ++c) {
    void *mem = nullptr;
    if (cudaMalloc(&mem, slot) != cudaSuccess)
      return fail(DS_ECUDA, "ds_fact_create_pool: out of device memory for " + std::to_string(nslots) +
                                " slots of " + std::to_string(slot) + " bytes");
    F->allocations.push_back(mem);
    F->slot_mem.push_back((cplx *)mem);
    F->slot_owner.push_back(-1);
    F->bytes_total += (int64_t)slot;
  }
  *out = F;
  return DS_OK;
}

extern "C" int ds_fact_pool_load_many(ds_ctx *ctx, ds_fact *F, int32_t n, const int32_t *idx,
                                      const int32_t *slots) {
  if (!ctx || !F || !F->pool || n < 0 || (n > 0 && (!idx || !slots)))
    return ds_fail(DS_ECONFIG, "ds_fact_pool_load: bad argument");
  std::vector<FactJob> jobs;
  std::vector<const cplx *> lh, uh;
  std::vector<std::pair<int, int>> todo;  // (operator, slot)
  for (int q = 0; q < n; ++q) {
    const int i = idx[q], slot = slots[q];
    if (i < 0 || i >= (int)F->facts.size() || slot < 0 || slot >= (int)F->slot_mem.size())
      return ds_fail(DS_ECONFIG, "ds_fact_pool_load: operator or slot out of range");
    for (int p = 0; p < q; ++p)
      if (slots[p] == slot || idx[p] == i)
        return ds_fail(DS_ECONFIG, "ds_fact_pool_load: repeated operator or slot in one batch");
    if (F->slot_owner[slot] == i) continue;
    if (F->facts[i].m <= DS_LARGE_SLAB)
      return ds_fail(DS_ECONFIG, "ds_fact_pool_load: pooled factors are for large (3D) slabs");
    todo.push_back({i, slot});
  }
  // evict first: previous owners of the target slots, and the operators'
  // other slots (an operator lives in at most one slot)
  for (auto &t : todo) {
    const int prev = F->slot_owner[t.second];
    if (prev >= 0) F->facts[prev].sinv = nullptr;
    F->slot_owner[t.second] = -1;
  }
  for (auto &t : todo)
    for (size_t c = 0; c < F->slot_owner.size(); ++c)
      if (F->slot_owner[c] == t.first) {
        F->slot_owner[c] = -1;
        F->facts[t.first].sinv = nullptr;
      }
  if (todo.empty()) return DS_OK;
  for (auto &t : todo) {
    FactJob job;
    memset(&job, 0, sizeof(job));
    job.op = F->ops[t.first]->dev;
    job.f = F->facts[t.first];
    job.f.sinv = F->slot_mem[t.second];
    job.sinv = F->slot_mem[t.second];
    jobs.push_back(job);
    lh.push_back(F->h_l[t.first].data());
    uh.push_back(F->h_u[t.first].data());
  }
  int *dst = nullptr;
  DS_CUDA(cudaMalloc(&dst, sizeof(int)));
  DS_CUDA(cudaMemsetAsync(dst, 0, sizeof(int), ctx->stream));
  // all chains of the batch advance together (ds_blocked_factor batches
  // every (operator, half) chain per step): the panel latency is shared
  int rc = ds_blocked_factor(ctx, jobs.data(), (int)jobs.size(), lh.data(), uh.data(), dst);
  int status = 0;
  if (!rc) {
    cudaError_t e = cudaMemcpyAsync(&status, dst, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) rc = ds_fail(DS_ECUDA, std::string("ds_fact_pool_load: ") + cudaGetErrorString(e));
  }
  cudaFree(dst);
  if (rc) return rc;
  if (status) return ds_fail(DS_ESOLVER, "blocked LU: zero or non-finite pivot in a Schur complement");
  for (auto &t : todo) {
    F->facts[t.first].sinv = F->slot_mem[t.second];
    F->slot_owner[t.second] = t.first;
    F->loads++;
  }
  return DS_OK;
}

extern "C" int ds_fact_pool_load(ds_ctx *ctx, ds_fact *F, int32_t i, int32_t slot) {
  return ds_fact_pool_load_many(ctx, F, 1, &i, &slot);
}

extern "C" int ds_fact_pool_state(const ds_fact *F, int32_t *nslots, int64_t *slot_bytes,
                                  int32_t *slot_owner, int64_t *loads) {
  if (!F || !F->pool) return ds_fail(DS_ECONFIG, "ds_fact_pool_state: not a factor pool");
  if (nslots) *nslots = (int32_t)F->slot_mem.size();
  if (slot_bytes) *slot_bytes = (int64_t)F->slot_bytes;
  if (slot_owner)
    for (size_t c = 0; c < F->slot_owner.size(); ++c) slot_owner[c] = F->slot_owner[c];
  if (loads) *loads = F->loads;
  return DS_OK;
}

const cplx *ds_fact_slot_mem(const ds_fact *F, int slot) {
  if (!F || !F->pool || slot < 0 || slot >= (int)F->slot_mem.size()) return nullptr;
  return F->slot_mem[slot];
}

extern "C" int ds_fact_info(const ds_fact *F, int32_t i, int32_t *ba, int32_t *nb, int32_t *m,
                            int64_t *bytes) {
  if (!F || i < 0 || i >= (int)F->facts.size()) return ds_fail(DS_ECONFIG, "ds_fact_info: bad index");
  if (ba) *ba = F->facts[i].block_axis;
  if (nb) *nb = F->facts[i].nb;
  if (m) *m = F->facts[i].m;
  if (bytes) *bytes = F->bytes[i];
  return DS_OK;
}

extern "C" int ds_fact_destroy(ds_fact *F) {
  if (!F) return DS_OK;
  for (void *p : F->allocations) cudaFree(p);
  delete F;
  return DS_OK;
}

// window C-order [W][R]  <->  block layout [nb][m][R]
__global__ void k_permute(FactDev f, const cplx *__restrict__ src, cplx *__restrict__ dst,
                          int nrhs, int to_block) {
  int64_t total = (int64_t)f.nb * f.m * nrhs;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total;
       q += (int64_t)gridDim.x * blockDim.x) {
    int r = q % nrhs;
    int64_t lin = q / nrhs;  // window C-order linear node
    int c[3];
    c[2] = lin % f.win_shape[2];
    int64_t tt = lin / f.win_shape[2];
    c[1] = tt % f.win_shape[1];
    c[0] = tt / f.win_shape[1];
    int64_t b = block_offset(f, c) * nrhs + r;
    if (to_block) dst[b] = src[q];
    else dst[q] = src[b];
  }
}


extern "C" int ds_fact_solve(ds_ctx *ctx, const ds_fact *F, int32_t i, const ds_cplx *rhs,
                             ds_cplx *x, int32_t nrhs) {
  if (!ctx || !F || !rhs || !x || nrhs < 1 || i < 0 || i >= (int)F->facts.size())
    return ds_fail(DS_ECONFIG, "ds_fact_solve: bad argument");
  const FactDev &f = F->facts[i];
  if (f.kind == 0 && !f.sinv)
    return ds_fail(DS_ECONFIG, "ds_fact_solve: operator's factors are not resident (ds_fact_pool_load)");
  size_t n = (size_t)f.nb * f.m * nrhs;
  cplx *tmp = nullptr;
  void *vis = nullptr;
  DS_CUDA(cudaMallocAsync((void **)&tmp, 6 * n * sizeof(cplx) + sizeof(FactDev) + 64, ctx->stream));
  cplx *bin = tmp, *bout = tmp + n, *xg = tmp + 2 * n;
  FactDev *fd = (FactDev *)(tmp + 6 * n);
  DS_CUDA(cudaMallocAsync(&vis, sizeof(SolveVisit), ctx->stream));
  SolveVisit hv{fd, bin, bout, nullptr, xg};
  DS_CUDA(cudaMemcpyAsync(fd, &f, sizeof(FactDev), cudaMemcpyHostToDevice, ctx->stream));
  DS_CUDA(cudaMemcpyAsync(vis, &hv, sizeof(hv), cudaMemcpyHostToDevice, ctx->stream));
  int blocks = (int)std::min<int64_t>((n + 255) / 256, (int64_t)ctx->num_sms * 8);
  k_permute<<<blocks, 256, 0, ctx->stream>>>(f, (const cplx *)rhs, bin, nrhs, 1);
  ctx->launches++;
  DS_CHECK_LAUNCH();
  int rc;
  if (f.kind == 1) {
    // modal: scratch = the exchange area (>= 4 n), one device job
    ModalJob hj{fd, bin, bout, xg, xg + n, nullptr};
    ModalJob *dj = nullptr;
    DS_CUDA(cudaMallocAsync((void **)&dj, sizeof(ModalJob), ctx->stream));
    DS_CUDA(cudaMemcpyAsync(dj, &hj, sizeof(hj), cudaMemcpyHostToDevice, ctx->stream));
    rc = ds_launch_modal(ctx, dj, &f, 1, nrhs);
    cudaFreeAsync(dj, ctx->stream);
  } else if (f.m > DS_LARGE_SLAB) {
    SolveVisit hvis{fd, bin, bout, nullptr, xg};
    const cplx *lh = F->h_l[i].data(), *uh = F->h_u[i].data();
    size_t cap = ds_stage_items_bytes(1, f.nb, f.m, nrhs);
    void *items = nullptr;
    DS_CUDA(cudaMallocAsync(&items, cap, ctx->stream));
    rc = ds_launch_solve_staged(ctx, &hvis, &f, &lh, &uh, 1, nrhs, items, cap);
    cudaFreeAsync(items, ctx->stream);
  } else {
    rc = ds_launch_solve_table(ctx, vis, 1, nrhs, f.m);
  }
  if (rc) return rc;
  k_permute<<<blocks, 256, 0, ctx->stream>>>(f, bout, (cplx *)x, nrhs, 0);
  ctx->launches++;
  DS_CHECK_LAUNCH();
  DS_CUDA(cudaFreeAsync(tmp, ctx->stream));
  DS_CUDA(cudaFreeAsync(vis, ctx->stream));
  return DS_OK;
}
