// Context, error handling, operators + stencil apply (K1), batched vector
// kernels for GMRES (K7) and layout conversion.
//
// K1 restates DiscreteOperator.apply (diagsweep/pml.py:135-159):
//   out = k2*v + sum_a [ -(c_lo+c_hi) v + c_lo[i] v[i-1] + c_hi[i] v[i+1] ]
// with zero Dirichlet data outside `region`.  HBM-bound: 32 B/node/RHS
// (+8 B for 'full' kappa^2); the RHS-minor layout makes every neighbour
// access a contiguous run of nrhs complex values.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <algorithm>
#include <string>

#include "ds_common.cuh"

static thread_local std::string g_last_error;

void ds_set_error(const std::string &msg) { g_last_error = msg; }
int ds_fail(int code, const std::string &msg) {
  g_last_error = msg;
  return code;
}
int ceil_div(int a, int b) { return (a + b - 1) / b; }

extern "C" int ds_abi_version(void) { return DS_ABI_VERSION; }
extern "C" const char *ds_last_error(void) { return g_last_error.c_str(); }

extern "C" int ds_ctx_create(int device, void *stream, ds_ctx **out) {
  if (!out) return ds_fail(DS_ECONFIG, "ds_ctx_create: null out");
  int ndev = 0;
  DS_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev)
    return ds_fail(DS_ECONFIG, "ds_ctx_create: bad device ordinal");
  DS_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  DS_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    return ds_fail(DS_ECONFIG, std::string("library built for sm_100a, device is ") +
                                   prop.name);
  ds_ctx *c = new ds_ctx();
  c->device = device;
  c->stream = (cudaStream_t)stream;
  c->num_sms = prop.multiProcessorCount;
  c->launches = 0;
  ds_options_from_env(c->opt);
  g_ds_pdl = c->opt.pdl;
  c->scratch_bytes = 1 << 20;
  if (cudaMalloc(&c->scratch, c->scratch_bytes) != cudaSuccess) {
    delete c;
    return ds_fail(DS_ECUDA, "ds_ctx_create: scratch allocation failed");
  }
  if (cudaMalloc((void **)&c->work, sizeof(unsigned long long)) != cudaSuccess ||
      cudaMemset(c->work, 0, sizeof(unsigned long long)) != cudaSuccess) {
    cudaFree(c->scratch);
    delete c;
    return ds_fail(DS_ECUDA, "ds_ctx_create: counter allocation failed");
  }
  *out = c;
  return DS_OK;
}

int g_ds_pdl = 1;

static int env_opt(const char *name, int dflt) {
  const char *v = getenv(name);
  return v && *v ? atoi(v) : dflt;
}

void ds_options_from_env(ds_options &o) {
  if (const char *v = getenv("DS_K1")) {
    if (*v == 't') o.k1 = 0;
    else if (*v == 'c') o.k1 = atoi(v + 1);
  }
  o.combine = env_opt("DS_COMBINE", 2) == 1 ? 1 : 2;
  if (const char *v = getenv("DS_K4"))
    if (*v == 'v') o.k4 = atoi(v + 1);
  o.k4_rv = env_opt("DS_K4_RV", o.k4_rv);
  o.k6_rv = env_opt("DS_K6_RV", o.k6_rv);
  o.pdl = env_opt("DS_PDL", 1) != 0;
  o.k5_side = env_opt("DS_K5_SIDE", 1) != 0;
  if (const char *v = getenv("DS_SOLVE_MODE")) o.staged = std::string(v) == "staged";
  o.k3g_mma = env_opt("DS_K3G_MMA", 1) != 0;
  o.stage_rows = env_opt("DS_STAGE_ROWS", 0);
  o.k3_warps = env_opt("DS_K3_NW", 4) >= 8 ? 8 : 4;
  o.k3_rc_min = std::max(1, env_opt("DS_K3_RCMIN", o.k3_rc_min));
  o.k3_rc_max = std::max(1, env_opt("DS_K3_RCMAX", o.k3_rc_max));
  o.k3_cluster = env_opt("DS_K3_CLUSTER", 0);
  o.hio_dstreams = std::max(2, env_opt("DS_HIO_DSTREAMS", 2));
  o.kskip = env_opt("DS_KSKIP", 1) != 0;
  o.k2b_groups = std::max(1, std::min(8, env_opt("DS_K2B_GROUPS", 2)));
  o.r3_cols = env_opt("DS_R3_COLS", 16) == 32 ? 32 : 16;
}

// name -> member of ds_options
static int *opt_field(ds_options &o, const std::string &k) {
  if (k == "k1") return &o.k1;
  if (k == "combine") return &o.combine;
  if (k == "k4") return &o.k4;
  if (k == "k4_rv") return &o.k4_rv;
  if (k == "k6_rv") return &o.k6_rv;
  if (k == "pdl") return &o.pdl;
  if (k == "k5_side") return &o.k5_side;
  if (k == "staged") return &o.staged;
  if (k == "k3g_mma") return &o.k3g_mma;
  if (k == "stage_rows") return &o.stage_rows;
  if (k == "k3_warps") return &o.k3_warps;
  if (k == "k3_rc_min") return &o.k3_rc_min;
  if (k == "k3_rc_max") return &o.k3_rc_max;
  if (k == "k3_cluster") return &o.k3_cluster;
  if (k == "hio_dstreams") return &o.hio_dstreams;
  if (k == "kskip") return &o.kskip;
  if (k == "count_work") return &o.count_work;
  if (k == "k2b_groups") return &o.k2b_groups;
  if (k == "r3_cols") return &o.r3_cols;
  return nullptr;
}

extern "C" int ds_ctx_set_option(ds_ctx *ctx, const char *name, int32_t value) {
  if (!ctx || !name) return ds_fail(DS_ECONFIG, "ds_ctx_set_option: null argument");
  int *f = opt_field(ctx->opt, name);
  if (!f) return ds_fail(DS_ECONFIG, std::string("ds_ctx_set_option: unknown option ") + name);
  const std::string k = name;
  bool ok = true;
  if (k == "k1") ok = value == 0 || value == 2 || value == 4 || value == 8 || value == 16;
  else if (k == "combine") ok = value == 1 || value == 2;
  else if (k == "k4") ok = value >= 0 && value <= 3;
  else if (k == "k6_rv" || k == "k4_rv") ok = value == 1 || value == 2 || value == 4 || value == 8;
  else if (k == "k3_warps") ok = value == 4 || value == 8;
  else if (k == "r3_cols") ok = value == 16 || value == 32;
  else if (k == "k2b_groups") ok = value >= 1 && value <= 8;
  else if (k == "k3_cluster") ok = value == 0 || (value >= 8 && value <= 16);
  else ok = value >= 0;
  if (!ok) return ds_fail(DS_ECONFIG, "ds_ctx_set_option: bad value for " + k);
  *f = value;
  if (k == "pdl") g_ds_pdl = value != 0;
  return DS_OK;
}

extern "C" int ds_ctx_get_option(const ds_ctx *ctx, const char *name, int32_t *value) {
  if (!ctx || !name || !value) return ds_fail(DS_ECONFIG, "ds_ctx_get_option: null argument");
  int *f = opt_field(const_cast<ds_ctx *>(ctx)->opt, name);
  if (!f) return ds_fail(DS_ECONFIG, std::string("ds_ctx_get_option: unknown option ") + name);
  *value = *f;
  return DS_OK;
}

extern "C" int ds_ctx_set_stream(ds_ctx *ctx, void *stream) {
  if (!ctx) return ds_fail(DS_ECONFIG, "null ctx");
  ctx->stream = (cudaStream_t)stream;
  return DS_OK;
}

extern "C" int ds_ctx_synchronize(ds_ctx *ctx) {
  if (!ctx) return ds_fail(DS_ECONFIG, "null ctx");
  DS_CUDA(cudaStreamSynchronize(ctx->stream));
  return DS_OK;
}

extern "C" int64_t ds_ctx_launches(const ds_ctx *ctx) { return ctx ? ctx->launches : -1; }

extern "C" int ds_ctx_work(ds_ctx *ctx, int64_t *cmacs, int32_t reset) {
  if (!ctx || !cmacs) return ds_fail(DS_ECONFIG, "ds_ctx_work: null argument");
  unsigned long long v = 0;
  DS_CUDA(cudaStreamSynchronize(ctx->stream));
  DS_CUDA(cudaMemcpy(&v, ctx->work, sizeof(v), cudaMemcpyDeviceToHost));
  if (reset) DS_CUDA(cudaMemset(ctx->work, 0, sizeof(v)));
  *cmacs = (int64_t)v;
  return DS_OK;
}

extern "C" int ds_ctx_destroy(ds_ctx *ctx) {
  if (!ctx) return DS_OK;
  cudaFree(ctx->scratch);
  cudaFree(ctx->work);
  delete ctx;
  return DS_OK;
}

// ------------------------------------------------------------------ ops

extern "C" int ds_op_create(ds_ctx *ctx, const ds_op_desc *d, ds_op **out) {
  if (!ctx || !d || !out) return ds_fail(DS_ECONFIG, "ds_op_create: null argument");
  if (d->dim != 2 && d->dim != 3) return ds_fail(DS_ECONFIG, "operator dim must be 2 or 3");
  int64_t nodes = 1;
  for (int a = 0; a < d->dim; ++a) {
    if (d->shape[a] < 1) return ds_fail(DS_ECONFIG, "operator shape must be positive");
    if (!d->c_lo[a] || !d->c_hi[a]) return ds_fail(DS_ECONFIG, "missing coupling array");
    nodes *= d->shape[a];
  }
  int64_t nk2;
  switch (d->kappa2_kind) {
    case 0: nk2 = 1; break;
    case 1:
      if (d->kappa2_axis < 0 || d->kappa2_axis >= d->dim)
        return ds_fail(DS_ECONFIG, "bad kappa2 axis");
      nk2 = d->shape[d->kappa2_axis];
      break;
    case 2: nk2 = nodes; break;
    default: return ds_fail(DS_ECONFIG, "bad kappa2 kind");
  }
  if (!d->kappa2) return ds_fail(DS_ECONFIG, "missing kappa2");
  int64_t ncoef = 0;
  for (int a = 0; a < d->dim; ++a) ncoef += 2 * d->shape[a];
  size_t bytes = ncoef * sizeof(cplx) + nk2 * sizeof(double);
  ds_op *op = new ds_op();
  if (cudaMalloc(&op->storage, bytes) != cudaSuccess) {
    delete op;
    return ds_fail(DS_ECUDA, "ds_op_create: allocation failed");
  }
  OpDev &o = op->dev;
  memset(&o, 0, sizeof(o));
  o.dim = d->dim;
  o.kappa2_kind = d->kappa2_kind;
  o.kappa2_axis = d->kappa2_kind == 1 ? d->kappa2_axis : -1;
  cplx *p = (cplx *)op->storage;
  for (int a = 0; a < d->dim; ++a) {
    o.shape[a] = d->shape[a];
    cudaMemcpy(p, d->c_lo[a], d->shape[a] * sizeof(cplx), cudaMemcpyHostToDevice);
    o.c_lo[a] = p;
    p += d->shape[a];
    cudaMemcpy(p, d->c_hi[a], d->shape[a] * sizeof(cplx), cudaMemcpyHostToDevice);
    o.c_hi[a] = p;
    p += d->shape[a];
    op->h_clo[a].assign((const cplx *)d->c_lo[a], (const cplx *)d->c_lo[a] + d->shape[a]);
    op->h_chi[a].assign((const cplx *)d->c_hi[a], (const cplx *)d->c_hi[a] + d->shape[a]);
  }
  for (int a = d->dim; a < 3; ++a) o.shape[a] = 1;
  double *k2 = (double *)p;
  DS_CUDA(cudaMemcpy(k2, d->kappa2, nk2 * sizeof(double), cudaMemcpyHostToDevice));
  o.kappa2 = k2;
  op->h_k2.assign(d->kappa2, d->kappa2 + nk2);
  *out = op;
  return DS_OK;
}

extern "C" int ds_op_destroy(ds_op *op) {
  if (!op) return DS_OK;
  cudaFree(op->storage);
  delete op;
  return DS_OK;
}

__device__ __forceinline__ double op_kappa2(const OpDev &o, const int *c) {
  if (o.kappa2_kind == 0) return o.kappa2[0];
  if (o.kappa2_kind == 1) return o.kappa2[c[o.kappa2_axis]];
  int64_t lin = c[0];
  for (int a = 1; a < o.dim; ++a) lin = lin * o.shape[a] + c[a];
  return o.kappa2[lin];
}

// One thread per (region node, rhs).  rlo = region offset inside the
// operator window.  Order of accumulation follows pml.py:144-158.
// layout 0: RHS-minor [nodes][nrhs]; layout 1: RHS-outer [nrhs][nodes].
// Index arithmetic is 32-bit (a region has < 2^31 nodes; RHS-outer: one
// grid row per RHS, RHS-minor: (node, rhs) pairs < 2^31 checked by the
// launcher) -- the first version's 64-bit div/mod per element made it
// instruction-bound at 34% of HBM (config 3, tools/k1_k7_bench.py).
__global__ void __launch_bounds__(256) k_apply(OpDev o, const cplx *__restrict__ v, cplx *__restrict__ out,
                        int nrhs, int rlo0, int rlo1, int rlo2, int rs0, int rs1,
                        int rs2, int outer) {
  const int nodes = rs0 * rs1 * rs2;
  const int ns = outer ? 1 : nrhs;  // node stride
  const int st2 = ns, st1 = rs2 * ns, st0 = rs1 * rs2 * ns;
  const int total = outer ? nodes : nodes * nrhs;
  const int64_t base = outer ? (int64_t)blockIdx.y * nodes : 0;
  const cplx *__restrict__ vb = v + base;
  cplx *__restrict__ ob = out + base;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < total; q += gridDim.x * blockDim.x) {
    const int node = outer ? q : q / nrhs;
    const int e2 = node % rs2, t = node / rs2;
    const int e1 = t % rs1, e0 = t / rs1;
    const int c[3] = {e0 + rlo0, e1 + rlo1, e2 + rlo2};
    const int e[3] = {e0, e1, e2};
    const int rs[3] = {rs0, rs1, rs2};
    const int str[3] = {st0, st1, st2};
    // all loads first: centre, neighbours, couplings, kappa^2
    const cplx vc = vb[q];
    cplx vm[3], vp[3], lo[3], hi[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      if (a >= o.dim) break;
      vm[a] = e[a] > 0 ? vb[q - str[a]] : vc;
      vp[a] = e[a] < rs[a] - 1 ? vb[q + str[a]] : vc;
      lo[a] = o.c_lo[a][c[a]];
      hi[a] = o.c_hi[a][c[a]];
    }
    double k2;
    if (o.kappa2_kind == 0) k2 = o.kappa2[0];
    else if (o.kappa2_kind == 1) k2 = o.kappa2[c[o.kappa2_axis]];
    else {
      int64_t lin = c[0];
      for (int a = 1; a < o.dim; ++a) lin = lin * o.shape[a] + c[a];
      k2 = o.kappa2[lin];
    }
    cplx acc = cscale(vc, k2);
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      if (a >= o.dim) break;
      acc = cadd(acc, cmul(make_double2(-(lo[a].x + hi[a].x), -(lo[a].y + hi[a].y)), vc));
      if (e[a] > 0) acc = cadd(acc, cmul(lo[a], vm[a]));
      if (e[a] < rs[a] - 1) acc = cadd(acc, cmul(hi[a], vp[a]));
    }
    ob[q] = acc;
  }
}

// K1 v2 (2D, RHS-outer): one block per 32 x 8 tile of one RHS plane; the
// tile and its one-node halo are staged in shared memory with coalesced row
// loads (1.33 loads per output instead of 5), couplings and kappa^2 read
// once per row / column.  Same arithmetic and accumulation order as
// k_apply (neighbours outside the region contribute nothing).
#define K1_TX 32
#ifndef K1_TY
#define K1_TY 8
#endif
#ifndef K1_RPB
#define K1_RPB 1  // RHS planes per block (couplings / kappa^2 loaded once)
#endif
__global__ void __launch_bounds__(K1_TX * K1_TY) k_apply2d_tiled(OpDev o, const cplx *__restrict__ v,
                                                                cplx *__restrict__ out, int rlo0,
                                                                int rlo1, int rs0, int rs1, int nrhs) {
  __shared__ cplx tile[2][K1_TY + 2][K1_TX + 2];
  const int64_t plane = (int64_t)rs0 * rs1;
  const int x0 = blockIdx.x * K1_TX, y0 = blockIdx.y * K1_TY;
  const int tx = threadIdx.x % K1_TX, ty = threadIdx.x / K1_TX;
  const int y = y0 + ty, x = x0 + tx;
  const bool in = y < rs0 && x < rs1;
  const int c0 = min(y, rs0 - 1) + rlo0, c1 = min(x, rs1 - 1) + rlo1;
  double k2;
  if (o.kappa2_kind == 0) k2 = o.kappa2[0];
  else if (o.kappa2_kind == 1) k2 = o.kappa2[o.kappa2_axis == 0 ? c0 : c1];
  else k2 = o.kappa2[(int64_t)c0 * o.shape[1] + c1];
  const cplx lo0 = o.c_lo[0][c0], hi0 = o.c_hi[0][c0], lo1 = o.c_lo[1][c1], hi1 = o.c_hi[1][c1];
  const cplx m0 = make_double2(-(lo0.x + hi0.x), -(lo0.y + hi0.y));
  const cplx m1 = make_double2(-(lo1.x + hi1.x), -(lo1.y + hi1.y));
  const int r0 = blockIdx.z * K1_RPB, r1 = min(nrhs, r0 + K1_RPB);
  auto stage = [&](int r, int b) {
    const cplx *__restrict__ vb = v + (int64_t)r * plane;
    for (int i = threadIdx.x; i < (K1_TY + 2) * (K1_TX + 2); i += K1_TX * K1_TY) {
      const int ly = i / (K1_TX + 2), lx = i % (K1_TX + 2);
      const int yy = y0 + ly - 1, xx = x0 + lx - 1;
      tile[b][ly][lx] = (yy >= 0 && yy < rs0 && xx >= 0 && xx < rs1) ? vb[(int64_t)yy * rs1 + xx]
                                                                      : make_double2(0.0, 0.0);
    }
  };
  stage(r0, 0);
  for (int r = r0; r < r1; ++r) {
    const int b = (r - r0) & 1;
    __syncthreads();                       // tile b complete, tile b^1 free
    if (r + 1 < r1) stage(r + 1, b ^ 1);  // next plane's loads in flight under this one
    if (!in) continue;
    const cplx vc = tile[b][ty + 1][tx + 1];
    cplx acc = cscale(vc, k2);
    acc = cadd(acc, cmul(m0, vc));
    if (y > 0) acc = cadd(acc, cmul(lo0, tile[b][ty][tx + 1]));
    if (y < rs0 - 1) acc = cadd(acc, cmul(hi0, tile[b][ty + 2][tx + 1]));
    acc = cadd(acc, cmul(m1, vc));
    if (x > 0) acc = cadd(acc, cmul(lo1, tile[b][ty + 1][tx]));
    if (x < rs1 - 1) acc = cadd(acc, cmul(hi1, tile[b][ty + 1][tx + 2]));
    out[(int64_t)r * plane + (int64_t)y * rs1 + x] = acc;
  }
}

// K1 v3 (2D, RHS-outer, the default): column marching.  A thread owns one x
// of a K1C_X-wide strip and walks K1C_YS rows down it with the rows above /
// below in registers; x neighbours come from the adjacent lanes by shuffle
// (lanes 0 and 31 load the one node across the warp edge).  All K1C_YS + 2
// row loads are independent and issued up front -- no shared memory, no
// barriers, 1 + 2/K1C_YS row reads per output.  Accumulation order as
// k_apply (pml.py:144-158), neighbours outside the region contribute nothing.
#ifndef K1C_X
#define K1C_X 64  // strip width: config 3's 441-wide regions fill 7 x 64 = 448 lanes (128: 512)
#endif
__device__ __forceinline__ cplx shfl_cplx(cplx v, int delta, bool up) {
  cplx r;
  r.x = up ? __shfl_up_sync(0xffffffffu, v.x, delta) : __shfl_down_sync(0xffffffffu, v.x, delta);
  r.y = up ? __shfl_up_sync(0xffffffffu, v.y, delta) : __shfl_down_sync(0xffffffffu, v.y, delta);
  return r;
}
#ifndef K1C_MINB
#define K1C_MINB (7 * 128 / K1C_X)  // rows <= 4: 72 registers, 28 warps per SM: config 3 K1 0.327 -> 0.272 ms at 128 wide (8 x 128 spills), 0.263 ms at 64 wide
#endif
template <int K1C_YS>
__global__ void __launch_bounds__(K1C_X, K1C_YS <= 4 ? K1C_MINB : 1) k_apply2d_cols(OpDev o, const cplx *__restrict__ v,
                                                       cplx *__restrict__ out, int rlo0, int rlo1, int rs0,
                                                       int rs1) {
  const int64_t plane = (int64_t)rs0 * rs1;
  const cplx *__restrict__ vb = v + (int64_t)blockIdx.z * plane;
  cplx *__restrict__ ob = out + (int64_t)blockIdx.z * plane;
  const int x = blockIdx.x * K1C_X + threadIdx.x, y0 = blockIdx.y * K1C_YS;
  const int lane = threadIdx.x & 31;
  const bool xin = x < rs1;
  const int xc = min(x, rs1 - 1);
  const cplx zero = make_double2(0.0, 0.0);
  // rows y0-1 .. y0+K1C_YS of my column (zero outside the region)
  cplx col[K1C_YS + 2], edge[K1C_YS];
#pragma unroll
  for (int i = 0; i < K1C_YS + 2; ++i) {
    const int y = y0 - 1 + i;
    col[i] = (xin && y >= 0 && y < rs0) ? vb[(int64_t)y * rs1 + x] : zero;
  }
  // across the warp edge: lane 0 needs x-1, lane 31 needs x+1
  const int xe = lane == 0 ? x - 1 : x + 1;
  const bool edge_lane = (lane == 0 || lane == 31) && xe >= 0 && xe < rs1;
#pragma unroll
  for (int i = 0; i < K1C_YS; ++i) {
    const int y = y0 + i;
    edge[i] = (edge_lane && y < rs0) ? vb[(int64_t)y * rs1 + xe] : zero;
  }
  const int c1 = xc + rlo1;
  const cplx lo1 = o.c_lo[1][c1], hi1 = o.c_hi[1][c1];
  const cplx m1 = make_double2(-(lo1.x + hi1.x), -(lo1.y + hi1.y));
#pragma unroll
  for (int i = 0; i < K1C_YS; ++i) {
    const int y = y0 + i;
    const cplx vc = col[i + 1];
    cplx left = shfl_cplx(vc, 1, true), right = shfl_cplx(vc, 1, false);
    if (lane == 0) left = edge[i];
    if (lane == 31) right = edge[i];
    if (!xin || y >= rs0) continue;
    const int c0 = y + rlo0;
    double k2;
    if (o.kappa2_kind == 0) k2 = o.kappa2[0];
    else if (o.kappa2_kind == 1) k2 = o.kappa2[o.kappa2_axis == 0 ? c0 : c1];
    else k2 = o.kappa2[(int64_t)c0 * o.shape[1] + c1];
    const cplx lo0 = o.c_lo[0][c0], hi0 = o.c_hi[0][c0];
    const cplx m0 = make_double2(-(lo0.x + hi0.x), -(lo0.y + hi0.y));
    cplx acc = cscale(vc, k2);
    acc = cadd(acc, cmul(m0, vc));
    if (y > 0) acc = cadd(acc, cmul(lo0, col[i]));
    if (y < rs0 - 1) acc = cadd(acc, cmul(hi0, col[i + 2]));
    acc = cadd(acc, cmul(m1, vc));
    if (x > 0) acc = cadd(acc, cmul(lo1, left));
    if (x < rs1 - 1) acc = cadd(acc, cmul(hi1, right));
    ob[(int64_t)y * rs1 + x] = acc;
  }
}

// K1 variant (option "k1"): rows per thread of the column-marching kernel
// (default 4: config 3 K1 0.287 ms = 74.5% of HBM vs 8 rows 61.8%, 16 rows
// 36.5%) or 0 = the 32 x 8 shared-memory tile (54.6%)
static int k1_variant(const ds_ctx *ctx) { return ctx->opt.k1; }

static int grid_for(ds_ctx *ctx, int64_t work, int threads) {
  int64_t blocks = (work + threads - 1) / threads;
  int64_t cap = (int64_t)ctx->num_sms * 16;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  return (int)blocks;
}

extern "C" int ds_op_apply(ds_ctx *ctx, const ds_op *op, const ds_cplx *v, ds_cplx *out,
                           int32_t nrhs, const int32_t *rlo, const int32_t *rs, int32_t layout) {
  if (!ctx || !op || !v || !out || nrhs < 1)
    return ds_fail(DS_ECONFIG, "ds_op_apply: bad argument");
  const OpDev &o = op->dev;
  int lo[3] = {0, 0, 0}, sh[3] = {1, 1, 1};
  for (int a = 0; a < o.dim; ++a) {
    lo[a] = rlo ? rlo[a] : 0;
    sh[a] = rs ? rs[a] : o.shape[a];
    if (lo[a] < 0 || sh[a] < 1 || lo[a] + sh[a] > o.shape[a])
      return ds_fail(DS_ECONFIG, "ds_op_apply: region outside the operator window");
  }
  const int64_t nodes = (int64_t)sh[0] * sh[1] * sh[2];
  if (nodes * (layout != 0 ? 1 : nrhs) >= (int64_t)1 << 31 || nrhs > 65535)
    return ds_fail(DS_ECONFIG, "ds_op_apply: region too large for one launch");
  if (layout != 0 && o.dim == 2 && nrhs <= 65535 && k1_variant(ctx) != 0) {
    const int ys = k1_variant(ctx);
    const dim3 grid((sh[1] + K1C_X - 1) / K1C_X, (sh[0] + ys - 1) / ys, nrhs);
    if (ys == 16)
      k_apply2d_cols<16><<<grid, K1C_X, 0, ctx->stream>>>(o, (const cplx *)v, (cplx *)out, lo[0], lo[1],
                                                         sh[0], sh[1]);
    else if (ys == 8)
      k_apply2d_cols<8><<<grid, K1C_X, 0, ctx->stream>>>(o, (const cplx *)v, (cplx *)out, lo[0], lo[1],
                                                        sh[0], sh[1]);
    else if (ys == 2)
      k_apply2d_cols<2><<<grid, K1C_X, 0, ctx->stream>>>(o, (const cplx *)v, (cplx *)out, lo[0], lo[1],
                                                        sh[0], sh[1]);
    else
      k_apply2d_cols<4><<<grid, K1C_X, 0, ctx->stream>>>(o, (const cplx *)v, (cplx *)out, lo[0], lo[1],
                                                        sh[0], sh[1]);
  } else if (layout != 0 && o.dim == 2 && nrhs <= 65535) {
    const dim3 grid((sh[1] + K1_TX - 1) / K1_TX, (sh[0] + K1_TY - 1) / K1_TY, (nrhs + K1_RPB - 1) / K1_RPB);
    k_apply2d_tiled<<<grid, K1_TX * K1_TY, 0, ctx->stream>>>(o, (const cplx *)v, (cplx *)out, lo[0], lo[1],
                                                             sh[0], sh[1], nrhs);
  } else if (layout != 0) {
    const int bx = (int)std::max<int64_t>(1, std::min<int64_t>((nodes + 255) / 256,
                                                               (int64_t)ctx->num_sms * 16 / nrhs + 1));
    k_apply<<<dim3(bx, nrhs), 256, 0, ctx->stream>>>(o, (const cplx *)v, (cplx *)out, nrhs, lo[0], lo[1],
                                                     lo[2], sh[0], sh[1], sh[2], 1);
  } else {
    k_apply<<<grid_for(ctx, nodes * nrhs, 256), 256, 0, ctx->stream>>>(
        o, (const cplx *)v, (cplx *)out, nrhs, lo[0], lo[1], lo[2], sh[0], sh[1], sh[2], 0);
  }
  ctx->launches++;
  DS_CHECK_LAUNCH();
  return DS_OK;
}

// ------------------------------------------------------- vector kernels
// GMRES vectors are RHS-outer [nrhs][n] (the reference's batch layout), so
// every per-RHS reduction runs over a contiguous vector.  Deterministic:
// grid (B, nrhs); block b of RHS r reduces a fixed chunk in a fixed tree
// order into partials[r][b]; a second kernel sums the B partials in order.

#define VEC_THREADS 256
#define VEC_BLOCKS_MAX 256

__device__ __forceinline__ cplx block_reduce(cplx v, cplx *red) {
  int t = threadIdx.x;
  red[t] = v;
  __syncthreads();
  for (int s = VEC_THREADS / 2; s > 0; s >>= 1) {
    if (t < s) red[t] = cadd(red[t], red[t + s]);
    __syncthreads();
  }
  return red[0];
}

// MODE 0: vdot(x, y); 1: |x|^2; 2: y -= a_prev*xprev then vdot(x, y);
// 3: y = x - xprev then |y|^2 (the residual r = b - A x and its norm)
template <int MODE>
__global__ void __launch_bounds__(VEC_THREADS)
    k_vec_reduce(int64_t n, const cplx *__restrict__ x, cplx *y, const cplx *__restrict__ a_prev,
                 const cplx *__restrict__ xprev, cplx *partials, int64_t chunk) {
  __shared__ cplx red[VEC_THREADS];
  const int r = blockIdx.y, B = gridDim.x;
  const int64_t base = (int64_t)r * n;
  int64_t i0 = blockIdx.x * chunk, i1 = min(n, i0 + chunk);
  cplx acc = make_double2(0.0, 0.0);
  cplx s = make_double2(0.0, 0.0);
  if (MODE == 2 && xprev) s = a_prev[r];
  for (int64_t i = i0 + threadIdx.x; i < i1; i += VEC_THREADS) {
    cplx a = x[base + i];
    if (MODE == 3) {
      a = csub(a, xprev[base + i]);
      y[base + i] = a;
    }
    if (MODE == 1 || MODE == 3) {
      acc.x = fma(a.x, a.x, acc.x);
      acc.x = fma(a.y, a.y, acc.x);
    } else {
      cplx yv = y[base + i];
      if (MODE == 2 && xprev) {
        yv = csub(yv, cmul(s, xprev[base + i]));
        y[base + i] = yv;
      }
      cfma_conj(acc, a, yv);
    }
  }
  cplx tot = block_reduce(acc, red);
  if (threadIdx.x == 0) partials[(int64_t)r * B + blockIdx.x] = tot;
}

__global__ void k_reduce_final(int nblocks, int nrhs, const cplx *partials, cplx *out_c,
                               double *out_norm) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrhs) return;
  cplx s = make_double2(0.0, 0.0);
  for (int b = 0; b < nblocks; ++b) s = cadd(s, partials[(int64_t)r * nblocks + b]);
  if (out_c) out_c[r] = s;
  if (out_norm) out_norm[r] = sqrt(s.x);
}

static int reduction_launch(ds_ctx *ctx, int mode, int64_t n, int nrhs, const cplx *x, cplx *y,
                            const cplx *a_prev, const cplx *xprev, cplx *out_c,
                            double *out_norm) {
  if (nrhs < 1 || nrhs > 65535 || n < 1) return ds_fail(DS_ECONFIG, "vector op: bad sizes");
  int64_t want = (int64_t)ctx->num_sms * 4 / nrhs;
  int B = (int)std::max<int64_t>(1, std::min<int64_t>(VEC_BLOCKS_MAX, want));
  int64_t chunk = (n + B - 1) / B;
  B = (int)((n + chunk - 1) / chunk);
  if ((size_t)B * nrhs * sizeof(cplx) > ctx->scratch_bytes)
    return ds_fail(DS_ECONFIG, "reduction scratch too small");
  cplx *partials = (cplx *)ctx->scratch;
  dim3 grid(B, nrhs);
  if (mode == 0)
    k_vec_reduce<0><<<grid, VEC_THREADS, 0, ctx->stream>>>(n, x, y, nullptr, nullptr, partials, chunk);
  else if (mode == 1)
    k_vec_reduce<1><<<grid, VEC_THREADS, 0, ctx->stream>>>(n, x, y, nullptr, nullptr, partials, chunk);
  else if (mode == 2)
    k_vec_reduce<2><<<grid, VEC_THREADS, 0, ctx->stream>>>(n, x, y, a_prev, xprev, partials, chunk);
  else
    k_vec_reduce<3><<<grid, VEC_THREADS, 0, ctx->stream>>>(n, x, y, nullptr, xprev, partials, chunk);
  k_reduce_final<<<ceil_div(nrhs, 128), 128, 0, ctx->stream>>>(B, nrhs, partials, out_c, out_norm);
  ctx->launches += 2;
  DS_CHECK_LAUNCH();
  return DS_OK;
}

extern "C" int ds_vec_dot(ds_ctx *ctx, int64_t n, int32_t nrhs, const ds_cplx *x,
                          const ds_cplx *y, ds_cplx *out) {
  if (!ctx) return ds_fail(DS_ECONFIG, "null ctx");
  return reduction_launch(ctx, 0, n, nrhs, (const cplx *)x, (cplx *)y, nullptr, nullptr,
                          (cplx *)out, nullptr);
}

extern "C" int ds_vec_norm(ds_ctx *ctx, int64_t n, int32_t nrhs, const ds_cplx *x,
                           double *out) {
  if (!ctx) return ds_fail(DS_ECONFIG, "null ctx");
  return reduction_launch(ctx, 1, n, nrhs, (const cplx *)x, nullptr, nullptr, nullptr, nullptr,
                          out);
}

extern "C" int ds_vec_axpy_dot(ds_ctx *ctx, int64_t n, int32_t nrhs, const ds_cplx *a_prev,
                               const ds_cplx *xprev, ds_cplx *y, const ds_cplx *x,
                               ds_cplx *out) {
  if (!ctx) return ds_fail(DS_ECONFIG, "null ctx");
  return reduction_launch(ctx, 2, n, nrhs, (const cplx *)x, (cplx *)y, (const cplx *)a_prev,
                          (const cplx *)xprev, (cplx *)out, nullptr);
}

__global__ void k_axpy(int64_t n, const cplx *__restrict__ a, double sgn,
                       const cplx *__restrict__ x, cplx *y) {
  const int r = blockIdx.y;
  cplx s = a[r];
  s.x *= sgn;
  s.y *= sgn;
  const int64_t base = (int64_t)r * n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[base + i] = cadd(y[base + i], cmul(s, x[base + i]));
}

extern "C" int ds_vec_sub_norm(ds_ctx *ctx, int64_t n, int32_t nrhs, const ds_cplx *b,
                               const ds_cplx *w, ds_cplx *out, double *norm_out) {
  if (!ctx || !b || !w || !out || !norm_out) return ds_fail(DS_ECONFIG, "ds_vec_sub_norm: null argument");
  return reduction_launch(ctx, 3, n, nrhs, (const cplx *)b, (cplx *)out, nullptr, (const cplx *)w,
                          nullptr, norm_out);
}

// rows of RHS-outer batches: dst[r] = src[map[r]] for map[r] >= 0, else 0
// (gather: map = selected rows; scatter into the full batch: map = inverse)
__global__ void k_rows_map(int64_t n, const int *__restrict__ map, const cplx *__restrict__ src,
                           cplx *__restrict__ dst) {
  const int r = blockIdx.y;
  const int q = map[r];
  const cplx *s = q >= 0 ? src + (int64_t)q * n : nullptr;
  cplx *d = dst + (int64_t)r * n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    d[i] = s ? s[i] : make_double2(0.0, 0.0);
}

static dim3 vec_grid(ds_ctx *ctx, int64_t n, int nrhs);

extern "C" int ds_vec_rows(ds_ctx *ctx, int64_t n, int32_t ndst, const int32_t *map_dev,
                           const ds_cplx *src, ds_cplx *dst) {
  if (!ctx || !map_dev || !src || !dst || ndst < 0 || ndst > 65535)
    return ds_fail(DS_ECONFIG, "ds_vec_rows: bad argument");
  if (ndst == 0 || n == 0) return DS_OK;
  k_rows_map<<<vec_grid(ctx, n, ndst), 256, 0, ctx->stream>>>(n, map_dev, (const cplx *)src, (cplx *)dst);
  ctx->launches++;
  DS_CHECK_LAUNCH();
  return DS_OK;
}

static dim3 vec_grid(ds_ctx *ctx, int64_t n, int nrhs) {
  int64_t per = std::max<int64_t>(1, (int64_t)ctx->num_sms * 8 / nrhs);
  int64_t need = (n + 255) / 256;
  return dim3((unsigned)std::max<int64_t>(1, std::min(per, need)), nrhs);
}

extern "C" int ds_vec_axpy(ds_ctx *ctx, int64_t n, int32_t nrhs, const ds_cplx *a,
                           double sgn, const ds_cplx *x, ds_cplx *y) {
  if (!ctx || nrhs < 1 || nrhs > 65535) return ds_fail(DS_ECONFIG, "ds_vec_axpy: bad argument");
  k_axpy<<<vec_grid(ctx, n, nrhs), 256, 0, ctx->stream>>>(n, (const cplx *)a, sgn,
                                                          (const cplx *)x, (cplx *)y);
  ctx->launches++;
  DS_CHECK_LAUNCH();
  return DS_OK;
}

#define MAX_COMBINE 64
struct CombineArgs {
  const cplx *x[MAX_COMBINE];
};

// y[r] += sum_j c[j][r] * X_j[r]   (krylov.py:139, x + Z^T y)
__global__ void k_combine(int64_t n, int nrhs, int nvec, CombineArgs args,
                          const cplx *__restrict__ c, cplx *y) {
  const int r = blockIdx.y;
  const int64_t base = (int64_t)r * n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    cplx acc = make_double2(0.0, 0.0);
    const cplx yv = y[base + i];
#pragma unroll 8
    for (int j = 0; j < nvec; ++j) acc = cadd(acc, cmul(__ldg(c + j * nrhs + r), args.x[j][base + i]));
    y[base + i] = cadd(yv, acc);
  }
}

// two elements per thread (i, i + stride): twice the independent loads in
// flight per thread, same per-element summation order as k_combine
__global__ void k_combine2(int64_t n, int nrhs, int nvec, CombineArgs args,
                           const cplx *__restrict__ c, cplx *y) {
  const int r = blockIdx.y;
  const int64_t base = (int64_t)r * n;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += 2 * stride) {
    const int64_t i2 = i + stride;
    const bool two = i2 < n;
    cplx acc = make_double2(0.0, 0.0), acc2 = make_double2(0.0, 0.0);
    const cplx yv = y[base + i];
    const cplx yv2 = two ? y[base + i2] : make_double2(0.0, 0.0);
#pragma unroll 8
    for (int j = 0; j < nvec; ++j) {
      const cplx cj = __ldg(c + j * nrhs + r);
      const cplx *xj = args.x[j] + base;
      acc = cadd(acc, cmul(cj, xj[i]));
      if (two) acc2 = cadd(acc2, cmul(cj, xj[i2]));
    }
    y[base + i] = cadd(yv, acc);
    if (two) y[base + i2] = cadd(yv2, acc2);
  }
}

extern "C" int ds_vec_combine(ds_ctx *ctx, int64_t n, int32_t nrhs, int32_t nvec,
                              const ds_cplx *const *xs, const ds_cplx *c, ds_cplx *y) {
  if (!ctx || nrhs < 1 || nrhs > 65535 || nvec < 0 || nvec > MAX_COMBINE)
    return ds_fail(DS_ECONFIG, "ds_vec_combine: bad argument");
  if (nvec == 0) return DS_OK;
  CombineArgs args;
  for (int j = 0; j < nvec; ++j) args.x[j] = (const cplx *)xs[j];
  if (ctx->opt.combine == 2)
    k_combine2<<<vec_grid(ctx, (n + 1) / 2, nrhs), 256, 0, ctx->stream>>>(n, nrhs, nvec, args,
                                                                        (const cplx *)c, (cplx *)y);
  else
    k_combine<<<vec_grid(ctx, n, nrhs), 256, 0, ctx->stream>>>(n, nrhs, nvec, args,
                                                               (const cplx *)c, (cplx *)y);
  ctx->launches++;
  DS_CHECK_LAUNCH();
  return DS_OK;
}

__global__ void k_scale(int64_t n, const cplx *__restrict__ x, const double *__restrict__ s,
                        cplx *y) {
  const int r = blockIdx.y;
  const double sc = s[r];
  const int64_t base = (int64_t)r * n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    cplx v = x[base + i];
    y[base + i] = sc == 0.0 ? make_double2(0.0, 0.0) : make_double2(v.x / sc, v.y / sc);
  }
}

extern "C" int ds_vec_scale(ds_ctx *ctx, int64_t n, int32_t nrhs, const ds_cplx *x,
                            const double *s, ds_cplx *y) {
  if (!ctx || nrhs < 1 || nrhs > 65535) return ds_fail(DS_ECONFIG, "ds_vec_scale: bad argument");
  k_scale<<<vec_grid(ctx, n, nrhs), 256, 0, ctx->stream>>>(n, (const cplx *)x, s, (cplx *)y);
  ctx->launches++;
  DS_CHECK_LAUNCH();
  return DS_OK;
}

// ----------------------------------------------------- layout transpose
// [R][n] <-> [n][R] through a 32x32 shared tile.
__global__ void k_transpose(int64_t rows, int64_t cols, int64_t ntc,
                            const cplx *__restrict__ src, cplx *__restrict__ dst) {
  // src is [rows][cols], dst is [cols][rows]; 1D grid over 32x32 tiles
  __shared__ cplx tile[32][33];
  int64_t tr = blockIdx.x / ntc, tc = blockIdx.x % ntc;
  int64_t r0 = tr * 32, c0 = tc * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    int64_t r = r0 + i, c = c0 + threadIdx.x;
    if (r < rows && c < cols) tile[i][threadIdx.x] = src[r * cols + c];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    int64_t c = c0 + i, r = r0 + threadIdx.x;
    if (r < rows && c < cols) dst[c * rows + r] = tile[threadIdx.x][i];
  }
}

static int transpose(ds_ctx *ctx, int64_t rows, int64_t cols, const cplx *src, cplx *dst) {
  if (rows < 1 || cols < 1) return DS_OK;
  if (rows == 1 || cols == 1) {
    DS_CUDA(cudaMemcpyAsync(dst, src, rows * cols * sizeof(cplx), cudaMemcpyDeviceToDevice,
                            ctx->stream));
    return DS_OK;
  }
  int64_t ntr = (rows + 31) / 32, ntc = (cols + 31) / 32;
  if (ntr * ntc > 0x7fffffffLL) return ds_fail(DS_ECONFIG, "transpose: too large");
  k_transpose<<<(unsigned)(ntr * ntc), dim3(32, 8), 0, ctx->stream>>>(rows, cols, ntc, src, dst);
  ctx->launches++;
  DS_CHECK_LAUNCH();
  return DS_OK;
}

extern "C" int ds_layout_to_minor(ds_ctx *ctx, int64_t n, int32_t nrhs, const ds_cplx *src,
                                  ds_cplx *dst) {
  if (!ctx || src == dst) return ds_fail(DS_ECONFIG, "ds_layout_to_minor: bad argument");
  // src [R][n] -> dst [n][R]
  return transpose(ctx, nrhs, n, (const cplx *)src, (cplx *)dst);
}

extern "C" int ds_layout_to_outer(ds_ctx *ctx, int64_t n, int32_t nrhs, const ds_cplx *src,
                                  ds_cplx *dst) {
  if (!ctx || src == dst) return ds_fail(DS_ECONFIG, "ds_layout_to_outer: bad argument");
  // src [n][R] -> dst [R][n]
  return transpose(ctx, n, nrhs, (const cplx *)src, (cplx *)dst);
}

// ------------------------------------------------------ cross-rank barrier
// Device-side barrier of a subdomain-sharded sweep (sharded.py): every rank
// owns an arrival array arrive[nranks] (uint64 generations) in its memory,
// mapped by its peers (NVLink P2P / CUDA IPC).  ds_barrier_wait enqueues one
// single-warp kernel: after a system-scope fence (the previous kernels'
// peer writes -- payloads, arrival flags -- become visible first), lane r
// stores the generation into arrive[rank] of rank r's array (release, system
// scope), then spins until its own arrive[r] reaches the generation
// (acquire).  No host round trip and no NCCL call between launches; the
// spin is bounded (~10 s of clock64) and traps instead of hanging.
struct ds_barrier {
  int nranks, rank;
  unsigned long long *arrive;            // own array, device memory
  unsigned long long **peers = nullptr;  // device table of every rank's array
  unsigned long long gen = 0;
};

__global__ void k_peer_barrier(unsigned long long *const *peers, unsigned long long *own, int nranks,
                               int rank, unsigned long long gen) {
  const int r = threadIdx.x;
  __threadfence_system();
  if (r < nranks) {
    unsigned long long *dst = peers[r] + rank;
    asm volatile("st.release.sys.global.u64 [%0], %1;\n" ::"l"(dst), "l"(gen) : "memory");
    unsigned long long v = 0;
    const long long t0 = clock64();
    do {
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];\n" : "=l"(v) : "l"(own + r) : "memory");
      if (v >= gen) break;
      if (clock64() - t0 > (1LL << 34)) __trap();  // a peer never arrived
    } while (true);
  }
  __syncwarp();
}

extern "C" int ds_barrier_create(ds_ctx *ctx, int32_t nranks, int32_t rank, ds_barrier **out) {
  if (!ctx || !out || nranks < 1 || nranks > 32 || rank < 0 || rank >= nranks)
    return ds_fail(DS_ECONFIG, "ds_barrier_create: bad argument");
  ds_barrier *B = new ds_barrier();
  B->nranks = nranks;
  B->rank = rank;
  if (cudaMalloc(&B->arrive, sizeof(unsigned long long) * nranks) != cudaSuccess ||
      cudaMemset(B->arrive, 0, sizeof(unsigned long long) * nranks) != cudaSuccess ||
      cudaMalloc(&B->peers, sizeof(void *) * nranks) != cudaSuccess) {
    cudaFree(B->arrive);
    delete B;
    return ds_fail(DS_ECUDA, "ds_barrier_create: allocation failed");
  }
  *out = B;
  return DS_OK;
}

extern "C" int ds_barrier_info(const ds_barrier *B, void **arrive, int64_t *bytes) {
  if (!B) return ds_fail(DS_ECONFIG, "null barrier");
  if (arrive) *arrive = B->arrive;
  if (bytes) *bytes = (int64_t)sizeof(unsigned long long) * B->nranks;
  return DS_OK;
}

extern "C" int ds_barrier_set_peers(ds_barrier *B, int32_t nranks, void *const *arrive) {
  if (!B || !arrive || nranks != B->nranks) return ds_fail(DS_ECONFIG, "ds_barrier_set_peers: bad argument");
  for (int r = 0; r < nranks; ++r)
    if (!arrive[r]) return ds_fail(DS_ECONFIG, "ds_barrier_set_peers: null peer array");
  DS_CUDA(cudaMemcpy(B->peers, arrive, sizeof(void *) * nranks, cudaMemcpyHostToDevice));
  return DS_OK;
}

extern "C" int ds_barrier_wait(ds_ctx *ctx, ds_barrier *B) {
  if (!ctx || !B) return ds_fail(DS_ECONFIG, "ds_barrier_wait: null argument");
  ++B->gen;
  k_peer_barrier<<<1, 32, 0, ctx->stream>>>(B->peers, B->arrive, B->nranks, B->rank, B->gen);
  ctx->launches++;
  DS_CHECK_LAUNCH();
  return DS_OK;
}

extern "C" int64_t ds_barrier_generation(const ds_barrier *B) { return B ? (int64_t)B->gen : -1; }

extern "C" int ds_barrier_destroy(ds_barrier *B) {
  if (!B) return DS_OK;
  cudaFree(B->arrive);
  cudaFree(B->peers);
  delete B;
  return DS_OK;
}
