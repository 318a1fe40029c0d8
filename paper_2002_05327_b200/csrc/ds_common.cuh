// Shared device/host helpers of the diagsweep_b200 library (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>

#include <string>
#include <vector>

#include "../../include/diagsweep_b200.h"

typedef double2 cplx;  // (re, im), same bytes as ds_cplx / complex128

#define DS_HD __host__ __device__ __forceinline__

DS_HD cplx cmk(double r, double i) { return make_double2(r, i); }
DS_HD cplx cadd(cplx a, cplx b) { return make_double2(a.x + b.x, a.y + b.y); }
DS_HD cplx csub(cplx a, cplx b) { return make_double2(a.x - b.x, a.y - b.y); }
DS_HD cplx cmul(cplx a, cplx b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
DS_HD cplx cscale(cplx a, double s) { return make_double2(a.x * s, a.y * s); }
// acc += a * b
DS_HD void cfma(cplx &acc, cplx a, cplx b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
}
// acc += conj(a) * b
DS_HD void cfma_conj(cplx &acc, cplx a, cplx b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(-a.y, b.x, acc.y);
}
DS_HD cplx cinv(cplx a) {
  // Smith's algorithm (robust reciprocal)
  if (fabs(a.x) >= fabs(a.y)) {
    double r = a.y / a.x, den = a.x + a.y * r;
    return make_double2(1.0 / den, -r / den);
  } else {
    double r = a.x / a.y, den = a.x * r + a.y;
    return make_double2(r / den, -1.0 / den);
  }
}
DS_HD bool cnonzero(cplx a) { return a.x != 0.0 || a.y != 0.0; }
DS_HD double cabs1(cplx a) { return fabs(a.x) + fabs(a.y); }

// ----------------------------------------------------------- status codes
enum {
  DS_OK = 0,
  DS_ECONFIG = -1,
  DS_EMODEL = -2,
  DS_ESOLVER = 1,
  DS_ECUDA = 2,
};

void ds_set_error(const std::string &msg);
int ds_fail(int code, const std::string &msg);

#define DS_CUDA(call)                                                      \
  do {                                                                     \
    cudaError_t _e = (call);                                               \
    if (_e != cudaSuccess)                                                 \
      return ds_fail(DS_ECUDA, std::string(#call) + ": " +                 \
                                   cudaGetErrorString(_e));                \
  } while (0)

#define DS_CHECK_LAUNCH()                                                  \
  do {                                                                     \
    cudaError_t _e = cudaGetLastError();                                   \
    if (_e != cudaSuccess)                                                 \
      return ds_fail(DS_ECUDA, std::string("kernel launch: ") +            \
                                   cudaGetErrorString(_e));                \
  } while (0)

// ---------------------------------------------- programmatic dependent launch
// Kernels on the sweep's critical path are launched with programmatic stream
// serialization: a kernel's CTAs may be scheduled while the previous
// kernel's last CTAs drain, read only static tables, and wait in
// griddepcontrol.wait until the previous grid has completed and flushed
// before touching data it produced.  The wait is a no-op without PDL.
// DS_PDL=0 disables it.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }

// programmatic dependent launch on/off: the "pdl" option of the last
// context that set it (launch_pdl has no context argument); default on
extern int g_ds_pdl;
inline bool ds_pdl_enabled() { return g_ds_pdl != 0; }

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = ds_pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, ((KArgs)args)...);
}

// ------------------------------------------------------------- handles
// Variant and tuning options of a context (ds_ctx_set_option).  Defaults are
// the measured-best choices; the environment variable named
// in each comment, read once when the context is created, overrides a
// default (A/B measurement tools).  Read at every launch, so tests switch
// variants in-process.
struct ds_options {
  int k1 = 4;          // DS_K1: stencil rows per thread (2, 4, 8, 16) or 0 = 32x8 shared tiles
  int combine = 2;     // DS_COMBINE: basis-update elements per thread (1 or 2)
  int k4 = 0;          // DS_K4: transfer kernel, 0 default (2D v3, 3D v2), 1 / 2 / 3 = v1 / v2 / v3
  int k4_rv = 1;       // DS_K4_RV: RHS columns per thread of transfer v1
  int k6_rv = 4;       // DS_K6_RV: RHS columns per thread of the assembly (1, 2, 4, 8)
  int pdl = 1;         // DS_PDL: programmatic dependent launch
  int k5_side = 1;     // DS_K5_SIDE: beta00 accumulation on a high-priority side stream
  int staged = 0;      // DS_SOLVE_MODE=staged: stage-per-launch block solve for small slabs too
  int k3g_mma = 1;     // DS_K3G_MMA: staged (3D) block product on DMMA
  int stage_rows = 0;  // DS_STAGE_ROWS: staged product rows per CTA (0 = auto)
  int k3_warps = 4;    // DS_K3_NW: warps per half of the cluster block solve (4 or 8)
  int k3_rc_min = 4;   // DS_K3_RCMIN / DS_K3_RCMAX: RHS chunk range of the cluster block solve
  int k3_rc_max = 16;
  int k3_cluster = 0;  // DS_K3_CLUSTER: force 8 or 16 CTAs per cluster (0 = choose)
  int hio_dstreams = 2;  // DS_HIO_DSTREAMS: download streams of the pinned-host path
  int kskip = 1;       // DS_KSKIP: forward transforms visit only the nonzero K-chunks (K6 masks)
  int r3_cols = 16;    // DS_R3_COLS: (mode, RHS) columns per block of the segmented recurrences (16 default, 32)
  int k2b_groups = 2;  // DS_K2B_GROUPS: concurrent groups of a blocked-factorization batch (1 .. 8)
  int count_work = 0;  // modal transforms add the complex multiply-adds they execute to ds_ctx::work
};
void ds_options_from_env(ds_options &o);

struct ds_ctx {
  int device;
  cudaStream_t stream;
  int num_sms;
  int64_t launches;  // kernel launches issued through this context
  ds_options opt;
  // scratch for reductions
  void *scratch = nullptr;
  size_t scratch_bytes = 0;
  // device counter of executed complex multiply-adds (option "count_work",
  // read by ds_ctx_work; measurement only)
  unsigned long long *work = nullptr;
};

// device-side operator view (coefficient arrays are device pointers)
struct OpDev {
  int dim;
  int shape[3];
  int kappa2_kind;
  int kappa2_axis;
  const cplx *c_lo[3];
  const cplx *c_hi[3];
  const double *kappa2;
};

struct ds_op {
  OpDev dev;
  void *storage;  // single allocation holding all coefficient arrays
  // host copies (used to assemble factor blocks)
  std::vector<cplx> h_clo[3], h_chi[3];
  std::vector<double> h_k2;
};

// per-operator factor layout
struct FactDev {
  int block_axis;
  int nb, m;
  int twist;          // middle block t: blocks k < t hold S_k^{-1} (top-down),
                      // k > t hold T_k^{-1} (bottom-up), k = t holds M_t^{-1}
  int other[2];       // the in-block axes in C order (unused entries = -1)
  int win_shape[3];
  const cplx *sinv;   // nb * m * m, row-major blocks (kind 0)
  const cplx *lcoef;  // nb: coupling of block k to k-1 (c_lo along axis)
  const cplx *ucoef;  // nb: coupling of block k to k+1 (c_hi along axis)
  // kind 1 (modal, separable operators): T_a = V_a diag(lambda_a) W_a for
  // the in-slab axes other[0..naxes) (W_a = V_a^{-1}, n_a x n_a row-major);
  // per (block k, mode j) the mode-wise tridiagonal LU along the block axis:
  // mmul[k][j] = l_k / piv_{k-1}(j) (k >= 1), minv[k][j] = 1 / piv_k(j)
  int kind;
  int naxes;
  int nax[2];
  const cplx *mW[2], *mV[2];
  const cplx *mmul, *minv;
};

struct ds_fact;
// device memory of slot `slot` of a factor pool (NULL if not a pool / bad slot)
const cplx *ds_fact_slot_mem(const ds_fact *F, int slot);

struct ds_fact {
  std::vector<FactDev> facts;
  std::vector<std::vector<cplx>> h_l, h_u;  // host copies of l_k, u_k per operator
  std::vector<void *> allocations;
  int64_t bytes_total = 0;
  std::vector<int64_t> bytes;
  // factor pool (ds_fact_create_pool, ABI 5): the operators' layouts without
  // resident factors; slot c holds the block inverses of operator
  // slot_owner[c] (-1: empty), facts[i].sinv points into its slot while
  // operator i is resident and is NULL otherwise
  bool pool = false;
  std::vector<cplx *> slot_mem;
  std::vector<int> slot_owner;
  std::vector<ds_op *> ops;
  size_t slot_bytes = 0;
  int64_t loads = 0;  // factorizations run by ds_fact_pool_load
};

// window-local linear (C-order) index <-> block layout offset
// perm offset of local coords c: (c[ba]*m + inblock(c)), inblock over the
// other axes in C order.
DS_HD int64_t block_offset(const FactDev &f, const int *c) {
  int64_t ib = 0;
  if (f.other[0] >= 0) ib = c[f.other[0]];
  if (f.other[1] >= 0) ib = ib * f.win_shape[f.other[1]] + c[f.other[1]];
  return (int64_t)c[f.block_axis] * f.m + ib;
}

// one (subdomain, step) solve of K3: rhs/x in block layout [nb][m][nrhs];
// nz: per-RHS nonzero flags (NULL = solve all); all-zero visits are skipped
struct SolveVisit {
  const FactDev *f;
  const cplx *rhs;
  cplx *x;
  const int *nz;
  cplx *xg;  // global exchange scratch: >= 4 * m * nrhs complex values
};

// launch K3 over a device table of visits (one cluster per visit x chunk)
int ds_launch_solve_table(ds_ctx *ctx, const void *visits_dev, int nvisit, int nrhs,
                          int max_m);

// modal solve (FactDev kind 1): per visit the in-slab transforms (batched
// complex GEMMs on DMMA) and the mode-wise tridiagonal solves; s0/s1 are
// scratch buffers of the visit's size (block layout, stride nrhs)
struct ModalJob {
  const FactDev *f;
  const cplx *rhs;
  cplx *x;
  cplx *s0, *s1;
  const int *nz;  // per-RHS nonzero flags (NULL = solve all)
  // nonzero K-chunks of the first forward pass's input (NULL = dense): one
  // word per input row (2D: block k; 3D: (k, i0)), bit c set when some node
  // with in-slab index 8c .. 8c+7 of that row is nonzero (written by K6)
  const uint32_t *km;
};
// launch the modal solve of njob visits (device job table; facts_host: the
// jobs' factor layouts, for grid sizing)
int ds_launch_modal(ds_ctx *ctx, const ModalJob *jobs_dev, const FactDev *facts_host, int njob,
                    int nrhs);
// one phase of it: 0 forward transforms, 1 recurrences, 2 inverse transforms
int ds_launch_modal_phase(ds_ctx *ctx, const ModalJob *jobs_dev, const FactDev *facts_host,
                          int njob, int nrhs, int phase);
void ds_fill_layout(const OpDev &o, FactDev &f);

int ceil_div(int a, int b);

// slabs above this size use the blocked factorization and the staged solve
#define DS_LARGE_SLAB 160

// K3g: staged solve (large slabs); host views of the visits and their
// factor layouts / block-axis couplings; items_dev: scratch of
// ds_stage_items_bytes(nvisit, max_nb) bytes
int ds_launch_solve_staged(ds_ctx *ctx, const SolveVisit *visits_host, const FactDev *facts_host,
                           const cplx *const *l_host, const cplx *const *u_host, int nvisit,
                           int nrhs, void *items_dev, size_t items_cap);
size_t ds_stage_items_bytes(int nvisit, int max_nb, int max_m, int nrhs);

// stage programs: all stage items of all steps of a plan, built once; one
// launch per stage (small slabs: fused PDL kernel; large: vin + GEMV)
struct StageProgram;
StageProgram *ds_stage_program_create(const std::vector<std::vector<SolveVisit>> &step_visits,
                                      const std::vector<std::vector<FactDev>> &step_facts,
                                      const std::vector<std::vector<const cplx *>> &step_l,
                                      const std::vector<std::vector<const cplx *>> &step_u,
                                      int nrhs_max, std::string *err);
int ds_stage_program_launch_step(ds_ctx *ctx, StageProgram *P, int step, int nrhs);
void ds_stage_program_destroy(StageProgram *P);
