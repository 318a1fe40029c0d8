// The diagonal-sweeping engine: static plan tables, the per-step kernels
// K6 (RHS assembly / restrict), K5 (beta00 accumulation), K4 (source
// transfer) and the host loop that issues, per anti-diagonal step,
//     assemble -> block solve (K3) -> accumulate -> transfer.
//
// Restates diagonal_sweep_solve (diagsweep/ddm.py:212-291):
//  * restrict_source (ddm.py:168-195): breakpoint nodes go to the lower
//    index, boundary subdomains own their collar (own window, host table);
//  * local RHS = own source (sweep 1) + queued payloads (ddm.py:242-254);
//    payloads live in per-(use sweep, target, direction) slots that the
//    consumer zeroes after reading;
//  * exact-zero flags and cut sets per (sweep, subdomain, RHS) evaluated on
//    the device: has_own = any(src != 0) (ddm.py:248), nonzero = any(rhs)
//    (ddm.py:256), solve_cuts = AND of arrival cuts unless has_own or no
//    arrivals (ddm.py:96-100), emits (ddm.py:103-110), content_cuts
//    (ddm.py:82-93) — cut bit (axis a, side s) = 1 << (2a + (s > 0));
//  * _accumulate (ddm.py:206-209) with a fixed owner order where supports
//    of same-step subdomains overlap (no atomics on field values);
//  * psi (transfer.py:100-155): payload = s * (rhs|band + L_nb((w - 1) v)|band)
//    with w = prod (1 - beta_a) on ext, evaluated node-wise with the
//    neighbour operator's couplings, zero outside ext.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <map>
#include <string>
#include <tuple>
#include <vector>

#include "ds_common.cuh"

#define RMAX 256
#define CUT_ALL 0x3f

struct SubDev {
  int win_lo[3], win_shape[3];
  int own_lo[3], own_shape[3];
  int sup_lo[3], sup_shape[3];
  const double *beta[3];
  const FactDev *f;
  const OpDev *op;
};

struct SlotRef {
  cplx *data;
  int lo[3], shape[3];
};

struct VisitDev {
  int sub, sweep, nslot, slot0;
  cplx *rhs, *x;
  int *nz;
  const int *arr;  // arrival counts of this visit [nrhs] (per-call stride)
  uint32_t *km;    // modal visits: nonzero K-chunk masks of the assembled rhs (ModalJob::km)
};

struct XferDev {
  int vidx;  // global visit index of the source visit
  int src, dst, use;
  int owner;  // rank owning dst (sharded plans; its slot and flags may be remote)
  int dirmask, content_base, keepmask;
  double sign;
  int band_lo[3], band_shape[3];
  int ext_lo[3], ext_shape[3];
  const double *fac[3];
  cplx *slot;
};

struct ds_plan {
  ds_ctx *ctx;
  int dim, nsub, nsweeps, nsteps, ndir, nrhs_max, gmax, max_m, max_w;
  int max_axis_sum = 0;  // max over windows of sum of extents (assemble masks)
  int gcounts[3];
  int64_t nnodes;
  std::vector<int> vstep_off, xstep_off;  // host copies, size nsweeps*nsteps+1
  // device tables
  SubDev *subs = nullptr;
  VisitDev *visits = nullptr;
  SolveVisit *solvetab = nullptr;
  SlotRef *slots = nullptr;
  XferDev *xfers = nullptr;
  FactDev *facts = nullptr;
  OpDev *ops = nullptr;
  // flags [nsweeps][nsub][nrhs] (stride = nrhs of the call)
  int *flags = nullptr;  // own_nz | nz | arr_cnt | arr_cut | emit_cnt | discard
  size_t flag_words = 0;
  std::vector<void *> allocs;
  int64_t workspace = 0;
  int64_t last_launches = 0;
  bool slots_dirty = false;
  std::vector<std::pair<cplx *, size_t>> slot_bufs;  // for re-zeroing
  // host copies of the visit tables; nz pointers are patched per nrhs stride
  std::vector<VisitDev> h_visits;
  std::vector<SolveVisit> h_solve;  // block-LU visits (compact, launch order)
  std::vector<int> blu_vidx, blu_off;  // visit index of each entry; per-launch offsets
  // modal visits (FactDev kind 1): job table, factor layouts, offsets
  ModalJob *mjobs = nullptr;
  std::vector<ModalJob> h_mjobs;
  std::vector<FactDev> h_mfacts;
  std::vector<int> mod_vidx, mod_off;
  // staged (large-slab) solve: host factor layouts and couplings per subdomain
  bool staged = false;
  std::vector<FactDev> h_facts;
  std::vector<const cplx *> h_l, h_u;
  void *stage_items = nullptr;
  size_t stage_cap = 0;
  StageProgram *program = nullptr;  // stage-per-launch solve (large slabs, or DS_SOLVE_MODE=staged)
  int patched_nrhs = 0;
  int nlaunch = 0;  // > 0: explicit launch schedule (visits of several sweeps per launch)
  // sharding: this plan is rank `rank` of `nranks`; subdomain s owned by owner[s]
  int nranks = 1, rank = 0;
  std::vector<int> owner;
  bool peers_set = false;
  std::vector<XferDev> h_xfers;
  // K4 v2 tables (rebuilt per nrhs stride in patch_tables)
  std::vector<SubDev> h_subs;
  std::vector<OpDev> h_ops;
  std::vector<int> h_op_of_sub;
  struct XferRec *recs = nullptr;
  int4 *tiles = nullptr;
  size_t tiles_cap = 0;
  std::vector<int> tile_off;  // per launch, size nq + 1
  std::vector<size_t> xfer_slot_off;  // element offset of each transfer's slot
  cplx *slot_base = nullptr;
  size_t slot_bytes = 0;
  std::map<std::tuple<int, int, int>, SlotRef> slot_by_key;  // (use-1, target, dir) -> slot (ds_plan_slot)
  int **d_flag_bases = nullptr;  // [nranks] flag words of every rank (device table)
  // K-chunk masks of the modal visits' rhs (K6 -> first forward transform),
  // zeroed with the flags at the start of every application
  uint32_t *kmask = nullptr;
  int64_t kmask_words = 0;
  int km_rows_max = 0;
  bool k5_pending[2] = {false, false};
  // graph
  bool use_graph = false;
  cudaGraphExec_t graph = nullptr;
  cudaStream_t gstream = nullptr;      // private stream for capture / replay
  cudaEvent_t gev_in = nullptr, gev_out = nullptr;
  // K5 (accumulate) runs on a side stream: nothing later in the application
  // reads u, so it leaves the critical path; ordering: K5 after its launch's
  // K3 (ev_k3), K5s serial among themselves (u summation order unchanged),
  // and the K3 that next overwrites a parity's solution buffers after the
  // K5 that read them (ev_k5[parity]); joined back at the end (ev_join)
  cudaStream_t side = nullptr;
  cudaEvent_t ev_k3 = nullptr, ev_k5[2] = {nullptr, nullptr}, ev_join = nullptr;
  const void *graph_f = nullptr;
  void *graph_u = nullptr;
  void *graph_partials = nullptr;
  int graph_nrhs = 0;
  bool graph_outer = false;
  // {f, u} of the current application, read by K6 / K5 / the zeroing: the
  // captured graphs replay for any field buffers (set by set_io before each
  // application, stream-ordered)
  cplx **d_io = nullptr;
  const void *io_f = nullptr;
  void *io_u = nullptr;
  // host-buffer application (ds_ddm_apply_host): node chunks along axis 0,
  // per launch the chunks of f its assembly needs, per chunk the launch of
  // the last accumulation touching it; device staging buffers; graph cache
  bool hio_ready = false;
  std::vector<struct HioBox> hio_boxes;   // upload boxes, in upload order
  std::vector<struct HioBox> hio_oboxes;  // download boxes
  std::vector<int> hio_need;             // per launch: chunks [0, need) resident
  std::vector<std::vector<int>> hio_out_at;  // per launch: chunks final after its K5
  std::vector<int> hio_out_early;        // chunks no K5 touches (zero rows)
  cplx *hio_fo = nullptr, *hio_fm = nullptr, *hio_uo = nullptr, *hio_um = nullptr;  // f/u staging: RHS-outer (copies), RHS-minor (sweep)
  cudaStream_t cstream = nullptr;
  cudaStream_t cstream2 = nullptr;  // second copy stream: boxes alternate between the two
  std::vector<cudaStream_t> cstream_x;  // further download streams (DS_HIO_DSTREAMS > 2)
  std::vector<cudaEvent_t> cjoin_x;
  cudaEvent_t hio_fork2 = nullptr, hio_join2 = nullptr;
  int side_priority = 0;  // K5 / copy stream priority
  std::vector<cudaEvent_t> hio_ev_in, hio_ev_out;
  cudaEvent_t hio_fork = nullptr, hio_join = nullptr;
  struct HGraph {
    const void *fh;
    void *uh;
    int nrhs;
    cudaGraphExec_t exec;
    int64_t launches;
  };
  std::vector<HGraph> hgraphs;
  // per-kernel-class timing (0 assemble, 1 solve, 2 accumulate, 3 transfer)
  bool profiling = false;
  std::vector<cudaEvent_t> ev;
  std::vector<int> ev_class;
  size_t ev_used = 0;
};

static int plan_alloc(ds_plan *P, void **ptr, size_t bytes) {
  if (bytes == 0) bytes = 16;
  if (cudaMalloc(ptr, bytes) != cudaSuccess)
    return ds_fail(DS_ECUDA, "ds_plan_create: out of device memory (" + std::to_string(bytes) +
                                 " bytes)");
  P->allocs.push_back(*ptr);
  P->workspace += bytes;
  return DS_OK;
}

// -------------------------------------------------------------- helpers
//
// All coordinate triples live in registers: every loop over the axes is
// unrolled with a compile-time index, and runtime axis numbers go through
// sel3 (a dynamically indexed local array would sit in local memory).
// Index arithmetic is 32-bit (a window or band has < 2^31 nodes); each thread
// owns one RHS column r of one node, so the node geometry is computed once
// per node and the nrhs lanes of a node read contiguous 16-byte values.

__device__ __forceinline__ int sel3(const int (&a)[3], int i) {
  return i == 0 ? a[0] : (i == 1 ? a[1] : a[2]);
}

__device__ __forceinline__ bool in_box(const int (&g)[3], const int *lo, const int *shape, int dim) {
  bool in = true;
#pragma unroll
  for (int a = 0; a < 3; ++a)
    if (a < dim) in = in && g[a] >= lo[a] && g[a] < lo[a] + shape[a];
  return in;
}

__device__ __forceinline__ int lin_of(const int (&e)[3], const int *shape, int dim) {
  int l = e[0];
#pragma unroll
  for (int a = 1; a < 3; ++a)
    if (a < dim) l = l * shape[a] + e[a];
  return l;
}

__device__ __forceinline__ int64_t lin_of64(const int (&e)[3], const int *shape, int dim) {
  int64_t l = e[0];
#pragma unroll
  for (int a = 1; a < 3; ++a)
    if (a < dim) l = l * shape[a] + e[a];
  return l;
}

__device__ __forceinline__ void unlin(int l, const int *shape, int dim, int (&e)[3]) {
  e[0] = e[1] = e[2] = 0;
  if (dim == 3) {
    e[2] = l % shape[2];
    l /= shape[2];
  }
  e[1] = l % shape[1];
  e[0] = l / shape[1];
}

// block layout offset -> window-local coordinates
__device__ __forceinline__ void block_coords(const FactDev &f, int blk, int (&c)[3]) {
  const int k = blk / f.m, i = blk % f.m;
  int j0 = i, j1 = 0;
  if (f.other[1] >= 0) {
    const int n1 = sel3(f.win_shape, f.other[1]);
    j0 = i / n1;
    j1 = i % n1;
  }
#pragma unroll
  for (int a = 0; a < 3; ++a)
    c[a] = a == f.block_axis ? k : (a == f.other[0] ? j0 : (a == f.other[1] ? j1 : 0));
}

// window-local coordinates -> block layout offset (registers only)
__device__ __forceinline__ int block_off(const FactDev &f, const int (&c)[3]) {
  int ib = f.other[0] >= 0 ? sel3(c, f.other[0]) : 0;
  if (f.other[1] >= 0) ib = ib * sel3(f.win_shape, f.other[1]) + sel3(c, f.other[1]);
  return sel3(c, f.block_axis) * f.m + ib;
}

// flags layout helpers (stride nrhs)
struct Flags {
  int *own_nz;    // [nsub][R]
  int *nz;        // [nsweeps][nsub][R]
  int *arr_cnt;   // [nsweeps][nsub][R]
  int *arr_cut;   // [nsweeps][nsub][R]
  int *emit_cnt;  // [nsweeps][nsub][R]
  int *discard;   // [R]
};

static Flags flags_view(ds_plan *P, int nrhs) {
  Flags F;
  size_t per = (size_t)P->nsweeps * P->nsub * nrhs;
  F.own_nz = P->flags;
  F.nz = F.own_nz + (size_t)P->nsub * nrhs;
  F.arr_cnt = F.nz + per;
  F.arr_cut = F.arr_cnt + per;
  F.emit_cnt = F.arr_cut + per;
  F.discard = F.emit_cnt + per;
  return F;
}

__device__ __forceinline__ int solve_cut(const Flags &F, int sweep, int sub, int nsub, int r,
                                         int nrhs) {
  size_t vi = ((size_t)(sweep - 1) * nsub + sub) * nrhs + r;
  if (sweep == 1 && F.own_nz[(size_t)sub * nrhs + r]) return 0;
  if (F.arr_cnt[vi] == 0) return 0;
  return F.arr_cut[vi] & CUT_ALL;
}

// arrival words (counts, cut masks) of a rank's flag block for stride nrhs
// (the layout of flags_view)
__device__ __forceinline__ void arrival_words(int *base, int nsweeps, int nsub, int nrhs,
                                              int *&arr_cnt, int *&arr_cut) {
  const size_t per = (size_t)nsweeps * nsub * nrhs;
  arr_cnt = base + (size_t)nsub * nrhs + per;
  arr_cut = arr_cnt + per;
}

#define SLOT_SMEM 32
// band nodes per thread and tile pass of k_transfer2, and its resident blocks per SM
#ifndef K4_NPT3
#define K4_NPT3 1
#endif
#define K4_NPT(dim) ((dim) == 2 ? 2 : K4_NPT3)
#define K4_MINB(dim) ((dim) == 2 ? 2 : K4_MINB3)
#ifndef K4_MINB3
#define K4_MINB3 2
#endif


// Thread mapping of K4/K5/K6: a thread owns RV RHS columns of one node --
// lane l of the node's LPN = nrhs / RV lanes takes columns l, l + LPN, ... --
// so the node's geometry (block coordinates, slot masks, stencil neighbours,
// beta) is computed once per RV values while every load instruction of the
// node's lanes still covers LPN consecutive 16-byte values (K4, K5); the
// store-dominated K6 instead gives each lane RV consecutive columns.  ncu on the 8-visit step of config 2
// showed the one-RHS-per-thread version instruction-bound (~140 instructions
// per value, IPC 0.6).

// u = 0 through the pointer table (graphs replay for any f / u buffers), and
// the application's flag words: 0, except the cut masks [cut0, cut1) which
// start all-ones (0x3f3f3f3f, the byte pattern of the former memsets) --
// one kernel instead of a kernel and three memset nodes (measured: a memset
// node at the head of the host-path graph cost ~0.3 ms end to end)
__global__ void k_zero_io(cplx *const *__restrict__ io, int64_t n, int *flags, int64_t nflags,
                          int64_t cut0, int64_t cut1, uint32_t *km, int64_t nkm) {
  cplx *u = io[1];
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride)
    u[i] = make_double2(0.0, 0.0);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nflags; i += stride)
    flags[i] = (i >= cut0 && i < cut1) ? 0x3f3f3f3f : 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nkm; i += stride) km[i] = 0u;
}

// ------------------------------------------------------------- K6 assemble
// rhs (block layout [nb][m][R]) = own restricted source (sweep 1) + the
// visit's queued payload slots in slot order; slots are zeroed as consumed.
// Slot membership is separable (boxes), so each block first builds, per
// window axis and coordinate, the bitmask of slots (bit 31: the own box)
// covering it; a node's slot set is then the AND of its axis masks.
template <int RV, bool OUTER>
__global__ void __launch_bounds__(256)
    k_assemble(const VisitDev *__restrict__ visits, const SubDev *__restrict__ subs,
               const SlotRef *__restrict__ slots, const cplx *__restrict__ f, int nrhs,
               int dim, int g0, int g1, int g2, Flags F, int64_t nnodes) {
  __shared__ int s_nz[RMAX], s_own[RMAX], s_live[RMAX];
  __shared__ SlotRef s_slot[SLOT_SMEM];
  extern __shared__ uint32_t s_mask[];  // [E0 | E1 | E2]
  const VisitDev V = visits[blockIdx.y];
  const SubDev &sd = subs[V.sub];
  const FactDev fd = *sd.f;
  const int t = threadIdx.x;
  // static part first (slot table, axis masks): under programmatic
  // dependent launch it overlaps the previous kernel's tail
  for (int r = t; r < nrhs; r += blockDim.x) s_nz[r] = s_own[r] = 0;
  const int ns = V.nslot;
  for (int k = t; k < min(ns, SLOT_SMEM); k += blockDim.x) s_slot[k] = slots[V.slot0 + k];
  const bool own = V.sweep == 1;
  const bool masks = ns <= 31;
  const int E0 = sd.win_shape[0], E1 = sd.win_shape[1], E2 = dim == 3 ? sd.win_shape[2] : 0;
  // modal visits: per input row of the first forward transform, the 8-wide
  // K-chunks holding a nonzero rhs value (ModalJob::km), OR-ed in shared memory
  uint32_t *s_km = s_mask + (E0 + E1 + E2);
  const int km_nl = V.km ? (fd.naxes == 2 ? fd.nax[1] : fd.m) : 0;
  const int km_rows = V.km ? fd.nb * (fd.m / km_nl) : 0;
  for (int x = t; x < km_rows; x += blockDim.x) s_km[x] = 0u;
  __syncthreads();
  if (masks) {
    for (int x = t; x < E0 + E1 + E2; x += blockDim.x) {
      const int a = x < E0 ? 0 : (x < E0 + E1 ? 1 : 2);
      const int gx = sd.win_lo[a] + x - (a == 0 ? 0 : (a == 1 ? E0 : E0 + E1));
      uint32_t mk = 0;
      for (int k = 0; k < ns; ++k)
        if (gx >= s_slot[k].lo[a] && gx < s_slot[k].lo[a] + s_slot[k].shape[a]) mk |= 1u << k;
      if (own && gx >= sd.own_lo[a] && gx < sd.own_lo[a] + sd.own_shape[a]) mk |= 1u << 31;
      s_mask[x] = mk;
    }
  }
  pdl_wait();
  // RHS columns that can be nonzero: an own source (sweep 1) or an arrival
  // (K4's counts).  The others are exactly zero: their rhs entries are not
  // written -- nothing reads them (the solves skip exact-zero columns, the
  // transfer only reads emitting ones)
  for (int r = t; r < nrhs; r += blockDim.x) s_live[r] = V.sweep == 1 || V.arr[r] > 0;
  __syncthreads();
  const int gc[3] = {g0, g1, g2};
  const int lpn = nrhs / RV;
  const int npb = blockDim.x / lpn, rl = (t % lpn) * RV, ln = t / lpn;  // consecutive columns (stores)
  const int nodes = fd.nb * fd.m;
  int wlo[3], olo[3], osh[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    wlo[a] = sd.win_lo[a];
    olo[a] = sd.own_lo[a];
    osh[a] = sd.own_shape[a];
  }
  bool any[RV] = {}, anyown[RV] = {};
  // warp-uniform trip count (the K-chunk mask aggregation below is a
  // full-warp collective); lanes past their own trips run it idle
  const int first = blockIdx.x * npb + ln, nstride = gridDim.x * npb;
  const int trips = (ln < npb && first < nodes) ? (nodes - first + nstride - 1) / nstride : 0;
  const int wtrips = __reduce_max_sync(0xffffffffu, trips);
  for (int it = 0; it < wtrips; ++it) {
    const int blk = first + it * nstride;
    int km_row = -1;
    uint32_t km_bit = 0u;
    if (it < trips) {
      int c[3], g[3];
      block_coords(fd, blk, c);
#pragma unroll
      for (int a = 0; a < 3; ++a) g[a] = wlo[a] + c[a];
      cplx val[RV];
#pragma unroll
      for (int j = 0; j < RV; ++j) val[j] = make_double2(0.0, 0.0);
      uint32_t mk;
      if (masks) {
        mk = s_mask[c[0]] & s_mask[E0 + c[1]];
        if (dim == 3) mk &= s_mask[E0 + E1 + c[2]];
      } else {
        mk = (own && in_box(g, olo, osh, dim)) ? 1u << 31 : 0u;
      }
      if (mk >> 31) {
        // f element (node, rhs): RHS-minor node * nrhs + rhs, RHS-outer rhs * N + node
        const int64_t lin = lin_of64(g, gc, dim);
        const cplx *src = OUTER ? f + rl * nnodes + lin : f + lin * nrhs + rl;
#pragma unroll
        for (int j = 0; j < RV; ++j) {
          const cplx sv = OUTER ? src[j * nnodes] : src[j];
          val[j] = cadd(val[j], sv);
          anyown[j] |= cnonzero(sv);
        }
      }
      if (masks) {
        mk &= 0x7fffffffu;
        while (mk) {
          const int k = __ffs(mk) - 1;
          mk &= mk - 1;
          const SlotRef &S = s_slot[k];
          int e[3];
#pragma unroll
          for (int a = 0; a < 3; ++a) e[a] = g[a] - S.lo[a];
          cplx *sp = S.data + (int64_t)lin_of(e, S.shape, dim) * nrhs + rl;
#pragma unroll
          for (int j = 0; j < RV; ++j) {
            val[j] = cadd(val[j], sp[j]);
            sp[j] = make_double2(0.0, 0.0);
          }
        }
      } else {
        for (int k = 0; k < ns; ++k) {
          const SlotRef &S = k < SLOT_SMEM ? s_slot[k] : slots[V.slot0 + k];
          if (!in_box(g, S.lo, S.shape, dim)) continue;
          int e[3];
#pragma unroll
          for (int a = 0; a < 3; ++a) e[a] = g[a] - S.lo[a];
          cplx *sp = S.data + (int64_t)lin_of(e, S.shape, dim) * nrhs + rl;
#pragma unroll
          for (int j = 0; j < RV; ++j) {
            val[j] = cadd(val[j], sp[j]);
            sp[j] = make_double2(0.0, 0.0);
          }
        }
      }
      cplx *dst = V.rhs + (int64_t)blk * nrhs + rl;
      bool nzn = false;
#pragma unroll
      for (int j = 0; j < RV; ++j) {
        if (s_live[rl + j]) dst[j] = val[j];
        const bool nzv = cnonzero(val[j]);
        any[j] |= nzv;
        nzn |= nzv;
      }
      if (km_nl && nzn) {
        // input row of the first forward pass and the node's K index: 2D
        // (row k, i); 3D (row (k, i0), i1)
        int kidx = sel3(c, fd.other[0]);
        km_row = sel3(c, fd.block_axis);
        if (fd.other[1] >= 0) {
          km_row = km_row * sel3(fd.win_shape, fd.other[0]) + kidx;
          kidx = sel3(c, fd.other[1]);
        }
        km_bit = 1u << (kidx >> 3);
      }
    }
    if (km_nl) {  // one shared atomic per distinct row of the warp (consecutive nodes: 1-2 rows)
      unsigned todo = __ballot_sync(0xffffffffu, km_bit != 0u);
      while (todo) {
        const int r0 = __shfl_sync(0xffffffffu, km_row, __ffs(todo) - 1);
        const uint32_t b = __reduce_or_sync(0xffffffffu, km_row == r0 ? km_bit : 0u);
        if ((int)(threadIdx.x & 31) == __ffs(todo) - 1 && (s_km[r0] & b) != b) atomicOr(&s_km[r0], b);
        todo &= ~__ballot_sync(0xffffffffu, km_row == r0);
      }
    }
  }
#pragma unroll
  for (int j = 0; j < RV; ++j) {
    if (any[j]) s_nz[rl + j] = 1;
    if (anyown[j]) s_own[rl + j] = 1;
  }
  __syncthreads();
  for (int q = t; q < nrhs; q += blockDim.x) {
    if (s_nz[q]) atomicOr(&V.nz[q], 1);
    if (s_own[q]) atomicOr(&F.own_nz[(size_t)V.sub * nrhs + q], 1);
  }
  for (int x = t; x < km_rows; x += blockDim.x)
    if (s_km[x]) atomicOr(&V.km[x], s_km[x]);
}

// ----------------------------------------------------------- K5 accumulate
// u += beta00 * x over the visit's support; where supports of same-step
// visits overlap the first visit owning the node sums all of them in visit
// order (deterministic, no atomics on field values).
template <int RV, bool OUTER>
__global__ void __launch_bounds__(256)
    k_accumulate(const VisitDev *__restrict__ visits, int G, const SubDev *__restrict__ subs,
                 cplx *const *__restrict__ io, int nrhs, int dim, int g0, int g1, int g2,
                 int64_t nnodes) {
  cplx *u = io[1];  // result field of this application (ds_plan::d_io)
  const int v = blockIdx.y;
  const SubDev &sd = subs[visits[v].sub];
  const int gc[3] = {g0, g1, g2};
  const int t = threadIdx.x;
  const int lpn = nrhs / RV;
  const int npb = blockDim.x / lpn, rl = t % lpn, ln = t / lpn;
  if (ln >= npb) return;
  const int nodes = sd.sup_shape[0] * sd.sup_shape[1] * (dim == 3 ? sd.sup_shape[2] : 1);
  for (int node = blockIdx.x * npb + ln; node < nodes; node += gridDim.x * npb) {
    int e[3], g[3];
    unlin(node, sd.sup_shape, dim, e);
#pragma unroll
    for (int a = 0; a < 3; ++a) g[a] = a < dim ? sd.sup_lo[a] + e[a] : 0;
    bool owner = true;
    for (int w = 0; w < v && owner; ++w) {
      const SubDev &so = subs[visits[w].sub];
      if (in_box(g, so.sup_lo, so.sup_shape, dim)) owner = false;
    }
    if (!owner) continue;
    const int64_t lin = lin_of64(g, gc, dim);
    cplx *up = OUTER ? u + rl * nnodes + lin : u + lin * nrhs + rl;  // RHS-outer / -minor
    const int64_t cstride = OUTER ? (int64_t)lpn * nnodes : lpn;  // column j * lpn
    cplx acc[RV];
#pragma unroll
    for (int j = 0; j < RV; ++j) acc[j] = up[j * cstride];
    bool touched = false;
    for (int w = v; w < G; ++w) {
      const VisitDev &W = visits[w];
      const SubDev &sw = subs[W.sub];
      if (w != v && !in_box(g, sw.sup_lo, sw.sup_shape, dim)) continue;
      double beta = 1.0;
      int c[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        if (a < dim) beta = beta * sw.beta[a][g[a] - sw.sup_lo[a]];
        c[a] = a < dim ? g[a] - sw.win_lo[a] : 0;
      }
      const cplx *xp = W.x + (int64_t)block_off(*sw.f, c) * nrhs + rl;
#pragma unroll
      for (int j = 0; j < RV; ++j) {
        if (!W.nz[rl + j * lpn]) continue;
        acc[j] = cadd(acc[j], cscale(xp[j * lpn], beta));
        touched = true;
      }
    }
    if (touched) {
#pragma unroll
      for (int j = 0; j < RV; ++j) up[j * cstride] = acc[j];
    }
  }
}

// ------------------------------------------------------------ K4 transfer
__device__ __forceinline__ double op_k2(const OpDev &o, const int (&c)[3]) {
  if (o.kappa2_kind == 0) return o.kappa2[0];
  if (o.kappa2_kind == 1) return o.kappa2[sel3(c, o.kappa2_axis)];
  int lin = c[0];
#pragma unroll
  for (int a = 1; a < 3; ++a)
    if (a < o.dim) lin = lin * o.shape[a] + c[a];
  return o.kappa2[lin];
}

// psi (transfer.py:100-155): payload = s * (rhs|band + L_nb((w - 1) v)|band),
// w = prod_a fac_a on ext; block 0 also does the arrival/emission bookkeeping
// (ddm.py:262-279), one thread per RHS.  RHS columns that do not emit
// (zero visit, or cut towards this direction) contribute nothing.
template <int RV, int DIM>
__global__ void __launch_bounds__(256)
    k_transfer(const XferDev *__restrict__ xfers, const VisitDev *__restrict__ visits,
               const SubDev *__restrict__ subs, int nsub, int nrhs, int dim_unused, Flags F,
               int *const *__restrict__ flag_bases, int nsweeps) {
  constexpr int dim = DIM, NP = 1 + 2 * DIM;  // stencil points
  const XferDev &X = xfers[blockIdx.y];
  const VisitDev &V = visits[X.vidx];
  const int sweep = V.sweep;  // a launch may hold visits of several sweeps
  if (blockIdx.x == 0) {
    // arrivals go to the flags of the rank owning the target (sharded plans:
    // a peer's memory over NVLink; otherwise this plan's own flags)
    int *arr_cnt = F.arr_cnt, *arr_cut = F.arr_cut;
    if (flag_bases) arrival_words(flag_bases[X.owner], nsweeps, nsub, nrhs, arr_cnt, arr_cut);
    for (int r = threadIdx.x; r < nrhs; r += blockDim.x) {
      if (!V.nz[r]) continue;
      int cut = solve_cut(F, sweep, X.src, nsub, r, nrhs);
      if (cut & X.dirmask) continue;
      if (X.use == 0) {
        atomicAdd(&F.discard[r], 1);
      } else {
        size_t ti = ((size_t)(X.use - 1) * nsub + X.dst) * nrhs + r;
        atomicAdd_system(&arr_cnt[ti], 1);
        atomicAnd_system(&arr_cut[ti], X.content_base | (cut & X.keepmask));
        atomicAdd(&F.emit_cnt[((size_t)(sweep - 1) * nsub + X.src) * nrhs + r], 1);
      }
    }
  }
  if (X.use == 0) return;
  const int t = threadIdx.x;
  const int lpn = nrhs / RV;
  const int npb = blockDim.x / lpn, rl = t % lpn, ln = t / lpn;
  if (ln >= npb) return;
  bool emit[RV];
  bool anyemit = false;
#pragma unroll
  for (int j = 0; j < RV; ++j) {
    emit[j] = V.nz[rl + j * lpn] && !(solve_cut(F, sweep, X.src, nsub, rl + j * lpn, nrhs) & X.dirmask);
    anyemit |= emit[j];
  }
  if (!anyemit) return;
  const SubDev &ss = subs[X.src];
  const SubDev &sn = subs[X.dst];
  const FactDev fs = *ss.f;
  const OpDev &on = *sn.op;
  int blo[3], elo[3], ehi[3], swlo[3], snlo[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    blo[a] = X.band_lo[a];
    elo[a] = X.ext_lo[a];
    ehi[a] = X.ext_lo[a] + X.ext_shape[a];
    swlo[a] = ss.win_lo[a];
    snlo[a] = sn.win_lo[a];
  }
  const int nodes = X.band_shape[0] * X.band_shape[1] * (dim == 3 ? X.band_shape[2] : 1);
  // (w(p) - 1) and the V.x column pointer of stencil point p (w = prod_a
  // fac_a(p_a) on ext)
  auto point = [&](const int (&p)[3], double &wm1, const cplx *&vp) {
    double wt = 1.0;
    int c[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      if (a < dim) wt = wt * X.fac[a][p[a] - elo[a]];
      c[a] = a < dim ? p[a] - swlo[a] : 0;
    }
    wm1 = wt - 1.0;
    vp = V.x + (int64_t)block_off(fs, c) * nrhs + rl;
  };
  for (int node = blockIdx.x * npb + ln; node < nodes; node += gridDim.x * npb) {
    int e[3], g[3], cn[3];
    unlin(node, X.band_shape, dim, e);
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      g[a] = a < dim ? blo[a] + e[a] : 0;
      cn[a] = a < dim ? g[a] - snlo[a] : 0;
    }
    // phase 1: every load of the node is issued before any arithmetic (the
    // gathers of the 2*dim+1 stencil points, couplings, rhs and slot);
    // neighbours outside ext load the centre and are skipped in phase 2
    double wm[NP];
    const cplx *vp[NP];
    bool ok[NP];
    point(g, wm[0], vp[0]);
    ok[0] = true;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      if (a >= dim) break;
      int pm[3] = {g[0], g[1], g[2]}, pp[3] = {g[0], g[1], g[2]};
      pm[a] -= 1;
      pp[a] += 1;
      ok[1 + 2 * a] = g[a] - 1 >= elo[a];
      ok[2 + 2 * a] = g[a] + 1 < ehi[a];
      if (ok[1 + 2 * a]) point(pm, wm[1 + 2 * a], vp[1 + 2 * a]);
      else { wm[1 + 2 * a] = 0.0; vp[1 + 2 * a] = vp[0]; }
      if (ok[2 + 2 * a]) point(pp, wm[2 + 2 * a], vp[2 + 2 * a]);
      else { wm[2 + 2 * a] = 0.0; vp[2 + 2 * a] = vp[0]; }
    }
    cplx v[NP][RV];
#pragma unroll
    for (int q = 0; q < NP; ++q) {
#pragma unroll
      for (int j = 0; j < RV; ++j) v[q][j] = vp[q][j * lpn];
    }
    cplx lo[3], hi[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      if (a >= dim) break;
      lo[a] = on.c_lo[a][cn[a]];
      hi[a] = on.c_hi[a][cn[a]];
    }
    const double k2 = op_k2(on, cn);
    int cs[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) cs[a] = a < dim ? g[a] - swlo[a] : 0;
    const cplx *rv = V.rhs + (int64_t)block_off(fs, cs) * nrhs + rl;
    cplx *sp = X.slot + (int64_t)node * nrhs + rl;
    cplx rvv[RV], spv[RV];
#pragma unroll
    for (int j = 0; j < RV; ++j) {
      rvv[j] = rv[j * lpn];
      spv[j] = sp[j * lpn];
    }
    // phase 2: the centre term k2*w0, then per axis -(lo+hi)*w0, lo*w(p-e_a),
    // hi*w(p+e_a) -- the same order as before the load hoisting
    cplx w0[RV], acc[RV];
#pragma unroll
    for (int j = 0; j < RV; ++j) {
      w0[j] = cscale(v[0][j], wm[0]);
      acc[j] = cscale(w0[j], k2);
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      if (a >= dim) break;
      const cplx mlh = make_double2(-(lo[a].x + hi[a].x), -(lo[a].y + hi[a].y));
#pragma unroll
      for (int j = 0; j < RV; ++j) acc[j] = cadd(acc[j], cmul(mlh, w0[j]));
      if (ok[1 + 2 * a]) {
#pragma unroll
        for (int j = 0; j < RV; ++j) acc[j] = cadd(acc[j], cmul(lo[a], cscale(v[1 + 2 * a][j], wm[1 + 2 * a])));
      }
      if (ok[2 + 2 * a]) {
#pragma unroll
        for (int j = 0; j < RV; ++j) acc[j] = cadd(acc[j], cmul(hi[a], cscale(v[2 + 2 * a][j], wm[2 + 2 * a])));
      }
    }
#pragma unroll
    for (int j = 0; j < RV; ++j)
      if (emit[j]) sp[j * lpn] = cadd(spv[j], cscale(cadd(rvv[j], acc[j]), X.sign));
  }
  if (flag_bases) __threadfence_system();  // sharded: peer-memory payloads before the barrier
}

// ------------------------------------------------------- K4 v2 (default)
// The same psi as k_transfer, restructured for latency (ncu on config 2:
// k_transfer was long-scoreboard bound, <1 node iteration per warp behind a
// 6-deep chain of dependent table loads, 95 registers, 3.9 waves):
//  * every transfer's geometry is flattened on the host into an XferRec of
//    pre-offset pointers and affine strides (block-layout offset of band
//    node e is sum_a str[a] e[a]; fac / couplings / kappa2 indexed by e) --
//    one level of table loads, staged through shared memory per tile;
//  * the launch's band nodes are cut into tiles of NPT x (256 / nrhs) nodes
//    (host list, discards have none), one tile per block pass, all loads
//    of the NPT nodes of a thread issued before the arithmetic;
//  * arrival / emission bookkeeping is spread over the first threads of
//    the grid (one thread per (transfer, RHS)).
// Summation order per value is that of k_transfer (bitwise equal results).
struct XferRec {
  const cplx *x, *rhs;  // source visit solution / rhs at the band origin
  cplx *slot;           // payload slot (band C-order, stride nrhs)
  const int *nz;        // source visit nonzero flags (per-call stride)
  const double *fac[3];           // (1 - beta) factors at band coordinate e
  const cplx *clo[3], *chi[3];    // neighbour couplings at band coordinate e
  const double *k2;               // neighbour kappa^2 at e = 0
  int str[3];    // block-layout stride (nodes) of band axis a
  int k2str[3];  // kappa^2 index stride per axis
  int shape[3];  // band shape
  int elo[3], ehi[3];  // ext bounds relative to the band origin
  int nodes, src, sweep, dirmask;
  double sign;
};
static_assert(sizeof(XferRec) % 8 == 0, "XferRec is copied as 8-byte words");

template <int DIM, int NPT>
__global__ void __launch_bounds__(256, K4_MINB(DIM))
    k_transfer2(const XferDev *__restrict__ xfers, const XferRec *__restrict__ recs,
                const int4 *__restrict__ tiles, int ntiles, int nx, int nsub, int nrhs, Flags F,
                int *const *__restrict__ flag_bases, int nsweeps) {
  constexpr int NP = 1 + 2 * DIM;
  __shared__ XferRec R;
  const int t = threadIdx.x;
  pdl_wait();
  // bookkeeping (ddm.py:262-279): one thread per (transfer, RHS) of the launch
  for (int gt = blockIdx.x * blockDim.x + t; gt < nx * nrhs; gt += gridDim.x * blockDim.x) {
    const int i = gt / nrhs, r = gt % nrhs;
    const XferRec &Q = recs[i];
    if (!Q.nz[r]) continue;
    const int cut = solve_cut(F, Q.sweep, Q.src, nsub, r, nrhs);
    const XferDev &X = xfers[i];
    if (cut & X.dirmask) continue;
    if (X.use == 0) {
      atomicAdd(&F.discard[r], 1);
    } else {
      int *arr_cnt = F.arr_cnt, *arr_cut = F.arr_cut;
      if (flag_bases) arrival_words(flag_bases[X.owner], nsweeps, nsub, nrhs, arr_cnt, arr_cut);
      const size_t ti = ((size_t)(X.use - 1) * nsub + X.dst) * nrhs + r;
      atomicAdd_system(&arr_cnt[ti], 1);
      atomicAnd_system(&arr_cut[ti], X.content_base | (cut & X.keepmask));
      atomicAdd(&F.emit_cnt[((size_t)(Q.sweep - 1) * nsub + X.src) * nrhs + r], 1);
    }
  }
  const int npb = blockDim.x / nrhs, r = t % nrhs, ln = t / nrhs;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int4 T = tiles[tile];  // (transfer, first node, end node)
    __syncthreads();
    if (t < (int)(sizeof(XferRec) / 8))
      reinterpret_cast<long long *>(&R)[t] = reinterpret_cast<const long long *>(recs + T.x)[t];
    __syncthreads();
    if (ln >= npb) continue;
    const bool emit = R.nz[r] && !(solve_cut(F, R.sweep, R.src, nsub, r, nrhs) & R.dirmask);
    if (!emit) continue;
    const int nodes = T.z;
    for (int n0 = T.y; n0 < nodes; n0 += NPT * npb) {
    // phase 1: all loads of the thread's NPT nodes
    cplx v[NPT][NP], rvv[NPT], spv[NPT], lo[NPT][DIM], hi[NPT][DIM];
    double wm[NPT][NP], k2[NPT];
    bool ok[NPT][NP], live[NPT];
    int node_of[NPT];
#pragma unroll
    for (int k = 0; k < NPT; ++k) {
      const int node = n0 + k * npb + ln;
      node_of[k] = node;
      live[k] = node < nodes;
      const int nd = live[k] ? node : n0;  // dead lanes reload a live node
      int e[3];
      if (DIM == 3) {
        e[2] = nd % R.shape[2];
        const int q = nd / R.shape[2];
        e[1] = q % R.shape[1];
        e[0] = q / R.shape[1];
      } else {
        e[1] = nd % R.shape[1];
        e[0] = nd / R.shape[1];
        e[2] = 0;
      }
      int off = 0, k2i = 0;
#pragma unroll
      for (int a = 0; a < DIM; ++a) {
        off += R.str[a] * e[a];
        k2i += R.k2str[a] * e[a];
      }
      double f0[DIM], fm[DIM], fp[DIM];
#pragma unroll
      for (int a = 0; a < DIM; ++a) {
        f0[a] = R.fac[a][e[a]];
        ok[k][1 + 2 * a] = e[a] - 1 >= R.elo[a];
        ok[k][2 + 2 * a] = e[a] + 1 < R.ehi[a];
        fm[a] = ok[k][1 + 2 * a] ? R.fac[a][e[a] - 1] : 0.0;
        fp[a] = ok[k][2 + 2 * a] ? R.fac[a][e[a] + 1] : 0.0;
        lo[k][a] = R.clo[a][e[a]];
        hi[k][a] = R.chi[a][e[a]];
      }
      ok[k][0] = true;
      v[k][0] = R.x[(int64_t)off * nrhs + r];
#pragma unroll
      for (int a = 0; a < DIM; ++a) {
        v[k][1 + 2 * a] = ok[k][1 + 2 * a] ? R.x[(int64_t)(off - R.str[a]) * nrhs + r] : v[k][0];
        v[k][2 + 2 * a] = ok[k][2 + 2 * a] ? R.x[(int64_t)(off + R.str[a]) * nrhs + r] : v[k][0];
      }
      rvv[k] = R.rhs[(int64_t)off * nrhs + r];
      spv[k] = R.slot[(int64_t)nd * nrhs + r];
      k2[k] = R.k2[k2i];
      // w(p) - 1 with w = prod_a fac_a in axis order (k_transfer's point())
#pragma unroll
      for (int q = 0; q < NP; ++q) {
        double wt = 1.0;
#pragma unroll
        for (int a = 0; a < DIM; ++a) {
          double fa = f0[a];
          if (q == 1 + 2 * a) fa = fm[a];
          if (q == 2 + 2 * a) fa = fp[a];
          wt = wt * fa;
        }
        wm[k][q] = (q == 0 || ok[k][q]) ? wt - 1.0 : 0.0;
      }
    }
    // phase 2: centre k2*w0, then per axis -(lo+hi)*w0, lo*w(p-e_a), hi*w(p+e_a)
#pragma unroll
    for (int k = 0; k < NPT; ++k) {
      const cplx w0 = cscale(v[k][0], wm[k][0]);
      cplx acc = cscale(w0, k2[k]);
#pragma unroll
      for (int a = 0; a < DIM; ++a) {
        const cplx mlh = make_double2(-(lo[k][a].x + hi[k][a].x), -(lo[k][a].y + hi[k][a].y));
        acc = cadd(acc, cmul(mlh, w0));
        if (ok[k][1 + 2 * a]) acc = cadd(acc, cmul(lo[k][a], cscale(v[k][1 + 2 * a], wm[k][1 + 2 * a])));
        if (ok[k][2 + 2 * a]) acc = cadd(acc, cmul(hi[k][a], cscale(v[k][2 + 2 * a], wm[k][2 + 2 * a])));
      }
      if (live[k])
        R.slot[(int64_t)node_of[k] * nrhs + r] = cadd(spv[k], cscale(cadd(rvv[k], acc), R.sign));
    }
    }
  }
  if (flag_bases) __threadfence_system();  // sharded: peer-memory payloads before the barrier
}

// K4 v3 (2D default): k_transfer2 with RV RHS columns per thread (lanes of a
// node take columns l, l + LPN, ...; every load instruction of a node's
// lanes still covers LPN consecutive 16-byte values) and the stencil
// accumulated point by point in psi's order, so the node geometry, the
// (1 - beta) factors and the couplings are computed once per RV columns and
// only one point's RV values are live at a time (k_transfer2 kept all seven
// points x NPT nodes in registers: 112 registers, 18% occupancy, 20% of
// HBM on config 4).
#ifndef K4V3_MINB
#define K4V3_MINB 2
#endif
template <int DIM, int RV>
__global__ void __launch_bounds__(256, K4V3_MINB)
    k_transfer3(const XferDev *__restrict__ xfers, const XferRec *__restrict__ recs,
                const int4 *__restrict__ tiles, int ntiles, int nx, int nsub, int nrhs, Flags F,
                int *const *__restrict__ flag_bases, int nsweeps) {
  __shared__ XferRec R;
  const int t = threadIdx.x;
  pdl_wait();
  for (int gt = blockIdx.x * blockDim.x + t; gt < nx * nrhs; gt += gridDim.x * blockDim.x) {
    const int i = gt / nrhs, r = gt % nrhs;
    const XferRec &Q = recs[i];
    if (!Q.nz[r]) continue;
    const int cut = solve_cut(F, Q.sweep, Q.src, nsub, r, nrhs);
    const XferDev &X = xfers[i];
    if (cut & X.dirmask) continue;
    if (X.use == 0) {
      atomicAdd(&F.discard[r], 1);
    } else {
      int *arr_cnt = F.arr_cnt, *arr_cut = F.arr_cut;
      if (flag_bases) arrival_words(flag_bases[X.owner], nsweeps, nsub, nrhs, arr_cnt, arr_cut);
      const size_t ti = ((size_t)(X.use - 1) * nsub + X.dst) * nrhs + r;
      atomicAdd_system(&arr_cnt[ti], 1);
      atomicAnd_system(&arr_cut[ti], X.content_base | (cut & X.keepmask));
      atomicAdd(&F.emit_cnt[((size_t)(Q.sweep - 1) * nsub + X.src) * nrhs + r], 1);
    }
  }
  const int lpn = nrhs / RV;
  const int npb = blockDim.x / lpn, rl = t % lpn, ln = t / lpn;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int4 T = tiles[tile];
    __syncthreads();
    if (t < (int)(sizeof(XferRec) / 8))
      reinterpret_cast<long long *>(&R)[t] = reinterpret_cast<const long long *>(recs + T.x)[t];
    __syncthreads();
    if (ln >= npb) continue;
    bool emit[RV];
    bool anyemit = false;
#pragma unroll
    for (int j = 0; j < RV; ++j) {
      const int r = rl + j * lpn;
      emit[j] = R.nz[r] && !(solve_cut(F, R.sweep, R.src, nsub, r, nrhs) & R.dirmask);
      anyemit |= emit[j];
    }
    if (!anyemit) continue;
    const cplx *__restrict__ xs = R.x;
    const int nodes = T.z;
    for (int node = T.y + ln; node < nodes; node += npb) {
      int e[3];
      if (DIM == 3) {
        e[2] = node % R.shape[2];
        const int q = node / R.shape[2];
        e[1] = q % R.shape[1];
        e[0] = q / R.shape[1];
      } else {
        e[1] = node % R.shape[1];
        e[0] = node / R.shape[1];
        e[2] = 0;
      }
      int off = 0, k2i = 0;
#pragma unroll
      for (int a = 0; a < DIM; ++a) {
        off += R.str[a] * e[a];
        k2i += R.k2str[a] * e[a];
      }
      double f0[DIM];
#pragma unroll
      for (int a = 0; a < DIM; ++a) f0[a] = R.fac[a][e[a]];
      double w0m1 = 1.0;
#pragma unroll
      for (int a = 0; a < DIM; ++a) w0m1 = w0m1 * f0[a];
      w0m1 -= 1.0;
      const double k2 = R.k2[k2i];
      const cplx *xc = xs + (int64_t)off * nrhs + rl;
      cplx acc[RV], w0[RV];
#pragma unroll
      for (int j = 0; j < RV; ++j) {
        w0[j] = cscale(xc[j * lpn], w0m1);
        acc[j] = cscale(w0[j], k2);
      }
#pragma unroll
      for (int a = 0; a < DIM; ++a) {
        const cplx lo = R.clo[a][e[a]], hi = R.chi[a][e[a]];
        const cplx mlh = make_double2(-(lo.x + hi.x), -(lo.y + hi.y));
#pragma unroll
        for (int j = 0; j < RV; ++j) acc[j] = cadd(acc[j], cmul(mlh, w0[j]));
#pragma unroll
        for (int side = 0; side < 2; ++side) {
          const int ea = e[a] + (side ? 1 : -1);
          if (side ? ea < R.ehi[a] : ea >= R.elo[a]) {
            // w(p +- e_a) - 1 with w = prod_b fac_b in axis order
            double wt = 1.0;
#pragma unroll
            for (int b = 0; b < DIM; ++b) wt = wt * (b == a ? R.fac[a][ea] : f0[b]);
            const double wm1 = wt - 1.0;
            const cplx cf = side ? hi : lo;
            const cplx *xp = xc + (int64_t)(side ? R.str[a] : -R.str[a]) * nrhs;
#pragma unroll
            for (int j = 0; j < RV; ++j) acc[j] = cadd(acc[j], cmul(cf, cscale(xp[j * lpn], wm1)));
          }
        }
      }
      const cplx *rv = R.rhs + (int64_t)off * nrhs + rl;
      cplx *sp = R.slot + (int64_t)node * nrhs + rl;
#pragma unroll
      for (int j = 0; j < RV; ++j)
        if (emit[j]) sp[j * lpn] = cadd(sp[j * lpn], cscale(cadd(rv[j * lpn], acc[j]), R.sign));
    }
  }
  if (flag_bases) __threadfence_system();
}

// ------------------------------------------------------------ plan create

extern "C" int ds_plan_create(ds_ctx *ctx, const ds_plan_desc *d, ds_plan **out) {
  if (!ctx || !d || !out) return ds_fail(DS_ECONFIG, "ds_plan_create: null argument");
  if (d->dim != 2 && d->dim != 3) return ds_fail(DS_ECONFIG, "plan dim must be 2 or 3");
  if (d->nrhs_max < 1 || d->nrhs_max > RMAX)
    return ds_fail(DS_ECONFIG, "nrhs_max must be in [1, 256]");
  if (!d->fact_of_sub || !d->fact_index) return ds_fail(DS_ECONFIG, "plan needs factorizations");
  const int dim = d->dim, nsub = d->nsub, nsw = d->nsweeps, nst = d->nsteps, ndir = d->ndir;
  ds_plan *P = new ds_plan();
  P->ctx = ctx;
  P->dim = dim;
  P->nsub = nsub;
  P->nsweeps = nsw;
  P->nsteps = nst;
  P->ndir = ndir;
  P->nrhs_max = d->nrhs_max;
  const bool sharded = d->nranks > 1;
  P->nranks = sharded ? d->nranks : 1;
  P->rank = sharded ? d->rank : 0;
  P->owner.assign(nsub, 0);
  if (sharded) {
    if (!d->owner || d->rank < 0 || d->rank >= d->nranks) {
      delete P;
      return ds_fail(DS_ECONFIG, "sharded plan: bad rank/owner table");
    }
    for (int s = 0; s < nsub; ++s) {
      P->owner[s] = d->owner[s];
      if (P->owner[s] < 0 || P->owner[s] >= d->nranks) {
        delete P;
        return ds_fail(DS_ECONFIG, "sharded plan: owner out of range");
      }
    }
  }
  P->nnodes = 1;
  for (int a = 0; a < 3; ++a) {
    P->gcounts[a] = a < dim ? d->grid_counts[a] : 1;
    P->nnodes *= P->gcounts[a];
  }
  auto fail = [&](int code) {
    for (void *p : P->allocs) cudaFree(p);
    delete P;
    return code;
  };
  // ---- operators and factor layouts in device memory
  void *mem;
  if (plan_alloc(P, &mem, sizeof(OpDev) * d->nops)) return fail(DS_ECUDA);
  P->ops = (OpDev *)mem;
  {
    std::vector<OpDev> h(d->nops);
    for (int i = 0; i < d->nops; ++i) h[i] = d->ops[i]->dev;
    cudaMemcpy(P->ops, h.data(), sizeof(OpDev) * d->nops, cudaMemcpyHostToDevice);
    P->h_ops = h;
  }
  // factor layout of every subdomain (device table, one entry per subdomain)
  std::vector<FactDev> hf(nsub);
  for (int s = 0; s < nsub; ++s) {
    const ds_fact *FA = d->fact_of_sub[s];
    int fi = d->fact_index[s];
    if (P->owner[s] != P->rank && !FA) {  // remote subdomain: no local factors
      memset(&hf[s], 0, sizeof(FactDev));
      continue;
    }
    if (!FA || fi < 0 || fi >= (int)FA->facts.size())
      return fail(ds_fail(DS_ECONFIG, "bad factorization handle/index for a subdomain"));
    hf[s] = FA->facts[fi];
  }
  if (plan_alloc(P, &mem, sizeof(FactDev) * nsub)) return fail(DS_ECUDA);
  P->facts = (FactDev *)mem;
  P->h_facts = hf;
  for (int s = 0; s < nsub; ++s) {
    const bool local = d->fact_of_sub[s] != nullptr;
    P->h_l.push_back(local ? d->fact_of_sub[s]->h_l[d->fact_index[s]].data() : nullptr);
    P->h_u.push_back(local ? d->fact_of_sub[s]->h_u[d->fact_index[s]].data() : nullptr);
  }
  cudaMemcpy(P->facts, hf.data(), sizeof(FactDev) * nsub, cudaMemcpyHostToDevice);
  // pooled factors (ABI 5): every visit (w, s) reads its factors from slot
  // visit_slot[w * nsub + s] of its factor pool (per-visit layout copies)
  std::vector<FactDev> hvf;
  FactDev *vfacts = nullptr;
  if (d->visit_slot) {
    hvf.resize((size_t)nsw * nsub);
    for (int w = 0; w < nsw; ++w)
      for (int s = 0; s < nsub; ++s) {
        FactDev fv = hf[s];
        if (P->owner[s] == P->rank) {
          const int slot = d->visit_slot[(size_t)w * nsub + s];
          const cplx *mem = ds_fact_slot_mem(d->fact_of_sub[s], slot);
          if (!mem || fv.kind != 0)
            return fail(ds_fail(DS_ECONFIG, "visit_slot: subdomain factors are not a block-LU pool"));
          fv.sinv = mem;
        }
        hvf[(size_t)w * nsub + s] = fv;
      }
    if (plan_alloc(P, &mem, sizeof(FactDev) * hvf.size())) return fail(DS_ECUDA);
    vfacts = (FactDev *)mem;
    cudaMemcpy(vfacts, hvf.data(), sizeof(FactDev) * hvf.size(), cudaMemcpyHostToDevice);
  }
  // ---- beta00 ramps
  int64_t nbeta = 0;
  for (int s = 0; s < nsub; ++s)
    for (int a = 0; a < dim; ++a)
      nbeta = std::max<int64_t>(nbeta, d->beta00_off[s * 3 + a] + d->sup_shape[s * 3 + a]);
  double *dbeta;
  if (plan_alloc(P, &mem, sizeof(double) * nbeta)) return fail(DS_ECUDA);
  dbeta = (double *)mem;
  cudaMemcpy(dbeta, d->beta00, sizeof(double) * nbeta, cudaMemcpyHostToDevice);
  // ---- subdomains
  std::vector<SubDev> hs(nsub);
  int max_w = 0;
  P->max_m = 0;
  for (int s = 0; s < nsub; ++s) {
    SubDev &S = hs[s];
    memset(&S, 0, sizeof(S));
    int oi = d->op_of_sub[s];
    if (oi < 0 || oi >= d->nops) return fail(ds_fail(DS_ECONFIG, "bad operator index"));
    const FactDev &fd = hf[s];
    int64_t wn = 1;
    for (int a = 0; a < 3; ++a) {
      bool ok = a < dim;
      S.win_lo[a] = ok ? d->win_lo[s * 3 + a] : 0;
      S.win_shape[a] = ok ? d->win_shape[s * 3 + a] : 1;
      S.own_lo[a] = ok ? d->own_lo[s * 3 + a] : 0;
      S.own_shape[a] = ok ? d->own_shape[s * 3 + a] : 1;
      S.sup_lo[a] = ok ? d->sup_lo[s * 3 + a] : 0;
      S.sup_shape[a] = ok ? d->sup_shape[s * 3 + a] : 1;
      S.beta[a] = ok ? dbeta + d->beta00_off[s * 3 + a] : nullptr;
      if (ok && P->owner[s] == P->rank && S.win_shape[a] != fd.win_shape[a])
        return fail(ds_fail(DS_ECONFIG, "window shape does not match its factorization"));
      wn *= S.win_shape[a];
    }
    S.f = P->facts + s;
    S.op = P->ops + oi;
    max_w = std::max<int>(max_w, (int)wn);
    P->max_w = max_w;
    P->max_axis_sum = std::max(P->max_axis_sum, S.win_shape[0] + S.win_shape[1] + S.win_shape[2]);
    if (P->owner[s] == P->rank && fd.kind == 0) P->max_m = std::max(P->max_m, fd.m);
  }
  if (plan_alloc(P, &mem, sizeof(SubDev) * nsub)) return fail(DS_ECUDA);
  P->subs = (SubDev *)mem;
  cudaMemcpy(P->subs, hs.data(), sizeof(SubDev) * nsub, cudaMemcpyHostToDevice);
  P->h_subs = hs;
  P->h_op_of_sub.assign(d->op_of_sub, d->op_of_sub + nsub);
  // ---- steps and visit buffers
  P->gmax = 0;
  int max_nb = 0;
  for (int s = 0; s < nsub; ++s) max_nb = std::max(max_nb, hf[s].nb);
  const bool sched = d->nlaunch > 0;
  if (sharded && !sched)
    return fail(ds_fail(DS_ECONFIG, "a sharded plan needs a launch schedule"));
  if (sched) {
    if (!d->launch_off || !d->launch_visits)
      return fail(ds_fail(DS_ECONFIG, "launch schedule without launch_off/launch_visits"));
    int nown = 0;
    for (int s = 0; s < nsub; ++s) nown += P->owner[s] == P->rank;
    if (d->launch_off[0] != 0 || d->launch_off[d->nlaunch] != nsw * nown)
      return fail(ds_fail(DS_ECONFIG, "launch schedule must cover every owned (sweep, subdomain) once"));
    std::vector<char> seen((size_t)nsw * nsub, 0);
    for (int l = 0; l < d->nlaunch; ++l) {
      P->gmax = std::max(P->gmax, d->launch_off[l + 1] - d->launch_off[l]);
      for (int i = d->launch_off[l]; i < d->launch_off[l + 1]; ++i) {
        int w = d->launch_visits[2 * i], s = d->launch_visits[2 * i + 1];
        if (w < 0 || w >= nsw || s < 0 || s >= nsub || P->owner[s] != P->rank ||
            seen[(size_t)w * nsub + s]++)
          return fail(ds_fail(DS_ECONFIG, "launch schedule: bad, remote or repeated visit"));
      }
    }
  } else {
    for (int w = 0; w < nsw; ++w)
      for (int t = 0; t < nst; ++t)
        P->gmax = std::max(P->gmax, d->step_off[w * (nst + 1) + t + 1] - d->step_off[w * (nst + 1) + t]);
  }
  P->nlaunch = d->nlaunch;
  size_t vbuf = (size_t)max_w * d->nrhs_max;
  cplx *bufs;
  if (plan_alloc(P, &mem, sizeof(cplx) * vbuf * 2 * 2 * P->gmax)) return fail(DS_ECUDA);
  bufs = (cplx *)mem;
  // K3 exchange scratch: 4 * m * nrhs per visit slot (2 parities x Gmax)
  size_t xgbuf = 4 * (size_t)P->max_m * d->nrhs_max;
  cplx *xgs;
  if (plan_alloc(P, &mem, sizeof(cplx) * std::max<size_t>(xgbuf, 1) * 2 * P->gmax)) return fail(DS_ECUDA);
  xgs = (cplx *)mem;
  bool any_modal = false;
  for (int s = 0; s < nsub; ++s) any_modal |= P->owner[s] == P->rank && hf[s].kind == 1;
  cplx *mscr = nullptr;  // modal scratch: 2 buffers per visit slot
  if (any_modal) {
    if (plan_alloc(P, &mem, sizeof(cplx) * vbuf * 2 * 2 * P->gmax)) return fail(DS_ECUDA);
    mscr = (cplx *)mem;
  }
  {
    P->staged = P->max_m > 0 && (P->max_m > DS_LARGE_SLAB || ctx->opt.staged);
  }
  (void)max_nb;
  // ---- flags
  P->flag_words = (size_t)nsub * d->nrhs_max + 4 * (size_t)nsw * nsub * d->nrhs_max + d->nrhs_max;
  if (plan_alloc(P, &mem, sizeof(int) * P->flag_words)) return fail(DS_ECUDA);
  P->flags = (int *)mem;
  // ---- payload slots keyed (use, target, direction)
  std::map<std::tuple<int, int, int>, int> slot_id;
  std::vector<SlotRef> hslots;
  std::vector<std::vector<int>> slots_of_visit((size_t)nsw * nsub);
  std::vector<int> slot_src_key;  // (s, k) that defines the band
  auto dir_of = [&](int k, int a) { return d->directions[k * 3 + a]; };
  auto sub_coords = [&](int s, int *idx) {
    int rem = s;
    for (int a = dim - 1; a >= 0; --a) {
      idx[a] = rem % d->part_counts[a];
      rem /= d->part_counts[a];
    }
  };
  auto sub_linear = [&](const int *idx) {
    int l = 0;
    for (int a = 0; a < dim; ++a) l = l * d->part_counts[a] + idx[a];
    return l;
  };
  size_t slot_elems = 0;
  std::vector<size_t> slot_off;
  for (int w = 0; w < nsw; ++w)
    for (int s = 0; s < nsub; ++s)
      for (int k = 0; k < ndir; ++k) {
        int use = d->xfer_use[((size_t)w * nsub + s) * ndir + k];
        if (use < 1) continue;
        int idx[3];
        sub_coords(s, idx);
        for (int a = 0; a < dim; ++a) idx[a] += dir_of(k, a);
        int dst = sub_linear(idx);
        auto key = std::make_tuple(use - 1, dst, k);
        if (slot_id.count(key)) continue;
        int id = (int)hslots.size();
        slot_id[key] = id;
        SlotRef R;
        memset(&R, 0, sizeof(R));
        int64_t n = 1;
        for (int a = 0; a < 3; ++a) {
          bool ok = a < dim;
          R.lo[a] = ok ? d->band_lo[((size_t)s * ndir + k) * 3 + a] : 0;
          R.shape[a] = ok ? d->band_shape[((size_t)s * ndir + k) * 3 + a] : 1;
          n *= R.shape[a];
        }
        slot_off.push_back(slot_elems);
        slot_elems += n * d->nrhs_max;
        hslots.push_back(R);
        slots_of_visit[(size_t)(use - 1) * nsub + dst].push_back(id);
      }
  cplx *slotmem;
  if (plan_alloc(P, &mem, sizeof(cplx) * std::max<size_t>(slot_elems, 1))) return fail(DS_ECUDA);
  slotmem = (cplx *)mem;
  cudaMemset(slotmem, 0, sizeof(cplx) * std::max<size_t>(slot_elems, 1));
  P->slot_bufs.push_back({slotmem, sizeof(cplx) * std::max<size_t>(slot_elems, 1)});
  for (size_t i = 0; i < hslots.size(); ++i) hslots[i].data = slotmem + slot_off[i];
  for (const auto &kv : slot_id) P->slot_by_key[kv.first] = hslots[kv.second];
  P->slot_base = slotmem;
  P->slot_bytes = sizeof(cplx) * std::max<size_t>(slot_elems, 1);
  // slot table ordered per visit (contiguous ranges)
  std::vector<SlotRef> hslot_tab;
  // ---- transfer (1 - beta) factors on ext
  int64_t nfac = 0;
  for (int s = 0; s < nsub; ++s)
    for (int k = 0; k < ndir; ++k)
      for (int a = 0; a < dim; ++a) {
        size_t o = ((size_t)s * ndir + k) * 3 + a;
        if (d->ext_shape[o] > 0) nfac = std::max<int64_t>(nfac, d->xfac_off[o] + d->ext_shape[o]);
      }
  double *dfac;
  if (plan_alloc(P, &mem, sizeof(double) * std::max<int64_t>(nfac, 1))) return fail(DS_ECUDA);
  dfac = (double *)mem;
  if (nfac) cudaMemcpy(dfac, d->xfac, sizeof(double) * nfac, cudaMemcpyHostToDevice);
  // ---- visits in execution order
  std::vector<VisitDev> hv;
  std::vector<std::pair<size_t, size_t>> km_at;  // (visit, mask word offset)
  std::vector<SolveVisit> hsv;
  P->blu_off.assign((size_t)(sched ? d->nlaunch : nsw * nst) + 1, 0);
  P->mod_off.assign(P->blu_off.size(), 0);
  std::vector<XferDev> hx;
  const int nq = sched ? d->nlaunch : nsw * nst;
  P->vstep_off.assign((size_t)nq + 1, 0);
  P->xstep_off.assign((size_t)nq + 1, 0);
  std::vector<int> visit_of((size_t)nsw * nsub, -1);
  // visit i of launch q: (sweep, subdomain)
  auto visit_at = [&](int q, int i, int &w, int &s) {
    if (sched) {
      w = d->launch_visits[2 * i];
      s = d->launch_visits[2 * i + 1];
    } else {
      w = q / nst;
      s = d->visit_sub[(size_t)w * nsub + i];
    }
  };
  int step_global = 0;
  for (int q = 0; q < nq; ++q, ++step_global) {
    {
      int b, e;
      if (sched) {
        b = d->launch_off[q];
        e = d->launch_off[q + 1];
      } else {
        const int w = q / nst, t = q % nst;
        b = d->step_off[w * (nst + 1) + t];
        e = d->step_off[w * (nst + 1) + t + 1];
      }
      P->vstep_off[step_global] = (int)hv.size();
      P->blu_off[step_global] = (int)hsv.size();
      P->mod_off[step_global] = (int)P->h_mjobs.size();
      int parity = step_global & 1;
      for (int g = b; g < e; ++g) {
        int w, s;
        visit_at(q, g, w, s);
        VisitDev V;
        memset(&V, 0, sizeof(V));
        V.sub = s;
        V.sweep = w + 1;
        V.slot0 = (int)hslot_tab.size();
        for (int id : slots_of_visit[(size_t)w * nsub + s]) hslot_tab.push_back(hslots[id]);
        V.nslot = (int)hslot_tab.size() - V.slot0;
        int gi = g - b;
        V.rhs = bufs + ((size_t)(parity * 2 + 0) * P->gmax + gi) * vbuf;
        V.x = bufs + ((size_t)(parity * 2 + 1) * P->gmax + gi) * vbuf;
        V.nz = nullptr;  // set per call (depends on nrhs stride)
        visit_of[(size_t)w * nsub + s] = (int)hv.size();
        hv.push_back(V);
        if (hf[s].kind == 1) {
          const int nl = hf[s].naxes == 2 ? hf[s].nax[1] : hf[s].m;  // K extent of forward pass 0
          const int rows = hf[s].nb * (hf[s].m / nl);
          if (nl <= 256 && rows <= 8192) {  // 32 chunks of 8 per mask word; K6 shared memory
            km_at.emplace_back(hv.size() - 1, (size_t)P->kmask_words);
            P->kmask_words += rows;
            P->km_rows_max = std::max(P->km_rows_max, rows);
          }
          cplx *s0 = mscr + ((size_t)(parity * 2 + 0) * P->gmax + gi) * vbuf;
          cplx *s1 = mscr + ((size_t)(parity * 2 + 1) * P->gmax + gi) * vbuf;
          P->h_mjobs.push_back(ModalJob{P->facts + s, V.rhs, V.x, s0, s1, nullptr});
          P->h_mfacts.push_back(hf[s]);
          P->mod_vidx.push_back((int)hv.size() - 1);
        } else {
          SolveVisit SV{vfacts ? vfacts + (size_t)w * nsub + s : P->facts + s, V.rhs, V.x, nullptr,
                        xgs + ((size_t)parity * P->gmax + gi) * xgbuf};
          hsv.push_back(SV);
          P->blu_vidx.push_back((int)hv.size() - 1);
        }
      }
      P->xstep_off[step_global] = (int)hx.size();
      for (int g = b; g < e; ++g) {
        int w, s;
        visit_at(q, g, w, s);
        for (int k = 0; k < ndir; ++k) {
          int use = d->xfer_use[((size_t)w * nsub + s) * ndir + k];
          if (use < 0) continue;  // target out of range: psi returns None
          XferDev X;
          memset(&X, 0, sizeof(X));
          X.vidx = visit_of[(size_t)w * nsub + s];
          X.src = s;
          int idx[3];
          sub_coords(s, idx);
          for (int a = 0; a < dim; ++a) idx[a] += dir_of(k, a);
          X.dst = sub_linear(idx);
          X.use = use;
          int order = 0;
          for (int a = 0; a < dim; ++a) {
            int c = dir_of(k, a);
            if (c) {
              order++;
              X.dirmask |= 1 << (2 * a + (c > 0));
              X.content_base |= 1 << (2 * a + (-c > 0));
            } else {
              X.keepmask |= 3 << (2 * a);
            }
          }
          X.sign = (order % 2 == 1) ? 1.0 : -1.0;
          for (int a = 0; a < 3; ++a) {
            bool ok = a < dim;
            size_t o = ((size_t)s * ndir + k) * 3 + a;
            X.band_lo[a] = ok ? d->band_lo[o] : 0;
            X.band_shape[a] = ok ? d->band_shape[o] : 1;
            X.ext_lo[a] = ok ? d->ext_lo[o] : 0;
            X.ext_shape[a] = ok ? d->ext_shape[o] : 1;
          }
          for (int a = 0; a < dim; ++a)
            X.fac[a] = dfac + d->xfac_off[((size_t)s * ndir + k) * 3 + a];
          X.slot = nullptr;
          X.owner = P->owner[X.dst];
          size_t soff = 0;
          if (use > 0) {
            const int sid = slot_id[std::make_tuple(use - 1, X.dst, k)];
            soff = slot_off[sid];
            // a remote target's slot lives on its owner: set by ds_plan_set_peers
            X.slot = X.owner == P->rank ? hslots[sid].data : nullptr;
          }
          P->xfer_slot_off.push_back(soff);
          hx.push_back(X);
        }
      }
    }
  }
  P->vstep_off[step_global] = (int)hv.size();
  P->xstep_off[step_global] = (int)hx.size();
  P->blu_off[step_global] = (int)hsv.size();
  P->mod_off[step_global] = (int)P->h_mjobs.size();
  // upload tables
  if (plan_alloc(P, &mem, sizeof(SlotRef) * std::max<size_t>(hslot_tab.size(), 1))) return fail(DS_ECUDA);
  P->slots = (SlotRef *)mem;
  cudaMemcpy(P->slots, hslot_tab.data(), sizeof(SlotRef) * hslot_tab.size(), cudaMemcpyHostToDevice);
  if (plan_alloc(P, &mem, sizeof(VisitDev) * hv.size())) return fail(DS_ECUDA);
  P->visits = (VisitDev *)mem;
  if (plan_alloc(P, &mem, sizeof(SolveVisit) * std::max<size_t>(hsv.size(), 1))) return fail(DS_ECUDA);
  P->solvetab = (SolveVisit *)mem;
  if (plan_alloc(P, &mem, sizeof(ModalJob) * std::max<size_t>(P->h_mjobs.size(), 1))) return fail(DS_ECUDA);
  P->mjobs = (ModalJob *)mem;
  if (plan_alloc(P, &mem, sizeof(XferDev) * std::max<size_t>(hx.size(), 1))) return fail(DS_ECUDA);
  P->xfers = (XferDev *)mem;
  cudaMemcpy(P->xfers, hx.data(), sizeof(XferDev) * hx.size(), cudaMemcpyHostToDevice);
  P->h_xfers = hx;
  if (plan_alloc(P, &mem, sizeof(XferRec) * std::max<size_t>(hx.size(), 1))) return fail(DS_ECUDA);
  P->recs = (XferRec *)mem;
  P->peers_set = !sharded;
  if (P->kmask_words > 0) {
    if (plan_alloc(P, &mem, sizeof(uint32_t) * P->kmask_words)) return fail(DS_ECUDA);
    P->kmask = (uint32_t *)mem;
    cudaMemset(P->kmask, 0, sizeof(uint32_t) * P->kmask_words);
    for (auto &e : km_at) hv[e.first].km = P->kmask + e.second;
    for (size_t j = 0; j < P->h_mjobs.size(); ++j) P->h_mjobs[j].km = hv[P->mod_vidx[j]].km;
  }
  P->h_visits = hv;
  P->h_solve = hsv;
  P->patched_nrhs = 0;
  if (P->staged) {
    std::vector<std::vector<SolveVisit>> sv;
    std::vector<std::vector<FactDev>> sf;
    std::vector<std::vector<const cplx *>> sl, su;
    for (size_t q = 0; q + 1 < P->vstep_off.size(); ++q) {
      sv.emplace_back();
      sf.emplace_back();
      sl.emplace_back();
      su.emplace_back();
      for (int e = P->blu_off[q]; e < P->blu_off[q + 1]; ++e) {
        const int i = P->blu_vidx[e];
        int sub = hv[i].sub;
        sv.back().push_back(hsv[e]);
        sf.back().push_back(hvf.empty() ? hf[sub] : hvf[(size_t)(hv[i].sweep - 1) * nsub + sub]);
        sl.back().push_back(P->h_l[sub]);
        su.back().push_back(P->h_u[sub]);
      }
    }
    std::string err;
    P->program = ds_stage_program_create(sv, sf, sl, su, d->nrhs_max, &err);
    if (!P->program) return fail(ds_fail(DS_ECUDA, err));
  }
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess)
    return fail(ds_fail(DS_ECUDA, std::string("ds_plan_create: ") + cudaGetErrorString(err)));
  if (ctx->opt.k5_side) {
    // the K5 and copy streams run at the highest priority (graphs are
    // instantiated with node priorities): their small grids take SMs as
    // soon as critical-path CTAs retire instead of queueing behind them
    int lo_pri = 0, hi_pri = 0;
    cudaDeviceGetStreamPriorityRange(&lo_pri, &hi_pri);
    P->side_priority = hi_pri;
    if (cudaStreamCreateWithPriority(&P->side, cudaStreamNonBlocking, P->side_priority) != cudaSuccess ||
        cudaEventCreateWithFlags(&P->ev_k3, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&P->ev_k5[0], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&P->ev_k5[1], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&P->ev_join, cudaEventDisableTiming) != cudaSuccess)
      return fail(ds_fail(DS_ECUDA, "ds_plan_create: side stream/events"));
  }
  *out = P;
  return DS_OK;
}

extern "C" int64_t ds_plan_workspace_bytes(const ds_plan *P) { return P ? P->workspace : -1; }
extern "C" int64_t ds_plan_last_launches(const ds_plan *P) { return P ? P->last_launches : -1; }

extern "C" int ds_plan_destroy(ds_plan *P) {
  if (!P) return DS_OK;
  if (P->graph) cudaGraphExecDestroy(P->graph);
  for (auto &g : P->hgraphs) cudaGraphExecDestroy(g.exec);
  if (P->cstream) cudaStreamDestroy(P->cstream);
  if (P->cstream2) cudaStreamDestroy(P->cstream2);
  for (auto x : P->cstream_x) cudaStreamDestroy(x);
  for (auto e : P->cjoin_x) cudaEventDestroy(e);
  if (P->hio_fork2) cudaEventDestroy(P->hio_fork2);
  if (P->hio_join2) cudaEventDestroy(P->hio_join2);
  for (auto e : P->hio_ev_in) cudaEventDestroy(e);
  for (auto e : P->hio_ev_out) cudaEventDestroy(e);
  if (P->hio_fork) cudaEventDestroy(P->hio_fork);
  if (P->hio_join) cudaEventDestroy(P->hio_join);
  if (P->gstream) cudaStreamDestroy(P->gstream);
  if (P->side) cudaStreamDestroy(P->side);
  for (cudaEvent_t e : {P->ev_k3, P->ev_k5[0], P->ev_k5[1], P->ev_join})
    if (e) cudaEventDestroy(e);
  if (P->gev_in) cudaEventDestroy(P->gev_in);
  if (P->gev_out) cudaEventDestroy(P->gev_out);
  for (auto e : P->ev) cudaEventDestroy(e);
  ds_stage_program_destroy(P->program);
  if (P->tiles) cudaFree(P->tiles);
  for (void *p : P->allocs) cudaFree(p);
  delete P;
  return DS_OK;
}

// point the per-visit nz flags at the [sweep][sub][nrhs] table of this stride
static int64_t g_patch_gen = 0;  // bumped whenever a plan's tables are rebuilt (grouped graphs)

static int patch_tables(ds_plan *P, int nrhs) {
  if (P->patched_nrhs == nrhs) return DS_OK;
  ++g_patch_gen;
  Flags F = flags_view(P, nrhs);
  for (size_t i = 0; i < P->h_visits.size(); ++i) {
    VisitDev &V = P->h_visits[i];
    V.nz = F.nz + ((size_t)(V.sweep - 1) * P->nsub + V.sub) * nrhs;
    V.arr = F.arr_cnt + ((size_t)(V.sweep - 1) * P->nsub + V.sub) * nrhs;
  }
  for (size_t e = 0; e < P->h_solve.size(); ++e) P->h_solve[e].nz = P->h_visits[P->blu_vidx[e]].nz;
  for (size_t e = 0; e < P->h_mjobs.size(); ++e) P->h_mjobs[e].nz = P->h_visits[P->mod_vidx[e]].nz;
  DS_CUDA(cudaMemcpyAsync(P->visits, P->h_visits.data(), sizeof(VisitDev) * P->h_visits.size(),
                          cudaMemcpyHostToDevice, P->ctx->stream));
  if (!P->h_solve.empty())
    DS_CUDA(cudaMemcpyAsync(P->solvetab, P->h_solve.data(), sizeof(SolveVisit) * P->h_solve.size(),
                            cudaMemcpyHostToDevice, P->ctx->stream));
  if (!P->h_mjobs.empty())
    DS_CUDA(cudaMemcpyAsync(P->mjobs, P->h_mjobs.data(), sizeof(ModalJob) * P->h_mjobs.size(),
                            cudaMemcpyHostToDevice, P->ctx->stream));
  // K4 v2: flattened transfer records and the per-launch band-node tiles
  std::vector<XferRec> hr(P->h_xfers.size());
  std::vector<int4> ht;
  const int npb = 256 / nrhs;
  const int pass_nodes = K4_NPT(P->dim) * npb;
  const int resident = P->ctx->num_sms * K4_MINB(P->dim);
  const int nq = (int)P->xstep_off.size() - 1;
  P->tile_off.assign((size_t)nq + 1, 0);
  for (int q = 0; q < nq; ++q) {
    P->tile_off[q] = (int)ht.size();
    // tile size of this launch: about one tile per resident block
    int64_t launch_nodes = 0;
    for (int i = P->xstep_off[q]; i < P->xstep_off[q + 1]; ++i) {
      const XferDev &X = P->h_xfers[i];
      if (X.use > 0) launch_nodes += (int64_t)X.band_shape[0] * X.band_shape[1] * X.band_shape[2];
    }
    int64_t tn = (launch_nodes + resident - 1) / resident;
    tn = std::max<int64_t>(1, (tn + pass_nodes - 1) / pass_nodes) * pass_nodes;
    for (int i = P->xstep_off[q]; i < P->xstep_off[q + 1]; ++i) {
      const XferDev &X = P->h_xfers[i];
      const VisitDev &V = P->h_visits[X.vidx];
      const FactDev &fs = P->h_facts[X.src];
      const SubDev &ss = P->h_subs[X.src], &sn = P->h_subs[X.dst];
      const OpDev &on = P->h_ops[P->h_op_of_sub[X.dst]];
      XferRec &Q = hr[i];
      memset(&Q, 0, sizeof(Q));
      int str[3] = {0, 0, 0};
      str[fs.block_axis] = fs.m;
      if (fs.other[0] >= 0) str[fs.other[0]] = fs.other[1] >= 0 ? fs.win_shape[fs.other[1]] : 1;
      if (fs.other[1] >= 0) str[fs.other[1]] = 1;
      int ostr[3] = {0, 0, 0};
      for (int a = P->dim - 1, acc = 1; a >= 0; --a) {
        ostr[a] = acc;
        acc *= on.shape[a];
      }
      int64_t base = 0, k2base = 0;
      Q.nodes = 1;
      for (int a = 0; a < P->dim; ++a) {
        const int blo = X.band_lo[a];
        base += (int64_t)str[a] * (blo - ss.win_lo[a]);
        Q.str[a] = str[a];
        Q.shape[a] = X.band_shape[a];
        Q.nodes *= X.band_shape[a];
        Q.elo[a] = X.ext_lo[a] - blo;
        Q.ehi[a] = X.ext_lo[a] + X.ext_shape[a] - blo;
        Q.fac[a] = X.fac[a] + (blo - X.ext_lo[a]);
        Q.clo[a] = on.c_lo[a] + (blo - sn.win_lo[a]);
        Q.chi[a] = on.c_hi[a] + (blo - sn.win_lo[a]);
        if (on.kappa2_kind == 2) {
          Q.k2str[a] = ostr[a];
          k2base += (int64_t)ostr[a] * (blo - sn.win_lo[a]);
        } else if (on.kappa2_kind == 1 && a == on.kappa2_axis) {
          Q.k2str[a] = 1;
          k2base += blo - sn.win_lo[a];
        }
      }
      Q.x = V.x + base * nrhs;
      Q.rhs = V.rhs + base * nrhs;
      Q.slot = X.slot;
      Q.nz = V.nz;
      Q.k2 = on.kappa2 + k2base;
      Q.src = X.src;
      Q.sweep = V.sweep;
      Q.dirmask = X.dirmask;
      Q.sign = X.sign;
      if (X.use > 0)
        for (int64_t n0 = 0; n0 < Q.nodes; n0 += tn)
          ht.push_back(make_int4(i - P->xstep_off[q], (int)n0, (int)std::min<int64_t>(Q.nodes, n0 + tn), 0));
    }
  }
  P->tile_off[nq] = (int)ht.size();
  if (!hr.empty())
    DS_CUDA(cudaMemcpyAsync(P->recs, hr.data(), sizeof(XferRec) * hr.size(), cudaMemcpyHostToDevice,
                            P->ctx->stream));
  if (ht.size() > P->tiles_cap) {
    DS_CUDA(cudaStreamSynchronize(P->ctx->stream));
    if (P->tiles) cudaFree(P->tiles);
    P->tiles = nullptr;
    P->tiles_cap = 0;
    DS_CUDA(cudaMalloc(&P->tiles, sizeof(int4) * ht.size()));
    P->tiles_cap = ht.size();
  }
  if (!ht.empty())
    DS_CUDA(cudaMemcpyAsync(P->tiles, ht.data(), sizeof(int4) * ht.size(), cudaMemcpyHostToDevice,
                            P->ctx->stream));
  DS_CUDA(cudaStreamSynchronize(P->ctx->stream));
  P->patched_nrhs = nrhs;
  if (P->graph) {
    cudaGraphExecDestroy(P->graph);
    P->graph = nullptr;
  }
  for (auto &g : P->hgraphs) cudaGraphExecDestroy(g.exec);  // tables may have moved
  P->hgraphs.clear();
  return DS_OK;
}

static int blocks_for(ds_ctx *ctx, int64_t work, int per_visit_cap) {
  int64_t b = (work + 255) / 256;
  if (b > per_visit_cap) b = per_visit_cap;
  if (b < 1) b = 1;
  (void)ctx;
  return (int)b;
}

static void prof_mark(ds_plan *P, int cls, cudaStream_t st) {
  if (!P->profiling) return;
  if (P->ev_used + 1 >= P->ev.size()) {
    size_t n = P->ev.size() ? P->ev.size() : 1024;
    for (size_t i = 0; i < n; ++i) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      P->ev.push_back(e);
      P->ev_class.push_back(-1);
    }
  }
  P->ev_class[P->ev_used] = cls;
  cudaEventRecord(P->ev[P->ev_used++], st);
}

// issue the whole application on ctx->stream (capturable)
// issue launches [q0, q1) of one application on ctx->stream (capturable);
// mode bit 0: zero u and the flags first; bit 1: join the K5 side stream
static int set_io(ds_plan *P, const void *f, void *u, cudaStream_t st) {
  if (!P->d_io) {
    void *mem;
    if (plan_alloc(P, &mem, 2 * sizeof(void *))) return DS_ECUDA;
    P->d_io = (cplx **)mem;
    P->io_f = nullptr;
    P->io_u = nullptr;
  }
  if (P->io_f == f && P->io_u == u) return DS_OK;
  const void *h[2] = {f, u};
  DS_CUDA(cudaMemcpyAsync(P->d_io, h, sizeof(h), cudaMemcpyHostToDevice, st));
  P->io_f = f;
  P->io_u = u;
  return DS_OK;
}

struct HostIO {
  const cplx *fh;  // pinned host sources, RHS-outer [R][N]
  cplx *uh;        // pinned host result, RHS-outer [R][N]
  // external mode (RHS groups, ds_ddm_apply_host_groups): the caller issues
  // the copies; the sweep only waits on the shared upload events and records
  // its per-box finalization events
  bool ext = false;
  const cudaEvent_t *ev_in = nullptr;
  cudaEvent_t *ev_out = nullptr;
};

// DS_HIO_TRACE (eager host path only): timestamps of uploads, launches and
// downloads, printed after the application (diagnostics)
static std::vector<std::pair<std::string, cudaEvent_t>> g_trace;
// DS_DIAG builds only: DS_HIO_TRACE=1 records a CUDA-event timeline of the
// pinned-host path (tools/ timeline probes)
static bool hio_trace_on() {
#ifdef DS_DIAG
  static const bool on = getenv("DS_HIO_TRACE") != nullptr;
  return on;
#else
  return false;
#endif
}
static void trace_mark(const std::string &what, cudaStream_t st) {
  if (!hio_trace_on()) return;
  cudaEvent_t e;
  cudaEventCreate(&e);
  cudaEventRecord(e, st);
  g_trace.push_back({what, e});
}
static int hio_in_chunks(ds_plan *P, const HostIO *hio, int nrhs, cudaStream_t cs);
static int hio_out_chunk(ds_plan *P, const HostIO *hio, int nrhs, int c, cudaStream_t cs);

static int issue_apply(ds_plan *P, const cplx *f, cplx *u, int nrhs, cplx *partials, int q0 = 0,
                       int q1 = -1, int mode = 3, const HostIO *hio = nullptr, bool outer = false) {
  // field layout of f and u: RHS-minor [N][R] or RHS-outer [R][N] (outer)
  ds_ctx *ctx = P->ctx;
  cudaStream_t st = ctx->stream;
  const int dim = P->dim;
  Flags F = flags_view(P, nrhs);
  int64_t launches0 = ctx->launches;
  size_t per = (size_t)P->nsweeps * P->nsub * nrhs;
  if (mode & 1) {
    {
      const int64_t n = P->nnodes * nrhs;
      const int64_t nflags = (int64_t)P->nsub * nrhs + 4 * (int64_t)per + nrhs;
      const int64_t cut0 = F.arr_cut - F.own_nz, cut1 = cut0 + (int64_t)per;
      k_zero_io<<<(unsigned)std::min<int64_t>((std::max(n, nflags) + 255) / 256, (int64_t)ctx->num_sms * 8),
                  256, 0, st>>>(P->d_io, n, F.own_nz, nflags, cut0, cut1, P->kmask, P->kmask_words);
      ctx->launches++;
      DS_CHECK_LAUNCH();
    }
    P->k5_pending[0] = P->k5_pending[1] = false;
  }
  // fork the copy streams after the zeroing (forking them first -- the
  // uploads need nothing from this call -- measured 2740 vs 3020 RHS/s end
  // to end on config 2: the graph's copies then start under the zeroing
  // kernel and the early launches)
  if (hio && !hio->ext) {
    DS_CUDA(cudaEventRecord(P->hio_fork, st));
    DS_CUDA(cudaStreamWaitEvent(P->cstream, P->hio_fork, 0));
    DS_CUDA(cudaStreamWaitEvent(P->cstream2, P->hio_fork, 0));
    for (auto x : P->cstream_x) DS_CUDA(cudaStreamWaitEvent(x, P->hio_fork, 0));
    if (int rc = hio_in_chunks(P, hio, nrhs, P->cstream)) return rc;
    for (int c : P->hio_out_early)
      if (int rc = hio_out_chunk(P, hio, nrhs, c, P->cstream)) return rc;
  }
  int hio_waited = 0, hio_nout = 0;
  // DS_DIAG builds only (wrong results): the DS_SKIP bitmask drops kernel
  // classes from the schedule to measure their marginal time under graph
  // replay (1 K6, 2 modal transforms, 4 modal recurrences, 8 K4, 16 K5)
#ifdef DS_DIAG
  static const int skip_cls = [] {
    const char *v = getenv("DS_SKIP");
    return v && *v ? atoi(v) : 0;
  }();
#else
  constexpr int skip_cls = 0;
#endif
  const int cap = std::max(1, ctx->num_sms * 4);
  // K6 runs 3 CTAs of 256 threads per SM (76 registers): in 2D a grid of
  // more than 3 x SMs leaves a partial second wave (ncu: 588 CTAs, 1.32
  // waves; capped: config 2 K6 0.814 -> 0.777 ms per application); the 3D
  // visits keep 4 x SMs (config 4: 5.63 vs 6.0 ms with the cap)
  const int cap6 = std::max(1, ctx->num_sms * (dim == 2 ? 3 : 4));
  if (partials && P->nlaunch > 0)
    return ds_fail(DS_ECONFIG, "per-sweep partials need the sweep-ordered plan (nlaunch = 0)");
  const int nq = q1 < 0 ? (int)P->vstep_off.size() - 1 : q1;
  // K5 stream (see ds_plan::side); single-stream when profiling or
  // collecting per-sweep partials (both read the stream in program order)
  const cudaStream_t s5 = (P->side && !P->profiling && !partials) ? P->side : st;
  bool *k5_pending = P->k5_pending;
  for (int q = q0; q < nq; ++q) {
    {
      int v0 = P->vstep_off[q], G = P->vstep_off[q + 1] - v0;
      if (G == 0) continue;
      const int64_t wmax = P->max_w, smax = P->max_w;
      int bx = blocks_for(ctx, wmax * nrhs / 4, std::max(1, cap6 / G));
      if (hio && P->hio_need[q] > hio_waited) {  // f boxes [0, need) this assembly may read:
        hio_waited = P->hio_need[q];               // the last of them on each copy stream
        const cudaEvent_t *evi = hio->ext ? hio->ev_in : P->hio_ev_in.data();
        DS_CUDA(cudaStreamWaitEvent(st, evi[hio_waited - 1], 0));
        if (hio_waited >= 2) DS_CUDA(cudaStreamWaitEvent(st, evi[hio_waited - 2], 0));
      }
      if (hio) trace_mark("launch " + std::to_string(q), st);
      prof_mark(P, 0, st);
      const int k6rv = ctx->opt.k6_rv;  // RHS columns per thread of K6 (default 4)
      if (skip_cls & 1) {
      } else if (k6rv == 8 && nrhs % 8 == 0)
        DS_CUDA(launch_pdl(outer ? k_assemble<8, true> : k_assemble<8, false>, dim3(bx, G), dim3(256),
                           sizeof(uint32_t) * (P->max_axis_sum + P->km_rows_max), st,
                           (const VisitDev *)(P->visits + v0), (const SubDev *)P->subs,
                           (const SlotRef *)P->slots, f, nrhs, dim,
                           P->gcounts[0], P->gcounts[1], P->gcounts[2], F, (int64_t)P->nnodes));
      else if (k6rv == 2 && nrhs % 2 == 0)
        DS_CUDA(launch_pdl(outer ? k_assemble<2, true> : k_assemble<2, false>, dim3(bx, G), dim3(256),
                           sizeof(uint32_t) * (P->max_axis_sum + P->km_rows_max), st,
                           (const VisitDev *)(P->visits + v0), (const SubDev *)P->subs,
                           (const SlotRef *)P->slots, f, nrhs, dim,
                           P->gcounts[0], P->gcounts[1], P->gcounts[2], F, (int64_t)P->nnodes));
      else if (k6rv >= 4 && nrhs % 4 == 0)
        DS_CUDA(launch_pdl(outer ? k_assemble<4, true> : k_assemble<4, false>, dim3(bx, G), dim3(256),
                           sizeof(uint32_t) * (P->max_axis_sum + P->km_rows_max), st,
                           (const VisitDev *)(P->visits + v0), (const SubDev *)P->subs,
                           (const SlotRef *)P->slots, f, nrhs, dim,
                           P->gcounts[0], P->gcounts[1], P->gcounts[2], F, (int64_t)P->nnodes));
      else
        DS_CUDA(launch_pdl(outer ? k_assemble<1, true> : k_assemble<1, false>, dim3(bx, G), dim3(256),
                           sizeof(uint32_t) * (P->max_axis_sum + P->km_rows_max), st,
                           (const VisitDev *)(P->visits + v0), (const SubDev *)P->subs,
                           (const SlotRef *)P->slots, f, nrhs, dim,
                           P->gcounts[0], P->gcounts[1], P->gcounts[2], F, (int64_t)P->nnodes));
      ctx->launches++;
      DS_CHECK_LAUNCH();
      prof_mark(P, 1, st);
      if (s5 != st && k5_pending[q & 1]) DS_CUDA(cudaStreamWaitEvent(st, P->ev_k5[q & 1], 0));
      int rc = DS_OK;
      const int b0 = P->blu_off[q], nbl = P->blu_off[q + 1] - b0;
      const int m0 = P->mod_off[q], nmo = P->mod_off[q + 1] - m0;
      if (nbl > 0) {
        if (P->program) rc = ds_stage_program_launch_step(ctx, P->program, q, nrhs);
        else rc = ds_launch_solve_table(ctx, P->solvetab + b0, nbl, nrhs, P->max_m);
      }
      if (rc) return rc;
      if (nmo > 0) {  // modal: transforms (class 1) / recurrences (class 4) / transforms
        for (int ph = 0; ph < 3 && !rc; ++ph) {
          if (ph > 0) prof_mark(P, ph == 1 ? 4 : 1, st);
          if (skip_cls & (ph == 1 ? 4 : 2)) continue;
          rc = ds_launch_modal_phase(ctx, P->mjobs + m0, P->h_mfacts.data() + m0, nmo, nrhs, ph);
        }
      }
      if (rc) return rc;
      DS_CHECK_LAUNCH();
      prof_mark(P, 2, st);
      int by = blocks_for(ctx, smax * nrhs / 4, std::max(1, cap / G));
      if (s5 != st) {
        DS_CUDA(cudaEventRecord(P->ev_k3, st));
        DS_CUDA(cudaStreamWaitEvent(s5, P->ev_k3, 0));
      }
      if (skip_cls & 16) {
      } else if (nrhs % 4 == 0)
        (outer ? k_accumulate<4, true> : k_accumulate<4, false>)<<<dim3(by, G), 256, 0, s5>>>(
            P->visits + v0, G, P->subs, P->d_io, nrhs, dim, P->gcounts[0], P->gcounts[1], P->gcounts[2],
            (int64_t)P->nnodes);
      else
        (outer ? k_accumulate<1, true> : k_accumulate<1, false>)<<<dim3(by, G), 256, 0, s5>>>(
            P->visits + v0, G, P->subs, P->d_io, nrhs, dim, P->gcounts[0], P->gcounts[1], P->gcounts[2],
            (int64_t)P->nnodes);
      ctx->launches++;
      DS_CHECK_LAUNCH();
      if (s5 != st) {
        DS_CUDA(cudaEventRecord(P->ev_k5[q & 1], s5));
        k5_pending[q & 1] = true;
      }
      if (hio && hio->ext)  // the caller downloads: mark the boxes this accumulation finalized
        for (int c : P->hio_out_at[q]) DS_CUDA(cudaEventRecord(hio->ev_out[c], s5));
      if (hio && !hio->ext)  // u chunks whose last accumulation this was: transpose + D2H
        for (int c : P->hio_out_at[q]) {
          const int nd = 2 + (int)P->cstream_x.size(), di = hio_nout++ % nd;
          cudaStream_t cs = di == 0 ? P->cstream : (di == 1 ? P->cstream2 : P->cstream_x[di - 2]);
          DS_CUDA(cudaEventRecord(P->hio_ev_out[c], s5));
          DS_CUDA(cudaStreamWaitEvent(cs, P->hio_ev_out[c], 0));
          trace_mark("  K5 done for box " + std::to_string(c) + " (launch " + std::to_string(q) + ")", cs);
          if (int rc = hio_out_chunk(P, hio, nrhs, c, cs)) return rc;
          trace_mark("  download done box " + std::to_string(c), cs);
        }
      int x0 = P->xstep_off[q], nx = P->xstep_off[q + 1] - x0;
      if (nx > 0 && !(skip_cls & 8)) {
        prof_mark(P, 3, st);
        int bz = std::max(1, std::min(64, 2 * cap / nx));
        const int k4rv = ctx->opt.k4_rv;  // v1: 1 measured fastest (config 2: 1.32 vs 1.51-1.59 ms)
#define K4_LAUNCH(RV_, D_)                                                                       \
  k_transfer<RV_, D_><<<dim3(bz, nx), 256, 0, st>>>(P->xfers + x0, P->visits, P->subs, P->nsub, \
                                                    nrhs, dim, F, P->d_flag_bases, P->nsweeps)
        const bool k4v1 = ctx->opt.k4 == 1;  // the original one-block-per-band kernel
        const int rv = (k4rv == 4 && nrhs % 4 == 0) ? 4 : ((k4rv >= 2 && nrhs % 2 == 0) ? 2 : 1);
        if (!k4v1) {
          const int t0 = P->tile_off[q], nt = P->tile_off[q + 1] - t0;
          const int resident = ctx->num_sms * K4_MINB(dim);
          const int gb = std::max(1, std::max(std::min(nt, resident), (nx * nrhs + 255) / 256));
          const XferDev *xd = P->xfers + x0;
          const XferRec *xr = P->recs + x0;
          const int4 *tl = P->tiles + t0;
          int *const *fb = P->d_flag_bases;
          const int k4v = ctx->opt.k4;
          // defaults (measured): 2D k_transfer3 (config 2 +3%), 3D k_transfer2
          // (config 4: 7.5 vs 7.9 ms per application with k_transfer3<3, 4>)
          const int v3rv = (dim == 3 && k4v == 3) ? (nrhs % 4 == 0 ? 4 : (nrhs % 2 == 0 ? 2 : 1)) : 0;
          if (dim == 2 && k4v != 2)
            DS_CUDA(launch_pdl(k_transfer3<2, 1>, dim3(gb), dim3(256), 0, st, xd, xr, tl, nt, nx,
                               P->nsub, nrhs, F, fb, P->nsweeps));
          else if (dim == 2)
            DS_CUDA(launch_pdl(k_transfer2<2, K4_NPT(2)>, dim3(gb), dim3(256), 0, st, xd, xr, tl, nt, nx,
                               P->nsub, nrhs, F, fb, P->nsweeps));
          else if (v3rv == 4)
            DS_CUDA(launch_pdl(k_transfer3<3, 4>, dim3(gb), dim3(256), 0, st, xd, xr, tl, nt, nx,
                               P->nsub, nrhs, F, fb, P->nsweeps));
          else if (v3rv == 2)
            DS_CUDA(launch_pdl(k_transfer3<3, 2>, dim3(gb), dim3(256), 0, st, xd, xr, tl, nt, nx,
                               P->nsub, nrhs, F, fb, P->nsweeps));
          else
            DS_CUDA(launch_pdl(k_transfer2<3, K4_NPT(3)>, dim3(gb), dim3(256), 0, st, xd, xr, tl, nt, nx,
                               P->nsub, nrhs, F, fb, P->nsweeps));
        } else if (dim == 2) {
          if (rv == 4) K4_LAUNCH(4, 2);
          else if (rv == 2) K4_LAUNCH(2, 2);
          else K4_LAUNCH(1, 2);
        } else {
          if (rv == 4) K4_LAUNCH(4, 3);
          else if (rv == 2) K4_LAUNCH(2, 3);
          else K4_LAUNCH(1, 3);
        }
#undef K4_LAUNCH
        ctx->launches++;
        DS_CHECK_LAUNCH();
      }
    }
    if (partials && (q + 1) % P->nsteps == 0)
      DS_CUDA(cudaMemcpyAsync(partials + (size_t)(q / P->nsteps) * P->nnodes * nrhs, u,
                              sizeof(cplx) * P->nnodes * nrhs, cudaMemcpyDeviceToDevice, st));
  }
  if ((mode & 2) && s5 != st && (k5_pending[0] || k5_pending[1])) {  // join: u complete on st
    DS_CUDA(cudaEventRecord(P->ev_join, s5));
    DS_CUDA(cudaStreamWaitEvent(st, P->ev_join, 0));
  }
  if (hio && !hio->ext) {  // join the copy stream: every u chunk is on the host
    DS_CUDA(cudaEventRecord(P->hio_join, P->cstream));
    DS_CUDA(cudaStreamWaitEvent(st, P->hio_join, 0));
    DS_CUDA(cudaEventRecord(P->hio_join2, P->cstream2));
    DS_CUDA(cudaStreamWaitEvent(st, P->hio_join2, 0));
    for (size_t i = 0; i < P->cstream_x.size(); ++i) {
      DS_CUDA(cudaEventRecord(P->cjoin_x[i], P->cstream_x[i]));
      DS_CUDA(cudaStreamWaitEvent(st, P->cjoin_x[i], 0));
    }
  }
  prof_mark(P, -1, st);
  P->last_launches = ctx->launches - launches0;
  return DS_OK;
}

// ------------------------------------------- host-buffer application
// Boxes of the grid (axis 0 x axis 1, axis 2 whole) moved between host and
// device as units.  Uploads go in the order the first sweep needs them; a
// box of u goes back as soon as the last accumulation touching it ran.
struct HioBox {
  int a0, a1, c0, c1;  // axis-0 rows, axis-1 columns
};

// box of RHS-outer [R][N] <-> RHS-minor [N][R]: run i (axis-0 row a0 + i) is
// the contiguous node range [base_i, base_i + L); to_minor: dst[n][r] =
// src[r][n], else dst[r][n] = src[n][r]; grid (32-tiles of R x L, runs)
__global__ void k_box_transpose(int R, int L, int64_t N, int64_t base0, int64_t run_stride,
                                const cplx *__restrict__ src, cplx *__restrict__ dst, int to_minor) {
  __shared__ cplx tile[32][33];
  const int ntc = (L + 31) / 32;
  const int r0 = (blockIdx.x / ntc) * 32, e0 = (blockIdx.x % ntc) * 32;
  const int64_t base = base0 + (int64_t)blockIdx.y * run_stride;
  if (to_minor) {
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
      const int r = r0 + i, e = e0 + threadIdx.x;
      if (r < R && e < L) tile[i][threadIdx.x] = src[(int64_t)r * N + base + e];
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
      const int e = e0 + i, r = r0 + threadIdx.x;
      if (r < R && e < L) dst[(base + e) * R + r] = tile[threadIdx.x][i];
    }
  } else {
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
      const int e = e0 + i, r = r0 + threadIdx.x;
      if (r < R && e < L) tile[threadIdx.x][i] = src[(base + e) * R + r];
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
      const int r = r0 + i, e = e0 + threadIdx.x;
      if (r < R && e < L) dst[(int64_t)r * N + base + e] = tile[i][threadIdx.x];
    }
  }
}

// chunk tables (nrhs-independent) and staging buffers (nrhs_max)
static std::vector<HioBox> hio_grid(const ds_plan *P, int a, int b) {
  const int B0 = std::min(std::max(1, a), P->gcounts[0]), B1 = std::min(std::max(1, b), P->gcounts[1]);
  std::vector<HioBox> boxes;
  for (int i = 0; i < B0; ++i)
    for (int j = 0; j < B1; ++j)
      boxes.push_back({(int)((int64_t)P->gcounts[0] * i / B0), (int)((int64_t)P->gcounts[0] * (i + 1) / B0),
                       (int)((int64_t)P->gcounts[1] * j / B1), (int)((int64_t)P->gcounts[1] * (j + 1) / B1)});
  return boxes;
}

static int hio_setup(ds_plan *P) {
  if (P->hio_ready) return DS_OK;
  // upload boxes (DS_HIO_IN, default 8x4) in first-use order and download
  // boxes (DS_HIO_BOXES, default 12x2) in finalization order; measured on
  // config 2 (tools/e2e_probe.py): whole-row bands 16x1 5.61 ms, 8x2 / 8x2
  // 5.29, 8x4 / 12x2 5.18 -- finer boxes start the sweep earlier, but 3D
  // copies of sub-4 KB rows run below the copy engine's rate
  // upload 8 x 4 and download 12 x 2 boxes (measured on config 2)
  const std::vector<HioBox> ib = hio_grid(P, 8, 4);
  const std::vector<HioBox> ob = hio_grid(P, 12, 2);
  const int CI = (int)ib.size(), CO = (int)ob.size();
  auto meets = [&](const HioBox &B, const int *lo, const int *sh) {
    return sh[0] > 0 && sh[1] > 0 && lo[0] < B.a1 && lo[0] + sh[0] > B.a0 && lo[1] < B.c1 &&
           lo[1] + sh[1] > B.c0;
  };
  const int nq = (int)P->vstep_off.size() - 1;
  std::vector<int> first(CI, nq), last(CO, -1);
  for (int q = 0; q < nq; ++q)
    for (int i = P->vstep_off[q]; i < P->vstep_off[q + 1]; ++i) {
      const VisitDev &V = P->h_visits[i];
      const SubDev &S = P->h_subs[V.sub];
      if (V.sweep == 1)
        for (int c = 0; c < CI; ++c)
          if (meets(ib[c], S.own_lo, S.own_shape)) first[c] = std::min(first[c], q);
      for (int c = 0; c < CO; ++c)
        if (meets(ob[c], S.sup_lo, S.sup_shape)) last[c] = q;
    }
  // upload order: by first use (boxes no assembly reads go last)
  std::vector<int> order(CI);
  for (int c = 0; c < CI; ++c) order[c] = c;
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return first[x] < first[y]; });
  P->hio_boxes.clear();
  for (int c : order) P->hio_boxes.push_back(ib[c]);
  std::vector<int> pos(CI);
  for (int k = 0; k < CI; ++k) pos[order[k]] = k;
  P->hio_need.assign(nq, 0);
  int need = 0;
  for (int q = 0; q < nq; ++q) {
    for (int c = 0; c < CI; ++c)
      if (first[c] == q) need = std::max(need, pos[c] + 1);
    P->hio_need[q] = need;
  }
  P->hio_oboxes = ob;
  P->hio_out_at.assign(nq, {});
  P->hio_out_early.clear();
  for (int c = 0; c < CO; ++c) {
    if (last[c] < 0) P->hio_out_early.push_back(c);
    else P->hio_out_at[last[c]].push_back(c);
  }
  const int C = std::max(CI, CO);
#ifdef DS_DIAG
  if (getenv("DS_HIO_DEBUG")) {
    fprintf(stderr, "hio: %d boxes, %d launches; uploads needed by launch:", C, nq);
    for (int q = 0; q < nq; ++q) fprintf(stderr, " %d", P->hio_need[q]);
    fprintf(stderr, "\nhio: boxes final after launch:");
    for (int q = 0; q < nq; ++q) fprintf(stderr, " %d", (int)P->hio_out_at[q].size());
    fprintf(stderr, "\n");
  }
#endif
  const size_t bytes = sizeof(cplx) * (size_t)P->nnodes * P->nrhs_max;
  void *mem;
  for (cplx **b : {&P->hio_fo, &P->hio_fm, &P->hio_uo, &P->hio_um}) {
    if (plan_alloc(P, &mem, bytes)) return DS_ECUDA;
    *b = (cplx *)mem;
  }
  DS_CUDA(cudaStreamCreateWithPriority(&P->cstream, cudaStreamNonBlocking, P->side_priority));
  DS_CUDA(cudaStreamCreateWithPriority(&P->cstream2, cudaStreamNonBlocking, P->side_priority));
  {
    const int nd = std::max(2, std::min(8, P->ctx->opt.hio_dstreams));
    for (int i = 2; i < nd; ++i) {
      cudaStream_t x;
      cudaEvent_t e;
      DS_CUDA(cudaStreamCreateWithPriority(&x, cudaStreamNonBlocking, P->side_priority));
      DS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      P->cstream_x.push_back(x);
      P->cjoin_x.push_back(e);
    }
  }
  DS_CUDA(cudaEventCreateWithFlags(&P->hio_fork2, cudaEventDisableTiming));
  DS_CUDA(cudaEventCreateWithFlags(&P->hio_join2, cudaEventDisableTiming));
  P->hio_ev_in.resize(C);
  P->hio_ev_out.resize(C);
  for (int c = 0; c < C; ++c) {
    DS_CUDA(cudaEventCreateWithFlags(&P->hio_ev_in[c], cudaEventDisableTiming));
    DS_CUDA(cudaEventCreateWithFlags(&P->hio_ev_out[c], cudaEventDisableTiming));
  }
  DS_CUDA(cudaEventCreateWithFlags(&P->hio_fork, cudaEventDisableTiming));
  DS_CUDA(cudaEventCreateWithFlags(&P->hio_join, cudaEventDisableTiming));
  P->hio_ready = true;
  return DS_OK;
}

// one box between pinned host [R][N] and the device staging copy (3D copy:
// R slices x box rows x box row bytes), plus the layout transpose
static int hio_box(ds_plan *P, const HostIO *hio, int nrhs, int k, cudaStream_t cs, bool in) {
#ifdef DS_DIAG
  static const int skip = [] {  // DS_DIAG only: 1 skips uploads, 2 downloads (wrong results)
    const char *v = getenv("DS_HIO_SKIP");
    return v && *v ? atoi(v) : 0;
  }();
  if ((skip & 1) && in) return DS_OK;
  if ((skip & 2) && !in) return DS_OK;
#endif
  const HioBox &B = in ? P->hio_boxes[k] : P->hio_oboxes[k];
  const int64_t N = P->nnodes, S1 = P->gcounts[2], S0 = (int64_t)P->gcounts[1] * S1;
  const int L = (int)((B.c1 - B.c0) * S1), runs = B.a1 - B.a0;
  if (L <= 0 || runs <= 0) return DS_OK;
  cudaMemcpy3DParms m = {};
  cplx *dev = in ? P->hio_fo : P->hio_uo;
  cplx *host = in ? (cplx *)hio->fh : hio->uh;
  cudaPitchedPtr hp = make_cudaPitchedPtr(host, sizeof(cplx) * S0, sizeof(cplx) * S0, P->gcounts[0]);
  cudaPitchedPtr dp = make_cudaPitchedPtr(dev, sizeof(cplx) * S0, sizeof(cplx) * S0, P->gcounts[0]);
  const cudaPos at = make_cudaPos(sizeof(cplx) * B.c0 * S1, B.a0, 0);
  m.extent = make_cudaExtent(sizeof(cplx) * L, runs, nrhs);
  const int64_t base0 = (int64_t)B.a0 * S0 + (int64_t)B.c0 * S1;
  const dim3 grid((unsigned)(((nrhs + 31) / 32) * ((L + 31) / 32)), runs);
  if (in) {
    m.srcPtr = hp;
    m.srcPos = at;
    m.dstPtr = dp;
    m.dstPos = at;
    m.kind = cudaMemcpyHostToDevice;
    DS_CUDA(cudaMemcpy3DAsync(&m, cs));
    k_box_transpose<<<grid, dim3(32, 8), 0, cs>>>(nrhs, L, N, base0, S0, P->hio_fo, P->hio_fm, 1);
  } else {
    k_box_transpose<<<grid, dim3(32, 8), 0, cs>>>(nrhs, L, N, base0, S0, P->hio_um, P->hio_uo, 0);
  }
  P->ctx->launches++;
  DS_CHECK_LAUNCH();
  if (!in) {
    m.srcPtr = dp;
    m.srcPos = at;
    m.dstPtr = hp;
    m.dstPos = at;
    m.kind = cudaMemcpyDeviceToHost;
    DS_CUDA(cudaMemcpy3DAsync(&m, cs));
  }
  return DS_OK;
}

// uploads of every source box in first-use order, one event per box
// box k goes on copy stream k % 2 (two boxes in flight: one box's layout
// transpose runs under the other's copy, and two copy engines share PCIe)
static int hio_in_chunks(ds_plan *P, const HostIO *hio, int nrhs, cudaStream_t cs) {
  for (int k = 0; k < (int)P->hio_boxes.size(); ++k) {
    cudaStream_t c = (k & 1) ? P->cstream2 : cs;
    if (int rc = hio_box(P, hio, nrhs, k, c, true)) return rc;
    DS_CUDA(cudaEventRecord(P->hio_ev_in[k], c));
    trace_mark("  upload done box " + std::to_string(k), c);
  }
  return DS_OK;
}

static int hio_out_chunk(ds_plan *P, const HostIO *hio, int nrhs, int k, cudaStream_t cs) {
  return hio_box(P, hio, nrhs, k, cs, false);
}

// One application from pinned host buffers (RHS-outer [R][N]) to pinned host
// buffers: the source H2D runs in axis-0 row chunks on a copy stream while
// the first sweep's launches start (each assembly waits only for the chunks
// it reads), and every chunk of u is transposed and copied back as soon as
// the last accumulation touching it has run.  CUDA-graph replay keyed on the
// host pointers (up to 4 cached graphs).
extern "C" int ds_ddm_apply_host(ds_ctx *ctx, ds_plan *P, const ds_cplx *f_host, ds_cplx *u_host,
                                 int32_t nrhs) {
  if (!ctx || !P || !f_host || !u_host) return ds_fail(DS_ECONFIG, "ds_ddm_apply_host: null argument");
  if (nrhs < 1 || nrhs > P->nrhs_max)
    return ds_fail(DS_ECONFIG, "ds_ddm_apply_host: nrhs exceeds the plan's nrhs_max");
  if (P->nranks > 1) return ds_fail(DS_ECONFIG, "ds_ddm_apply_host: sharded plans run through ds_ddm_apply_range");
  if (ctx != P->ctx) P->ctx = ctx;
  int rc = patch_tables(P, nrhs);
  if (rc) return rc;
  if ((rc = hio_setup(P))) return rc;
  if (P->slots_dirty) {
    for (auto &b : P->slot_bufs) DS_CUDA(cudaMemsetAsync(b.first, 0, b.second, ctx->stream));
    P->slots_dirty = false;
  }
  HostIO hio{(const cplx *)f_host, (cplx *)u_host};
  if ((rc = set_io(P, P->hio_fm, P->hio_um, ctx->stream))) return rc;
  if (!P->use_graph || P->profiling) {
    trace_mark("start", ctx->stream);
    rc = issue_apply(P, P->hio_fm, P->hio_um, nrhs, nullptr, 0, -1, 3, &hio);
    trace_mark("end", ctx->stream);
    if (rc) P->slots_dirty = true;
    if (hio_trace_on() && !g_trace.empty()) {
      cudaDeviceSynchronize();
      for (auto &t : g_trace) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, g_trace.front().second, t.second);
        fprintf(stderr, "hio %8.3f ms  %s\n", ms, t.first.c_str());
      }
      for (auto &t : g_trace) cudaEventDestroy(t.second);
      g_trace.clear();
    }
    return rc;
  }
  if (!P->gstream) {
    DS_CUDA(cudaStreamCreateWithFlags(&P->gstream, cudaStreamNonBlocking));
    DS_CUDA(cudaEventCreateWithFlags(&P->gev_in, cudaEventDisableTiming));
    DS_CUDA(cudaEventCreateWithFlags(&P->gev_out, cudaEventDisableTiming));
  }
  cudaStream_t user = ctx->stream;
  ds_plan::HGraph *G = nullptr;
  for (auto &g : P->hgraphs)
    if (g.fh == f_host && g.uh == u_host && g.nrhs == nrhs) G = &g;
  DS_CUDA(cudaEventRecord(P->gev_in, user));
  DS_CUDA(cudaStreamWaitEvent(P->gstream, P->gev_in, 0));
  if (!G) {
    if (P->hgraphs.size() >= 4) {
      cudaGraphExecDestroy(P->hgraphs.front().exec);
      P->hgraphs.erase(P->hgraphs.begin());
    }
    cudaGraph_t g;
    ctx->stream = P->gstream;
    DS_CUDA(cudaStreamBeginCapture(P->gstream, cudaStreamCaptureModeThreadLocal));
    const int64_t l0 = ctx->launches;
    rc = issue_apply(P, P->hio_fm, P->hio_um, nrhs, nullptr, 0, -1, 3, &hio);
    cudaError_t e = cudaStreamEndCapture(P->gstream, &g);
    ctx->stream = user;
    if (rc) {
      P->slots_dirty = true;
      return rc;
    }
    if (e != cudaSuccess) return ds_fail(DS_ECUDA, std::string("graph capture: ") + cudaGetErrorString(e));
    ds_plan::HGraph h{f_host, u_host, nrhs, nullptr, ctx->launches - l0};
    DS_CUDA(cudaGraphInstantiate(&h.exec, g, cudaGraphInstantiateFlagUseNodePriority));
    cudaGraphDestroy(g);
    ctx->launches = l0;
    P->hgraphs.push_back(h);
    G = &P->hgraphs.back();
  }
  DS_CUDA(cudaGraphLaunch(G->exec, P->gstream));
  DS_CUDA(cudaEventRecord(P->gev_out, P->gstream));
  DS_CUDA(cudaStreamWaitEvent(user, P->gev_out, 0));
  ctx->launches += G->launches;
  P->last_launches = G->launches;
  return DS_OK;
}

static int ddm_apply(ds_ctx *ctx, ds_plan *P, const ds_cplx *f, ds_cplx *u, int32_t nrhs,
                     ds_cplx *partials, bool outer) {
  if (ctx && P && f && u)
    if (int rc0 = set_io(P, f, u, ctx->stream)) return rc0;
  if (!ctx || !P || !f || !u) return ds_fail(DS_ECONFIG, "ds_ddm_apply: null argument");
  if (nrhs < 1 || nrhs > P->nrhs_max)
    return ds_fail(DS_ECONFIG, "ds_ddm_apply: nrhs exceeds the plan's nrhs_max");
  if (P->nranks > 1)
    return ds_fail(DS_ECONFIG, "ds_ddm_apply: a sharded plan runs through ds_ddm_apply_range");
  if (ctx != P->ctx) P->ctx = ctx;
  int rc = patch_tables(P, nrhs);
  if (rc) return rc;
  if (P->slots_dirty) {
    for (auto &b : P->slot_bufs) DS_CUDA(cudaMemsetAsync(b.first, 0, b.second, ctx->stream));
    P->slots_dirty = false;
  }
  if (P->use_graph && !P->profiling && !partials) {  // per-sweep partials: fresh buffers, eager
    // capture / replay on a private stream (the caller's stream may be the
    // legacy default stream, which cannot be captured), ordered by events
    if (!P->gstream) {
      DS_CUDA(cudaStreamCreateWithFlags(&P->gstream, cudaStreamNonBlocking));
      DS_CUDA(cudaEventCreateWithFlags(&P->gev_in, cudaEventDisableTiming));
      DS_CUDA(cudaEventCreateWithFlags(&P->gev_out, cudaEventDisableTiming));
    }
    cudaStream_t user = ctx->stream;
    // the graph reads u through d_io and f as a kernel parameter
    bool match = P->graph && P->graph_f == f && P->graph_nrhs == nrhs &&
                 P->graph_partials == partials && P->graph_outer == outer;
    DS_CUDA(cudaEventRecord(P->gev_in, user));
    DS_CUDA(cudaStreamWaitEvent(P->gstream, P->gev_in, 0));
    if (!match) {
      if (P->graph) {
        cudaGraphExecDestroy(P->graph);
        P->graph = nullptr;
      }
      cudaGraph_t g;
      ctx->stream = P->gstream;
      DS_CUDA(cudaStreamBeginCapture(P->gstream, cudaStreamCaptureModeThreadLocal));
      int64_t l0 = ctx->launches;
      rc = issue_apply(P, (const cplx *)f, (cplx *)u, nrhs, (cplx *)partials, 0, -1, 3, nullptr, outer);
      cudaError_t e = cudaStreamEndCapture(P->gstream, &g);
      ctx->stream = user;
      if (rc) {
        P->slots_dirty = true;
        return rc;
      }
      if (e != cudaSuccess) return ds_fail(DS_ECUDA, std::string("graph capture: ") + cudaGetErrorString(e));
      DS_CUDA(cudaGraphInstantiate(&P->graph, g, cudaGraphInstantiateFlagUseNodePriority));
      cudaGraphDestroy(g);
      P->graph_f = f;
      P->graph_u = u;
      P->graph_nrhs = nrhs;
      P->graph_partials = partials;
      P->graph_outer = outer;
      ctx->launches = l0;
    }
    DS_CUDA(cudaGraphLaunch(P->graph, P->gstream));
    DS_CUDA(cudaEventRecord(P->gev_out, P->gstream));
    DS_CUDA(cudaStreamWaitEvent(user, P->gev_out, 0));
    ctx->launches += P->last_launches;
    return DS_OK;
  }
  rc = issue_apply(P, (const cplx *)f, (cplx *)u, nrhs, (cplx *)partials, 0, -1, 3, nullptr, outer);
  if (rc) P->slots_dirty = true;
  return rc;
}

extern "C" int ds_ddm_apply(ds_ctx *ctx, ds_plan *P, const ds_cplx *f, ds_cplx *u, int32_t nrhs,
                            ds_cplx *partials) {
  return ddm_apply(ctx, P, f, u, nrhs, partials, false);
}

// the same on RHS-outer [R][N] device buffers (no layout transposes)
extern "C" int ds_ddm_apply_outer(ds_ctx *ctx, ds_plan *P, const ds_cplx *f, ds_cplx *u,
                                  int32_t nrhs) {
  return ddm_apply(ctx, P, f, u, nrhs, nullptr, true);
}

extern "C" int ds_plan_shard_info(const ds_plan *P, void **slot_base, int64_t *slot_bytes,
                                  void **flag_base, int64_t *flag_bytes) {
  if (!P) return ds_fail(DS_ECONFIG, "null plan");
  if (slot_base) *slot_base = P->slot_base;
  if (slot_bytes) *slot_bytes = (int64_t)P->slot_bytes;
  if (flag_base) *flag_base = P->flags;
  if (flag_bytes) *flag_bytes = (int64_t)(P->flag_words * sizeof(int));
  return DS_OK;
}

extern "C" int ds_plan_set_peers(ds_ctx *ctx, ds_plan *P, int32_t nranks, void *const *slot_bases,
                                 void *const *flag_bases) {
  if (!ctx || !P || !slot_bases || !flag_bases) return ds_fail(DS_ECONFIG, "ds_plan_set_peers: null argument");
  if (nranks != P->nranks) return ds_fail(DS_ECONFIG, "ds_plan_set_peers: rank count mismatch");
  for (int r = 0; r < nranks; ++r)
    if (!slot_bases[r] || !flag_bases[r]) return ds_fail(DS_ECONFIG, "ds_plan_set_peers: null peer pointer");
  std::vector<XferDev> hx = P->h_xfers;
  for (size_t i = 0; i < hx.size(); ++i)
    if (hx[i].use > 0) hx[i].slot = (cplx *)slot_bases[hx[i].owner] + P->xfer_slot_off[i];
  DS_CUDA(cudaMemcpy(P->xfers, hx.data(), sizeof(XferDev) * hx.size(), cudaMemcpyHostToDevice));
  P->h_xfers = hx;
  P->patched_nrhs = 0;  // XferRec slot pointers are rebuilt from h_xfers
  if (!P->d_flag_bases) {
    void *mem;
    if (plan_alloc(P, &mem, sizeof(int *) * nranks)) return ds_fail(DS_ECUDA, "ds_plan_set_peers: alloc");
    P->d_flag_bases = (int **)mem;
  }
  DS_CUDA(cudaMemcpy(P->d_flag_bases, flag_bases, sizeof(int *) * nranks, cudaMemcpyHostToDevice));
  P->peers_set = true;
  return DS_OK;
}

extern "C" int ds_plan_slot(ds_ctx *ctx, const ds_plan *P, int32_t use_sweep, int32_t target,
                            int32_t dir, int32_t *lo, int32_t *shape, ds_cplx *out_dev,
                            int64_t out_elems, int32_t nrhs) {
  if (!ctx || !P || !lo || !shape) return ds_fail(DS_ECONFIG, "ds_plan_slot: null argument");
  auto it = P->slot_by_key.find(std::make_tuple(use_sweep - 1, target, dir));
  if (it == P->slot_by_key.end()) return ds_fail(DS_ECONFIG, "ds_plan_slot: no such payload slot");
  int64_t n = 1;
  for (int a = 0; a < 3; ++a) {
    lo[a] = it->second.lo[a];
    shape[a] = it->second.shape[a];
    n *= shape[a];
  }
  if (!out_dev) return DS_OK;
  if (nrhs < 1 || nrhs > P->nrhs_max || out_elems < n * nrhs)
    return ds_fail(DS_ECONFIG, "ds_plan_slot: output buffer too small or bad nrhs");
  DS_CUDA(cudaMemcpyAsync(out_dev, it->second.data, sizeof(cplx) * n * nrhs,
                          cudaMemcpyDeviceToDevice, ctx->stream));
  return DS_OK;
}

extern "C" int32_t ds_plan_nlaunch(const ds_plan *P) {
  return P ? (int32_t)P->vstep_off.size() - 1 : -1;
}

extern "C" int ds_ddm_apply_range(ds_ctx *ctx, ds_plan *P, const ds_cplx *f, ds_cplx *u, int32_t nrhs,
                                  int32_t l0, int32_t l1, int32_t mode) {
  if (!ctx || !P || !f || !u) return ds_fail(DS_ECONFIG, "ds_ddm_apply_range: null argument");
  if (nrhs < 1 || nrhs > P->nrhs_max)
    return ds_fail(DS_ECONFIG, "ds_ddm_apply_range: nrhs exceeds the plan's nrhs_max");
  const int nq = (int)P->vstep_off.size() - 1;
  if (l0 < 0 || l1 < l0 || l1 > nq) return ds_fail(DS_ECONFIG, "ds_ddm_apply_range: bad launch range");
  if (!P->peers_set) return ds_fail(DS_ECONFIG, "ds_ddm_apply_range: ds_plan_set_peers not called");
  if (ctx != P->ctx) P->ctx = ctx;
  if (int rc0 = set_io(P, f, u, ctx->stream)) return rc0;
  int rc = patch_tables(P, nrhs);
  if (rc) return rc;
  if (P->slots_dirty) {
    for (auto &b : P->slot_bufs) DS_CUDA(cudaMemsetAsync(b.first, 0, b.second, ctx->stream));
    P->slots_dirty = false;
  }
  rc = issue_apply(P, (const cplx *)f, (cplx *)u, nrhs, nullptr, l0, l1, mode);
  if (rc) P->slots_dirty = true;
  return rc;
}

extern "C" int ds_ddm_enable_graph(ds_ctx *ctx, ds_plan *P, int32_t enable) {
  if (!P) return ds_fail(DS_ECONFIG, "null plan");
  (void)ctx;
  P->use_graph = enable != 0;
  if (!P->use_graph && P->graph) {
    cudaGraphExecDestroy(P->graph);
    P->graph = nullptr;
  }
  return DS_OK;
}

extern "C" int ds_ddm_counters(ds_ctx *ctx, ds_plan *P, int32_t nrhs, int32_t *nonzero,
                               int32_t *discarded, int32_t *visit_nonzero,
                               int32_t *visit_consumed, int32_t *visit_emitted,
                               int32_t *visit_cut) {
  if (!ctx || !P || nrhs < 1 || nrhs > P->nrhs_max)
    return ds_fail(DS_ECONFIG, "ds_ddm_counters: bad argument");
  // the flag block (own | nz | arr_cnt | arr_cut | emit_cnt | discard) is
  // contiguous for this stride: one device-to-host copy (ordered after the
  // application on the context stream)
  Flags F = flags_view(P, nrhs);
  const size_t per = (size_t)P->nsweeps * P->nsub * nrhs;
  const size_t own_n = (size_t)P->nsub * nrhs;
  const size_t words = own_n + 4 * per + nrhs;
  std::vector<int> h(words);
  DS_CUDA(cudaMemcpyAsync(h.data(), F.own_nz, sizeof(int) * words, cudaMemcpyDeviceToHost, ctx->stream));
  DS_CUDA(cudaStreamSynchronize(ctx->stream));
  const int *own = h.data(), *nz = own + own_n, *cnt2 = nz + per, *cut = cnt2 + per,
            *em = cut + per, *disc = em + per;
  if (nonzero) {
    for (int r = 0; r < nrhs; ++r) nonzero[r] = 0;
    for (size_t i = 0; i < per; ++i) nonzero[i % nrhs] += nz[i] ? 1 : 0;
  }
  if (discarded) memcpy(discarded, disc, sizeof(int) * nrhs);
  if (visit_nonzero)
    for (size_t i = 0; i < per; ++i) visit_nonzero[i] = nz[i] ? 1 : 0;
  if (visit_consumed) memcpy(visit_consumed, cnt2, sizeof(int) * per);
  if (visit_emitted) memcpy(visit_emitted, em, sizeof(int) * per);
  if (visit_cut) {
    for (size_t i = 0; i < per; ++i) {
      size_t w = i / own_n, rem = i % own_n;
      bool has_own = (w == 0) && own[rem];
      visit_cut[i] = (has_own || cnt2[i] == 0) ? 0 : (cut[i] & CUT_ALL);
    }
  }
  return DS_OK;
}

extern "C" int ds_plan_set_profiling(ds_plan *P, int32_t enable) {
  if (!P) return ds_fail(DS_ECONFIG, "null plan");
  P->profiling = enable != 0;
  P->ev_used = 0;
  return DS_OK;
}

// Sum of event-bracketed durations per kernel class since the last reset
// (blocks the host).  ms[5], count[5]: assemble, solve (K3 / modal
// transforms), accumulate, transfer, modal recurrences.
extern "C" int ds_plan_kernel_times(ds_plan *P, double *ms, int64_t *count, int32_t reset) {
  if (!P) return ds_fail(DS_ECONFIG, "null plan");
  for (int c = 0; c < 5; ++c) {
    if (ms) ms[c] = 0.0;
    if (count) count[c] = 0;
  }
  if (P->ev_used > 0) DS_CUDA(cudaEventSynchronize(P->ev[P->ev_used - 1]));
  for (size_t i = 0; i + 1 < P->ev_used; ++i) {
    int c = P->ev_class[i];
    if (c < 0 || c > 4) continue;
    float t = 0.f;
    DS_CUDA(cudaEventElapsedTime(&t, P->ev[i], P->ev[i + 1]));
    if (ms) ms[c] += t;
    if (count) count[c] += 1;
  }
  if (reset) P->ev_used = 0;
  return DS_OK;
}


// ---------------------------------------------------------------------
// One application of an RHS-grouped batch from pinned host buffers: groups
// g = 0..G-1 (identical plans over contiguous RHS ranges) sweep concurrently
// on their own streams (the device path's GroupedPlan), while one shared
// copy pipeline moves each source box once (all RHS) and transposes its
// rows into every group's RHS-minor buffer, and downloads each result box
// once both groups have finalized it.
struct GroupHost {
  cplx *fo = nullptr, *uo = nullptr;  // RHS-outer staging [R][N]
  size_t cap = 0;                     // complex elements
  std::vector<cudaStream_t> gs;
  std::vector<cudaEvent_t> gjoin;
  struct G {
    const void *fh;
    void *uh;
    int nrhs, groups;
    cudaGraphExec_t exec;
    int64_t launches;
    int64_t gen;  // g_patch_gen at capture
    std::vector<const ds_plan *> plans;
  };
  std::vector<G> graphs;
};
static GroupHost *g_group_host = nullptr;  // one per process (plans of one device)

static int box_transpose(ds_plan *P0, const HioBox &B, int R, const cplx *src, cplx *dst, int to_minor,
                         cudaStream_t cs) {
  const int64_t N = P0->nnodes, S1 = P0->gcounts[2], S0 = (int64_t)P0->gcounts[1] * S1;
  const int L = (int)((B.c1 - B.c0) * S1), runs = B.a1 - B.a0;
  if (L <= 0 || runs <= 0 || R <= 0) return DS_OK;
  const int64_t base0 = (int64_t)B.a0 * S0 + (int64_t)B.c0 * S1;
  const dim3 grid((unsigned)(((R + 31) / 32) * ((L + 31) / 32)), runs);
  k_box_transpose<<<grid, dim3(32, 8), 0, cs>>>(R, L, N, base0, S0, src, dst, to_minor);
  P0->ctx->launches++;
  DS_CHECK_LAUNCH();
  return DS_OK;
}

static int box_copy(ds_plan *P0, const HioBox &B, int R, cplx *host, cplx *dev, bool h2d, cudaStream_t cs) {
  const int64_t S1 = P0->gcounts[2], S0 = (int64_t)P0->gcounts[1] * S1;
  const int L = (int)((B.c1 - B.c0) * S1), runs = B.a1 - B.a0;
  if (L <= 0 || runs <= 0) return DS_OK;
  cudaMemcpy3DParms m = {};
  cudaPitchedPtr hp = make_cudaPitchedPtr(host, sizeof(cplx) * S0, sizeof(cplx) * S0, P0->gcounts[0]);
  cudaPitchedPtr dp = make_cudaPitchedPtr(dev, sizeof(cplx) * S0, sizeof(cplx) * S0, P0->gcounts[0]);
  const cudaPos at = make_cudaPos(sizeof(cplx) * B.c0 * S1, B.a0, 0);
  m.extent = make_cudaExtent(sizeof(cplx) * L, runs, R);
  m.srcPtr = h2d ? hp : dp;
  m.dstPtr = h2d ? dp : hp;
  m.srcPos = at;
  m.dstPos = at;
  m.kind = h2d ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost;
  DS_CUDA(cudaMemcpy3DAsync(&m, cs));
  return DS_OK;
}

static int issue_groups(ds_ctx *ctx, ds_plan *const *plans, int G, const cplx *fh, cplx *uh, int nrhs,
                        GroupHost *GH) {
  ds_plan *P0 = plans[0];
  cudaStream_t st = ctx->stream;
  const int64_t N = P0->nnodes;
  std::vector<int> r0(G + 1);
  for (int g = 0; g <= G; ++g) r0[g] = (int)((int64_t)nrhs * g / G);
  DS_CUDA(cudaEventRecord(P0->hio_fork, st));
  DS_CUDA(cudaStreamWaitEvent(P0->cstream, P0->hio_fork, 0));
  DS_CUDA(cudaStreamWaitEvent(P0->cstream2, P0->hio_fork, 0));
  for (int g = 0; g < G; ++g) DS_CUDA(cudaStreamWaitEvent(GH->gs[g], P0->hio_fork, 0));
  // uploads: each box once (all RHS), transposed into every group's buffer
  for (int k = 0; k < (int)P0->hio_boxes.size(); ++k) {
    cudaStream_t cs = (k & 1) ? P0->cstream2 : P0->cstream;
    const HioBox &B = P0->hio_boxes[k];
    if (int rc = box_copy(P0, B, nrhs, (cplx *)fh, GH->fo, true, cs)) return rc;
    for (int g = 0; g < G; ++g)
      if (int rc = box_transpose(P0, B, r0[g + 1] - r0[g], GH->fo + (int64_t)r0[g] * N, plans[g]->hio_fm, 1, cs))
        return rc;
    DS_CUDA(cudaEventRecord(P0->hio_ev_in[k], cs));
  }
  // the groups' sweeps
  for (int g = 0; g < G; ++g) {
    HostIO h{fh, uh};
    h.ext = true;
    h.ev_in = P0->hio_ev_in.data();
    h.ev_out = plans[g]->hio_ev_out.data();
    ctx->stream = GH->gs[g];
    plans[g]->ctx = ctx;
    int rc = issue_apply(plans[g], plans[g]->hio_fm, plans[g]->hio_um, r0[g + 1] - r0[g], nullptr, 0, -1, 3, &h);
    ctx->stream = st;
    if (rc) return rc;
    DS_CUDA(cudaEventRecord(GH->gjoin[g], GH->gs[g]));
  }
  // downloads: each box once every group has finalized it
  int nout = 0;
  auto download = [&](int c, bool after_groups) -> int {
    cudaStream_t cs = (nout++ & 1) ? P0->cstream2 : P0->cstream;
    for (int g = 0; g < G; ++g)
      DS_CUDA(cudaStreamWaitEvent(cs, after_groups ? GH->gjoin[g] : plans[g]->hio_ev_out[c], 0));
    const HioBox &B = P0->hio_oboxes[c];
    for (int g = 0; g < G; ++g)
      if (int rc = box_transpose(P0, B, r0[g + 1] - r0[g], plans[g]->hio_um, GH->uo + (int64_t)r0[g] * N, 0, cs))
        return rc;
    return box_copy(P0, B, nrhs, uh, GH->uo, false, cs);
  };
  const int nq = (int)P0->vstep_off.size() - 1;
  for (int q = 0; q < nq; ++q)
    for (int c : P0->hio_out_at[q])
      if (int rc = download(c, false)) return rc;
  for (int c : P0->hio_out_early)
    if (int rc = download(c, true)) return rc;
  for (int g = 0; g < G; ++g) DS_CUDA(cudaStreamWaitEvent(st, GH->gjoin[g], 0));
  DS_CUDA(cudaEventRecord(P0->hio_join, P0->cstream));
  DS_CUDA(cudaStreamWaitEvent(st, P0->hio_join, 0));
  DS_CUDA(cudaEventRecord(P0->hio_join2, P0->cstream2));
  DS_CUDA(cudaStreamWaitEvent(st, P0->hio_join2, 0));
  return DS_OK;
}

extern "C" int ds_ddm_apply_host_groups(ds_ctx *ctx, ds_plan *const *plans, int32_t G,
                                        const ds_cplx *f_host, ds_cplx *u_host, int32_t nrhs) {
  if (!ctx || !plans || G < 1 || G > 16 || !f_host || !u_host)
    return ds_fail(DS_ECONFIG, "ds_ddm_apply_host_groups: bad argument");
  ds_plan *P0 = plans[0];
  for (int g = 0; g < G; ++g) {
    ds_plan *P = plans[g];
    if (!P || P->nranks > 1 || P->vstep_off.size() != P0->vstep_off.size() || P->nnodes != P0->nnodes)
      return ds_fail(DS_ECONFIG, "ds_ddm_apply_host_groups: plans must be identical unsharded plans");
    const int Rg = (int)((int64_t)nrhs * (g + 1) / G - (int64_t)nrhs * g / G);
    if (Rg < 1 || Rg > P->nrhs_max) return ds_fail(DS_ECONFIG, "ds_ddm_apply_host_groups: group too large");
    P->ctx = ctx;
    if (int rc = patch_tables(P, Rg)) return rc;
    if (int rc = hio_setup(P)) return rc;
    if (P->slots_dirty) {
      for (auto &b : P->slot_bufs) DS_CUDA(cudaMemsetAsync(b.first, 0, b.second, ctx->stream));
      P->slots_dirty = false;
    }
    if (int rc = set_io(P, P->hio_fm, P->hio_um, ctx->stream)) return rc;
  }
  if (!g_group_host) g_group_host = new GroupHost();
  GroupHost *GH = g_group_host;
  const size_t need = (size_t)P0->nnodes * nrhs;
  if (need > GH->cap) {
    DS_CUDA(cudaStreamSynchronize(ctx->stream));
    for (auto &gg : GH->graphs) cudaGraphExecDestroy(gg.exec);
    GH->graphs.clear();
    if (GH->fo) cudaFree(GH->fo);
    if (GH->uo) cudaFree(GH->uo);
    GH->fo = GH->uo = nullptr;
    GH->cap = 0;
    DS_CUDA(cudaMalloc(&GH->fo, sizeof(cplx) * need));
    DS_CUDA(cudaMalloc(&GH->uo, sizeof(cplx) * need));
    GH->cap = need;
  }
  while ((int)GH->gs.size() < G) {
    cudaStream_t s;
    cudaEvent_t e;
    DS_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    DS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    GH->gs.push_back(s);
    GH->gjoin.push_back(e);
  }
  if (!P0->use_graph || P0->profiling) return issue_groups(ctx, plans, G, (const cplx *)f_host, (cplx *)u_host, nrhs, GH);
  if (!P0->gstream) {
    DS_CUDA(cudaStreamCreateWithFlags(&P0->gstream, cudaStreamNonBlocking));
    DS_CUDA(cudaEventCreateWithFlags(&P0->gev_in, cudaEventDisableTiming));
    DS_CUDA(cudaEventCreateWithFlags(&P0->gev_out, cudaEventDisableTiming));
  }
  cudaStream_t user = ctx->stream;
  GroupHost::G *hit = nullptr;
  for (auto &gg : GH->graphs)
    if (gg.fh == f_host && gg.uh == u_host && gg.nrhs == nrhs && gg.groups == G && gg.gen == g_patch_gen &&
        std::equal(gg.plans.begin(), gg.plans.end(), plans))
      hit = &gg;
  DS_CUDA(cudaEventRecord(P0->gev_in, user));
  DS_CUDA(cudaStreamWaitEvent(P0->gstream, P0->gev_in, 0));
  if (!hit) {
    if (GH->graphs.size() >= 4) {
      cudaGraphExecDestroy(GH->graphs.front().exec);
      GH->graphs.erase(GH->graphs.begin());
    }
    cudaGraph_t gr;
    ctx->stream = P0->gstream;
    DS_CUDA(cudaStreamBeginCapture(P0->gstream, cudaStreamCaptureModeThreadLocal));
    const int64_t l0 = ctx->launches;
    int rc = issue_groups(ctx, plans, G, (const cplx *)f_host, (cplx *)u_host, nrhs, GH);
    cudaError_t e = cudaStreamEndCapture(P0->gstream, &gr);
    ctx->stream = user;
    if (rc) {
      for (int g = 0; g < G; ++g) plans[g]->slots_dirty = true;
      return rc;
    }
    if (e != cudaSuccess) return ds_fail(DS_ECUDA, std::string("graph capture: ") + cudaGetErrorString(e));
    GroupHost::G h{f_host, u_host, nrhs, G, nullptr, ctx->launches - l0, g_patch_gen,
                   std::vector<const ds_plan *>(plans, plans + G)};
    DS_CUDA(cudaGraphInstantiate(&h.exec, gr, cudaGraphInstantiateFlagUseNodePriority));
    cudaGraphDestroy(gr);
    ctx->launches = l0;
    GH->graphs.push_back(h);
    hit = &GH->graphs.back();
  }
  DS_CUDA(cudaGraphLaunch(hit->exec, P0->gstream));
  DS_CUDA(cudaEventRecord(P0->gev_out, P0->gstream));
  DS_CUDA(cudaStreamWaitEvent(user, P0->gev_out, 0));
  ctx->launches += hit->launches;
  return DS_OK;
}
