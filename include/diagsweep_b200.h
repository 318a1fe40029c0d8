/*
 * diagsweep_b200.h — C-ABI of the B200-native diagonal-sweeping DDM hot path.
 *
 * Plain C types only (no torch / C++ types cross this boundary).  Every
 * buffer argument named `*_dev` is a device pointer owned by the caller;
 * the library owns factor storage and plan workspaces behind opaque
 * handles and frees them in the matching *_destroy call.  All calls are
 * asynchronous on the context's stream unless stated; they block the host
 * only where a result must be read back (ds_fact_create's pivot check,
 * ds_ddm_counters, ds_*_host helpers).
 *
 * Status codes: 0 ok; < 0 configuration error (bad shape/window/argument,
 * maps to diagsweep.errors.ConfigurationError; -2 = model error, e.g. a
 * nonpositive velocity, maps to ModelError); > 0 solver error (zero
 * pivot, non-finite factor, CUDA failure; maps to SolverError).  The
 * message of the last failure on the calling thread is ds_last_error().
 *
 * Complex values are complex128: interleaved (re, im) float64, i.e. the
 * memory layout of numpy.complex128 / torch.complex128.
 *
 * Layout convention ("RHS-minor"): a batched field over a window of shape
 * (n0, n1[, n2]) with R right-hand sides is stored [n0][n1][n2][R], node
 * C-order outermost, the RHS index fastest.  The Python host converts from
 * the reference's [R, *counts] batches at the API boundary.
 *
 * Reference interfaces replaced (the reference is pure Python; these are the
 * calls a ctypes binding of its hot path makes — see INTEGRATION.md):
 *   ds_op_*        <- DiscreteOperator / assemble_operator / .apply
 *                     (diagsweep/pml.py:75-188, :216-266)
 *   ds_fact_*      <- factorize / FactorizationCache.get(op).solve(rhs)
 *                     (diagsweep/subdomain.py:43-179)
 *   ds_plan_*,
 *   ds_ddm_apply   <- diagonal_sweep_solve (diagsweep/ddm.py:212-291) incl.
 *                     restrict_source (:168-195), _accumulate (:206-209),
 *                     cut bookkeeping (:82-110), psi (transfer.py:100-155)
 *   ds_vec_*       <- the vector kernels of gmres (diagsweep/krylov.py:40-147)
 */
#ifndef DIAGSWEEP_B200_H
#define DIAGSWEEP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DS_ABI_VERSION 7

#if defined(__GNUC__)
#define DS_API __attribute__((visibility("default")))
#else
#define DS_API
#endif

typedef struct ds_ctx ds_ctx;
typedef struct ds_op ds_op;
typedef struct ds_fact ds_fact;
typedef struct ds_plan ds_plan;

typedef struct {
  double re, im;
} ds_cplx;

/* ---------------------------------------------------------------- context */

DS_API int ds_abi_version(void);
DS_API const char *ds_last_error(void);

/* `stream` is a cudaStream_t (NULL = legacy default stream). */
DS_API int ds_ctx_create(int device, void *stream, ds_ctx **out);
DS_API int ds_ctx_set_stream(ds_ctx *ctx, void *stream);
DS_API int ds_ctx_synchronize(ds_ctx *ctx);
DS_API int ds_ctx_destroy(ds_ctx *ctx);
/* Kernels this library has launched on `ctx` so far (graph replays count
 * their captured launches).  Diagnostic: bench.py's `gpu_launches`. */
DS_API int64_t ds_ctx_launches(const ds_ctx *ctx);
/* (ABI 7) Complex multiply-adds the modal transforms (K3m-T) executed on
 * `ctx` while the option "count_work" was 1: per tile, valid rows x valid
 * columns x the K extent actually multiplied (exact-zero RHS columns and
 * skipped all-zero K-chunks not counted).  Synchronizes the context's
 * stream; `reset` != 0 zeroes the counter.  Measurement only: bench.py's
 * roofline numerator (the reference has no counterpart). */
DS_API int ds_ctx_work(ds_ctx *ctx, int64_t *cmacs, int32_t reset);
/* Variant / tuning options of a context (ABI 5), read at every launch (a
 * plan's captured CUDA graph keeps the choices it was recorded with).
 * Defaults are the measured-best choices; a DS_<NAME> environment variable
 * read at ds_ctx_create overrides a default.  Names and values:
 *   "k1" stencil rows per thread 2 / 4 (default) / 8 / 16, 0 = 32x8 tiles;
 *   "combine" basis-update elements per thread 1 / 2 (default);
 *   "k4" transfer kernel 0 (default: 2D v3, 3D v2) / 1 / 2 / 3;
 *   "k4_rv", "k6_rv" RHS columns per thread (1, 2, 4, 8);
 *   "pdl" programmatic dependent launch 1 / 0 (process-wide);
 *   "k5_side" beta00 accumulation on a side stream 1 / 0;
 *   "staged" stage-per-launch block solve for small slabs too 0 / 1;
 *   "k3g_mma" staged block product on DMMA 1 / 0; "stage_rows";
 *   "k3_warps" 4 / 8, "k3_rc_min", "k3_rc_max", "k3_cluster" 0 / 8 / 16:
 *     the cluster block solve's configuration search;
 *   "hio_dstreams" download streams of ds_ddm_apply_host (>= 2);
 *   "kskip" forward transforms skip all-zero K-chunks 1 / 0;
 *   "r3_cols" (mode, RHS) columns per block of the segmented mode-wise
 *     recurrences 16 (default) / 32;
 *   "k2b_groups" concurrent groups of a blocked-factorization batch 1 .. 8
 *     (default 2);
 *   "count_work" 0 / 1 (see ds_ctx_work).
 * Unknown names or values: < 0. */
DS_API int ds_ctx_set_option(ds_ctx *ctx, const char *name, int32_t value);
DS_API int ds_ctx_get_option(const ds_ctx *ctx, const char *name, int32_t *value);

/* --------------------------------------------------------------- operator
 * One assembled PML Helmholtz operator on a window (pml.py:75-188).
 * c_lo[a], c_hi[a]: host arrays of length shape[a] (complex128) — the
 * couplings 1/(alpha_node*alpha_face*h^2) computed on the host bit-exactly.
 * kappa2_kind: 0 'const' (1 value), 1 'axis' (shape[kappa2_axis] values),
 * 2 'full' (prod(shape) values, C-order).  Host pointers; copied. */
typedef struct {
  int32_t dim;
  int32_t shape[3];
  const ds_cplx *c_lo[3];
  const ds_cplx *c_hi[3];
  int32_t kappa2_kind;
  int32_t kappa2_axis;
  const double *kappa2;
} ds_op_desc;

DS_API int ds_op_create(ds_ctx *ctx, const ds_op_desc *desc, ds_op **out);
DS_API int ds_op_destroy(ds_op *op);

/* out = L v on `region` (zero outside region), pml.py:135-159.
 * region_lo: offsets of the region inside the operator window;
 * region_shape: its shape.  layout 0: v_dev/out_dev are RHS-minor
 * [*region_shape][nrhs]; layout 1: RHS-outer [nrhs][*region_shape]. */
DS_API int ds_op_apply(ds_ctx *ctx, const ds_op *op, const ds_cplx *v_dev,
                ds_cplx *out_dev, int32_t nrhs, const int32_t *region_lo,
                const int32_t *region_shape, int32_t layout);

/* ---------------------------------------------------------- factorization
 * Block-tridiagonal LU of n operators along each window's longest axis
 * (first on ties): S_0 = D_0, S_k = D_k - (l_k u_{k-1}) S_{k-1}^{-1}; the
 * dense inverses S_k^{-1} (complex128, Gauss-Jordan with partial pivoting)
 * are stored.  Replaces SeparableFactorization / SparseLuFactorization
 * (subdomain.py:43-133).  Blocks until done; returns > 0 on a zero pivot or
 * a non-finite inverse. */
DS_API int ds_fact_create(ds_ctx *ctx, ds_op *const *ops, int32_t n, ds_fact **out);
/* Per-operator layout info: block axis, number of blocks, block size,
 * factor bytes. */
DS_API int ds_fact_info(const ds_fact *fact, int32_t i, int32_t *block_axis,
                 int32_t *nb, int32_t *m, int64_t *bytes);
/* x = A_i^{-1} rhs for one operator; rhs_dev/x_dev: [*window][nrhs]
 * (subdomain.py:77-106 `.solve`). */
DS_API int ds_fact_solve(ds_ctx *ctx, const ds_fact *fact, int32_t i,
                  const ds_cplx *rhs_dev, ds_cplx *x_dev, int32_t nrhs);
DS_API int ds_fact_destroy(ds_fact *fact);

/* Modal factorization of separable operators (kappa^2 'const' or 'axis'):
 * the drop-in for SeparableFactorization (subdomain.py:43-96), which
 * triangularizes the per-axis 1D tridiagonals (Schur) and solves a
 * triangular Sylvester equation.  Here the 1D tridiagonal T_a of every
 * in-slab axis a (the window axes other than the block axis, C order; one in
 * 2D, two in 3D; T_a includes kappa^2 when kappa^2 varies along a) is
 * diagonalised, T_a = V_a diag(lambda_a) V_a^{-1}, so the operator becomes
 * one scalar tridiagonal system along the block axis per in-slab mode j:
 *     (T_ba + kappa^2 + mu_j) y_j = (W g)_j,   mu_j = sum_a lambda_a(j_a).
 * The device computes and stores the mode-wise LU pivots; a solve is two
 * (2D) or four (3D) batched complex GEMMs on the FP64 tensor cores plus the
 * mode-wise recurrences.  The host supplies the eigen-decompositions
 * (row-major n_a x n_a V_a, V_a^{-1}, and lambda_a; host arrays, copied).
 * block_axis must be the layout's (longest axis, first on ties).  Returns
 * > 0 on a zero or non-finite pivot. */
typedef struct {
  int32_t block_axis;
  int32_t naxes;              /* dim - 1 */
  const ds_cplx *v[2];        /* V_a */
  const ds_cplx *vinv[2];     /* V_a^{-1} */
  const ds_cplx *lambda[2];   /* eigenvalues of T_a */
} ds_modal_desc;

DS_API int ds_fact_create_modal(ds_ctx *ctx, ds_op *const *ops, int32_t n,
                                const ds_modal_desc *descs, ds_fact **out);
/* 0: block-LU factors (ds_fact_create), 1: modal (ds_fact_create_modal) */
DS_API int ds_fact_kind(const ds_fact *fact, int32_t i);

/* Factor pool (ABI 5; out-of-core block LU for factor sets larger than HBM,
 * e.g. config 5: 638 GB of dense block inverses).  Lays out the n operators
 * (block axis, blocks, block size as ds_fact_create) without factoring them
 * and allocates nslots factor slots of the largest operator's size.
 * ds_fact_pool_load factors operator i into `slot` (the K2b blocked path,
 * bitwise the factors ds_fact_create computes), evicting the slot's previous
 * operator; it blocks and returns > 0 on a zero / non-finite pivot.
 * ds_fact_solve works on resident operators only.  3D (large-slab)
 * operators only. */
DS_API int ds_fact_create_pool(ds_ctx *ctx, ds_op *const *ops, int32_t n, int32_t nslots,
                               ds_fact **out);
DS_API int ds_fact_pool_load(ds_ctx *ctx, ds_fact *fact, int32_t i, int32_t slot);
/* n loads at once (operators idx[q] into slots[q], distinct): every chain of
 * the batch advances together, sharing the panel steps' latency. */
DS_API int ds_fact_pool_load_many(ds_ctx *ctx, ds_fact *fact, int32_t n, const int32_t *idx,
                                  const int32_t *slots);
/* slots, slot size, slot_owner[nslots] (operator index or -1; may be NULL),
 * factorizations run so far */
DS_API int ds_fact_pool_state(const ds_fact *fact, int32_t *nslots, int64_t *slot_bytes,
                              int32_t *slot_owner, int64_t *loads);

/* ------------------------------------------------------------- sweep plan
 * Static schedule of one diagonal-sweeping application (ddm.py:212-291),
 * built once by the host from the bit-exact partition / routing metadata.
 * All arrays are host arrays; copied into device tables.
 *
 * Subdomain s (C-order linear id over 1-based indices):
 *   win_lo/win_shape   [nsub*3]  its window (partition.py:83-90)
 *   own_lo/own_shape   [nsub*3]  restricted-source region (ddm.py:185-194)
 *   sup_lo/sup_shape   [nsub*3]  beta00 support (partition.py:135-150)
 *   beta00             concatenated per-axis beta00 ramps over the support,
 *                      axis a of s at beta00 + beta00_off[s*3+a]
 *   op_of_sub[s]       index into `ops`
 *   fact_of_sub[s], fact_index[s]  the factorization handle of subdomain s
 *                      and the operator index inside that handle
 * Sweeps (2^dim) and steps: visit order of sweep w is
 *   visit_sub[w*nsub + step_off[w*(nsteps+1)+t] ...
 *             w*nsub + step_off[w*(nsteps+1)+t+1]) for step t (sorted).
 * Transfers: for every (sweep w, subdomain s, direction k) with an in-range
 * target, xfer_use[(w*nsub+s)*ndir+k] = use sweep (1-based, 0 = discarded,
 * -1 = target out of range).  directions[ndir*3] in itertools.product
 * order (ddm.py:75-79).  Geometry per (s, k): band_lo/band_shape/ext_lo/
 * ext_shape [(s*ndir+k)*3], and the (1-beta) factors on ext per axis at
 * xfac + xfac_off[(s*ndir+k)*3+a] (ones on zero axes).
 * Launch schedule (optional, ABI 2): nlaunch = 0 runs the visits sweep by
 * sweep, step by step (the reference order).  nlaunch > 0 runs launch l over
 * the visits launch_visits[2*i] (0-based sweep), launch_visits[2*i+1]
 * (subdomain) for i in [launch_off[l], launch_off[l+1]); every visit exactly
 * once, each after the visits it depends on (its step predecessors and the
 * sources routed to it) and after any earlier writer of the same payload
 * slot (the host's list scheduler, _engine.launch_schedule).  Per-sweep
 * partials need nlaunch = 0.
 * Subdomain sharding (optional, ABI 3): nranks > 1
 * makes this plan rank `rank` of a sweep whose subdomain s is owned by rank
 * owner[s].  fact_of_sub may be NULL for subdomains this rank does not own;
 * the launch schedule (required) lists only owned visits, with the same
 * launch boundaries on every rank.  Payload slots live on the rank owning
 * their target; after ds_plan_set_peers, the transfer kernel writes payloads
 * and arrival flags of remote targets directly into the owner's memory
 * (peer / IPC-mapped pointers over NVLink) -- no separate exchange step.
 * Arrays are int32 unless noted. */
typedef struct {
  int32_t dim, nsub, nsweeps, nsteps, ndir, nrhs_max;
  int32_t grid_counts[3];
  int32_t part_counts[3];
  const int32_t *win_lo, *win_shape;
  const int32_t *own_lo, *own_shape;
  const int32_t *sup_lo, *sup_shape;
  const double *beta00;
  const int64_t *beta00_off;
  int32_t nops;
  ds_op *const *ops;
  const int32_t *op_of_sub;
  ds_fact *const *fact_of_sub;
  const int32_t *fact_index;
  const int32_t *visit_sub;
  const int32_t *step_off;
  const int32_t *directions;
  const int32_t *xfer_use;
  const int32_t *band_lo, *band_shape, *ext_lo, *ext_shape;
  const double *xfac;
  const int64_t *xfac_off;
  int32_t nlaunch;
  const int32_t *launch_off;
  const int32_t *launch_visits;
  int32_t nranks, rank;
  const int32_t *owner;
  /* Pooled factors (optional, ABI 5): when non-NULL, fact_of_sub[s] is a
   * factor pool (ds_fact_create_pool) and visit (sweep w, subdomain s) reads
   * its block inverses from pool slot visit_slot[w * nsub + s]; the caller
   * makes the slot hold s's factors (ds_fact_pool_load) before the launch
   * containing the visit runs (ds_ddm_apply_range, launch by launch). */
  const int32_t *visit_slot;
} ds_plan_desc;

DS_API int ds_plan_create(ds_ctx *ctx, const ds_plan_desc *desc, ds_plan **out);
DS_API int64_t ds_plan_workspace_bytes(const ds_plan *plan);
DS_API int ds_plan_destroy(ds_plan *plan);

/* One application of the diagonal-sweeping DDM to nrhs sources at once.
 * f_dev, u_dev: [*grid_counts][nrhs] (RHS-minor).  u = sum of beta00-blended
 * local solutions.  Emission masks (cuts, exact-zero flags) are evaluated on
 * the device with the reference semantics (ddm.py:82-110, :242-279).
 * partials_dev: NULL, or [nsweeps][*grid_counts][nrhs] receiving a copy of
 * the running sum after each sweep (collect_partials). */
DS_API int ds_ddm_apply(ds_ctx *ctx, ds_plan *plan, const ds_cplx *f_dev,
                 ds_cplx *u_dev, int32_t nrhs, ds_cplx *partials_dev);

/* Per-RHS counters of the last ds_ddm_apply (blocks the host):
 *   nonzero[r], discarded[r] (DdmReport fields, ddm.py:149-165), and when
 *   the arrays are non-NULL the per-visit tables [nsweeps][nsub][nrhs]:
 *   visit_nonzero, visit_consumed, visit_emitted and visit_cut (the solve
 *   cut mask, bit 2a+(side>0) for cut (axis a, side)). */
DS_API int ds_ddm_counters(ds_ctx *ctx, ds_plan *plan, int32_t nrhs,
                    int32_t *nonzero, int32_t *discarded,
                    int32_t *visit_nonzero, int32_t *visit_consumed,
                    int32_t *visit_emitted, int32_t *visit_cut);

/* Record / replay the whole application as one CUDA graph (same f/u
 * pointers and nrhs); ds_ddm_apply uses the graph when it matches. */
DS_API int ds_ddm_enable_graph(ds_ctx *ctx, ds_plan *plan, int32_t enable);

/* ds_ddm_apply_host for a batch split into G contiguous RHS groups, one
 * identical plan per group (plans[g] covers RHS [nrhs g / G, nrhs (g+1) / G)):
 * the groups sweep concurrently on their own streams while one shared copy
 * pipeline uploads each source box once and downloads each result box once
 * every group has finalized it.  Results are bitwise those of one plan. */
DS_API int ds_ddm_apply_host_groups(ds_ctx *ctx, ds_plan *const *plans, int32_t ngroups,
                                    const ds_cplx *f_host, ds_cplx *u_host, int32_t nrhs);

/* ds_ddm_apply on RHS-outer device buffers f_dev / u_dev ([nrhs][N], the
 * batched API layout): the assembly reads and the accumulation writes that
 * layout directly (no layout transposes); no per-sweep partials. */
DS_API int ds_ddm_apply_outer(ds_ctx *ctx, ds_plan *plan, const ds_cplx *f_dev,
                              ds_cplx *u_dev, int32_t nrhs);

/* One application from pinned HOST buffers: f_host / u_host are RHS-outer
 * [nrhs][N] complex128 in page-locked memory.  The source upload runs in
 * axis-0 row chunks on a copy stream overlapped with the first sweep (each
 * assembly waits only for the chunks it reads) and every chunk of u is
 * copied back as soon as the last accumulation touching it has run; the
 * call is asynchronous on the context stream (synchronize before reading
 * u_host).  CUDA-graph replay keyed on (f_host, u_host, nrhs). */
DS_API int ds_ddm_apply_host(ds_ctx *ctx, ds_plan *plan, const ds_cplx *f_host,
                             ds_cplx *u_host, int32_t nrhs);

/* Per-kernel-class timing: when enabled, ds_ddm_apply brackets every
 * launch with CUDA events on the context stream (graph replay is bypassed).
 * ds_plan_kernel_times returns summed milliseconds and launch counts for
 * classes {0 assemble (K6), 1 block solve (K3) / modal transforms (K3m-T),
 * 2 accumulate (K5), 3 transfer (K4), 4 modal recurrences (K3m-R)} since
 * the last reset (ms[5], count[5]); blocks the host. */
DS_API int ds_plan_set_profiling(ds_plan *plan, int32_t enable);
DS_API int ds_plan_kernel_times(ds_plan *plan, double *ms, int64_t *count,
                                int32_t reset);

/* Launch count of the last ds_ddm_apply (kernel nodes issued). */
DS_API int64_t ds_plan_last_launches(const ds_plan *plan);

/* ---------------------------------------------------------- sharded sweep
 * Device memory a sharded plan exposes to its peers: the payload slots and
 * the flag words ([own_nz | nz | arrivals | cuts | emitted | discards],
 * stride nrhs of the call).  Every rank's layout is identical. */
DS_API int ds_plan_shard_info(const ds_plan *plan, void **slot_base, int64_t *slot_bytes,
                              void **flag_base, int64_t *flag_bytes);
/* Pointers (valid in this process: local, peer or IPC-mapped) to every
 * rank's slot and flag memory, index = rank; must be called before the
 * first ds_ddm_apply_range of a sharded plan. */
DS_API int ds_plan_set_peers(ds_ctx *ctx, ds_plan *plan, int32_t nranks,
                             void *const *slot_bases, void *const *flag_bases);
/* Number of launches of the plan's schedule. */
DS_API int32_t ds_plan_nlaunch(const ds_plan *plan);
/* Launches [l0, l1) of one application (eager, on the context stream).
 * mode bit 0: initialise (zero u and this rank's flags) before l0;
 * bit 1: finalise (join the side stream into the context stream) after l1.
 * A sharded application is: init on every rank, then per launch every rank
 * runs [l, l+1) with a cross-rank barrier between launches, then finalise;
 * u of the sweep is the sum over ranks of their u. */
DS_API int ds_ddm_apply_range(ds_ctx *ctx, ds_plan *plan, const ds_cplx *f_dev, ds_cplx *u_dev,
                              int32_t nrhs, int32_t l0, int32_t l1, int32_t mode);

/* Inspection (ABI 5; used by the per-step parity tests of psi and
 * _accumulate): the payload slot that queues sources of direction `dir`
 * (index into `directions`) for visit (use_sweep 1-based, target subdomain).
 * lo / shape receive its band (grid coordinates); when out_dev is non-NULL
 * its contents, [band nodes, C-order][nrhs] as left by the last call with
 * that nrhs, are copied there (out_elems >= band nodes * nrhs; async on the
 * context stream).  Between the producing transfer and the consuming
 * assembly a slot holds the sum of the payloads queued for it
 * (transfer.py:100-155, ddm.py:276).  < 0 if no routing fills that slot. */
DS_API int ds_plan_slot(ds_ctx *ctx, const ds_plan *plan, int32_t use_sweep, int32_t target,
                        int32_t dir, int32_t *lo, int32_t *shape, ds_cplx *out_dev,
                        int64_t out_elems, int32_t nrhs);

/* Cross-rank device barrier of a sharded sweep (ABI 5): rank `rank` of
 * `nranks` owns an arrival array (ds_barrier_info: device pointer + bytes, to
 * be mapped by its peers); ds_barrier_set_peers takes every rank's array
 * (index = rank, local / peer / IPC-mapped pointers); ds_barrier_wait
 * enqueues the barrier on the context stream: all prior work of this rank is
 * made visible system-wide, then it waits on the device until every rank has
 * arrived at the same generation.  Replaces a per-launch collective between
 * the launches of ds_ddm_apply_range. */
typedef struct ds_barrier ds_barrier;
DS_API int ds_barrier_create(ds_ctx *ctx, int32_t nranks, int32_t rank, ds_barrier **out);
DS_API int ds_barrier_info(const ds_barrier *b, void **arrive, int64_t *bytes);
DS_API int ds_barrier_set_peers(ds_barrier *b, int32_t nranks, void *const *arrive);
DS_API int ds_barrier_wait(ds_ctx *ctx, ds_barrier *b);
DS_API int64_t ds_barrier_generation(const ds_barrier *b);
DS_API int ds_barrier_destroy(ds_barrier *b);

/* ---------------------------------------------------------- vector kernels
 * Batched complex vector ops for GMRES (krylov.py:80, :97-106, :139-142);
 * vectors are RHS-outer [nrhs][n] (the reference's batch layout), one
 * scalar per RHS.  Reductions are deterministic (fixed two-level order). */
/* out[r] = sum_i conj(x[r,i]) * y[r,i] (np.vdot semantics) */
DS_API int ds_vec_dot(ds_ctx *ctx, int64_t n, int32_t nrhs, const ds_cplx *x_dev,
               const ds_cplx *y_dev, ds_cplx *out_dev);
/* out[r] = ||x[r,:]||_2 */
DS_API int ds_vec_norm(ds_ctx *ctx, int64_t n, int32_t nrhs, const ds_cplx *x_dev,
                double *out_dev);
/* y[r,:] += alpha_sign * a[r] * x[r,:]  (alpha_sign = +1 or -1) */
DS_API int ds_vec_axpy(ds_ctx *ctx, int64_t n, int32_t nrhs, const ds_cplx *a_dev,
                double alpha_sign, const ds_cplx *x_dev, ds_cplx *y_dev);
/* fused MGS step: y -= a_prev * xprev (if xprev != NULL), then
 * out[r] = vdot(x, y).  Same arithmetic as the unfused pair. */
DS_API int ds_vec_axpy_dot(ds_ctx *ctx, int64_t n, int32_t nrhs,
                    const ds_cplx *a_prev_dev, const ds_cplx *xprev_dev,
                    ds_cplx *y_dev, const ds_cplx *x_dev, ds_cplx *out_dev);
/* y[r] += sum_j c[j*nrhs+r] * X_j[r]   (basis update x += Z^T y) */
DS_API int ds_vec_combine(ds_ctx *ctx, int64_t n, int32_t nrhs, int32_t nvec,
                   const ds_cplx *const *x_dev_list, const ds_cplx *c_dev,
                   ds_cplx *y_dev);
/* y[r] = x[r] / s[r]  (s real; rows with s[r] == 0 are set to zero) —
 * the normalisations V[0] = r/beta and V[k+1] = w/norm_w of krylov.py */
DS_API int ds_vec_scale(ds_ctx *ctx, int64_t n, int32_t nrhs, const ds_cplx *x_dev,
                 const double *s_dev, ds_cplx *y_dev);

/* out[r] = b[r] - w[r] and norm_out[r] = ||out[r]||_2 in one pass (the
 * residual r = b - A x of krylov.py:80, :140-141; ABI 5). */
DS_API int ds_vec_sub_norm(ds_ctx *ctx, int64_t n, int32_t nrhs, const ds_cplx *b_dev,
                           const ds_cplx *w_dev, ds_cplx *out_dev, double *norm_out_dev);
/* Row gather / scatter of RHS-outer batches (ABI 5): dst[r] = src[map[r]]
 * for r < ndst, zero where map[r] < 0 (device int32 map) -- the active-row
 * selection of the batched GMRES. */
DS_API int ds_vec_rows(ds_ctx *ctx, int64_t n, int32_t ndst, const int32_t *map_dev,
                       const ds_cplx *src_dev, ds_cplx *dst_dev);

/* RHS-outer [R][n] <-> RHS-minor [n][R] layout conversion. */
DS_API int ds_layout_to_minor(ds_ctx *ctx, int64_t n, int32_t nrhs,
                       const ds_cplx *src_dev, ds_cplx *dst_dev);
DS_API int ds_layout_to_outer(ds_ctx *ctx, int64_t n, int32_t nrhs,
                       const ds_cplx *src_dev, ds_cplx *dst_dev);

/* ------------------------------------------------ assembly on the device
 * (ABI 6).  Replace the host-O(N) steps of building a
 * problem: assemble_operator's raster kappa^2 (pml.py:197-213 with
 * RasterModel.speed_at, media.py:75-101) and Gaussian source batches
 * (media.py:147-167 / the configs' seeded sources).
 *
 * ds_raster_kappa2: out[node] = (omega / c(node))^2 over a window of
 * win_counts[dim] nodes (C order), c the multilinear interpolation of the
 * raster samples (raster_counts[dim], C order, as float64 -- float32 rasters
 * widened exactly) with the per-axis tables
 * base_dev[a][i] (lower raster index of window coordinate i along axis a)
 * and frac_dev[a][i] (its fraction), as the reference computes them; bitwise
 * the reference's values.  Returns -2 (model error) if some c <= 0.  Blocks
 * until done (reads the error flag). */
DS_API int ds_raster_kappa2(ds_ctx *ctx, int32_t dim, const int32_t *win_counts,
                            const int32_t *raster_counts, const double *samples_dev,
                            const int32_t *const *base_dev, const double *const *frac_dev,
                            double omega, double *out_dev);
/* ds_gaussian_fields: out[r][node] = amp[r] * exp(arg), RHS-outer, complex
 * with zero imaginary part; r2 = sum over axes (in order) of the per-axis
 * tables d2_dev[a][r * counts[a] + i]; arg = scale[r] * r2, or -r2 / scale[r]
 * when divide != 0.  CUDA exp: values within ~2 ulp of NumPy's. */
DS_API int ds_gaussian_fields(ds_ctx *ctx, int32_t dim, const int32_t *counts, int32_t nrhs,
                              const double *const *d2_dev, const double *amp_dev,
                              const double *scale_dev, int32_t divide, ds_cplx *out_dev);

#ifdef __cplusplus
}
#endif

#endif /* DIAGSWEEP_B200_H */
