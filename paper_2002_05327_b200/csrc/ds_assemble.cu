// K8: operator assembly and source generation on the device (SURVEY §8(f)
// rank 3) -- the host-O(N) parts of building a problem.
//
// K8a  raster kappa^2 of an operator window (pml.py _kappa2 "full" kind,
//      reference pml.py:197-213 with RasterModel.speed_at, media.py:75-101):
//      per node the multilinear interpolation of the speed raster (float32
//      or float64 samples, widened exactly to float64 on upload)
//      at the node's clamped coordinates, then kappa^2 = (omega / c)^2.
//      Everything that depends on one axis only -- the clamped coordinate,
//      t, the lower raster index and its fraction -- is a 1D table built on
//      the host by the same NumPy expressions; the device does the O(N)
//      part: per node 2^dim gathers and the weight products, in the
//      reference's corner order (corner bits = axes, axis 0 first) with
//      explicitly rounded multiplies and adds (no FMA contraction), so the
//      result is bitwise NumPy's (tests/test_gpu_assemble.py).
// K8b  Gaussian source batches (configs.sources / media.gaussian_source):
//      f[r][node] = amp_r * exp(scale_r * r2)  (gaussian_source: -rate * r2)
//      or amp_r * exp(-r2 / scale_r)           (configs.sources, divide = 1),
//      r2 summed over axes in order
//      from per-axis squared distances (host 1D tables, exact as NumPy's).
//      The exponential is CUDA's exp (<= 1 ulp, not NumPy's), so fields
//      agree to ~2 ulp; the exact-zero set (underflow) is what the DDM
//      masks read and is compared exactly in the tests.
#include <cuda_runtime.h>

#include <algorithm>

#include "ds_common.cuh"

struct RasterAxes {
  const int32_t *base[3];  // lower raster index per window node along the axis
  const double *frac[3];   // t - base
  int n[3];                // window extent per axis (1 past dim)
  int rc[3];               // raster count per axis
  int64_t rstride[3];      // raster strides (C order, elements)
};

__global__ void k_raster_kappa2(RasterAxes X, int dim, const double *__restrict__ samples,
                                double omega, int64_t total, double *__restrict__ out,
                                int *__restrict__ bad) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int i[3] = {0, 0, 0};
    int64_t rem = e;
    for (int a = dim - 1; a >= 0; --a) {
      i[a] = (int)(rem % X.n[a]);
      rem /= X.n[a];
    }
    double acc = 0.0;
    for (int corner = 0; corner < (1 << dim); ++corner) {
      double w = 1.0;
      int64_t off = 0;
      for (int a = 0; a < dim; ++a) {
        const bool up = (corner >> a) & 1;
        const int b0 = X.base[a][i[a]];
        const double fr = X.frac[a][i[a]];
        if (up && X.rc[a] > 1) {
          off += (int64_t)(b0 + 1) * X.rstride[a];
          w = __dmul_rn(w, fr);
        } else {
          off += (int64_t)b0 * X.rstride[a];
          if (X.rc[a] > 1) w = __dmul_rn(w, __dsub_rn(1.0, fr));
          else if (up) w = __dmul_rn(w, 0.0);
        }
      }
      acc = __dadd_rn(acc, __dmul_rn(w, samples[off]));
    }
    if (!(acc > 0.0)) atomicExch(bad, 1);
    const double q = __ddiv_rn(omega, acc);
    out[e] = __dmul_rn(q, q);
  }
}

extern "C" int ds_raster_kappa2(ds_ctx *ctx, int32_t dim, const int32_t *win_counts,
                                const int32_t *raster_counts, const double *samples_dev,
                                const int32_t *const *base_dev, const double *const *frac_dev,
                                double omega, double *out_dev) {
  if (!ctx || dim < 1 || dim > 3 || !win_counts || !raster_counts || !samples_dev || !base_dev ||
      !frac_dev || !out_dev)
    return ds_fail(DS_ECONFIG, "ds_raster_kappa2: bad argument");
  RasterAxes X;
  int64_t total = 1, st = 1;
  for (int a = 2; a >= 0; --a) {
    X.base[a] = a < dim ? base_dev[a] : nullptr;
    X.frac[a] = a < dim ? frac_dev[a] : nullptr;
    X.n[a] = a < dim ? win_counts[a] : 1;
    X.rc[a] = a < dim ? raster_counts[a] : 1;
    if (X.n[a] < 1 || X.rc[a] < 1) return ds_fail(DS_ECONFIG, "ds_raster_kappa2: empty axis");
    X.rstride[a] = st;
    st *= X.rc[a];
    total *= X.n[a];
  }
  int *bad = (int *)ctx->scratch;
  DS_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), ctx->stream));
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, (int64_t)ctx->num_sms * 8);
  k_raster_kappa2<<<std::max(1, blocks), 256, 0, ctx->stream>>>(X, dim, samples_dev, omega,
                                                                 total, out_dev, bad);
  ctx->launches++;
  DS_CHECK_LAUNCH();
  int hbad = 0;
  DS_CUDA(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  DS_CUDA(cudaStreamSynchronize(ctx->stream));
  if (hbad) return ds_fail(DS_EMODEL, "nonpositive velocity inside operator window");
  return DS_OK;
}

// f[r][e] = amp[r] * exp(scale[r] * r2), r2 = ((0 + d2_0) + d2_1) + d2_2 with
// d2_a[r][i] the per-axis squared distance tables (RHS-major, length n_a)
struct GaussAxes {
  const double *d2[3];
  int n[3];
};

__global__ void k_gauss_fields(GaussAxes X, int dim, int nrhs, const double *__restrict__ amp,
                               const double *__restrict__ scale, int divide, int64_t total,
                               cplx *__restrict__ out) {
  const int r = blockIdx.y;
  if (r >= nrhs) return;
  const double am = amp[r], sc = scale[r];
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t rem = e;
    int i[3] = {0, 0, 0};
    for (int a = dim - 1; a >= 0; --a) {
      i[a] = (int)(rem % X.n[a]);
      rem /= X.n[a];
    }
    double r2 = 0.0;
    for (int a = 0; a < dim; ++a) r2 = __dadd_rn(r2, X.d2[a][(int64_t)r * X.n[a] + i[a]]);
    const double arg = divide ? __ddiv_rn(-r2, sc) : __dmul_rn(sc, r2);
    // below exp's normal range CUDA's exp does not round into the subnormals
    // as NumPy's does: exp(arg) = exp(A) (1 + B) 2^-64 with A = arg + 64 ln2_hi
    // (exact: Cody-Waite split, ln2_hi has 32 significant bits) and
    // B = 64 ln2_lo, rounded once into the subnormal range by scalbn -- same
    // exact-zero (underflow) set as NumPy and a few ulp apart
    double ex;
    if (arg >= -708.0) {
      ex = exp(arg);
    } else {
      const double A = arg + 64.0 * 6.93147180369123816490e-01;
      const double B = 64.0 * 1.90821492927058770002e-10;
      ex = scalbn(exp(A) * (1.0 + B + 0.5 * B * B), -64);
    }
    out[(int64_t)r * total + e] = make_double2(__dmul_rn(am, ex), 0.0);
  }
}

extern "C" int ds_gaussian_fields(ds_ctx *ctx, int32_t dim, const int32_t *counts, int32_t nrhs,
                                  const double *const *d2_dev, const double *amp_dev,
                                  const double *scale_dev, int32_t divide, ds_cplx *out_dev) {
  if (!ctx || dim < 1 || dim > 3 || !counts || nrhs < 0 || !d2_dev || !amp_dev || !scale_dev ||
      (!out_dev && nrhs > 0))
    return ds_fail(DS_ECONFIG, "ds_gaussian_fields: bad argument");
  if (nrhs == 0) return DS_OK;
  GaussAxes X;
  int64_t total = 1;
  for (int a = 0; a < 3; ++a) {
    X.d2[a] = a < dim ? d2_dev[a] : nullptr;
    X.n[a] = a < dim ? counts[a] : 1;
    if (X.n[a] < 1) return ds_fail(DS_ECONFIG, "ds_gaussian_fields: empty axis");
    total *= X.n[a];
  }
  const int bx = (int)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256,
                                                             (int64_t)ctx->num_sms * 8 / std::max(1, nrhs) + 1));
  k_gauss_fields<<<dim3(bx, nrhs), 256, 0, ctx->stream>>>(X, dim, nrhs, amp_dev, scale_dev, divide != 0,
                                                          total, (cplx *)out_dev);
  ctx->launches++;
  DS_CHECK_LAUNCH();
  return DS_OK;
}
