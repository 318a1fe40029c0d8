// Microbenchmark: K3's per-stage block product in isolation (no exchange, no
// TMA traffic).  One CTA of 256 threads = 2 halves x 4 warps, each warp runs
// mma_product<MT, NT> over a quarter of K for an (8*MT)-row, rc-RHS tile of
// an m-column factor slice, exactly as k_block_solve8 does; the split-K
// partials go to shared memory and a __syncthreads closes the "stage".
// Reports cycles per stage for several (rows, rc) shapes, with 1 CTA/SM on
// every SM (the K3 occupancy).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2002_05327_b200/csrc -o /tmp/pm tools/product_micro.cu
#include <cuda_runtime.h>
#include <cstdio>

#include "ds_mma.cuh"

template <int MT, int NT>
__global__ void __launch_bounds__(256, 1) k_product(int m, int rc, int stages, long long *out, double *sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int rows = 8 * MT;
  cplx *A = (cplx *)sm;                 // [2 halves][rows][m]
  cplx *X = A + 2 * rows * m;           // [2 halves][m][rc]
  cplx *red = X + 2 * m * rc;           // [2][4][rows*rc]
  const int t = threadIdx.x, hh = t >> 7, tl = t & 127;
  for (int i = t; i < 2 * rows * m; i += 256) A[i] = make_double2(1e-3 * (i % 97), 1e-3 * (i % 89));
  for (int i = t; i < 2 * m * rc; i += 256) X[i] = make_double2(1e-3 * (i % 83), -1e-3 * (i % 79));
  __syncthreads();
  const int warp = tl >> 5, lane = t & 31, g = lane >> 2, tg = lane & 3;
  const int nk = (m + 3) >> 2, kb = (warp * nk) >> 2, ke = ((warp + 1) * nk) >> 2;
  const int rstride = rows * rc;
  cplx *rp = red + ((size_t)hh * 4 + warp) * rstride;
  double acc = 0;
  long long t0 = clock64(), tp = 0, tr = 0, ts = 0;
  for (int s = 0; s < stages; ++s) {
    double cr[2][2][2] = {}, ci[2][2][2] = {};
    long long a0 = clock64();
    mma_product<MT, NT, false>(A + hh * rows * m, m, X + hh * m * rc, nullptr, rc, m, kb, ke, g, tg, cr, ci);
    // force completion of the product before the timestamp
    acc += cr[0][0][0];
    long long a1 = clock64();
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int row = mt * 8 + g, col = nt * 8 + 2 * tg + e;
          if (col < rc) rp[row * rc + col] = make_double2(cr[mt][nt][e], ci[mt][nt][e]);
        }
    long long a2 = clock64();
    __syncthreads();
    long long a3 = clock64();
    acc += red[tl].x;
    __syncthreads();
    tp += a1 - a0;
    tr += a2 - a1;
    ts += a3 - a2;
  }
  long long t1 = clock64();
  if (t == 0 && blockIdx.x == 0) {
    out[0] = (t1 - t0) / stages;
    printf("   warp0: product %lld  red-store %lld  barrier-wait %lld (cycles/stage)\n", tp / stages, tr / stages,
           ts / stages);
  }
  if (acc == 12345.0) sink[0] = acc;
}

// mma_product alone (no split-K stores, no barriers): the loop's own cost
template <int MT, int NT>
__global__ void __launch_bounds__(256, 1) k_product_only(int m, int rc, int stages, long long *out,
                                                       double *sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int rows = 8 * MT;
  cplx *A = (cplx *)sm;
  cplx *X = A + 2 * rows * m;
  const int t = threadIdx.x, hh = t >> 7, tl = t & 127;
  for (int i = t; i < 2 * rows * m; i += 256) A[i] = make_double2(1e-3 * (i % 97), 1e-3 * (i % 89));
  for (int i = t; i < 2 * m * rc; i += 256) X[i] = make_double2(1e-3 * (i % 83), -1e-3 * (i % 79));
  __syncthreads();
  const int warp = tl >> 5, lane = t & 31, g = lane >> 2, tg = lane & 3;
  const int nk = (m + 3) >> 2, kb = (warp * nk) >> 2, ke = ((warp + 1) * nk) >> 2;
  double acc = 0;
  long long t0 = clock64();
  for (int s = 0; s < stages; ++s) {
    double cr[2][2][2] = {}, ci[2][2][2] = {};
    mma_product<MT, NT, false>(A + hh * rows * m, m, X + hh * m * rc, nullptr, rc, m, kb, ke, g, tg, cr, ci);
    acc += cr[0][0][0] + ci[0][0][1];
  }
  long long t1 = clock64();
  if (t == 0 && blockIdx.x == 0) out[0] = (t1 - t0) / stages;
  if (acc == 12345.0) sink[0] = acc;
}

template <int MT, int NT>
void run_product_only(int m, int rc) {
  long long *o;
  double *sink;
  cudaMalloc(&o, 8);
  cudaMalloc(&sink, 8);
  const int rows = 8 * MT;
  size_t smem = (size_t)(2 * rows * m + 2 * m * rc) * 16;
  cudaFuncSetAttribute(k_product_only<MT, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  k_product_only<MT, NT><<<sms, 256, smem>>>(m, rc, 10, o, sink);
  k_product_only<MT, NT><<<sms, 256, smem>>>(m, rc, 200, o, sink);
  cudaDeviceSynchronize();
  long long h;
  cudaMemcpy(&h, o, 8, cudaMemcpyDeviceToHost);
  int nk = (m + 3) / 4, steps = (nk + 3) / 4;
  long floor_c = 2L * steps * 3 * MT * NT * 16;
  printf("product only rows %2d rc %2d : %6lld cycles/stage (floor %ld, %.0f%%)\n", rows, rc, h, floor_c,
         100.0 * floor_c / h);
}

// the same DMMA sequence with register-resident fragments (no shared loads)
template <int MT, int NT>
__global__ void __launch_bounds__(256, 1) k_dmma_only(int m, int stages, long long *out, double *sink) {
  const int t = threadIdx.x, tl = t & 127, warp = tl >> 5;
  const int nk = (m + 3) >> 2, kb = (warp * nk) >> 2, ke = ((warp + 1) * nk) >> 2;
  double a = 1e-3 * t, b = 2e-3 * t, as = a + b, bs = a - b;
  double p1[MT][NT][2] = {}, p2[MT][NT][2] = {}, p3[MT][NT][2] = {};
  long long t0 = clock64();
  for (int s = 0; s < stages; ++s) {
    for (int kq = kb; kq < ke; ++kq) {
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          dmma(p1[mt][nt], a, b);
          dmma(p2[mt][nt], b, a);
          dmma(p3[mt][nt], as, bs);
        }
    }
    __syncthreads();
  }
  long long t1 = clock64();
  double acc = 0;
  for (int mt = 0; mt < MT; ++mt)
    for (int nt = 0; nt < NT; ++nt) acc += p1[mt][nt][0] + p2[mt][nt][1] + p3[mt][nt][0];
  if (t == 0 && blockIdx.x == 0) out[0] = (t1 - t0) / stages;
  if (acc == 12345.0) sink[0] = acc;
}

// DMMAs on register operands plus 3 unrelated LDS.128 per k-step (the
// product's load traffic), barrier per stage: structural LDS/DMMA conflict?
__global__ void __launch_bounds__(256, 1) k_dmma_lds(int m, int stages, long long *out, double *sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  double2 *buf = (double2 *)sm;
  const int t = threadIdx.x, tl = t & 127, warp = tl >> 5;
  for (int i = t; i < 8192; i += 256) buf[i] = make_double2(i, -i);
  __syncthreads();
  const int nk = (m + 3) >> 2, kb = (warp * nk) >> 2, ke = ((warp + 1) * nk) >> 2;
  double a = 1e-3 * t, b = 2e-3 * t, as = a + b, bs = a - b;
  double p[6][2] = {};
  double2 sacc = make_double2(0, 0);
  long long t0 = clock64();
  for (int s = 0; s < stages; ++s) {
    for (int kq = kb; kq < ke; ++kq) {
      const double2 l0 = buf[(kq * 96 + t) & 8191], l1 = buf[(kq * 96 + t + 256) & 8191],
                    l2 = buf[(kq * 96 + t + 512) & 8191];
      dmma(p[0], a, b);
      dmma(p[1], b, a);
      dmma(p[2], as, bs);
      dmma(p[3], a, bs);
      dmma(p[4], b, as);
      dmma(p[5], as, a);
      sacc.x += l0.x + l1.x + l2.x;
      sacc.y += l0.y + l1.y + l2.y;
    }
    __syncthreads();
  }
  long long t1 = clock64();
  double acc = sacc.x + sacc.y;
  for (int i = 0; i < 6; ++i) acc += p[i][0];
  if (t == 0 && blockIdx.x == 0) out[0] = (t1 - t0) / stages;
  if (acc == 12345.0) sink[0] = acc;
}

template <int MT, int NT>
void run_dmma_only(int m) {
  long long *o;
  double *sink;
  cudaMalloc(&o, 8);
  cudaMalloc(&sink, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  k_dmma_only<MT, NT><<<sms, 256>>>(m, 10, o, sink);
  k_dmma_only<MT, NT><<<sms, 256>>>(m, 200, o, sink);
  cudaDeviceSynchronize();
  long long h;
  cudaMemcpy(&h, o, 8, cudaMemcpyDeviceToHost);
  int nk = (m + 3) / 4, steps = (nk + 3) / 4;
  long floor_c = 2L * steps * 3 * MT * NT * 16;
  printf("DMMA only rows %2d NT %d m %3d : %6lld cycles/stage (floor %ld, %.0f%%)\n", 8 * MT, NT, m, h, floor_c,
         100.0 * floor_c / h);
}

template <int MT, int NT>
void run(int m, int rc) {
  long long *o;
  double *sink;
  cudaMalloc(&o, 8);
  cudaMalloc(&sink, 8);
  const int rows = 8 * MT;
  size_t smem = (size_t)(2 * rows * m + 2 * m * rc + 8 * rows * rc) * 16;
  cudaFuncSetAttribute(k_product<MT, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  k_product<MT, NT><<<sms, 256, smem>>>(m, rc, 10, o, sink);
  k_product<MT, NT><<<sms, 256, smem>>>(m, rc, 200, o, sink);
  cudaError_t e = cudaDeviceSynchronize();
  long long h;
  cudaMemcpy(&h, o, 8, cudaMemcpyDeviceToHost);
  // DMMA pipe floor: per SMSP 2 warps x ceil(nk/4) k-steps x 3*MT*NT DMMAs x 16 cycles
  int nk = (m + 3) / 4, steps = (nk + 3) / 4;
  long floor_c = 2L * steps * 3 * MT * NT * 16;
  printf("rows %2d  rc %2d  m %3d : %6lld cycles/stage  (DMMA pipe floor %ld, %.0f%%)  %s\n", rows, rc, m, h,
         floor_c, 100.0 * floor_c / h, cudaGetErrorString(e));
  cudaFree(o);
  cudaFree(sink);
}

int main() {
  run<1, 2>(115, 16);
  run<1, 1>(115, 8);
  run<1, 1>(115, 4);
  run<2, 2>(115, 16);
  run<2, 1>(115, 8);
  run<1, 2>(230, 16);
  {
    long long *o;
    double *sink;
    cudaMalloc(&o, 8);
    cudaMalloc(&sink, 8);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaFuncSetAttribute(k_dmma_lds, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192 * 16);
    k_dmma_lds<<<sms, 256, 8192 * 16>>>(115, 10, o, sink);
    k_dmma_lds<<<sms, 256, 8192 * 16>>>(115, 200, o, sink);
    cudaDeviceSynchronize();
    long long h;
    cudaMemcpy(&h, o, 8, cudaMemcpyDeviceToHost);
    printf("DMMA + 3 LDS.128 per k-step, barrier/stage: %lld cycles/stage (DMMA floor 1536)\n", h);
  }
  run_product_only<1, 2>(115, 16);
  run_product_only<1, 1>(115, 8);
  run_dmma_only<1, 2>(115);
  run_dmma_only<1, 1>(115);
  run_dmma_only<2, 2>(115);
  return 0;
}
