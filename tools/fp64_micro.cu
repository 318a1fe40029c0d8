// FP64 pipe microbenchmark on sm_100a: DFMA vs DMMA (mma.sync m8n8k4 f64)
// throughput per SM, plus DSMEM push / cluster barrier latencies are
// measured elsewhere (tools/trace_solve.py).  nvcc -arch=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_loop(double *out, int iters) {
  double a[8], b = 1.0000001, c = 0.9999999;
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.0) out[0] = s;
}

__global__ void dmma_loop(double *out, int iters) {
  double acc[4][2];
  for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = 0;
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int i = 0; i < 4; ++i) s += acc[i][0] + acc[i][1];
  if (s == 12345.0) out[0] = s;
}

int main() {
  double *d;
  cudaMalloc(&d, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int iters = 20000;
  for (int warps : {4, 8, 16, 32}) {
    dfma_loop<<<sms, warps * 32>>>(d, 100);
    cudaEventRecord(e0);
    dfma_loop<<<sms, warps * 32>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 8 * iters * (double)warps * 32 * sms;
    printf("DFMA  warps/SM %2d: %.2f TFLOP/s\n", warps, fl / ms / 1e9);
    dmma_loop<<<sms, warps * 32>>>(d, 100);
    cudaEventRecord(e0);
    dmma_loop<<<sms, warps * 32>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    fl = 2.0 * 256 * 4 * iters * (double)warps * sms;
    printf("DMMA  warps/SM %2d: %.2f TFLOP/s\n", warps, fl / ms / 1e9);
  }
  return 0;
}
