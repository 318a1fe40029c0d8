// Microbenchmark: (1) dependent-issue latency of DMMA.8x8x4 (f64) and DFMA,
// (2) issue cost of TMA bulk copies (cp.async.bulk global->shared, 14.7 KB,
// and the cluster multicast of 2 KB) as seen by the issuing thread, i.e.
// how long the issuing warp is held before its next instruction.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ilm tools/issue_latency_micro.cu
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstring>

namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k_dmma_lat(double *out, int n, int chains) {
  double c[8][2];
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = threadIdx.x * 1e-3;
  double a = 1.0 + threadIdx.x * 1e-6, b = 0.999;
  long long t0 = clock64();
  if (chains == 1) {
    for (int i = 0; i < n; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[0][0]), "+d"(c[0][1]) : "d"(a), "d"(b));
  } else if (chains == 3) {
    for (int i = 0; i < n; ++i) {
#pragma unroll
      for (int j = 0; j < 3; ++j)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
    }
  } else {
    for (int i = 0; i < n; ++i) {
#pragma unroll
      for (int j = 0; j < 8; ++j)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
    }
  }
  long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (threadIdx.x == 0) {
    out[0] = (double)(t1 - t0) / n;
    out[1] = s;
  }
}

__global__ void k_dfma_lat(double *out, int n) {
  double x = threadIdx.x * 1e-3, a = 1.0000001, b = 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(x) : "d"(a), "d"(b));
  long long t1 = clock64();
  if (threadIdx.x == 0) {
    out[0] = (double)(t1 - t0) / n;
    out[1] = x;
  }
}

// issue cost of bulk copies: thread 0 issues `n` copies back to back and
// times the issue loop; completion is waited for afterwards (not timed)
__global__ void k_bulk_issue(const char *src, double *out, int n, uint32_t bytes, int multicast) {
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t *bar = (uint64_t *)sm;
  char *dst = (char *)(sm + 128);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cl.sync();
  if (threadIdx.x == 0) {
    uint32_t total = (multicast ? cl.num_blocks() : 1) * 0 + bytes * n;
    if (multicast && cl.block_rank() != 0) total = bytes * n;  // every CTA receives all copies of rank 0
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)),
                 "r"(multicast ? bytes * n : bytes * n)
                 : "memory");
  }
  cl.sync();
  long long t0 = clock64(), t1 = t0;
  if (threadIdx.x == 0 && (!multicast || cl.block_rank() == 0)) {
    for (int i = 0; i < n; ++i) {
      if (multicast)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], "
            "%4;" ::"r"(su32(dst)),
            "l"(src + (size_t)i * bytes), "r"(bytes), "r"(su32(bar)), "h"((uint16_t)((1u << cl.num_blocks()) - 1))
            : "memory");
      else
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         su32(dst)),
                     "l"(src + ((size_t)blockIdx.x * n + i) * bytes), "r"(bytes), "r"(su32(bar))
                     : "memory");
    }
    t1 = clock64();
  }
  if (threadIdx.x == 0) {
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0,1,0,p;\n}\n"
                   : "=r"(ok) : "r"(su32(bar)) : "memory");
  }
  long long t2 = clock64();
  cl.sync();
  if (threadIdx.x == 0 && cl.block_rank() == 0 && blockIdx.x == 0) {
    out[0] = (double)(t1 - t0) / n;
    out[1] = (double)(t2 - t0);
  }
}

int main() {
  double *d, h[2];
  cudaMalloc(&d, 64);
  for (int ch : {1, 3, 8}) {
    k_dmma_lat<<<1, 32>>>(d, 1000, ch);
    k_dmma_lat<<<1, 32>>>(d, 1000, ch);
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("DMMA 8x8x4, 1 warp, %d independent chain(s): %.1f cycles per iteration (%.1f per DMMA)\n", ch, h[0],
           h[0] / ch);
  }
  k_dfma_lat<<<1, 32>>>(d, 1000);
  k_dfma_lat<<<1, 32>>>(d, 1000);
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.1f cycles\n", h[0]);

  char *src;
  size_t sbytes = (size_t)1 << 30;
  cudaMalloc(&src, sbytes);
  cudaMemset(src, 1, sbytes);
  cudaFuncSetAttribute(k_bulk_issue, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k_bulk_issue, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int mc : {0, 1}) {
    for (uint32_t bytes : {2048u, 14720u, 29440u}) {
      if (mc && bytes > 4096) continue;
      for (int n : {1, 2, 4}) {
        cudaLaunchConfig_t cfg;
        memset(&cfg, 0, sizeof(cfg));
        cfg.gridDim = dim3(16);
        cfg.blockDim = dim3(32);
        cfg.dynamicSmemBytes = 128 + 32 * 1024;
        cudaLaunchAttribute a[1];
        a[0].id = cudaLaunchAttributeClusterDimension;
        a[0].val.clusterDim.x = 16;
        a[0].val.clusterDim.y = 1;
        a[0].val.clusterDim.z = 1;
        cfg.attrs = a;
        cfg.numAttrs = 1;
        for (int rep = 0; rep < 2; ++rep)
          cudaLaunchKernelEx(&cfg, k_bulk_issue, (const char *)(src + (size_t)rep * 64 * 1024 * 1024), d, n, bytes, mc);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        printf("%s %5u B x %d: issue %.0f cycles per copy, issue->complete %.0f cycles  (%s)\n",
               mc ? "multicast x16" : "bulk g2s     ", bytes, n, h[0], h[1], cudaGetErrorString(e));
      }
    }
  }
  return 0;
}
