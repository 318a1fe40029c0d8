// Microbenchmark: chained all-gather rounds inside one thread-block cluster
// (the exchange step of K3).  Each of C CTAs owns `rows` rows x `rc`
// complex values and every round must deliver all rows to every CTA before
// the next round starts.  Reports cycles per round for
//   mode 0: bulk copies shared::cta -> shared::cluster, one lane per peer,
//           completion by mbarrier complete_tx on the receiver;
//   mode 1: remote st.shared::cluster by every thread + remote mbarrier
//           arrive (release.cluster) by one lane per peer;
//   mode 2: rows written to global, then one multicast TMA bulk load
//           global -> all CTAs (issuer = CTA 0 loads the whole vector).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o cluster_exchange_micro cluster_exchange_micro.cu
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstring>

namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t par) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(su32(b)), "r"(par) : "memory");
}
__device__ __forceinline__ uint32_t mapa(const void *p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(su32(p)), "r"(rank));
  return r;
}

template <int MODE>
__global__ void k_exchange(int rounds, int rows, int rc, double2 *gbuf, long long *out) {
  cg::cluster_group cl = cg::this_cluster();
  const int rank = cl.block_rank(), C = cl.num_blocks();
  const int t = threadIdx.x;
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t *bar = (uint64_t *)sm;               // [2]
  double2 *vec = (double2 *)(sm + 128);         // [2][C*rows*rc]
  const int n = C * rows * rc;
  double2 *stg = vec + 2 * n;                   // [2][rows*rc]
  const uint32_t mine = rows * rc * 16, all = n * 16;
  if (t == 0) {
    mbar_init(&bar[0], MODE == 1 ? C : 1);
    mbar_init(&bar[1], MODE == 1 ? C : 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cl.sync();
  if (MODE != 1 && t == 0) {
    mbar_expect_tx(&bar[0], all);
    mbar_expect_tx(&bar[1], all);
  }
  long long t0 = clock64();
  for (int r = 0; r < rounds; ++r) {
    const int b = r & 1;
    // produce my rows (depends on the previous round's vector)
    double2 seed = r ? vec[((r - 1) & 1) * n + (t % n)] : make_double2(rank, t);
    for (int e = t; e < rows * rc; e += blockDim.x) stg[b * rows * rc + e] = make_double2(seed.x + e, seed.y);
    if (MODE == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (t < C) {
        uint32_t dst = mapa(vec + b * n + rank * rows * rc, t), rb = mapa(&bar[b], t);
        asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(dst), "r"(su32(stg + b * rows * rc)), "r"(mine), "r"(rb) : "memory");
      }
    } else if (MODE == 1) {
      for (int e = t; e < rows * rc; e += blockDim.x) {
        double2 v = stg[b * rows * rc + e];
        for (int q = 0; q < C; ++q) {
          uint32_t dst = mapa(vec + b * n + rank * rows * rc + e, q);
          asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(dst), "d"(v.x), "d"(v.y) : "memory");
        }
      }
      __syncthreads();
      if (t < C) {
        uint32_t rb = mapa(&bar[b], t);
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(rb) : "memory");
      }
    } else if (MODE == 4) {
      // st.async: every thread stores its values straight into each peer's
      // buffer; completion is counted by the peer's mbarrier (complete_tx)
      for (int e = t; e < rows * rc; e += blockDim.x) {
        double2 v = stg[b * rows * rc + e];
        for (int q = 0; q < C; ++q) {
          uint32_t dst = mapa(vec + b * n + rank * rows * rc + e, q), rb = mapa(&bar[b], q);
          asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];"
                       ::"r"(dst), "d"(v.x), "d"(v.y), "r"(rb) : "memory");
        }
      }
    } else if (MODE == 3) {
      // own rows -> global, then one multicast bulk load of my rows to all CTAs
      double2 *g = gbuf + (size_t)blockIdx.y * 2 * n + b * n + rank * rows * rc;
      for (int e = t; e < rows * rc; e += blockDim.x) g[e] = stg[b * rows * rc + e];
      asm volatile("fence.proxy.async.global;" ::: "memory");
      __syncthreads();
      if (t == 0) {
        uint16_t mask = (uint16_t)((1u << C) - 1);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;"
                     ::"r"(su32(vec + b * n + rank * rows * rc)), "l"(g), "r"(mine), "r"(su32(&bar[b])), "h"(mask) : "memory");
      }
    } else {
      double2 *g = gbuf + (size_t)blockIdx.y * 2 * n + b * n;
      for (int e = t; e < rows * rc; e += blockDim.x) g[rank * rows * rc + e] = stg[b * rows * rc + e];
      asm volatile("fence.proxy.async.global;" ::: "memory");
      __syncthreads();
      cl.sync();  // everyone's rows are in global
      if (rank == 0 && t == 0) {
        uint16_t mask = (uint16_t)((1u << C) - 1);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;"
                     ::"r"(su32(vec + b * n)), "l"(g), "r"(all), "r"(su32(&bar[b])), "h"(mask) : "memory");
      }
    }
    mbar_wait(&bar[b], (r >> 1) & 1);
    if (MODE != 1 && t == 0 && r + 2 < rounds) mbar_expect_tx(&bar[b], all);
  }
  long long t1 = clock64();
  cl.sync();
  if (t == 0 && rank == 0) out[blockIdx.y] = (t1 - t0) / rounds;
}

template <int MODE>
void run(int C, int rows, int rc, int nclusters) {
  int rounds = 2000;
  size_t smem = 128 + (2 * (size_t)C * rows * rc + 2 * rows * rc) * 16;
  auto k = k_exchange<MODE>;
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  double2 *g;
  cudaMalloc(&g, (size_t)nclusters * 2 * C * rows * rc * 16);
  long long *out;
  cudaMalloc(&out, 8 * nclusters);
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3(C, nclusters);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute a[1];
  a[0].id = cudaLaunchAttributeClusterDimension;
  a[0].val.clusterDim.x = C;
  a[0].val.clusterDim.y = 1;
  a[0].val.clusterDim.z = 1;
  cfg.attrs = a;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k, rounds, rows, rc, g, out);
  cudaError_t e2 = cudaDeviceSynchronize();
  long long h = -1;
  cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
  printf("mode %d  C=%2d rows=%2d rc=%2d clusters=%d : %lld cycles/round  (%s %s)\n", MODE, C, rows, rc,
         nclusters, h, cudaGetErrorString(e), cudaGetErrorString(e2));
  cudaFree(g);
  cudaFree(out);
}

int main() {
  run<4>(16, 8, 16, 1);
  run<4>(16, 8, 16, 7);
  run<4>(16, 8, 8, 1);
  run<4>(8, 15, 16, 1);
  run<3>(16, 8, 16, 1);
  run<3>(16, 8, 16, 7);
  run<0>(16, 8, 4, 1);
  run<3>(16, 8, 4, 1);
  run<0>(16, 8, 1, 1);
  run<3>(16, 8, 1, 1);
  run<3>(8, 15, 16, 1);
  run<3>(4, 29, 4, 1);
  for (int nc : {1}) {
    if (nc) break;
    run<0>(16, 8, 16, nc);
    run<1>(16, 8, 16, nc);
    run<2>(16, 8, 16, nc);
    run<0>(4, 29, 4, nc);
    run<1>(4, 29, 4, nc);
    run<2>(4, 29, 4, nc);
    run<0>(8, 15, 16, nc);
    run<1>(8, 15, 16, nc);
  }
  return 0;
}
