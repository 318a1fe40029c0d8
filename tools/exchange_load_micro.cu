// Microbenchmark: the data movement of one K3 stage without the arithmetic.
// Each round (stage) every CTA of a cluster
//   * streams a factor tile of `tile` bytes from a large HBM buffer into
//     shared memory with one TMA bulk copy, one round ahead (as K3 does);
//   * writes its rows of `nv` vectors (rows x rc complex each) to global,
//     fences the async proxy and multicasts them to the CTAs of its group
//     (group = the whole cluster, or halves of it when `split`);
//   * waits until all rows of the round have landed.
// Reports cycles per round.  It answers: is the K3 exchange bound by the
// per-SM ingress (multicast + tile bytes) rather than by latency?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/elm tools/exchange_load_micro.cu
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstring>

namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t par) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
                   su32(b)),
               "r"(par)
               : "memory");
}

struct Cfg {
  int C, rows, rc, nv, split;
  uint32_t tile;
};

__global__ void k_stage_io(Cfg c, int rounds, double2 *gbuf, const char *hbm, size_t hbm_bytes, long long *out) {
  cg::cluster_group cl = cg::this_cluster();
  const int rank = cl.block_rank();
  const int t = threadIdx.x;
  const int G = c.split ? c.C / 2 : c.C;           // CTAs per exchange group
  const int grp = c.split ? rank / G : 0, gr = rank % G;
  const uint16_t mask = (uint16_t)(((1u << G) - 1) << (grp * G));
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t *vbar = (uint64_t *)sm;   // [2]
  uint64_t *fbar = vbar + 2;         // [2]
  const int per = c.rows * c.rc;      // my rows of one vector
  const int n = G * per;              // one vector
  double2 *vec = (double2 *)(sm + 128);       // [2 parity][nv][n]
  char *tile = (char *)(vec + 2 * c.nv * n);  // [2][tile]
  const uint32_t vbytes = (uint32_t)(n * 16) * c.nv;
  double2 *g = gbuf + ((size_t)(blockIdx.y * gridDim.x + blockIdx.x)) * 2 * c.nv * per;
  if (t == 0) {
    mbar_init(&vbar[0], 1);
    mbar_init(&vbar[1], 1);
    mbar_init(&fbar[0], 1);
    mbar_init(&fbar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cl.sync();
  const size_t stride = (size_t)gridDim.x * gridDim.y * c.tile;
  auto load_tile = [&](int r) {
    if (!c.tile) return;
    size_t off = ((size_t)r * stride + (size_t)(blockIdx.y * gridDim.x + blockIdx.x) * c.tile) % (hbm_bytes - c.tile);
    off &= ~(size_t)127;
    mbar_expect_tx(&fbar[r & 1], c.tile);
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     su32(tile + (r & 1) * c.tile)),
                 "l"(hbm + off), "r"(c.tile), "r"(su32(&fbar[r & 1]))
                 : "memory");
  };
  if (t == 0) {
    mbar_expect_tx(&vbar[0], vbytes);
    mbar_expect_tx(&vbar[1], vbytes);
    load_tile(0);
  }
  long long t0 = clock64();
  for (int r = 0; r < rounds; ++r) {
    const int b = r & 1;
    if (t == 0 && r + 1 < rounds) load_tile(r + 1);
    // my rows depend on the previous round's vectors
    double2 seed = r ? vec[((r - 1) & 1) * c.nv * n + (t % n)] : make_double2(rank, t);
    for (int e = t; e < c.nv * per; e += blockDim.x) g[b * c.nv * per + e] = make_double2(seed.x + e, seed.y);
    asm volatile("fence.proxy.async.global;" ::: "memory");
    __syncthreads();
    if (t == 0) {
      for (int v = 0; v < c.nv; ++v)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], "
            "%4;" ::"r"(su32(vec + (b * c.nv + v) * n + gr * per)),
            "l"(g + b * c.nv * per + v * per), "r"((uint32_t)(per * 16)), "r"(su32(&vbar[b])), "h"(mask)
            : "memory");
    }
    if (c.tile) mbar_wait(&fbar[b], (r >> 1) & 1);
    mbar_wait(&vbar[b], (r >> 1) & 1);
    __syncthreads();
    if (t == 0 && r + 2 < rounds) mbar_expect_tx(&vbar[b], vbytes);
  }
  long long t1 = clock64();
  cl.sync();
  if (t == 0 && rank == 0) out[blockIdx.y] = (t1 - t0) / rounds;
}

static char *g_hbm;
static size_t g_hbm_bytes = (size_t)4 << 30;

void run(Cfg c, int nclusters, const char *label) {
  const int rounds = 2000;
  const int G = c.split ? c.C / 2 : c.C;
  size_t smem = 128 + (size_t)2 * c.nv * G * c.rows * c.rc * 16 + 2 * (size_t)c.tile;
  cudaFuncSetAttribute(k_stage_io, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k_stage_io, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  double2 *gb;
  cudaMalloc(&gb, (size_t)nclusters * c.C * 2 * c.nv * c.rows * c.rc * 16);
  long long *out;
  cudaMalloc(&out, 8 * nclusters);
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3(c.C, nclusters);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute a[1];
  a[0].id = cudaLaunchAttributeClusterDimension;
  a[0].val.clusterDim.x = c.C;
  a[0].val.clusterDim.y = 1;
  a[0].val.clusterDim.z = 1;
  cfg.attrs = a;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k_stage_io, c, rounds, gb, (const char *)g_hbm, g_hbm_bytes, out);
  cudaError_t e2 = cudaDeviceSynchronize();
  long long h[16] = {0};
  cudaMemcpy(h, out, 8 * nclusters, cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < nclusters; ++i) mx = h[i] > mx ? h[i] : mx;
  double in_kb = (c.nv * G * c.rows * c.rc * 16.0 + c.tile) / 1024.0;
  printf("%-44s C=%2d grp=%2d rows=%2d rc=%2d nv=%d tile=%5u clusters=%d : %5lld cycles/round  ingress %.1f KB/round "
         "(%.1f B/clk)  %s\n",
         label, c.C, G, c.rows, c.rc, c.nv, c.tile, nclusters, mx, in_kb, in_kb * 1024 / (mx ? mx : 1),
         e != cudaSuccess ? cudaGetErrorString(e) : cudaGetErrorString(e2));
  cudaFree(gb);
  cudaFree(out);
}

int main() {
  cudaMalloc(&g_hbm, g_hbm_bytes);
  cudaMemset(g_hbm, 1, g_hbm_bytes);
  const uint32_t tile8 = 8 * 115 * 16, tile15 = 15 * 115 * 16;
  for (int ncl : {1, 7}) {
    run({16, 8, 16, 1, 0, 0}, ncl, "one vector, no tile");
    run({16, 8, 16, 2, 0, 0}, ncl, "two vectors (v5 halves), no tile");
    run({16, 8, 16, 1, 0, 2 * tile8}, ncl, "one vector + 2x8-row tiles");
    run({16, 8, 16, 2, 0, 2 * tile8}, ncl, "two vectors + 2x8-row tiles (v5 stage)");
    run({16, 15, 16, 1, 1, tile15}, ncl, "split: 8-CTA groups, one vector + 15-row tile");
    run({16, 15, 16, 1, 1, 0}, ncl, "split: 8-CTA groups, one vector, no tile");
    run({16, 8, 8, 2, 0, 2 * tile8}, ncl, "two vectors rc=8 + tiles");
  }
  return 0;
}
