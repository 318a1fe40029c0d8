// PCIe copy-shape probe: D2H / H2D GB/s for contiguous copies vs 2D copies
// with the row lengths the pinned host path uses (config 2: 3.5 KB rows).
#include <cstdio>
#include <cuda_runtime.h>
int main() {
  const size_t total = 48ull << 20;
  void *d, *h;
  cudaMalloc(&d, total * 2);
  cudaMallocHost(&h, total * 2);
  cudaStream_t s[2];
  for (auto &x : s) cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const size_t rows_list[] = {0, 577, 1750, 3500, 7000, 14000};
  for (int dir = 0; dir < 2; ++dir)
    for (int ns = 1; ns <= 2; ++ns)
      for (size_t w : rows_list) {
        float best = 1e9;
        for (int rep = 0; rep < 5; ++rep) {
          cudaEventRecord(a, s[0]);
          if (ns == 2) { cudaStreamWaitEvent(s[1], a, 0); }
          const int nchunk = 24;
          const size_t cb = total / nchunk;
          for (int c = 0; c < nchunk; ++c) {
            cudaStream_t st = s[c % ns];
            char *dp = (char *)d + c * cb, *hp = (char *)h + c * cb;
            if (w == 0) {
              if (dir == 0) cudaMemcpyAsync(hp, dp, cb, cudaMemcpyDeviceToHost, st);
              else cudaMemcpyAsync(dp, hp, cb, cudaMemcpyHostToDevice, st);
            } else {
              size_t rows = cb / w;  // pitch 2w: half-width rows
              if (dir == 0) cudaMemcpy2DAsync(hp, 2 * w, dp, 2 * w, w, rows / 2, cudaMemcpyDeviceToHost, st);
              else cudaMemcpy2DAsync(dp, 2 * w, hp, 2 * w, w, rows / 2, cudaMemcpyHostToDevice, st);
            }
          }
          if (ns == 2) { cudaEvent_t j; cudaEventCreate(&j); cudaEventRecord(j, s[1]); cudaStreamWaitEvent(s[0], j, 0); }
          cudaEventRecord(b, s[0]);
          cudaEventSynchronize(b);
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          if (ms < best) best = ms;
        }
        size_t bytes = w == 0 ? total : (total / 2);
        printf("%s streams %d row %6zu B: %.1f GB/s\n", dir == 0 ? "D2H" : "H2D", ns, w,
               bytes / best / 1e6);
      }
  // bidirectional: contiguous D2H and H2D at once
  {
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(a, s[0]);
      cudaStreamWaitEvent(s[1], a, 0);
      cudaMemcpyAsync(h, d, total, cudaMemcpyDeviceToHost, s[0]);
      cudaMemcpyAsync((char *)d + total, (char *)h + total, total, cudaMemcpyHostToDevice, s[1]);
      cudaEvent_t j; cudaEventCreate(&j); cudaEventRecord(j, s[1]); cudaStreamWaitEvent(s[0], j, 0);
      cudaEventRecord(b, s[0]);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    printf("bidirectional 48 MB each way: %.3f ms (%.1f GB/s per direction)\n", best, total / best / 1e6);
  }
  return 0;
}
