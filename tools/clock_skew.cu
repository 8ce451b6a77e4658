// clock64 across the warps of one CTA: every warp stamps right after the
// same named barrier; the spread is the skew between the SM sub-partitions'
// counters (measurement tool: nvcc -gencode arch=compute_100a,code=sm_100a
// -o clock_skew tools/clock_skew.cu).
#include <cstdio>
__global__ void k(long long *out, int rounds) {
  for (int r = 0; r < rounds; ++r) {
    asm volatile("barrier.sync 1, %0;" ::"r"(blockDim.x));
    long long c;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(c)::"memory");
    if ((threadIdx.x & 31) == 0)
      out[r * 32 + threadIdx.x / 32] = c;
  }
}
int main() {
  long long *d, h[8 * 32];
  cudaMalloc(&d, sizeof(h));
  for (int threads : {64, 128, 256}) {
    k<<<1, threads>>>(d, 8);
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("threads %d:", threads);
    for (int r = 4; r < 6; ++r) {
      printf(" [");
      for (int w = 0; w < threads / 32; ++w)
        printf(" %lld", h[r * 32 + w] - h[r * 32]);
      printf(" ]");
    }
    printf("\n");
  }
  return 0;
}
