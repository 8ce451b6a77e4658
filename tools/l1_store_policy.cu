// Does a global store leave its line in L1 for a later load by the same
// warp?  A dependent chain: store v to p[i], then load p[i] (the value feeds
// the next address), for several store cache qualifiers; cycles per step.
// Stores and loads are separated by `gap` independent ALU ops so the load is
// not forwarded from the store queue (measurement tool:
// nvcc -gencode arch=compute_100a,code=sm_100a -o l1p tools/l1_store_policy.cu).
#include <cstdio>
template <int M>
__global__ void chain(unsigned *buf, int steps, long long *out, unsigned seed) {
  const unsigned lane = threadIdx.x & 31;
  unsigned v = seed + lane, idx = lane;
  __syncwarp();
  long long t0 = clock64();
  for (int s = 0; s < steps; ++s) {
    unsigned *p = buf + ((idx * 32 + lane) & 0xffff);
    if (M == 0)
      asm volatile("st.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
    else if (M == 1)
      asm volatile("st.global.L1::evict_last.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
    else if (M == 2)
      asm volatile("st.global.wb.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
    else if (M == 3)
      asm volatile("st.global.L1::evict_normal.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
    // independent work so the load issues well after the store
#pragma unroll
    for (int k = 0; k < 64; ++k)
      v = v * 1664525u + 1013904223u;
    unsigned r;
    if (M == 4)
      asm volatile("ld.global.L1::evict_last.u32 %0, [%1];" : "=r"(r) : "l"(p) : "memory");
    else
      asm volatile("ld.global.u32 %0, [%1];" : "=r"(r) : "l"(p) : "memory");
    idx = (r ^ v) & 0x7ff;
  }
  long long t1 = clock64();
  if (lane == 0)
    out[0] = t1 - t0, out[1] = idx;
}
template <int M> double run(unsigned *b, long long *o, int steps) {
  chain<M><<<1, 32>>>(b, steps, o, 1);
  long long h[2];
  cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
  chain<M><<<1, 32>>>(b, steps, o, 1);
  cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
  return double(h[0]) / steps;
}
int main() {
  unsigned *b;
  long long *o;
  cudaMalloc(&b, 1 << 20);
  cudaMemset(b, 0, 1 << 20);
  cudaMalloc(&o, 16);
  const int n = 4096;
  printf("cycles per step (64 dependent IMADs + store + load):\n");
  printf("  st.global                 %.1f\n", run<0>(b, o, n));
  printf("  st.global.L1::evict_last  %.1f\n", run<1>(b, o, n));
  printf("  st.global.wb              %.1f\n", run<2>(b, o, n));
  printf("  st.global.L1::evict_normal %.1f\n", run<3>(b, o, n));
  printf("  st.global + ld.L1::evict_last %.1f\n", run<4>(b, o, n));
  return 0;
}
