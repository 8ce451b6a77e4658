// Per-launch floor of kernels with the config-2 team geometry (296 x 512
// threads, 2281 B dynamic smem), queued back to back: an empty kernel, one
// that only synchronises the CTA a few times, and one that also reads 2 KB
// from global into smem -- what a team kernel's fixed cost is made of
// (measurement tool: nvcc -gencode arch=compute_100a,code=sm_100a -o lf
// tools/launch_floor.cu && ./lf).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void empty_k(double *) {}
__global__ void bars_k(double *p, int nb) {
  for (int i = 0; i < nb; ++i)
    asm volatile("barrier.sync 1, %0;" ::"r"(blockDim.x));
}
__global__ void __launch_bounds__(1024, 1) stage_k(double *p, int nb) {
  extern __shared__ double sm[];
  if (threadIdx.x < 256)
    sm[threadIdx.x] = p[threadIdx.x];
  for (int i = 0; i < nb; ++i)
    asm volatile("barrier.sync 1, %0;" ::"r"(blockDim.x));
  if (threadIdx.x == 0 && sm[5] == 123.0)
    p[0] = 1;
}

template <class F> float time_it(F f, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 10; ++i)
    f();
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i)
    f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms * 1000.f / reps;
}

int main() {
  double *p;
  cudaMalloc(&p, 1 << 20);
  cudaMemset(p, 0, 1 << 20);
  const int reps = 2000;
  for (int threads : {128, 512}) {
    for (int teams : {148, 296, 1036}) {
      printf("teams %4d x %3d: empty %.2f us, 4 barriers %.2f us, stage+4 barriers %.2f us, "
             "+2281 B smem %.2f us\n",
             teams, threads, time_it([&] { empty_k<<<teams, threads>>>(p); }, reps),
             time_it([&] { bars_k<<<teams, threads>>>(p, 4); }, reps),
             time_it([&] { stage_k<<<teams, threads, 2048>>>(p, 4); }, reps),
             time_it([&] { stage_k<<<teams, threads, 2281>>>(p, 4); }, reps));
    }
  }
  return 0;
}
