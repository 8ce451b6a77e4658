// stack_cost.cu -- measurement tool (not product): cost of a data-sharing
// stack push + pop pair (DsStack, csrc/ompds_device.cuh) on one worker warp,
// in SM cycles (clock64), with the frame in the shared-memory slot or on the
// global overflow chain.  Each iteration pushes a lane-strided frame (40
// bytes per lane, the config-3 level-1 frame), stores and reloads one value
// in it, and pops; the baseline does the same store/load at a fixed address.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I paper_1711_10413_b200/csrc tools/stack_cost.cu -o tools/stack_cost.bin
#include "ompds_device.cuh"

#include <cstdio>

using namespace ompds;

constexpr int N = 4096;

template <int mode>
__global__ void stack_cost(unsigned char *chain, long long *out) {
  __shared__ __align__(16) unsigned char slot[4096];
  const uint32_t lane = threadIdx.x & 31;
  DsStack ds;
  // mode 0: baseline (no push/pop); 1: frames in the slot; 2: on the chain
  ds.init(slot, mode == 2 ? 0 : 4096, chain, 1 << 16);
  int32_t acc = 0;
  __syncwarp();
  const long long t0 = clock64();
  for (int i = 0; i < N; ++i) {
    unsigned char *base;
    Frame f{};
    if constexpr (mode == 0) {
      base = slot;
    } else {
      f = ds.push(40, kWarp);
      base = f.base;
    }
    volatile int32_t *e = reinterpret_cast<volatile int32_t *>(base + lane * 40);
    *e = i + acc;
    acc += *e;
    if constexpr (mode != 0)
      acc += ds.pop(f);
  }
  const long long t1 = clock64();
  if (lane == 0) {
    out[2 * mode] = t1 - t0;
    out[2 * mode + 1] = acc;
  }
}

int main() {
  unsigned char *chain;
  long long *out;
  cudaMalloc(&chain, 1 << 16);
  cudaMalloc(&out, 64);
  const char *names[] = {"store+load at a fixed smem address (baseline)",
                         "push + store/load in the frame + pop, smem slot",
                         "push + store/load in the frame + pop, global chain"};
  long long h[6];
  for (int rep = 0; rep < 2; ++rep) {
    stack_cost<0><<<1, 32>>>(chain, out);
    stack_cost<1><<<1, 32>>>(chain, out);
    stack_cost<2><<<1, 32>>>(chain, out);
  }
  cudaMemcpy(h, out, sizeof h, cudaMemcpyDeviceToHost);
  for (int mode = 0; mode < 3; ++mode)
    printf("%-52s %7.1f cycles/iteration\n", names[mode], double(h[2 * mode]) / N);
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
