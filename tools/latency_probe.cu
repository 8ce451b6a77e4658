// latency_probe.cu -- measurement tool (not product): where does a config-1
// parallel region's time go?  Replays the generic-mode handoff of
// csrc/ompds_kernels.cu (same device runtime, same barriers) for one team of
// 32 workers and records %globaltimer-free clock64() stamps at each step of
// the master's and worker 0's critical paths.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I paper_1711_10413_b200/csrc tools/latency_probe.cu -o /tmp/probe
#include "ompds_device.cuh"

#include <cstdio>
#include <vector>

using namespace ompds;

constexpr int R = 256;
constexpr int NS = 12;

__global__ void probe(int32_t *a, long long *ts, int variant) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int depot = 56, prealloc = 20;
  TeamCtx t = make_team(smem, depot, prealloc, 0, nullptr, 0, nullptr, 0);
  for (int i = threadIdx.x; i < team_region_bytes(depot, prealloc); i += blockDim.x)
    smem[i] = 0;
  __syncthreads();
  if (threadIdx.x == 0)
    t.work_fn() = -1;
  __syncthreads();
  const uint32_t nthr = blockDim.x;
  if (threadIdx.x < 32) { // worker warp
    const bool mine = true;
    for (int r = 0;; ++r) {
      long long *T = ts + (r < R ? r : R - 1) * NS;
      bar_sync(kBarHandoff, nthr);
      long long t0 = clock64();
      Fetch f = begin_parallel_warp(t, mine);
      long long t1 = clock64();
      if (f.fn < 0)
        break;
      SharedVars sv = get_shared_variables(f.args, f.nargs);
      int32_t old = a[threadIdx.x];
      int32_t c1 = shared_value<int32_t>(sv, 0), c2 = shared_value<int32_t>(sv, 1);
      int32_t c3 = shared_value<int32_t>(sv, 2), c4 = shared_value<int32_t>(sv, 3);
      long long t2 = clock64();
      a[threadIdx.x] = old + c1 + c2 + c3 + c4;
      long long t3 = clock64();
      end_parallel_warp(t, mine, f);
      long long t4 = clock64();
      if (threadIdx.x == 0) {
        T[0] = t0; T[1] = t1; T[2] = t2; T[3] = t3; T[4] = t4;
      }
      bar_sync(kBarHandoff, nthr);
      if (threadIdx.x == 0)
        T[5] = clock64();
    }
  } else {
    const bool leader = (threadIdx.x & 31) == 0;
    if (leader)
      kernel_init(t, kMaster, 32);
    unsigned char *d = smem;
    if (leader) {
      *reinterpret_cast<int32_t *>(d) = 1; *reinterpret_cast<int32_t *>(d + 8) = 2;
      *reinterpret_cast<int32_t *>(d + 16) = 3; *reinterpret_cast<int32_t *>(d + 24) = 4;
    }
    void *mine = (threadIdx.x & 31) < 4 ? d + 8 * (threadIdx.x & 31) : nullptr;
    for (int r = 0; r < R; ++r) {
      long long *T = ts + r * NS;
      long long m0 = clock64();
      void **list = nullptr;
      int32_t s = 0;
      if (leader)
        s = prepare_parallel(t, kMaster, 0, 4, &list);
      s = __shfl_sync(0xffffffffu, s, 0);
      list = reinterpret_cast<void **>(__shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(list), 0));
      if ((threadIdx.x & 31) < 4)
        list[threadIdx.x & 31] = mine;
      long long m1 = clock64();
      bar_sync(kBarHandoff, nthr);
      long long m2 = clock64();
      bar_sync(kBarHandoff, nthr);
      long long m3 = clock64();
      if (leader)
        *reinterpret_cast<int32_t *>(d + 24) += 1;
      if (leader) {
        T[6] = m0; T[7] = m1; T[8] = m2; T[9] = m3;
      }
    }
    if (leader)
      kernel_deinit(t, kMaster);
    __syncwarp();
    bar_sync(kBarHandoff, nthr);
  }
}

int main() {
  int32_t *a;
  long long *ts;
  cudaMalloc(&a, 32 * 4);
  cudaMemset(a, 0, 128);
  cudaMalloc(&ts, R * NS * 8);
  cudaMemset(ts, 0, R * NS * 8);
  probe<<<1, 64, team_region_bytes(56, 20)>>>(a, ts, 0);
  cudaError_t e = cudaDeviceSynchronize();
  if (e) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
  std::vector<long long> h(R * NS);
  cudaMemcpy(h.data(), ts, R * NS * 8, cudaMemcpyDeviceToHost);
  // average over regions 16..R-2 of each interval
  const char *names[] = {"worker: fetch (begin_parallel_warp)", "worker: gsv + capture values + body load",
                         "worker: body store", "worker: end_parallel_warp", "worker: end -> join released",
                         "master: prepare+publish", "master: release bar", "master: release -> join released",
                         "region period (master m0 -> next m0)", "master: after join -> next m0",
                         "release: master m1 -> worker t0"};
  double acc[11] = {0};
  int n = 0;
  for (int r = 16; r < R - 2; ++r) {
    long long *T = h.data() + r * NS, *U = h.data() + (r + 1) * NS;
    acc[0] += T[1] - T[0]; acc[1] += T[2] - T[1]; acc[2] += T[3] - T[2]; acc[3] += T[4] - T[3];
    acc[4] += T[5] - T[4]; acc[5] += T[7] - T[6]; acc[6] += T[8] - T[7]; acc[7] += T[9] - T[8];
    acc[8] += U[6] - T[6]; acc[9] += U[6] - T[9]; acc[10] += T[0] - T[7];
    ++n;
  }
  for (int i = 0; i < 11; ++i)
    printf("%-45s %8.1f cycles\n", names[i], acc[i] / n);
  int32_t ha[32];
  cudaMemcpy(ha, a, 128, cudaMemcpyDeviceToHost);
  printf("a[0]=%d\n", ha[0]);
  return 0;
}
