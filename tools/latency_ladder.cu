// latency_ladder.cu -- measurement tool (not product): marginal cost of each
// piece of a generic-mode parallel region on B200 (1 team, 32 workers).
// Variant k adds step k on top of variant k-1:
//   0 bare handoff: release + join named barriers only
//   1 + master prepare_parallel / publish list, worker fetch (smem state)
//   2 + get-shared-variables (list entry, capture values, shuffles)
//   3 + the body's global read-modify-write
//   4 + end_parallel (warp-aggregated retire, last-retire bookkeeping)
//   5 the product kernel's path (= 4 with the master's c4 += 1 and r store)
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I paper_1711_10413_b200/csrc tools/latency_ladder.cu -o tools/latency_ladder.bin
#include "ompds_device.cuh"

#include <cstdio>

using namespace ompds;

struct Opaque {
  int prealloc, fail, workers, maxev;
  ompds_event *ev;
  unsigned char *slab;
};
template <int V>
__global__ void ladder(int32_t *a, int R, long long *cycles, const __grid_constant__ Opaque o) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int depot = 56, prealloc = V >= 6 ? o.prealloc : 20;
  TeamCtx t = V >= 6 ? make_team(smem, depot, prealloc, o.fail, o.slab, 4096, o.ev, o.maxev)
                     : make_team(smem, depot, prealloc, 0, nullptr, 0, nullptr, 0);
  const bool mine = V >= 7 ? int(threadIdx.x) < o.workers : true;
  for (int i = threadIdx.x; i < team_region_bytes(depot, prealloc); i += blockDim.x)
    smem[i] = 0;
  __syncthreads();
  if (threadIdx.x == 0)
    t.work_fn() = -1;
  __syncthreads();
  const uint32_t nthr = blockDim.x;
  if (threadIdx.x < 32) {
    int32_t acc = 0;
    for (;;) {
      bar_sync(kBarHandoff, nthr);
      int32_t fn = 0;
      void **args = nullptr;
      int32_t nargs = 0;
      Fetch f{};
      if (V >= 1) {
        f = begin_parallel_warp(t, mine);
        fn = f.fn;
        args = f.args;
        nargs = f.nargs;
      } else {
        fn = t.phase() == kTerminated ? -1 : 0;
      }
      if (fn < 0)
        break;
      int32_t sum = 1;
      if (V >= 2) {
        SharedVars sv = get_shared_variables(args, nargs);
        sum = shared_value<int32_t>(sv, 0) + shared_value<int32_t>(sv, 1) +
              shared_value<int32_t>(sv, 2) + shared_value<int32_t>(sv, 3);
      }
      if (V >= 3)
        a[threadIdx.x] += sum;
      else
        acc += sum;
      if (V >= 4)
        end_parallel_warp(t, mine, f);
      bar_sync(kBarHandoff, nthr);
    }
    if (V < 3)
      a[threadIdx.x] = acc;
  } else {
    const bool leader = (threadIdx.x & 31) == 0;
    if (leader)
      kernel_init(t, kMaster, 32);
    unsigned char *d = smem;
    if (leader) {
      *reinterpret_cast<int32_t *>(d) = 1;
      *reinterpret_cast<int32_t *>(d + 8) = 2;
      *reinterpret_cast<int32_t *>(d + 16) = 3;
      *reinterpret_cast<int32_t *>(d + 24) = 4;
    }
    void *mine = (threadIdx.x & 31) < 4 ? d + 8 * (threadIdx.x & 31) : nullptr;
    __syncwarp();
    long long t0 = clock64();
    for (int r = 0; r < R; ++r) {
      if (V >= 1) {
        void **list = nullptr;
        unsigned long long packed = 0;
        if (leader) {
          int32_t s = prepare_parallel(t, kMaster, 0, 4, &list);
          packed = s ? (1ull << 63) : reinterpret_cast<unsigned long long>(list);
        }
        packed = __shfl_sync(0xffffffffu, packed, 0);
        list = reinterpret_cast<void **>(packed);
        if ((threadIdx.x & 31) < 4)
          list[threadIdx.x & 31] = mine;
      }
      bar_sync(kBarHandoff, nthr);
      bar_sync(kBarHandoff, nthr);
      if (V < 4 && V >= 1 && leader) // no end_parallel: reset by hand
        retire_last(t);
      if (V >= 5 && leader) {
        *reinterpret_cast<int32_t *>(d + 24) += 1;
        *reinterpret_cast<int32_t *>(d + 32) = r;
      }
    }
    long long t1 = clock64();
    if (leader) {
      *cycles = t1 - t0;
      t.phase() = kTerminated;
    }
    __syncwarp();
    bar_sync(kBarHandoff, nthr);
  }
}

template <int V> void run(int32_t *a, long long *c, int R) {
  Opaque o{20, 0, 32, 0, nullptr, nullptr};
  ladder<V><<<1, 64, team_region_bytes(56, 20)>>>(a, 64, c, o); // warm
  ladder<V><<<1, 64, team_region_bytes(56, 20)>>>(a, R, c, o);
  cudaDeviceSynchronize();
  long long h = 0;
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  ladder<V><<<1, 64, team_region_bytes(56, 20)>>>(a, R, c, o);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("variant %d: %7.1f cycles/region (clock64)  %7.1f ns/region (events)\n", V,
         double(h) / R, ms * 1e6 / R);
}

int main() {
  int32_t *a;
  long long *c;
  cudaMalloc(&a, 128);
  cudaMemset(a, 0, 128);
  cudaMalloc(&c, 8);
  const int R = 20000;
  run<0>(a, c, R);
  run<1>(a, c, R);
  run<2>(a, c, R);
  run<3>(a, c, R);
  run<4>(a, c, R);
  run<5>(a, c, R);
  run<6>(a, c, R);
  run<7>(a, c, R);
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  int main_product(void);
  return main_product();
}

// ---------------------------------------------------------------------------
// Variant P: the product kernel template (generic_mode_kernel) with the
// config-1 program, timed inside the master loop with clock64.
#include "ompds_kernels.cu"

namespace ompds {
struct ProbeProg {
  struct Args {
    int32_t *a;
    int32_t regions;
    long long *cycles;
  };
  __device__ static void master(Master &m, const Args &a) {
    RegionsProg<int32_t>::Args ra{a.a, 64};
    RegionsProg<int32_t>::master(m, ra); // warm
    long long t0 = clock64();
    RegionsProg<int32_t>::Args rb{a.a, a.regions};
    RegionsProg<int32_t>::master(m, rb);
    long long t1 = clock64();
    if (m.leader)
      *a.cycles = t1 - t0;
  }
  __device__ static void region(int32_t fn, const SharedVars &sv, Worker &w,
                                const Args &a) {
    RegionsProg<int32_t>::Args ra{a.a, 0};
    RegionsProg<int32_t>::region(fn, sv, w, ra);
  }
};
// worker side replaced by the ladder's body
struct ProbeProgW {
  using Args = ProbeProg::Args;
  __device__ static void master(Master &m, const Args &a) { ProbeProg::master(m, a); }
  __device__ static void region(int32_t, const SharedVars &sv, Worker &w, const Args &a) {
    int32_t sum = shared_value<int32_t>(sv, 0) + shared_value<int32_t>(sv, 1) +
                  shared_value<int32_t>(sv, 2) + shared_value<int32_t>(sv, 3);
    a.a[threadIdx.x] += sum;
  }
};
// master side replaced by the ladder's loop
struct ProbeProgM {
  using Args = ProbeProg::Args;
  __device__ static void loop(Master &m, int R) {
    const bool leader = m.leader;
    unsigned char *d = m.t.region;
    void *mine = (threadIdx.x & 31) < 4 ? d + 8 * (threadIdx.x & 31) : nullptr;
    for (int r = 0; r < R; ++r) {
      void **list = nullptr;
      unsigned long long packed = 0;
      if (leader) {
        int32_t s = prepare_parallel(m.t, kMaster, 0, 4, &list);
        packed = s ? (1ull << 63) : reinterpret_cast<unsigned long long>(list);
      }
      packed = __shfl_sync(0xffffffffu, packed, 0);
      list = reinterpret_cast<void **>(packed);
      if ((threadIdx.x & 31) < 4)
        list[threadIdx.x & 31] = mine;
      bar_sync(kBarHandoff, m.team_threads);
      bar_sync(kBarHandoff, m.team_threads);
      if (leader) {
        *reinterpret_cast<int32_t *>(d + 24) += 1;
        *reinterpret_cast<int32_t *>(d + 32) = r;
      }
    }
  }
  __device__ static void master(Master &m, const Args &a) {
    loop(m, 64);
    long long t0 = clock64();
    loop(m, a.regions);
    long long t1 = clock64();
    if (m.leader)
      *a.cycles = t1 - t0;
  }
  __device__ static void region(int32_t fn, const SharedVars &sv, Worker &w, const Args &a) {
    ProbeProg::region(fn, sv, w, a);
  }
};
// ladder loop, but the handoff through Master::parallel_with
struct ProbeProgPW {
  using Args = ProbeProg::Args;
  __device__ static void loop(Master &m, int R) {
    const bool leader = m.leader;
    unsigned char *d = m.t.region;
    void *mine = (threadIdx.x & 31) < 4 ? d + 8 * (threadIdx.x & 31) : nullptr;
    for (int r = 0; r < R; ++r) {
      if (m.parallel_with(0, 4, [mine](int) { return mine; }) != OMPDS_OK)
        return;
      if (leader) {
        *reinterpret_cast<int32_t *>(d + 24) += 1;
        *reinterpret_cast<int32_t *>(d + 32) = r;
      }
    }
  }
  __device__ static void master(Master &m, const Args &a) {
    loop(m, 64);
    long long t0 = clock64();
    loop(m, a.regions);
    long long t1 = clock64();
    if (m.leader)
      *a.cycles = t1 - t0;
  }
  __device__ static void region(int32_t fn, const SharedVars &sv, Worker &w, const Args &a) {
    ProbeProg::region(fn, sv, w, a);
  }
};
} // namespace ompds

template <class P> void product_variant(const char *name) {
  int32_t *a;
  long long *c;
  cudaMalloc(&a, 128);
  cudaMalloc(&c, 8);
  const int R = 20000;
  ompds_launch l{1, 32, 20, 0, -1, 0, 0, nullptr};
  FixedLayout lay;
  build_fixed_layout({4, 4, 4, 4}, 4, &lay);
  launch_generic<P>(&l, lay, 4, typename P::Args{a, R, c}, nullptr, nullptr);
  cudaDeviceSynchronize();
  long long h = 0;
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("%s: %7.1f cycles/region\n", name, double(h) / R);
}

int main_product() {
  product_variant<ProbeProgW>("product master + ladder worker body");
  product_variant<ProbeProgM>("ladder master loop + product worker");
  product_variant<ProbeProgPW>("ladder master loop via Master::parallel_with");
  int32_t *a;
  long long *c;
  cudaMalloc(&a, 128);
  cudaMalloc(&c, 8);
  const int R = 20000;
  ompds_launch l{1, 32, 20, 0, -1, 0, 0, nullptr};
  FixedLayout lay;
  build_fixed_layout({4, 4, 4, 4}, 4, &lay);
  for (int k = 0; k < 2; ++k) {
    int32_t s = launch_generic<ProbeProg>(&l, lay, 4, ProbeProg::Args{a, R, c}, nullptr, nullptr);
    cudaDeviceSynchronize();
    long long h = 0;
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("product kernel (status %d): %7.1f cycles/region inside the master loop\n", s,
           double(h) / R);
  }
  // several worker warps: the retire takes the atomic path
  int32_t *a2;
  cudaMalloc(&a2, 4 * 1024);
  cudaMemset(a2, 0, 4 * 1024);
  for (int w : {64, 96, 224, 480, 992}) {
    ompds_launch l2{1, w, 20, 0, -1, 0, 0, nullptr};
    int32_t s = launch_generic<ProbeProg>(&l2, lay, 4, ProbeProg::Args{a2, R, c}, nullptr, nullptr);
    cudaDeviceSynchronize();
    long long h = 0;
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("product kernel W=%d (status %d): %7.1f cycles/region\n", w, s, double(h) / R);
  }
  return 0;
}
