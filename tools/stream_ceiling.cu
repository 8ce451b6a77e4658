// stream_ceiling.cu -- measurement tool (not product): how fast can B200
// stream the config-4 body y = fma(c1, x, y) + s over 2^28 doubles
// (24 B/element) outside the data-sharing runtime?  Bounds what the
// generic-mode kernel can reach.  Variants:
//   ldg<U>    grid-stride over 16-byte units, U units of x and y in flight
//   bulk<S>   per-CTA tiles staged with cp.async.bulk (TMA) into shared
//             memory, S-stage mbarrier pipeline, result written back with
//             cp.async.bulk shared->global
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/stream_ceiling.cu -o tools/stream_ceiling.bin
#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ double op(double c1, double x, double y, double s) {
  return __dadd_rn(__fma_rn(c1, x, y), s);
}

template <int U>
__global__ void __launch_bounds__(1024) ldg(const double2 *__restrict__ x, double2 *__restrict__ y,
                                            int64_t units, double c1, double s) {
  const int64_t pool = int64_t(gridDim.x) * blockDim.x;
  int64_t u = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; u + (U - 1) * pool < units; u += U * pool) {
    double2 xs[U], ys[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      xs[k] = __ldcs(x + u + k * pool);
      ys[k] = __ldcs(y + u + k * pool);
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      ys[k].x = op(c1, xs[k].x, ys[k].x, s);
      ys[k].y = op(c1, xs[k].y, ys[k].y, s);
      __stcs(y + u + k * pool, ys[k]);
    }
  }
  for (; u < units; u += pool) {
    double2 a = __ldcs(x + u), b = __ldcs(y + u);
    b.x = op(c1, a.x, b.x, s);
    b.y = op(c1, a.y, b.y, s);
    __stcs(y + u, b);
  }
}

// K consecutive 16-byte units per thread (16K bytes contiguous per thread),
// cyclic over threads: unit block b = gid + j * pool covers units [K*b, K*b+K)
template <int K>
__global__ void __launch_bounds__(1024) ldg_blk(const double2 *__restrict__ x,
                                                double2 *__restrict__ y, int64_t units,
                                                double c1, double s) {
  const int64_t pool = int64_t(gridDim.x) * blockDim.x;
  const int64_t blocks = units / K;
  for (int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; b < blocks; b += pool) {
    double2 xs[K], ys[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      xs[k] = __ldcs(x + b * K + k);
      ys[k] = __ldcs(y + b * K + k);
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
      ys[k].x = op(c1, xs[k].x, ys[k].x, s);
      ys[k].y = op(c1, xs[k].y, ys[k].y, s);
      __stcs(y + b * K + k, ys[k]);
    }
  }
}

__device__ __forceinline__ uint32_t sa(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// TMA bulk pipeline: tile = T doubles of x and of y; S stages.  Warp 0 lane 0
// issues loads; all threads compute; the tile is stored back with one bulk
// store by thread 0 after a __syncthreads.
template <int S, int T>
__global__ void __launch_bounds__(256) bulk(const double *__restrict__ x, double *__restrict__ y,
                                            int64_t n, double c1, double s) {
  extern __shared__ __align__(128) unsigned char sm[];
  double *xs = reinterpret_cast<double *>(sm);
  double *ys = xs + S * T;
  __shared__ __align__(8) uint64_t full[S];
  const int64_t tiles = n / T;
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  auto issue = [&](int64_t tile, int st) {
    const uint32_t bytes = T * 8;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[st])),
                 "r"(2 * bytes));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(sa(xs + st * T)), "l"(x + tile * T), "r"(bytes), "r"(sa(&full[st])) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(sa(ys + st * T)), "l"(y + tile * T), "r"(bytes), "r"(sa(&full[st])) : "memory");
  };
  int64_t t0 = blockIdx.x;
  if (threadIdx.x == 0)
    for (int i = 0; i < S; ++i)
      if (t0 + int64_t(i) * gridDim.x < tiles)
        issue(t0 + int64_t(i) * gridDim.x, i);
  uint32_t phase = 0;
  int st = 0;
  for (int64_t t = t0; t < tiles; t += gridDim.x) {
    asm volatile("{\n.reg .pred P;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W_%=;\n}"
                 ::"r"(sa(&full[st])), "r"(phase) : "memory");
    double2 *x2 = reinterpret_cast<double2 *>(xs + st * T);
    double2 *y2 = reinterpret_cast<double2 *>(ys + st * T);
    for (int i = threadIdx.x; i < T / 2; i += blockDim.x) {
      double2 a = x2[i], b = y2[i];
      b.x = op(c1, a.x, b.x, s);
      b.y = op(c1, a.y, b.y, s);
      y2[i] = b;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                   ::"l"(y + t * T), "r"(sa(ys + st * T)), "r"(T * 8) : "memory");
      asm volatile("cp.async.bulk.commit_group;");
      // the stage is reused by the load S tiles ahead: its store must have
      // read shared memory first
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      const int64_t nt = t + int64_t(S) * gridDim.x;
      if (nt < tiles)
        issue(nt, st);
    }
    __syncthreads();
    if (++st == S) {
      st = 0;
      phase ^= 1;
    }
  }
  if (threadIdx.x == 0)
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  const int64_t n = int64_t(1) << 28;
  double *x, *y;
  cudaMalloc(&x, n * 8);
  cudaMalloc(&y, n * 8);
  cudaMemset(x, 0, n * 8);
  cudaMemset(y, 0, n * 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](const char *name, auto launch) {
    for (int i = 0; i < 3; ++i)
      launch();
    cudaEventRecord(e0);
    const int R = 50;
    for (int i = 0; i < R; ++i)
      launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double gbs = 24.0 * n * R / (ms * 1e-3) / 1e9;
    printf("%-44s %8.1f GB/s  (%s)\n", name, gbs, cudaGetErrorString(cudaGetLastError()));
  };
  const int64_t units = n / 2;
  for (int bps : {2, 16}) {
    for (int thr : {128, 1024}) {
      if (bps * thr > 2048)
        continue;
      char nm[96];
      snprintf(nm, sizeof nm, "ldg<2>  %d blocks/SM x %d", bps, thr);
      timeit(nm, [&] { ldg<2><<<sms * bps, thr>>>((const double2 *)x, (double2 *)y, units, 0.125, 4.375); });
      snprintf(nm, sizeof nm, "ldg<4>  %d blocks/SM x %d", bps, thr);
      timeit(nm, [&] { ldg<4><<<sms * bps, thr>>>((const double2 *)x, (double2 *)y, units, 0.125, 4.375); });
    }
  }
  // repeatability: the product geometry vs the best contiguous-block one
  for (int rep = 0; rep < 4; ++rep) {
    timeit("rep ldg<2> 1184 x 96 (product geometry)", [&] {
      ldg<2><<<sms * 8, 96>>>((const double2 *)x, (double2 *)y, units, 0.125, 4.375); });
    timeit("rep ldg_blk<4> 888 x 96", [&] {
      ldg_blk<4><<<sms * 6, 96>>>((const double2 *)x, (double2 *)y, units, 0.125, 4.375); });
    timeit("rep ldg_blk<2> 888 x 96", [&] {
      ldg_blk<2><<<sms * 6, 96>>>((const double2 *)x, (double2 *)y, units, 0.125, 4.375); });
  }
  // contiguous per-thread blocks of K units
  for (int k : {6, 8, 12, 16}) {
    for (int thr : {96, 128, 256}) {
      char nm[96];
      snprintf(nm, sizeof nm, "ldg_blk<2> %d x %d", sms * k, thr);
      timeit(nm, [&] { ldg_blk<2><<<sms * k, thr>>>((const double2 *)x, (double2 *)y, units, 0.125, 4.375); });
      snprintf(nm, sizeof nm, "ldg_blk<4> %d x %d", sms * k, thr);
      timeit(nm, [&] { ldg_blk<4><<<sms * k, thr>>>((const double2 *)x, (double2 *)y, units, 0.125, 4.375); });
    }
  }
  // pool-size sensitivity: the generic-mode kernel runs 96 workers per
  // 128-thread team; here a plain grid of 148*k blocks of t threads
  for (int k : {6, 7, 8, 9, 10}) {
    for (int thr : {64, 96, 128, 160, 192, 224}) {
      if (k * thr > 2048)
        continue;
      char nm[96];
      snprintf(nm, sizeof nm, "ldg<2>  %d x %d threads (pool %d)", sms * k, thr, sms * k * thr);
      timeit(nm, [&] { ldg<2><<<sms * k, thr>>>((const double2 *)x, (double2 *)y, units, 0.125, 4.375); });
    }
  }
  {
    constexpr int T = 2048, S = 4; // 16 KB x + 16 KB y per stage
    const size_t smem = size_t(2) * S * T * 8;
    cudaFuncSetAttribute(bulk<S, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    for (int bps : {1, 2, 3}) {
      char nm[96];
      snprintf(nm, sizeof nm, "bulk<4 stages, 16 KB tiles> %d blocks/SM", bps);
      timeit(nm, [&] { bulk<S, T><<<sms * bps, 256, smem>>>(x, y, n, 0.125, 4.375); });
    }
  }
  {
    constexpr int T = 4096, S = 3; // 32 KB x + 32 KB y per stage
    const size_t smem = size_t(2) * S * T * 8;
    cudaFuncSetAttribute(bulk<S, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    char nm[96];
    snprintf(nm, sizeof nm, "bulk<3 stages, 32 KB tiles> 1 block/SM");
    timeit(nm, [&] { bulk<S, T><<<sms, 256, smem>>>(x, y, n, 0.125, 4.375); });
  }
  {
    constexpr int T = 1024, S = 6; // 8 KB x + 8 KB y per stage
    const size_t smem = size_t(2) * S * T * 8;
    cudaFuncSetAttribute(bulk<S, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    for (int bps : {2, 4}) {
      char nm[96];
      snprintf(nm, sizeof nm, "bulk<6 stages, 8 KB tiles> %d blocks/SM", bps);
      timeit(nm, [&] { bulk<S, T><<<sms * bps, 256, smem>>>(x, y, n, 0.125, 4.375); });
    }
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
