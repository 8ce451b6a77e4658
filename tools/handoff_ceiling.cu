// handoff_ceiling.cu -- measurement tool (not product): the whole-GPU ceiling
// of the config-1 handoff alone.  Teams of 64 threads (one worker warp + the
// master warp) run R "regions" of nothing but the two named-barrier
// handoffs (release + join, barrier id 1, 64 threads), optionally with the
// lean protocol's shared-memory traffic around them (mode 1: master one
// staging STS.64 + one list STS.64; workers one LDS + two LDS.128), so the
// config-1 kernel's regions/s can be read against what the barriers (and
// the shared-memory instructions) alone allow per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o handoff_ceiling tools/handoff_ceiling.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int kMode>
__global__ void __launch_bounds__(64, 32) handoff(int R, unsigned long long *sink) {
  __shared__ __align__(16) unsigned long long w[8];
  const int warp = threadIdx.x >> 5;
  const unsigned lane = threadIdx.x & 31;
  if (threadIdx.x < 8)
    w[threadIdx.x] = threadIdx.x;
  __syncthreads();
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(w));
  unsigned long long acc = 0;
  if (warp == 1) { // master
    for (int r = 0; r < R; ++r) {
      if (kMode == 1 || kMode == 2) { // predicated, as the product's staging (no divergence)
        asm volatile("{\n\t.reg .pred p, q;\n\tsetp.eq.u32 p, %2, 0;\n\tsetp.lt.u32 q, %2, 4;\n\t"
                     "@p st.shared.u64 [%0], %1;\n\t@q st.shared.u64 [%3], %1;\n\t}"
                     ::"r"(sa), "l"((unsigned long long)r), "r"(lane), "r"(sa + 16 + 8 * lane)
                     : "memory");
      }
      if (kMode == 6) // every lane stores (no predicate)
        asm volatile("st.shared.u64 [%0], %1;" ::"r"(sa + 8 * (lane & 7)), "l"((unsigned long long)r) : "memory");
      if (kMode == 7) { // lane-0 predicated store, then the master reads it back before the release
        unsigned long long v;
        asm volatile("{\n\t.reg .pred p;\n\tsetp.eq.u32 p, %2, 0;\n\t"
                     "@p st.shared.u64 [%0], %1;\n\t}" ::"r"(sa), "l"((unsigned long long)r), "r"(lane) : "memory");
        asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(sa) : "memory");
        acc += v;
      }
      if (kMode == 4) { // one store, then ~100 cycles of independent work before the release
        if (lane == 0)
          asm volatile("st.shared.u64 [%0], %1;" ::"r"(sa), "l"((unsigned long long)r) : "memory");
        unsigned x = r;
#pragma unroll
        for (int k = 0; k < 24; ++k)
          x = x * 1664525u + 1013904223u;
        acc += x;
      }
      asm volatile("bar.sync 1, 64;" ::: "memory");
      asm volatile("bar.sync 1, 64;" ::: "memory");
    }
  } else {
    for (int r = 0; r < R; ++r) {
      asm volatile("bar.sync 1, 64;" ::: "memory");
      if (kMode == 1 || kMode == 3) {
        unsigned long long s, a, b, c, d;
        asm volatile("ld.volatile.shared.u64 %0, [%5];\n\t"
                     "ld.volatile.shared.v2.u64 {%1, %2}, [%5+16];\n\t"
                     "ld.volatile.shared.v2.u64 {%3, %4}, [%5+32];"
                     : "=l"(s), "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "r"(sa) : "memory");
        acc += s + a + b + c + d;
      }
      if (kMode == 5) { // one dependent LDS after the release
        unsigned long long v;
        asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(sa) : "memory");
        acc += v;
      }
      asm volatile("bar.sync 1, 64;" ::: "memory");
    }
  }
  if (acc == 42)
    *sink = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long *sink;
  cudaMalloc(&sink, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int R = 20000;
  const char *names[] = {"barriers only", "barriers + master 2 STS + worker 3 LDS",
                         "barriers + master 2 STS", "barriers + worker 3 LDS",
                         "barriers + master STS 100 cycles before release",
                         "barriers + worker 1 LDS", "barriers + master STS, every lane",
                         "barriers + master STS then LDS before release"};
  for (int mode = 0; mode < 8; ++mode)
    for (int per_sm : {1, 16, 32}) {
      const int teams = sms * per_sm;
      float best = 1e30f;
      for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(a);
        switch (mode) {
        case 0: handoff<0><<<teams, 64>>>(R, sink); break;
        case 1: handoff<1><<<teams, 64>>>(R, sink); break;
        case 2: handoff<2><<<teams, 64>>>(R, sink); break;
        case 3: handoff<3><<<teams, 64>>>(R, sink); break;
        case 4: handoff<4><<<teams, 64>>>(R, sink); break;
        case 5: handoff<5><<<teams, 64>>>(R, sink); break;
        case 6: handoff<6><<<teams, 64>>>(R, sink); break;
        case 7: handoff<7><<<teams, 64>>>(R, sink); break;
        }
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (rep && ms < best)
          best = ms;
      }
      printf("mode %d (%-48s) teams/SM %2d: %7.2f ns per region per team, %6.2f G regions/s\n",
             mode, names[mode], per_sm, best * 1e6 / R, double(teams) * R / (best * 1e-3) / 1e9);
    }
  return 0;
}
