// micro_lat.cu -- measurement tool (not product): latencies of the
// primitives a generic-mode region handoff is built from, on B200 (sm_100a),
// in SM clock cycles (clock64 inside one CTA).  Each test is a dependent
// chain or a ping-pong, so the number is a latency, not a throughput.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/micro_lat.cu -o tools/micro_lat.bin
#include <cstdint>
#include <cstdio>

constexpr int N = 4096;

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void k_chain(long long *out, int *gbuf, int test) {
  __shared__ __align__(16) uint32_t s[1024];
  __shared__ __align__(8) unsigned long long sp[64];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x)
    s[i] = (i + 1) & 1023;
  for (int i = threadIdx.x; i < 64; i += blockDim.x)
    sp[i] = reinterpret_cast<unsigned long long>(&sp[(i + 1) & 63]);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = 0;
  long long t0 = 0, t1 = 0;
  switch (test) {
  case 0: // LDS dependent chain
    if (warp == 0) {
      t0 = clock64();
      for (int i = 0; i < N; ++i)
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(x) : "r"(smem_u32(s) + 4 * x));
      t1 = clock64();
    }
    break;
  case 1: { // generic LD of a shared address, dependent chain
    if (warp == 0) {
      unsigned long long p = reinterpret_cast<unsigned long long>(&sp[0]);
      t0 = clock64();
      for (int i = 0; i < N; ++i)
        asm volatile("ld.u64 %0, [%0];" : "+l"(p));
      t1 = clock64();
      x = static_cast<uint32_t>(p);
    }
    break;
  }
  case 2: // ATOMS.ADD with return, dependent chain
    if (warp == 0) {
      t0 = clock64();
      for (int i = 0; i < N; ++i)
        x = atomicAdd(&s[x & 1], 0u);
      t1 = clock64();
    }
    break;
  case 3: // SHFL dependent chain
    if (warp == 0) {
      x = lane;
      t0 = clock64();
      for (int i = 0; i < N; ++i)
        x = __shfl_sync(0xffffffffu, x, (x + 1) & 31);
      t1 = clock64();
    }
    break;
  case 4: // barrier.sync 1, 64 ping-pong between two warps (no memory ops)
    if (warp < 2) {
      t0 = clock64();
      for (int i = 0; i < N; ++i)
        asm volatile("barrier.sync 1, 64;" ::: "memory");
      t1 = clock64();
    }
    break;
  case 5: // bar.sync (aligned) 1, 64 ping-pong
    if (warp < 2) {
      t0 = clock64();
      for (int i = 0; i < N; ++i)
        asm volatile("bar.sync 1, 64;" ::: "memory");
      t1 = clock64();
    }
    break;
  case 6: // STS by lane 0 + barrier.sync 1,64 + LDS by the other warp, chain
    if (warp < 2) {
      t0 = clock64();
      for (int i = 0; i < N; ++i) {
        if (warp == (i & 1) && lane == 0)
          asm volatile("st.shared.u32 [%0], %1;" ::"r"(smem_u32(s)), "r"(x + 1));
        asm volatile("barrier.sync 1, 64;" ::: "memory");
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(x) : "r"(smem_u32(s)));
      }
      t1 = clock64();
    }
    break;
  case 7: // RED.ADD (no return) by lane 0 then barrier.sync 1, 64
    if (warp < 2) {
      t0 = clock64();
      for (int i = 0; i < N; ++i) {
        if (lane == 0)
          atomicAdd(&s[warp], 1u);
        asm volatile("barrier.sync 1, 64;" ::: "memory");
      }
      t1 = clock64();
    }
    break;
  case 8: // atom.acq_rel.cta with return, lane 0, then barrier
    if (warp < 2) {
      t0 = clock64();
      for (int i = 0; i < N; ++i) {
        if (lane == 0) {
          uint32_t o;
          asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;"
                       : "=r"(o) : "r"(smem_u32(&s[warp])) : "memory");
          x += o;
        }
        asm volatile("barrier.sync 1, 64;" ::: "memory");
      }
      t1 = clock64();
    }
    break;
  case 9: // STG by every lane then barrier.sync 1, 64
    if (warp < 2) {
      t0 = clock64();
      for (int i = 0; i < N; ++i) {
        gbuf[threadIdx.x] = i;
        asm volatile("barrier.sync 1, 64;" ::: "memory");
      }
      t1 = clock64();
    }
    break;
  case 10: // LDG+STG read-modify-write of own element, then barrier (config-1 body)
    if (warp < 2) {
      t0 = clock64();
      for (int i = 0; i < N; ++i) {
        gbuf[threadIdx.x] += 1;
        asm volatile("barrier.sync 1, 64;" ::: "memory");
      }
      t1 = clock64();
    }
    break;
  case 11: // LDG dependent chain on the same address (L1 hit after first)
    if (warp == 0) {
      int *p = gbuf + 4096;
      t0 = clock64();
      for (int i = 0; i < N; ++i)
        x = *reinterpret_cast<volatile int *>(p + (x & 1));
      t1 = clock64();
    }
    break;
  case 12: // __syncwarp cost in a chain with STS
    if (warp == 0) {
      t0 = clock64();
      for (int i = 0; i < N; ++i)
        __syncwarp();
      t1 = clock64();
    }
    break;
  case 13: // fence.acq_rel.cta (MEMBAR.CTA) after an STG, lane 0
    if (warp == 0) {
      t0 = clock64();
      for (int i = 0; i < N; ++i) {
        gbuf[threadIdx.x] = i;
        asm volatile("fence.acq_rel.cta;" ::: "memory");
      }
      t1 = clock64();
    }
    break;
  case 14: // vote.ballot + popc chain
    if (warp == 0) {
      t0 = clock64();
      for (int i = 0; i < N; ++i)
        x = __popc(__ballot_sync(0xffffffffu, (x + lane) & 1));
      t1 = clock64();
    }
    break;
  case 15: // alternating handoff: warp 0 runs 8 dependent LDS while warp 1
            // waits, then warp 1 runs 8 while warp 0 waits (2 barriers/iter)
  case 16:  // same with 32 dependent LDS per side
    if (warp < 2) {
      const int K = test == 15 ? 8 : 32;
      t0 = clock64();
      for (int i = 0; i < N / 8; ++i) {
        if (warp == 0)
          for (int k = 0; k < K; ++k)
            asm volatile("ld.shared.u32 %0, [%1];" : "=r"(x) : "r"(smem_u32(s) + 4 * (x & 1023)));
        asm volatile("barrier.sync 1, 64;" ::: "memory");
        if (warp == 1)
          for (int k = 0; k < K; ++k)
            asm volatile("ld.shared.u32 %0, [%1];" : "=r"(x) : "r"(smem_u32(s) + 4 * (x & 1023)));
        asm volatile("barrier.sync 1, 64;" ::: "memory");
      }
      t1 = clock64();
      t1 = t0 + (t1 - t0) * 8; // reported per N/8 iterations below
    }
    break;
  case 17: // alternating handoff with no work (2 barriers/iter)
    if (warp < 2) {
      t0 = clock64();
      for (int i = 0; i < N / 8; ++i) {
        asm volatile("barrier.sync 1, 64;" ::: "memory");
        asm volatile("barrier.sync 1, 64;" ::: "memory");
      }
      t1 = clock64();
      t1 = t0 + (t1 - t0) * 8;
    }
    break;
  case 18: // divergent lane-0 STS + __syncwarp + barrier + LDS + shfl chain
    if (warp < 2) {
      t0 = clock64();
      for (int i = 0; i < N; ++i) {
        if (lane == 0 && warp == (i & 1))
          asm volatile("st.shared.u32 [%0], %1;" ::"r"(smem_u32(s)), "r"(x + 1));
        __syncwarp();
        asm volatile("barrier.sync 1, 64;" ::: "memory");
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(x) : "r"(smem_u32(s)));
        x = __shfl_sync(0xffffffffu, x, 0);
      }
      t1 = clock64();
    }
    break;
  }
  if (threadIdx.x == 0) {
    out[2 * test] = t1 - t0;
    out[2 * test + 1] = x;
  }
}

int main() {
  long long *out;
  int *g;
  cudaMalloc(&out, 64 * 8);
  cudaMalloc(&g, 1 << 20);
  cudaMemset(g, 0, 1 << 20);
  const char *names[] = {
      "LDS dependent chain (per load)",
      "generic LD to shared, dependent chain",
      "ATOMS.ADD with return, dependent chain",
      "SHFL.IDX dependent chain",
      "barrier.sync 1,64 two warps (per barrier)",
      "bar.sync (aligned) 1,64 two warps",
      "STS -> barrier.sync -> LDS handoff (per barrier)",
      "RED.ADD lane0 + barrier.sync (per iter)",
      "atom.acq_rel.cta with return + barrier.sync",
      "STG all lanes + barrier.sync",
      "LDG+STG RMW own element + barrier.sync",
      "LDG dependent chain, same address",
      "__syncwarp (per call)",
      "STG + fence.acq_rel.cta (per iter)",
      "ballot+popc dependent chain",
      "alternating 8 LDS per side, per iter/8 (2 bars)",
      "alternating 32 LDS per side, per iter/8 (2 bars)",
      "alternating no work, per iter/8 (2 bars)",
      "lane0 STS+syncwarp+bar+LDS+shfl (per iter)",
  };
  for (int t = 0; t < 19; ++t) {
    k_chain<<<1, 128>>>(out, g, t);
    k_chain<<<1, 128>>>(out, g, t);
    cudaDeviceSynchronize();
    long long h[2];
    cudaMemcpy(h, out + 2 * t, 16, cudaMemcpyDeviceToHost);
    printf("%-50s %8.1f cycles\n", names[t], double(h[0]) / N);
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
