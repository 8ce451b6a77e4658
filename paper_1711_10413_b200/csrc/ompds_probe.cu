// ompds_probe.cu -- ompds_probe_overheads: the cost of the runtime's building
// blocks on one SM, for BASELINE.json's "push/pop + handoff overhead in ns
// per parallel region".
//
// Data-sharing stack (DsStack, ompds_device.cuh; the reference's
// pushActivation / popActivation, proj/src/Simulator.cpp:439-479).  One warp
// runs `iterations` iterations; iteration i pushes d_i frames of
// `frame_bytes` x `lanes` bytes, where d_i in [1, max_depth] comes from a
// hash of (i, seed), touches one 4-byte word per lane in every frame (a weak
// store then a load, the value folded into a running sum) and pops them in
// LIFO order.  Frame size, lane count, slot capacity, depth pattern and seed
// are kernel arguments, so the stack's `top` and the frame addresses are
// run-time values: the bookkeeping cannot be folded away (the SASS excerpt
// in profiles/ shows it inside the loop).  Each stack mode has a baseline
// that makes the same accesses at the same addresses computed without the
// stack:
//
//   mode 0  smem baseline   frame k at slot + k*stride, LDS/STS
//   mode 1  slot            push/pop, frames in the warp's smem slot, LDS/STS
//   mode 2  global baseline frame k at chain + k*stride, weak LDG/STG
//   mode 3  chain           push/pop with a 0-byte slot: every frame on the
//                           global overflow chain, weak LDG/STG
//   mode 4  bookkeeping     push/pop with no frame access, each frame's
//                           offset folded into the sum (the dependent chain of
//                           the bookkeeping instructions alone)
//   mode 5  its baseline    the same loop with k*stride instead of the stack
//
// push+pop pair cost = (mode - baseline) / pairs executed.  A 2-warp kernel
// then times the bare region handoff (release + join on named barrier 1).
#include "ompds_generic.cuh"

namespace ompds {
namespace {

constexpr int kProbeMaxDepth = 4;   // frames per iteration at most
constexpr int kProbeSlot = 8192;    // static smem slot (bytes)

struct ProbeArgs {
  int32_t iters;
  int32_t frame_bytes; // per lane
  int32_t lanes;
  int32_t max_depth;
  uint32_t seed;
  uint32_t slot_cap;
  unsigned char *chain;
  int64_t chain_bytes;
  uint32_t zero; // always 0 (see touch_shared)
};

__device__ __forceinline__ int32_t probe_depth(uint32_t i, uint32_t seed, int32_t maxd) {
  uint32_t h = (i ^ seed) * 0x9E3779B1u;
  h ^= h >> 15;
  h *= 0x85EBCA6Bu;
  h ^= h >> 13;
  // multiply-shift range reduction to [0, maxd) (no integer division)
  return 1 + static_cast<int32_t>(((h >> 16) * static_cast<uint32_t>(maxd)) >> 16);
}

// Weak (non-volatile) accesses.  The load reads `p + zero`, where `zero` is
// a kernel argument that is always 0: ptxas cannot prove the two addresses
// equal, so it cannot forward the stored value to the load in registers (it
// does for a plain store/load pair at one address, even inside asm).
__device__ __forceinline__ int32_t touch_shared(unsigned char *p, uint32_t zero, int32_t v) {
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(p));
  int32_t r;
  asm volatile("st.shared.u32 [%1], %3;\n\tld.shared.u32 %0, [%2];"
               : "=r"(r) : "r"(a), "r"(a + zero), "r"(v) : "memory");
  return r;
}
__device__ __forceinline__ int32_t touch_global(unsigned char *p, uint32_t zero, int32_t v) {
  int32_t r;
  asm volatile("st.global.u32 [%1], %3;\n\tld.global.u32 %0, [%2];"
               : "=r"(r) : "l"(p), "l"(p + zero), "r"(v) : "memory");
  return r;
}

template <int kMode>
__device__ __forceinline__ int32_t probe_loop(const ProbeArgs a, unsigned char *slot,
                                              long long &cyc, long long &ns, long long &pairs) {
  const uint32_t lane = lane_id();
  const uint32_t fb = static_cast<uint32_t>(a.frame_bytes);
  const uint32_t stride = (fb * static_cast<uint32_t>(a.lanes) + 7u) & ~7u;
  DsStack ds;
  ds.init(slot, kMode == 3 ? 0 : a.slot_cap, a.chain, a.chain_bytes);
  unsigned char *fixed = kMode == 2 || kMode == 3 ? a.chain : slot;
  int32_t acc = 0;
  long long np = 0;
  __syncwarp();
  const long long t0 = clock64();
  const int64_t g0 = globaltimer_ns();
  for (int32_t i = 0; i < a.iters; ++i) {
    const int32_t d = probe_depth(static_cast<uint32_t>(i), a.seed, a.max_depth);
    Frame f[kProbeMaxDepth];
#pragma unroll
    for (int k = 0; k < kProbeMaxDepth; ++k) {
      if (k < d) {
        unsigned char *base;
        int32_t in_smem;
        if constexpr (kMode == 1 || kMode == 3 || kMode == 4) {
          f[k] = ds.push(fb, a.lanes);
          base = f[k].base;
          in_smem = f[k].in_smem;
        } else {
          base = fixed + k * stride;
          in_smem = kMode == 0 || kMode == 5;
        }
        if constexpr (kMode == 4)
          acc += f[k].offset ^ in_smem;
        else if constexpr (kMode == 5)
          acc += static_cast<int32_t>(k * stride) ^ in_smem;
        else if (lane < static_cast<uint32_t>(a.lanes)) // the frame's lanes only
          acc += in_smem ? touch_shared(base + lane * fb, a.zero, i + acc)
                         : touch_global(base + lane * fb, a.zero, i + acc);
      }
    }
#pragma unroll
    for (int k = kProbeMaxDepth - 1; k >= 0; --k)
      if (k < d) {
        if constexpr (kMode == 1 || kMode == 3 || kMode == 4)
          acc += ds.pop(f[k]);
      }
    np += d;
  }
  __syncwarp();
  cyc = clock64() - t0;
  ns = globaltimer_ns() - g0;
  pairs = np;
  return acc + ds.depth + static_cast<int32_t>(ds.high_water);
}

// One kernel per stack mode (a separate function each, so its loop is one
// contiguous block of SASS -- profiles/ holds the excerpt): one warp, the
// mode's loop, cycles / ns / pairs to out[3*mode ..].
template <int kMode>
__global__ void __launch_bounds__(32) probe_stack_kernel(ProbeArgs a, long long *out) {
  __shared__ __align__(16) unsigned char slot[kProbeSlot];
  long long c = 0, t = 0, p = 0;
  const int32_t acc = probe_loop<kMode>(a, slot, c, t, p);
  if (threadIdx.x == 0) {
    out[3 * kMode] = c;
    out[3 * kMode + 1] = t;
    out[3 * kMode + 2] = p;
    out[21 + kMode] = acc; // keeps the loop's result live
  }
}

// Region handoff without the runtime: warp 0 (worker) and warp 1 (master),
// release + join on named barrier 1 per iteration.  A few untimed handoffs
// first bring both warps into step; thread 0 reports.
__global__ void __launch_bounds__(64) probe_handoff_kernel(int32_t iters, long long *out) {
  for (int i = 0; i < 16; ++i) {
    bar_sync(kBarHandoff, 64);
    bar_sync(kBarHandoff, 64);
  }
  const long long h0 = clock64();
  const int64_t hg0 = globaltimer_ns();
  for (int32_t i = 0; i < iters; ++i) {
    bar_sync(kBarHandoff, 64);
    bar_sync(kBarHandoff, 64);
  }
  const long long hc = clock64() - h0;
  const int64_t ht = globaltimer_ns() - hg0;
  if (threadIdx.x == 0) {
    out[18] = hc;
    out[19] = ht;
  }
}

} // namespace
} // namespace ompds

using namespace ompds;

extern "C" int32_t ompds_probe_overheads(ompds_overhead_probe *io, void *stream) {
  if (!io)
    return OMPDS_ERR_INVALID;
  ompds_overhead_probe r = *io;
  if (r.frame_bytes == 0)
    r.frame_bytes = 40;
  if (r.max_depth == 0)
    r.max_depth = 2;
  if (r.lanes == 0)
    r.lanes = kWarp;
  if (r.iterations < 1 || r.iterations > (1 << 20) || r.frame_bytes < 4 || r.frame_bytes > 256 ||
      (r.frame_bytes & 3) || r.max_depth < 1 || r.max_depth > kProbeMaxDepth || r.lanes < 1 ||
      r.lanes > kWarp)
    return OMPDS_ERR_INVALID;
  const int64_t frame = round_up(int64_t(r.frame_bytes) * r.lanes, 8);
  if (frame * r.max_depth > kProbeSlot) // the deepest iteration fits the slot
    return OMPDS_ERR_INVALID;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t chain_bytes = frame * r.max_depth;
  unsigned char *chain = nullptr;
  long long h[27] = {};
  OMPDS_CUDA(cudaMalloc(&chain, round_up(chain_bytes, 256) + sizeof h));
  long long *dev = reinterpret_cast<long long *>(chain + round_up(chain_bytes, 256));
  ProbeArgs a{r.iterations, r.frame_bytes, r.lanes, r.max_depth, r.seed,
              static_cast<uint32_t>(kProbeSlot), chain, chain_bytes, 0u};
  cudaError_t z = cudaMemsetAsync(dev, 0, sizeof h, st); // every slot defined
  if (z != cudaSuccess) {
    cudaFree(chain);
    return cuda_fail(z, "ompds_probe_overheads");
  }
  ProbeArgs warm = a; // the chain's first touch (TLB, L2) is not a push/pop cost
  warm.iters = a.iters < 256 ? a.iters : 256;
  probe_stack_kernel<3><<<1, 32, 0, st>>>(warm, dev);
  probe_stack_kernel<0><<<1, 32, 0, st>>>(a, dev);
  probe_stack_kernel<1><<<1, 32, 0, st>>>(a, dev);
  probe_stack_kernel<2><<<1, 32, 0, st>>>(a, dev);
  probe_stack_kernel<3><<<1, 32, 0, st>>>(a, dev);
  probe_stack_kernel<4><<<1, 32, 0, st>>>(a, dev);
  probe_stack_kernel<5><<<1, 32, 0, st>>>(a, dev);
  probe_handoff_kernel<<<1, 64, 0, st>>>(a.iters, dev);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(h, dev, sizeof h, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess)
    e = cudaStreamSynchronize(st);
  cudaFree(chain);
  OMPDS_CUDA(e);
  long long cyc = 0, ns = 0;
  for (int k = 0; k < 6; ++k) {
    cyc += h[3 * k];
    ns += h[3 * k + 1];
  }
  r.sm_clock_mhz = ns > 0 ? 1e3 * double(cyc) / double(ns) : 0.0;
  r.pairs = double(h[3 * 1 + 2]);
  const double it = r.iterations;
  r.smem_baseline_cycles = double(h[0]) / it;
  r.slot_cycles = double(h[3]) / it;
  r.global_baseline_cycles = double(h[6]) / it;
  r.chain_cycles = double(h[9]) / it;
  r.bookkeeping_cycles = double(h[12]) / it;
  r.bookkeeping_baseline_cycles = double(h[15]) / it;
  r.handoff_cycles = double(h[18]) / it;
  *io = r;
  return OMPDS_OK;
}
