// reduction_region.cu -- a user-defined region program on the B200 runtime.
//
// What a compiler targeting this runtime would emit for
//
//   #pragma omp target teams map(to: x[0:n]) map(from: out[0:2*teams])
//   {
//     long sum = 0, thr, cnt = 0;              // kernel locals, captured below
//     #pragma omp parallel                     // region 0 shares {sum}
//     { long s = 0; for (i = mine) s += x[i];  #pragma omp atomic  sum += s; }
//     thr = sum / n_team;                       // sequential code reads sum
//     #pragma omp parallel                     // region 1 shares {thr, cnt}
//     { long c = 0; for (i = mine) c += x[i] > thr;  #pragma omp atomic  cnt += c; }
//     long wsum[32], tot;                        // captured array + scalar
//     #pragma omp parallel                     // region 2 shares {wsum, tot}
//     { warp partial of x -> wsum[warp];  #pragma omp barrier
//       if (omp_get_thread_num() == 0) tot = sum over wsum; }
//     out[3*team] = sum; out[3*team+1] = cnt; out[3*team+2] = tot;
//   }
//
// The locals are implicitly shared: they live in the team's depot in
// shared memory, the workers reach them through get-shared-variables, and
// their writes (the atomics) are what the master reads after each join --
// the data-sharing semantics of arXiv 1711.10413 end to end.  Each team
// reduces its own contiguous slice of x; the host checks every team's sum
// and count against numpy, and the barrier region's total against the first
// region's sum (tests/test_example_region.py).
//
// Built by paper_1711_10413_b200/build.py into _build/libompds_example.so
// against the runtime headers and libompds_b200.so.
#include "ompds_generic.cuh"

namespace {

using namespace ompds;

struct ReductionProg {
  struct Args {
    const int32_t *x;
    int64_t n;
    long long *out; // 3 per team: sum, count above the team's mean, total
  };
  __device__ static void team_range(const Args &a, int64_t *lo, int64_t *hi) {
    *lo = a.n * blockIdx.x / gridDim.x;
    *hi = a.n * (blockIdx.x + 1) / gridDim.x;
  }
  __device__ static void master(Master &m, const Args &a) {
    long long *sum = reinterpret_cast<long long *>(m.cap(0));
    long long *thr = reinterpret_cast<long long *>(m.cap(1));
    long long *cnt = reinterpret_cast<long long *>(m.cap(2));
    if (m.leader) {
      *sum = 0;
      *cnt = 0;
    }
    __syncwarp();
    if (m.parallel(0, 1) != OMPDS_OK) // shares {sum}
      return;
    int64_t lo, hi;
    team_range(a, &lo, &hi);
    if (m.leader) // sequential code between the regions reads the shared sum
      *thr = hi > lo ? *sum / (hi - lo) : 0;
    __syncwarp();
    if (m.parallel_with(1, 2, [&](int j) -> void * { return m.cap(1 + j); }) !=
        OMPDS_OK) // shares {thr, cnt}
      return;
    long long *wsum = reinterpret_cast<long long *>(m.cap(3));
    if (m.parallel_with(2, 2, [&](int j) -> void * { return m.cap(3 + j); }) !=
        OMPDS_OK) // shares {wsum, tot}
      return;
    if (m.leader) {
      a.out[3 * blockIdx.x] = *sum;
      a.out[3 * blockIdx.x + 1] = *cnt;
      a.out[3 * blockIdx.x + 2] = *reinterpret_cast<long long *>(m.cap(4));
    }
    (void)wsum;
  }
  __device__ static void region(int32_t fn, const SharedVars &sv, Worker &w,
                                const Args &a) {
    int64_t lo, hi;
    team_range(a, &lo, &hi);
    long long *s0 = static_cast<long long *>(sv.get(0));
    long long *s1 = static_cast<long long *>(sv.get(1));
    long long part = 0;
    if (fn == 2) { // per-warp partials, an omp barrier, one worker totals them
      for (int64_t i = lo + w.wid; w.mine && i < hi; i += w.workers)
        part += a.x[i];
      for (int o = 16; o > 0; o >>= 1)
        part += __shfl_xor_sync(0xffffffffu, part, o);
      if ((threadIdx.x & 31) == 0)
        s0[w.warp] = part;
      w.barrier();
      if (w.wid == 0) {
        long long tot = 0;
        for (uint32_t k = 0; k < w.worker_threads / 32; ++k)
          tot += s0[k];
        *s1 = tot;
      }
      return;
    }
    if (fn == 0) {
      for (int64_t i = lo + w.wid; w.mine && i < hi; i += w.workers)
        part += a.x[i];
    } else {
      const long long thr = *s0;
      for (int64_t i = lo + w.wid; w.mine && i < hi; i += w.workers)
        part += a.x[i] > thr ? 1 : 0;
    }
    for (int o = 16; o > 0; o >>= 1)
      part += __shfl_xor_sync(0xffffffffu, part, o);
    if ((threadIdx.x & 31) == 0) // one atomic per warp on the shared variable
      atomicAdd(reinterpret_cast<unsigned long long *>(fn == 0 ? s0 : s1),
                static_cast<unsigned long long>(part));
  }
};

// A program that stages more captures than its launch declared (n_caps):
// region 0 shares one variable, region 1 asks for `nargs2` entries.  With
// n_caps within the window the launcher picks the lean instantiation, whose
// prepare refuses a list past the window (it has no list allocator): the
// team traps, the workers
// see no staged region and do not run region 0's body again
// (tests/test_example_region.py: the lean instantiation's refused prepare).
struct MisdeclaredProg {
  struct Args {
    unsigned long long *runs; // per team: region-0 bodies run (one per worker)
    int32_t nargs2;
  };
  __device__ static void master(Master &m, const Args &a) {
    if (m.parallel(0, 1) != OMPDS_OK)
      return;
    m.parallel(0, a.nargs2); // refused when it does not fit what the launch declared
  }
  __device__ static void region(int32_t, const SharedVars &, Worker &w, const Args &a) {
    if (w.mine)
      atomicAdd(a.runs + blockIdx.x, 1ull);
  }
};

} // namespace

extern "C" int32_t example_misdeclared(const ompds_launch *launch, int32_t nargs2,
                                       unsigned long long *runs, ompds_team_stats *stats) {
  if (!runs)
    return OMPDS_ERR_INVALID;
  FixedLayout lay;
  const int32_t s = build_fixed_layout({8, 8}, 0, &lay);
  if (s)
    return s;
  // declares one capture: the lean instantiation when it fits the window
  return launch_generic<MisdeclaredProg>(launch, lay, 1, {runs, nargs2}, stats, nullptr);
}

extern "C" int32_t example_reduction(const ompds_launch *launch, const int32_t *x,
                                     int64_t n, long long *out,
                                     ompds_team_stats *stats) {
  if (!x || !out || n < 0)
    return OMPDS_ERR_INVALID;
  FixedLayout lay;
  // kernel frame group: sum, thr, cnt (captured, 8 B each), wsum[32]
  // (256 B), tot (8 B), then __omp_worker's wf.addr / args.addr -- 304 B,
  // team footprint 513 B
  const int32_t s = build_fixed_layout({8, 8, 8, 256, 8}, 0, &lay);
  if (s)
    return s;
  return launch_generic<ReductionProg>(launch, lay, 5, {x, n, out}, stats, nullptr);
}
