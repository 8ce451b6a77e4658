// nested_region.cu -- nested parallel regions written against the device
// API (Worker::push_frame / pop_frame / parallel_serialized): what a
// compiler targeting this runtime would emit for the config-3 program of
// DESIGN.md §7,
//
//   int c = 1; double s[8] = {1..8};               // kernel locals, shared
//   for (r = 0; r < R; ++r) {
//     #pragma omp parallel                          // L1 shares {c, s}
//     { int me = omp_get_thread_num(), e = me + c; double v[4] = s[me%8]*(j+1);
//       #pragma omp parallel                        // L2 (nested) shares {e, v, c, me}
//       { double f = e + v[3];
//         #pragma omp parallel                      // L3 (nested) shares {f, c, me}
//         { a[team*W + me] += f + c; f = f * 2; }
//         v[0] = f; e += 1; }
//       a[team*W + me] += v[0] + e; }
//     c += 1;
//   }
//
// L1's locals that L2 and L3 capture are globalized onto the warp's
// data-sharing stack (push_frame, one lane-strided frame per warp); each
// nested region is serialized on its lane and receives its captures through a
// list frame on the same stack (parallel_serialized).  The result equals the
// hand-fused NestedProg kernel's and the C oracle's orc_nested
// (tests/test_example_region.py).
#include "ompds_generic.cuh"

namespace {

using namespace ompds;

struct NestedApiProg {
  struct Args {
    double *a;
    int32_t regions;
  };
  __device__ static void master(Master &m, const Args &a) {
    if (m.leader) {
      *reinterpret_cast<int32_t *>(m.cap(0)) = 1;
      double *s = reinterpret_cast<double *>(m.cap(1));
      for (int k = 0; k < 8; ++k)
        s[k] = double(k + 1);
    }
    __syncwarp();
    for (int32_t r = 0; r < a.regions; ++r) {
      if (m.parallel(0, 2) != OMPDS_OK) // L1 shares {c, s}
        return;
      if (m.leader)
        *reinterpret_cast<int32_t *>(m.cap(0)) += 1;
      __syncwarp();
    }
  }
  __device__ static void region(int32_t, const SharedVars &sv, Worker &w, const Args &a) {
    int32_t *c = static_cast<int32_t *>(sv.get(0));
    const double *s = static_cast<const double *>(sv.get(1));
    const uint32_t lane = lane_id();
    // L1's frame: me, e (int) and v[4] (double), globalized: L2/L3 capture them
    struct L1 {
      double v[4];
      int32_t me, e;
    };
    const Frame f1 = w.push_frame(sizeof(L1));
    if (f1.status != OMPDS_OK) {
      w.t->trap(f1.status);
      return;
    }
    L1 *l1 = reinterpret_cast<L1 *>(f1.base) + lane;
    l1->me = w.wid;
    l1->e = w.wid + *c;
    for (int j = 0; j < 4; ++j)
      l1->v[j] = s[w.wid % 8] * double(j + 1);
    double *dst = a.a + size_t(w.team) * w.workers + (w.mine ? w.wid : 0);
    void *l2caps[4] = {&l1->e, l1->v, c, &l1->me};
    int32_t st = w.parallel_serialized(4, [&](int j) { return l2caps[j]; },
                                       [&](const Worker::NestedVars &v2) {
      int32_t *e = static_cast<int32_t *>(v2.get(0));
      double *v = static_cast<double *>(v2.get(1));
      const int32_t *c2 = static_cast<const int32_t *>(v2.get(2));
      // L2's frame: f, globalized (L3 captures it)
      const Frame f2 = w.push_frame(sizeof(double));
      if (f2.status != OMPDS_OK)
        return;
      double *f = reinterpret_cast<double *>(f2.base) + lane;
      *f = double(*e) + v[3];
      void *l3caps[3] = {f, const_cast<int32_t *>(c2), v2.get(3)};
      w.parallel_serialized(3, [&](int j) { return l3caps[j]; },
                            [&](const Worker::NestedVars &v3) {
        double *f3 = static_cast<double *>(v3.get(0));
        const int32_t c3 = *static_cast<const int32_t *>(v3.get(1));
        const int32_t me = *static_cast<const int32_t *>(v3.get(2));
        if (w.mine)
          a.a[size_t(w.team) * w.workers + me] += *f3 + double(c3);
        *f3 = *f3 * 2.0;
      });
      v[0] = *f;
      *e = *e + 1;
      w.pop_frame(f2);
    });
    if (st != OMPDS_OK)
      w.t->trap(st);
    if (w.mine)
      *dst = *dst + (l1->v[0] + double(l1->e));
    w.pop_frame(f1);
  }
};

} // namespace

extern "C" int32_t example_nested(const ompds_launch *launch, double *a, int32_t regions,
                                  int64_t warp_slot_bytes, int64_t warp_overflow_bytes,
                                  ompds_team_stats *stats) {
  if (!a || regions < 0 || warp_slot_bytes < 0 || warp_overflow_bytes < 0)
    return OMPDS_ERR_INVALID;
  FixedLayout lay;
  // kernel frame group: c (int, captured), s[8] (double, captured)
  const int32_t s = build_fixed_layout({4, 64}, 0, &lay);
  if (s)
    return s;
  return launch_generic<NestedApiProg>(launch, lay, 2, {a, regions}, stats, nullptr,
                                       warp_slot_bytes, warp_overflow_bytes);
}
