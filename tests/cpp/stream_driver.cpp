// stream_driver.cpp -- C++ host code calling the B200 runtime through the C
// ABI only (no Python, no torch): config 4's target region on device
// buffers and through the host-buffer entry point, a team-range-sharded
// config-1 grid, and the args-list statistics; every result is checked on
// the host.  Built and run by tests/test_cpp_adapter.py:
//
//   g++ -std=c++20 -I include tests/cpp/stream_driver.cpp \
//       -L paper_1711_10413_b200/_build -lompds_b200 -lcudart ...
#include "ompds.h"

#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#define CHECK(c)                                                               \
  do {                                                                         \
    if (!(c)) {                                                                \
      std::fprintf(stderr, "FAILED %s:%d: %s (%s)\n", __FILE__, __LINE__, #c,  \
                   ompds_last_error());                                        \
      return 1;                                                                \
    }                                                                          \
  } while (0)

static ompds_launch launch_of(int32_t teams, int32_t workers) {
  ompds_launch l;
  std::memset(&l, 0, sizeof l);
  l.teams = teams;
  l.workers = workers;
  l.prealloc_entries = OMPDS_DEFAULT_PREALLOC_ENTRIES;
  l.depot_capacity = -1;
  return l;
}

int main() {
  if (ompds_device_count() < 1) {
    std::printf("no GPU\n");
    return 2;
  }
  // --- config 4 on device buffers: y = fma(c1, x, y) + (c2+...+c8) ---------
  const int64_t n = (int64_t(1) << 20) + 3;
  double *x = nullptr, *y = nullptr;
  CHECK(cudaMalloc(&x, n * 8) == cudaSuccess && cudaMalloc(&y, n * 8) == cudaSuccess);
  CHECK(ompds_fill_uniform(1, x, n, 0x5eed01ab, 0, nullptr) == OMPDS_OK);
  CHECK(ompds_fill_uniform(1, y, n, 0x5eed01ac, 0, nullptr) == OMPDS_OK);
  std::vector<double> hx(n), hy(n), want(n);
  CHECK(cudaMemcpy(hx.data(), x, n * 8, cudaMemcpyDeviceToHost) == cudaSuccess);
  CHECK(cudaMemcpy(hy.data(), y, n * 8, cudaMemcpyDeviceToHost) == cudaSuccess);
  double coef[8], s = 0;
  for (int k = 0; k < 8; ++k)
    coef[k] = (k + 1) / 8.0;
  for (int k = 1; k < 8; ++k)
    s += coef[k];
  for (int64_t i = 0; i < n; ++i)
    want[i] = std::fma(coef[0], hx[i], hy[i]) + s;
  const int32_t teams = 148 * 8;
  ompds_launch l = launch_of(teams, 96);
  std::vector<ompds_team_stats> st(teams);
  ompds_team_stats *dst = nullptr;
  CHECK(cudaMalloc(&dst, teams * sizeof(ompds_team_stats)) == cudaSuccess);
  CHECK(ompds_run_stream(&l, 1, n, x, y, coef, dst, nullptr) == OMPDS_OK);
  CHECK(cudaMemcpy(hy.data(), y, n * 8, cudaMemcpyDeviceToHost) == cudaSuccess);
  CHECK(cudaMemcpy(st.data(), dst, teams * sizeof(ompds_team_stats),
                   cudaMemcpyDeviceToHost) == cudaSuccess);
  for (int64_t i = 0; i < n; ++i)
    CHECK(std::memcmp(&hy[i], &want[i], 8) == 0);
  for (const ompds_team_stats &t : st)
    CHECK(t.trap == 0 && t.regions == 1 && t.master_barriers == 2 &&
          t.barrier_releases == 3 && t.smem_bytes == 289);

  // --- the same region from host buffers (H2D, region, D2H) -----------------
  std::vector<double> hx2(hx), hy2(n);
  CHECK(ompds_fill_uniform(1, y, n, 0x5eed01ac, 0, nullptr) == OMPDS_OK);
  CHECK(cudaMemcpy(hy2.data(), y, n * 8, cudaMemcpyDeviceToHost) == cudaSuccess);
  CHECK(ompds_run_stream_host(&l, 1, n, hx2.data(), hy2.data(), coef, x, y) == OMPDS_OK);
  for (int64_t i = 0; i < n; ++i)
    CHECK(std::memcmp(&hy2[i], &want[i], 8) == 0);

  // --- config 1, a 6-team grid in two team-range shards ---------------------
  const int32_t T = 6, W = 40, R = 3;
  int32_t *a = nullptr;
  CHECK(cudaMalloc(&a, T * W * 4) == cudaSuccess);
  CHECK(cudaMemset(a, 0, T * W * 4) == cudaSuccess);
  for (int32_t g = 0; g < 2; ++g) {
    ompds_launch lr = launch_of(T / 2, W);
    lr.first_team = g * (T / 2);
    lr.total_teams = T;
    CHECK(ompds_run_regions(&lr, 0, R, a, nullptr, nullptr) == OMPDS_OK);
  }
  std::vector<int32_t> ha(T * W);
  CHECK(cudaMemcpy(ha.data(), a, T * W * 4, cudaMemcpyDeviceToHost) == cudaSuccess);
  // a[t*W + w] after R regions of a += c1 + c2 + c3 + c4 with c4 += 1 in
  // between (c1..c4 = 1, 2, 3, 4): sum over r of (10 + r)
  for (int32_t i = 0; i < T * W; ++i)
    CHECK(ha[i] == 10 * R + R * (R - 1) / 2);

  // --- an args list past a 2-entry window, device malloc (paper scheme) -----
  ompds_launch lm = launch_of(2, 32);
  lm.prealloc_entries = 2;
  lm.list_allocator = OMPDS_LIST_MALLOC;
  std::vector<ompds_team_stats> st2(2);
  CHECK(ompds_run_regions(&lm, 0, R, a, dst, nullptr) == OMPDS_OK);
  CHECK(cudaMemcpy(st2.data(), dst, 2 * sizeof(ompds_team_stats),
                   cudaMemcpyDeviceToHost) == cudaSuccess);
  for (const ompds_team_stats &t : st2)
    CHECK(t.trap == 0 && t.dynamic_allocs == R && t.dynamic_frees == R &&
          t.dynamic_alloc_bytes == R * 4 * 8);
  std::printf("stream driver ok\n");
  return 0;
}
