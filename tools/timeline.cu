// timeline.cu -- measurement tool (not product): per-step timeline of the
// config-1 parallel region inside the PRODUCT kernel
// (generic_mode_kernel<RegionsProg<int>>, built with -DOMPDS_TIMELINE=256 so
// the OMPDS_TL stamps in csrc/ompds_kernels.cu record clock64 for the master
// lane and worker warp 0 of team 0).  Stamps mark instruction issue, not the
// completion of loads still in flight.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DOMPDS_TIMELINE=256 \
//        -I paper_1711_10413_b200/csrc -I include tools/timeline.cu \
//        paper_1711_10413_b200/csrc/ompds_host.cpp -o paper_1711_10413_b200/_build/timeline.bin
//   timeline.bin [W] [int|f64]
#include "ompds_kernels.cu"

#include <algorithm>
#include <string>
#include <vector>

int main(int argc, char **argv) {
  const int W = argc > 1 ? atoi(argv[1]) : 32;
  const int R = 300;
  int32_t *a;
  cudaMalloc(&a, 4096 * 8);
  cudaMemset(a, 0, 4096 * 8);
  ompds_launch l{1, W, 20, 0, -1, 0, 0, nullptr};
  FixedLayout lay;
  build_fixed_layout({4, 4, 4, 4}, 4, &lay);
  const bool f64 = argc > 2 && std::string(argv[2]) == "f64";
  for (int rep = 0; rep < 2; ++rep) {
    int32_t s = f64 ? launch_generic<RegionsProg<double>>(
                          &l, lay, 4, RegionsProg<double>::Args{reinterpret_cast<double *>(a), R},
                          nullptr, nullptr)
                    : launch_generic<RegionsProg<int32_t>>(
                          &l, lay, 4, RegionsProg<int32_t>::Args{a, R}, nullptr, nullptr);
    cudaError_t e = cudaDeviceSynchronize();
    if (s || e) {
      printf("launch status %d %s\n", s, cudaGetErrorString(e));
      return 1;
    }
  }
  const int T = OMPDS_TIMELINE;
  std::vector<long long> h(T * 16);
  cudaMemcpyFromSymbol(h.data(), g_timeline, T * 16 * 8);
  const char *names[16] = {"M parallel_with entry", "M prepare checks done", "M before release bar",
                           "M release bar passed", "M join bar passed", "W release bar passed",
                           "W fetch done", "W get-shared-variables", "W region body done",
                           "W end_parallel done", "W join bar passed"};
  // order of events within region r, relative to the master's entry stamp
  const int order[] = {0, 1, 2, 5, 3, 6, 7, 8, 9, 10, 4};
  double mean[16] = {};
  int cnt = 0;
  for (int r = 32; r < T - 1; ++r) {
    for (int k = 0; k < 11; ++k)
      mean[k] += double(h[r * 16 + k] - h[r * 16 + 0]);
    ++cnt;
  }
  double per = 0;
  for (int r = 32; r < T - 1; ++r)
    per += double(h[(r + 1) * 16] - h[r * 16]);
  printf("W=%d %s: %.1f cycles per region (master entry to next entry)\n", W, f64 ? "f64" : "int", per / cnt);
  for (int k : order)
    printf("  %-28s %8.1f\n", names[k], mean[k] / cnt);
  // raw: every stamp of regions 100..102 in time order, relative to the
  // master's entry into region 100
  if (argc > 3) {
    std::vector<std::pair<long long, std::string>> ev;
    for (int r = 100; r < 103; ++r)
      for (int k = 0; k < 11; ++k)
        ev.push_back({h[r * 16 + k] - h[100 * 16], std::string(names[k]) + " #" + std::to_string(r)});
    std::sort(ev.begin(), ev.end());
    for (auto &e : ev)
      printf("    %6lld  %s\n", e.first, e.second.c_str());
  }
  return 0;
}
