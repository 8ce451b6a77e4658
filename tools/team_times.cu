// team_times.cu -- measurement tool (not product): per-team %globaltimer
// stamps of the config-2 launch (296 teams x 480 workers, 2^24 fp64, d[]
// staged by TMA) inside the PRODUCT kernel built with -DOMPDS_TEAM_TIMES:
// when teams start, release their region, pass the join and finish,
// relative to the first team's start.  L2 is evicted before the launch.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DOMPDS_TEAM_TIMES=4096 \
//        -I paper_1711_10413_b200/csrc -I include tools/team_times.cu \
//        paper_1711_10413_b200/csrc/ompds_host.cpp -o paper_1711_10413_b200/_build/team_times.bin
#include "ompds_kernels.cu"

#include <algorithm>
#include <string>
#include <vector>

static void pct(const char *name, std::vector<long long> v) {
  std::sort(v.begin(), v.end());
  auto q = [&](double f) { return v[size_t(f * (v.size() - 1))]; };
  printf("  %-26s min %7lld  p10 %7lld  p50 %7lld  p90 %7lld  max %7lld ns\n", name, v.front(),
         q(0.1), q(0.5), q(0.9), v.back());
}

int main(int argc, char **argv) {
  const int teams = argc > 1 ? atoi(argv[1]) : 296, W = argc > 2 ? atoi(argv[2]) : 480;
  const int64_t n = int64_t(1) << 24;
  double *a, *d;
  int *flush;
  cudaMalloc(&a, n * 8);
  cudaMalloc(&d, 256 * 8);
  cudaMalloc(&flush, size_t(256) << 20);
  cudaMemset(a, 0, n * 8);
  std::vector<double> hd(256);
  for (int k = 0; k < 256; ++k)
    hd[k] = 3 * k + 1;
  cudaMemcpy(d, hd.data(), 256 * 8, cudaMemcpyHostToDevice);
  // "stream": config 4 (2^28 fp64 x, y) instead of config 2
  const bool stream = argc > 3 && std::string(argv[3]) == "stream";
  // "noflush": no L2 eviction between launches (the kernel's code stays in L2)
  const bool noflush = argc > 4 && std::string(argv[4]) == "noflush";
  const int64_t n4 = int64_t(1) << 28;
  double *x4 = nullptr, *y4 = nullptr;
  const double coef[8] = {1, 1, 1, 1, 1, 1, 1, 1};
  if (stream) {
    cudaMalloc(&x4, n4 * 8);
    cudaMalloc(&y4, n4 * 8);
    cudaMemset(x4, 0, n4 * 8);
    cudaMemset(y4, 0, n4 * 8);
  }
  ompds_launch l{};
  l.teams = teams;
  l.workers = W;
  l.prealloc_entries = 20;
  l.depot_capacity = -1;
  std::vector<long long> h(size_t(OMPDS_TEAM_TIMES) * 8);
  for (int rep = 0; rep < 4; ++rep) {
    if (!noflush)
      cudaMemset(flush, rep, size_t(256) << 20); // evict a[] from L2 (writes, then drained)
    cudaDeviceSynchronize();
    std::fill(h.begin(), h.end(), 0);
    cudaMemcpyToSymbol(g_team_times, h.data(), h.size() * 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    int32_t s = stream ? ompds_run_stream(&l, 1, n4, x4, y4, coef, nullptr, nullptr)
                       : ompds_run_shared_array(&l, 1, n, a, d, nullptr, nullptr);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (s) {
      printf("status %d: %s\n", s, ompds_last_error());
      return 1;
    }
    cudaMemcpyFromSymbol(h.data(), g_team_times, h.size() * 8);
    long long t0 = h[0];
    for (int t = 0; t < teams; ++t)
      t0 = std::min(t0, h[t * 8]);
    std::vector<long long> c[8];
    for (int t = 0; t < teams; ++t)
      for (int k = 0; k < 8; ++k)
        c[k].push_back(h[t * 8 + k] - t0);
    std::vector<long long> body;
    for (int t = 0; t < teams; ++t)
      body.push_back(h[t * 8 + 3] - h[t * 8 + 2]);
    printf("rep %d: %s, %d teams x %d, event-bracketed %.1f us\n", rep, stream ? "config 4" : "config 2", teams, W, ms * 1e3);
    pct("kernel entry", c[0]);
    pct("prologue (zeroing) done", c[5]);
    pct("kernel_init done", c[6]);
    pct("master ready (init+depot)", c[1]);
    pct("release (before barrier)", c[2]);
    pct("join passed", c[3]);
    pct("master done", c[4]);
    pct("release -> join (region)", body);
  }
  return 0;
}
