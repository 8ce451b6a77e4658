// team_handle_cost.cu -- measurement tool (not product): the C-level cost of
// one reference-facing TeamRuntime operation through the team handle
// (ompds_team_*), beside the floor of one empty-kernel launch + stream
// synchronisation on the same stream kind.  The Python bench figure adds
// ctypes and the adapter's event bookkeeping on top.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I include tools/team_handle_cost.cu \
//        -L paper_1711_10413_b200/_build -lompds_b200 -Xlinker -rpath,$PWD/paper_1711_10413_b200/_build \
//        -o tools/team_handle_cost.bin
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>

#include "ompds.h"

__global__ void empty_kernel() {}
__global__ void flag_kernel(volatile unsigned *flag, unsigned v) {
  __threadfence_system();
  *flag = v;
}

int main() {
  cudaFree(nullptr);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  const int N = 3000;
  for (int w = 0; w < 100; ++w) {
    empty_kernel<<<1, 32, 0, s>>>();
    cudaStreamSynchronize(s);
  }
  auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < N; ++i) {
    empty_kernel<<<1, 32, 0, s>>>();
    cudaStreamSynchronize(s);
  }
  auto t1 = std::chrono::steady_clock::now();
  const double floor_us = std::chrono::duration<double, std::micro>(t1 - t0).count() / N;
  // the same launch, completion observed by spinning on a mapped host word
  unsigned *hflag = nullptr, *dflag = nullptr;
  cudaHostAlloc(reinterpret_cast<void **>(&hflag), 64, cudaHostAllocMapped);
  cudaHostGetDevicePointer(reinterpret_cast<void **>(&dflag), hflag, 0);
  *hflag = 0;
  t0 = std::chrono::steady_clock::now();
  for (int i = 1; i <= N; ++i) {
    flag_kernel<<<1, 1, 0, s>>>(dflag, unsigned(i));
    while (*reinterpret_cast<volatile unsigned *>(hflag) != unsigned(i)) {
    }
  }
  t1 = std::chrono::steady_clock::now();
  const double spin_us = std::chrono::duration<double, std::micro>(t1 - t0).count() / N;
  cudaStreamSynchronize(s);
  // launch cost alone (the host side of one launch, no wait)
  t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < N; ++i)
    empty_kernel<<<1, 32, 0, s>>>();
  t1 = std::chrono::steady_clock::now();
  const double launch_us = std::chrono::duration<double, std::micro>(t1 - t0).count() / N;
  cudaStreamSynchronize(s);

  ompds_runtime_config cfg{20, 0};
  ompds_team *h = nullptr;
  if (ompds_team_create(&cfg, 0x2000, nullptr, nullptr, nullptr, &h) != 0) {
    printf("create failed\n");
    return 1;
  }
  ompds_team_kernel_init(h, OMPDS_ROLE_MASTER, 1);
  uint64_t addr;
  int32_t fn, part;
  for (int i = 0; i < 100; ++i) {
    ompds_team_prepare_parallel(h, OMPDS_ROLE_MASTER, 0, 4, &addr);
    ompds_team_kernel_parallel(h, OMPDS_ROLE_WORKER, &fn, &addr, &part);
    ompds_team_end_parallel(h, OMPDS_ROLE_WORKER);
  }
  t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < N; ++i) {
    int32_t r = ompds_team_prepare_parallel(h, OMPDS_ROLE_MASTER, 0, 4, &addr);
    r |= ompds_team_kernel_parallel(h, OMPDS_ROLE_WORKER, &fn, &addr, &part);
    r |= ompds_team_end_parallel(h, OMPDS_ROLE_WORKER);
    if (r) {
      printf("call failed %d\n", r);
      return 1;
    }
  }
  t1 = std::chrono::steady_clock::now();
  const double call_us = std::chrono::duration<double, std::micro>(t1 - t0).count() / (3.0 * N);
  printf("{\"team_handle_us_per_call_c\": %.2f, \"empty_launch_sync_us\": %.2f, "
         "\"launch_spin_on_mapped_flag_us\": %.2f, \"launch_only_us\": %.2f, \"calls\": %d}\n",
         call_us, floor_us, spin_us, launch_us, 3 * N);
  ompds_team_destroy(h);
  return 0;
}
