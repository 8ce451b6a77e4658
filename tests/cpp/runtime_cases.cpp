// The reference's TeamRuntime unit cases (proj/tests/RuntimeTests.cpp),
// written against the C++ adapter include/ompds.hpp -- i.e. as a reference
// user would after switching to the B200 runtime.  Exit code 0 = all passed.
#include "ompds.hpp"

#include <cstdio>
#include <random>

using namespace ompds_cpp;

static int Failures = 0;
#define CHECK(c)                                                               \
  do {                                                                         \
    if (!(c)) {                                                                \
      std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c);                  \
      ++Failures;                                                              \
    }                                                                          \
  } while (0)

static constexpr uint64_t PreallocBase = 0x2000;

static TeamRuntime makeLive(int Workers = 8, RuntimeConfig Cfg = {}) {
  TeamRuntime Rt(Cfg, PreallocBase);
  CHECK(Rt.kernelInit(RtRole::Master, Workers).Ok);
  return Rt;
}

static void drain(TeamRuntime &Rt) {
  std::string Wf;
  uint64_t Args = 0;
  bool P = false;
  CHECK(Rt.kernelParallel(RtRole::Worker, Wf, Args, P).Ok);
  CHECK(P);
  CHECK(Rt.endParallel(RtRole::Worker).Ok);
}

int main() {
  { // init accepts one master call and nothing else
    TeamRuntime Rt({}, PreallocBase);
    CHECK(!Rt.kernelInit(RtRole::Worker, 8).Ok);
    CHECK(!Rt.kernelInit(RtRole::Master, 0).Ok);
    CHECK(Rt.kernelInit(RtRole::Master, 8).Ok);
    CHECK(!Rt.kernelInit(RtRole::Master, 8).Ok);
    CHECK(Rt.workerCount() == 8);
  }
  { // small capture lists use the preallocated window
    TeamRuntime Rt = makeLive();
    for (int64_t N : {0, 1, 19, 20}) {
      uint64_t Addr = 0;
      CHECK(Rt.prepareParallel(RtRole::Master, "wf", N, Addr).Ok);
      CHECK(Addr == PreallocBase);
      drain(Rt);
    }
    CHECK(Rt.dynamicAllocs() == 0);
  }
  { // oversized lists fall back to global memory, freed on last retire
    TeamRuntime Rt = makeLive();
    for (auto [N, Bytes] : {std::pair<int64_t, int64_t>{21, 168}, {32, 256}, {64, 512}, {128, 1024}}) {
      uint64_t Addr = 0;
      CHECK(Rt.prepareParallel(RtRole::Master, "wf", N, Addr).Ok);
      CHECK(Addr != PreallocBase);
      CHECK(Rt.events().back().K == RuntimeEvent::PrepareDynamic && Rt.events().back().Bytes == Bytes);
      drain(Rt);
      CHECK(Rt.events().back().K == RuntimeEvent::DynamicFree && Rt.events().back().Bytes == Bytes);
    }
    CHECK(Rt.dynamicAllocs() == 4 && Rt.dynamicFrees() == 4 && Rt.leakedBlocks() == 0);
  }
  { // failing allocation is a trap
    RuntimeConfig Cfg;
    Cfg.FailDynamicAlloc = true;
    TeamRuntime Rt = makeLive(8, Cfg);
    uint64_t Addr = 0;
    RtResult R = Rt.prepareParallel(RtRole::Master, "wf", 21, Addr);
    CHECK(!R.Ok && R.TrapReason == "shared-args-alloc-failed");
  }
  { // protocol violations with exact reasons
    uint64_t Addr = 0;
    TeamRuntime A({}, PreallocBase);
    CHECK(A.prepareParallel(RtRole::Master, "wf", 1, Addr).TrapReason ==
          "protocol error: prepare_parallel before init");
    TeamRuntime B = makeLive();
    CHECK(B.prepareParallel(RtRole::Master, "wf", 1, Addr).Ok);
    CHECK(B.prepareParallel(RtRole::Master, "wf", 1, Addr).TrapReason ==
          "protocol error: prepare_parallel while a region is in flight");
    TeamRuntime C = makeLive();
    std::string Wf;
    bool P = false;
    CHECK(C.kernelParallel(RtRole::Worker, Wf, Addr, P).TrapReason ==
          "protocol error: kernel_parallel with no staged region");
    CHECK(C.endParallel(RtRole::Worker).TrapReason ==
          "protocol error: end_parallel with no active region");
    CHECK(C.kernelDeinit(RtRole::Master).Ok);
    CHECK(!C.kernelDeinit(RtRole::Master).Ok);
  }
  { // termination sentinel + event order
    TeamRuntime Rt = makeLive();
    uint64_t Addr = 0;
    CHECK(Rt.prepareParallel(RtRole::Master, "region0", 21, Addr).Ok);
    std::string Wf;
    bool P = false;
    CHECK(Rt.kernelParallel(RtRole::Worker, Wf, Addr, P).Ok && Wf == "region0");
    CHECK(Rt.endParallel(RtRole::Worker).Ok);
    CHECK(Rt.kernelDeinit(RtRole::Master).Ok);
    Wf = "stale";
    Addr = 99;
    P = true;
    CHECK(Rt.kernelParallel(RtRole::Worker, Wf, Addr, P).Ok);
    CHECK(Wf.empty() && Addr == 0 && !P && Rt.terminated());
    std::vector<RuntimeEvent::Kind> K;
    for (auto &E : Rt.events())
      K.push_back(E.K);
    CHECK((K == std::vector<RuntimeEvent::Kind>{RuntimeEvent::Init, RuntimeEvent::PrepareDynamic,
                                                RuntimeEvent::Fetch, RuntimeEvent::Retire,
                                                RuntimeEvent::DynamicFree, RuntimeEvent::Deinit}));
  }
  { // byte law (mt19937(1234), N in [0,128])
    std::mt19937 Rng(1234);
    std::uniform_int_distribution<int64_t> Dist(0, 128);
    for (int Round = 0; Round < 60; ++Round) {
      int64_t N = Dist(Rng);
      TeamRuntime Rt = makeLive();
      uint64_t Addr = 0;
      CHECK(Rt.prepareParallel(RtRole::Master, "wf", N, Addr).Ok);
      CHECK(Rt.events().back().Bytes == dynamicArgsBytes(static_cast<int>(N)));
      CHECK((Addr == PreallocBase) == (N <= DefaultPreallocEntries));
    }
  }
  std::printf("%s (%d failures)\n", Failures ? "FAILED" : "ok", Failures);
  return Failures ? 1 : 0;
}
