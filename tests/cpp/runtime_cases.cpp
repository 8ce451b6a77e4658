// The reference's TeamRuntime unit cases (proj/tests/RuntimeTests.cpp:19-252),
// written against the C++ adapter include/ompds.hpp exactly as a reference
// user would after switching includes: `omplab::TeamRuntime(Config,
// PreallocBase, Heap)` with a RecordingHeap allocator that checks every
// allocate / release address.  Each runtime is one GPU-resident team handle.
// Exit code 0 = all passed.
#include "ompds.hpp"

#include <cstdio>
#include <map>
#include <random>

using namespace omplab;

static int Failures = 0;
#define CHECK(c)                                                               \
  do {                                                                         \
    if (!(c)) {                                                                \
      std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c);                  \
      ++Failures;                                                              \
    }                                                                          \
  } while (0)

namespace {

/// Heap double that hands out distinct addresses and records traffic
/// (RuntimeTests.cpp:19-42).
class RecordingHeap : public SharedArgsAllocator {
public:
  uint64_t allocate(int64_t Bytes) override {
    if (FailAll)
      return 0;
    uint64_t Addr = Next;
    Next += static_cast<uint64_t>(Bytes) + 64;
    LiveBytes[Addr] = Bytes;
    ++Allocs;
    return Addr;
  }
  void release(uint64_t Addr) override {
    CHECK(LiveBytes.count(Addr) == 1);
    LiveBytes.erase(Addr);
    ++Frees;
  }
  bool FailAll = false;
  uint64_t Next = 0x1000;
  std::map<uint64_t, int64_t> LiveBytes;
  int Allocs = 0;
  int Frees = 0;
};

constexpr uint64_t PreallocBase = 0x2000;

TeamRuntime makeLive(RecordingHeap &Heap, int Workers = 8, RuntimeConfig Cfg = {}) {
  TeamRuntime Rt(Cfg, PreallocBase, Heap);
  CHECK(Rt.kernelInit(RtRole::Master, Workers).Ok);
  return Rt;
}

/// One worker fetches and retires the staged region.
void drainRegion(TeamRuntime &Rt) {
  std::string Wf;
  uint64_t Args = 0;
  bool Participate = false;
  CHECK(Rt.kernelParallel(RtRole::Worker, Wf, Args, Participate).Ok);
  CHECK(Participate);
  CHECK(Rt.endParallel(RtRole::Worker).Ok);
}

} // namespace

int main() {
  { // init accepts one master call and nothing else
    RecordingHeap Heap;
    TeamRuntime Rt({}, PreallocBase, Heap);
    CHECK(!Rt.kernelInit(RtRole::Worker, 8).Ok);
    CHECK(!Rt.kernelInit(RtRole::Master, 0).Ok);
    CHECK(Rt.kernelInit(RtRole::Master, 8).Ok);
    CHECK(!Rt.kernelInit(RtRole::Master, 8).Ok);
    CHECK(Rt.workerCount() == 8);
  }
  { // small capture lists use the preallocated window
    RecordingHeap Heap;
    TeamRuntime Rt = makeLive(Heap);
    for (int64_t N : {0, 1, 19, 20}) {
      uint64_t Addr = 0;
      CHECK(Rt.prepareParallel(RtRole::Master, "wf", N, Addr).Ok);
      CHECK(Addr == PreallocBase);
      CHECK(Heap.Allocs == 0);
      drainRegion(Rt);
    }
    CHECK(Rt.dynamicAllocs() == 0);
  }
  { // oversized capture lists fall back to the device heap
    RecordingHeap Heap;
    TeamRuntime Rt = makeLive(Heap);
    for (auto [N, Bytes] : {std::pair<int64_t, int64_t>{21, 168}, {32, 256}, {64, 512}, {128, 1024}}) {
      uint64_t Addr = 0;
      CHECK(Rt.prepareParallel(RtRole::Master, "wf", N, Addr).Ok);
      CHECK(Addr != PreallocBase);
      CHECK(Heap.LiveBytes.size() == 1);
      CHECK(Heap.LiveBytes.begin()->first == Addr); // the allocator's own block
      CHECK(Heap.LiveBytes.begin()->second == Bytes);
      drainRegion(Rt);
      // the block is freed when the last worker retires the region
      CHECK(Heap.LiveBytes.empty());
    }
    CHECK(Rt.dynamicAllocs() == 4);
    CHECK(Rt.dynamicFrees() == 4);
    CHECK(Rt.leakedBlocks() == 0);
    CHECK(Heap.Allocs == 4 && Heap.Frees == 4);
  }
  { // the window boundary is exactly the entry count
    RecordingHeap Heap;
    RuntimeConfig Cfg;
    Cfg.PreallocEntries = 4;
    TeamRuntime Rt = makeLive(Heap, 8, Cfg);
    uint64_t Addr = 0;
    CHECK(Rt.prepareParallel(RtRole::Master, "wf", 4, Addr).Ok);
    CHECK(Addr == PreallocBase);
    drainRegion(Rt);
    CHECK(Rt.prepareParallel(RtRole::Master, "wf", 5, Addr).Ok);
    CHECK(Addr != PreallocBase);
    CHECK(Heap.LiveBytes.begin()->second == 40);
  }
  { // a failing device heap is a trap, not a silent corruption
    RecordingHeap Heap;
    RuntimeConfig Cfg;
    Cfg.FailDynamicAlloc = true;
    TeamRuntime Rt = makeLive(Heap, 8, Cfg);
    uint64_t Addr = 0;
    RtResult R = Rt.prepareParallel(RtRole::Master, "wf", 21, Addr);
    CHECK(!R.Ok && R.TrapReason == "shared-args-alloc-failed");
    CHECK(Heap.Allocs == 0); // the hook short-circuits the heap (DeviceRuntime.cpp:67)
  }
  { // an exhausted heap (allocate returns 0) is the same trap; state unchanged
    RecordingHeap Heap;
    Heap.FailAll = true;
    TeamRuntime Rt = makeLive(Heap);
    uint64_t Addr = 7;
    RtResult R = Rt.prepareParallel(RtRole::Master, "wf", 30, Addr);
    CHECK(!R.Ok && R.TrapReason == "shared-args-alloc-failed" && Addr == 7);
    Heap.FailAll = false;
    CHECK(Rt.prepareParallel(RtRole::Master, "wf", 30, Addr).Ok); // still Idle
    drainRegion(Rt);
    CHECK(Rt.dynamicAllocs() == 1 && Rt.dynamicFrees() == 1 && Heap.LiveBytes.empty());
  }
  { // protocol violations trap with specific reasons
    RecordingHeap Heap;
    uint64_t Addr = 0;
    { // prepare before init
      TeamRuntime Rt({}, PreallocBase, Heap);
      RtResult R = Rt.prepareParallel(RtRole::Master, "wf", 1, Addr);
      CHECK(!R.Ok && R.TrapReason == "protocol error: prepare_parallel before init");
    }
    { // worker prepares
      TeamRuntime Rt = makeLive(Heap);
      RtResult R = Rt.prepareParallel(RtRole::Worker, "wf", 1, Addr);
      CHECK(!R.Ok && R.TrapReason == "protocol error: prepare_parallel from a worker thread");
    }
    { // double prepare
      TeamRuntime Rt = makeLive(Heap);
      CHECK(Rt.prepareParallel(RtRole::Master, "wf", 1, Addr).Ok);
      RtResult R = Rt.prepareParallel(RtRole::Master, "wf", 1, Addr);
      CHECK(!R.Ok && R.TrapReason == "protocol error: prepare_parallel while a region is in flight");
    }
    { // prepare while workers are still inside the previous region
      TeamRuntime Rt = makeLive(Heap);
      CHECK(Rt.prepareParallel(RtRole::Master, "wf", 1, Addr).Ok);
      std::string Wf;
      bool P = false;
      CHECK(Rt.kernelParallel(RtRole::Worker, Wf, Addr, P).Ok);
      CHECK(!Rt.prepareParallel(RtRole::Master, "wf", 1, Addr).Ok);
    }
    { // fetch with nothing staged
      TeamRuntime Rt = makeLive(Heap);
      std::string Wf;
      bool P = false;
      RtResult R = Rt.kernelParallel(RtRole::Worker, Wf, Addr, P);
      CHECK(!R.Ok && R.TrapReason == "protocol error: kernel_parallel with no staged region");
    }
    { // master fetches work
      TeamRuntime Rt = makeLive(Heap);
      CHECK(Rt.prepareParallel(RtRole::Master, "wf", 1, Addr).Ok);
      std::string Wf;
      bool P = false;
      RtResult R = Rt.kernelParallel(RtRole::Master, Wf, Addr, P);
      CHECK(!R.Ok && R.TrapReason == "protocol error: kernel_parallel from the master thread");
    }
    { // end with no active region
      TeamRuntime Rt = makeLive(Heap);
      RtResult R = Rt.endParallel(RtRole::Worker);
      CHECK(!R.Ok && R.TrapReason == "protocol error: end_parallel with no active region");
    }
    { // deinit while a region is in flight
      TeamRuntime Rt = makeLive(Heap);
      CHECK(Rt.prepareParallel(RtRole::Master, "wf", 1, Addr).Ok);
      RtResult R = Rt.kernelDeinit(RtRole::Master);
      CHECK(!R.Ok && R.TrapReason == "protocol error: kernel_deinit while a region is in flight");
    }
    { // double deinit
      TeamRuntime Rt = makeLive(Heap);
      CHECK(Rt.kernelDeinit(RtRole::Master).Ok);
      RtResult R = Rt.kernelDeinit(RtRole::Master);
      CHECK(!R.Ok && R.TrapReason == "protocol error: kernel_deinit called twice");
    }
  }
  { // after deinit workers receive the termination sentinel
    RecordingHeap Heap;
    TeamRuntime Rt = makeLive(Heap);
    CHECK(Rt.kernelDeinit(RtRole::Master).Ok);
    std::string Wf = "stale";
    uint64_t Args = 99;
    bool P = true;
    CHECK(Rt.kernelParallel(RtRole::Worker, Wf, Args, P).Ok);
    CHECK(Wf.empty() && Args == 0 && !P && Rt.terminated());
  }
  { // event log keeps the lifecycle in order
    RecordingHeap Heap;
    TeamRuntime Rt = makeLive(Heap);
    uint64_t Addr = 0;
    CHECK(Rt.prepareParallel(RtRole::Master, "region0", 21, Addr).Ok);
    std::string Wf;
    bool P = false;
    CHECK(Rt.kernelParallel(RtRole::Worker, Wf, Addr, P).Ok);
    CHECK(Wf == "region0");
    CHECK(Rt.endParallel(RtRole::Worker).Ok);
    CHECK(Rt.kernelDeinit(RtRole::Master).Ok);
    std::vector<RuntimeEvent::Kind> K;
    for (const auto &E : Rt.events())
      K.push_back(E.K);
    CHECK((K == std::vector<RuntimeEvent::Kind>{RuntimeEvent::Init, RuntimeEvent::PrepareDynamic,
                                                RuntimeEvent::Fetch, RuntimeEvent::Retire,
                                                RuntimeEvent::DynamicFree, RuntimeEvent::Deinit}));
    CHECK(Rt.events()[1].str() == "prepare region0 nargs=21 dynamic bytes=168");
    CHECK(Rt.events()[4].str() == "free bytes=168");
  }
  { // dynamic allocation follows the byte law for every count
    std::mt19937 Rng(1234);
    std::uniform_int_distribution<int64_t> Dist(0, 128);
    for (int Round = 0; Round < 200; ++Round) {
      int64_t N = Dist(Rng);
      RecordingHeap Heap;
      TeamRuntime Rt = makeLive(Heap);
      uint64_t Addr = 0;
      CHECK(Rt.prepareParallel(RtRole::Master, "wf", N, Addr).Ok);
      int64_t Dynamic = Heap.LiveBytes.empty() ? 0 : Heap.LiveBytes.begin()->second;
      CHECK(Dynamic == dynamicArgsBytes(static_cast<int>(N)));
      CHECK((Dynamic == 0) == (N <= DefaultPreallocEntries));
      if (N > DefaultPreallocEntries)
        CHECK(Dynamic == SharedArgEntryBytes * N);
    }
  }
  { // long histories: O(1) per call (no replay), W workers per region
    RecordingHeap Heap;
    TeamRuntime Rt = makeLive(Heap, 3);
    for (int R = 0; R < 300; ++R) {
      uint64_t Addr = 0;
      const int64_t N = R % 3 == 0 ? 25 : 2;
      CHECK(Rt.prepareParallel(RtRole::Master, R % 2 ? "odd" : "even", N, Addr).Ok);
      for (int W = 0; W < 3; ++W) {
        std::string Wf;
        uint64_t A = 0;
        bool P = false;
        CHECK(Rt.kernelParallel(RtRole::Worker, Wf, A, P).Ok && P && A == Addr);
        CHECK(Wf == (R % 2 ? "odd" : "even"));
      }
      for (int W = 0; W < 3; ++W)
        CHECK(Rt.endParallel(RtRole::Worker).Ok);
    }
    CHECK(Rt.kernelDeinit(RtRole::Master).Ok);
    CHECK(Rt.dynamicAllocs() == 100 && Rt.dynamicFrees() == 100 && Heap.LiveBytes.empty());
    CHECK(Rt.events().size() == 1 + 300 * 7 + 100 + 1); // init, per region 1+3+3, frees, deinit
  }
  std::printf("%s (%d failures)\n", Failures ? "FAILED" : "ok", Failures);
  return Failures ? 1 : 0;
}
