// ompds.hpp -- header-only C++ adapter with the reference's class shapes
// (omplab::TeamRuntime / SharedArgsAllocator / RtResult / RuntimeConfig /
// RuntimeEvent, proj/include/omplab/DeviceRuntime.h:26-119) over the C ABI
// in ompds.h.
//
// Drop-in for code written against omplab::TeamRuntime: same constructor
// (RuntimeConfig, PreallocBase, SharedArgsAllocator&), method names,
// argument meaning and error behaviour (RtResult with the reference's exact
// trap strings, no exceptions on protocol errors).  Each TeamRuntime owns
// one ompds_team handle whose state lives on the GPU; every call runs the
// team's __device__ protocol function once (O(1) per call).  The allocator
// is called where the reference calls it -- allocate() after prepare's
// checks pass for a list past the window (never with FailDynamicAlloc),
// release() by the last retirement of that region.  Work functions are
// named by strings as in the reference; the adapter interns them as the
// integer ids the device stages.
//
// `namespace omplab` is an alias of `ompds_cpp` (define
// OMPDS_NO_OMPLAB_ALIAS to drop it), so `omplab::TeamRuntime` code compiles
// unchanged against this header.
#ifndef OMPDS_HPP
#define OMPDS_HPP

#include "ompds.h"

#include <cstdint>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <utility>
#include <vector>

namespace ompds_cpp {

inline constexpr int DefaultPreallocEntries = OMPDS_DEFAULT_PREALLOC_ENTRIES;
inline constexpr int64_t SharedArgEntryBytes = OMPDS_SHARED_ARG_ENTRY_BYTES;
inline constexpr int64_t RuntimePrivateBytes = OMPDS_RUNTIME_PRIVATE_BYTES;

constexpr int64_t dynamicArgsBytes(int NArgs, int PreallocEntries = DefaultPreallocEntries) {
  return NArgs <= PreallocEntries ? 0 : int64_t(NArgs) * SharedArgEntryBytes;
}

struct RuntimeConfig {
  int PreallocEntries = DefaultPreallocEntries;
  bool FailDynamicAlloc = false; // test hook: dynamic requests report failure
};

/// Device-heap hooks the runtime uses for oversized shared-args lists
/// (DeviceRuntime.h:46-52).
class SharedArgsAllocator {
public:
  virtual ~SharedArgsAllocator() = default;
  /// Returns the block address, or 0 when the heap is exhausted.
  virtual uint64_t allocate(int64_t Bytes) = 0;
  virtual void release(uint64_t Addr) = 0;
};

enum class RtRole { Master, Worker };

struct RtResult {
  bool Ok = true;
  std::string TrapReason;
  static RtResult ok() { return {}; }
  static RtResult trap(std::string R) { return {false, std::move(R)}; }
};

struct RuntimeEvent {
  enum Kind { Init, PreparePrealloc, PrepareDynamic, Fetch, Retire, DynamicFree, Deinit } K;
  std::string Fn;
  int64_t NArgs = 0;
  int64_t Bytes = 0;
  std::string str() const {
    switch (K) {
    case Init: return "init workers=" + std::to_string(NArgs);
    case PreparePrealloc: return "prepare " + Fn + " nargs=" + std::to_string(NArgs) + " prealloc";
    case PrepareDynamic:
      return "prepare " + Fn + " nargs=" + std::to_string(NArgs) +
             " dynamic bytes=" + std::to_string(Bytes);
    case Fetch: return "fetch " + Fn;
    case Retire: return "retire remaining=" + std::to_string(NArgs);
    case DynamicFree: return "free bytes=" + std::to_string(Bytes);
    case Deinit: return "deinit";
    }
    return "?";
  }
};

class TeamRuntime {
public:
  /// Throws std::runtime_error only if the device handle cannot be created
  /// (no usable GPU): there is no host fallback.
  TeamRuntime(RuntimeConfig Config, uint64_t PreallocBase, SharedArgsAllocator &Heap)
      : Heap(&Heap) {
    ompds_runtime_config C{Config.PreallocEntries, Config.FailDynamicAlloc ? 1 : 0};
    // the allocator itself is the callbacks' user pointer: it outlives the
    // runtime (the reference keeps a reference) and survives moves
    int32_t S = ompds_team_create(&C, PreallocBase, &TeamRuntime::allocThunk,
                                  &TeamRuntime::releaseThunk, &Heap, &H);
    if (S != OMPDS_OK)
      throw std::runtime_error(std::string("ompds_team_create: ") + ompds_last_error());
  }
  TeamRuntime(const TeamRuntime &) = delete;
  TeamRuntime &operator=(const TeamRuntime &) = delete;
  TeamRuntime(TeamRuntime &&O) noexcept { *this = std::move(O); }
  TeamRuntime &operator=(TeamRuntime &&O) noexcept {
    if (this != &O) {
      ompds_team_destroy(H);
      H = std::exchange(O.H, nullptr);
      Heap = O.Heap;
      Fns = std::move(O.Fns);
      FnIds = std::move(O.FnIds);
      Events = std::move(O.Events);
      Summary = O.Summary;
    }
    return *this;
  }
  ~TeamRuntime() { ompds_team_destroy(H); }

  RtResult kernelInit(RtRole Role, int WorkerCount) {
    return done(ompds_team_kernel_init(H, role(Role), WorkerCount));
  }
  RtResult prepareParallel(RtRole Role, const std::string &Fn, int64_t NArgs,
                           uint64_t &ArgsAddr) {
    uint64_t A = 0;
    RtResult R = done(ompds_team_prepare_parallel(H, role(Role), intern(Fn), NArgs, &A));
    if (R.Ok)
      ArgsAddr = A;
    return R;
  }
  /// WfName comes back empty once the kernel is torn down.
  RtResult kernelParallel(RtRole Role, std::string &WfName, uint64_t &ArgsAddr,
                          bool &Participate) {
    int32_t Fn = -1, P = 0;
    uint64_t A = 0;
    RtResult R = done(ompds_team_kernel_parallel(H, role(Role), &Fn, &A, &P));
    if (R.Ok) {
      WfName = Fn >= 0 ? Fns.at(static_cast<size_t>(Fn)) : std::string();
      ArgsAddr = A;
      Participate = P != 0;
    }
    return R;
  }
  RtResult endParallel(RtRole Role) { return done(ompds_team_end_parallel(H, role(Role))); }
  RtResult kernelDeinit(RtRole Role) { return done(ompds_team_kernel_deinit(H, role(Role))); }

  int workerCount() const { return Summary.workers; }
  int64_t dynamicAllocs() const { return Summary.dynamic_allocs; }
  int64_t dynamicFrees() const { return Summary.dynamic_frees; }
  int64_t leakedBlocks() const { return Summary.leaked_blocks; }
  bool terminated() const { return Summary.terminated != 0; }
  const std::vector<RuntimeEvent> &events() const { return Events; }

private:
  static uint64_t allocThunk(int64_t Bytes, void *Heap) {
    return static_cast<SharedArgsAllocator *>(Heap)->allocate(Bytes);
  }
  static void releaseThunk(uint64_t Addr, void *Heap) {
    static_cast<SharedArgsAllocator *>(Heap)->release(Addr);
  }
  static int32_t role(RtRole R) { return R == RtRole::Master ? OMPDS_ROLE_MASTER : OMPDS_ROLE_WORKER; }
  int32_t intern(const std::string &Fn) {
    auto It = FnIds.find(Fn);
    if (It != FnIds.end())
      return It->second;
    const int32_t Id = static_cast<int32_t>(Fns.size());
    Fns.push_back(Fn);
    FnIds.emplace(Fn, Id);
    return Id;
  }
  RtResult done(int32_t S) {
    if (S >= OMPDS_ERR_CUDA)
      throw std::runtime_error(std::string("ompds_team: ") + ompds_trap_reason(S) + ": " +
                               ompds_last_error());
    if (S != OMPDS_OK)
      return RtResult::trap(ompds_trap_reason(S));
    ompds_team_summary(H, &Summary);
    // pull the events this call logged (O(new events))
    int32_t Total = 0;
    ompds_event Buf[8];
    for (;;) {
      const int32_t First = static_cast<int32_t>(Events.size());
      int32_t St = ompds_team_events(H, First, Buf, 8, &Total);
      for (int32_t I = 0; I < 8 && First + I < Total; ++I) {
        const ompds_event &E = Buf[I];
        Events.push_back({static_cast<RuntimeEvent::Kind>(E.kind),
                          E.fn >= 0 && size_t(E.fn) < Fns.size() ? Fns[E.fn] : std::string(),
                          E.nargs, E.bytes});
      }
      if (St != OMPDS_ERR_CAPACITY)
        break;
    }
    return RtResult::ok();
  }

  ompds_team *H = nullptr;
  SharedArgsAllocator *Heap = nullptr;
  std::vector<std::string> Fns;
  std::unordered_map<std::string, int32_t> FnIds;
  std::vector<RuntimeEvent> Events;
  ompds_rt_summary Summary{};
};

} // namespace ompds_cpp

#ifndef OMPDS_NO_OMPLAB_ALIAS
namespace omplab = ompds_cpp;
#endif

#endif // OMPDS_HPP
