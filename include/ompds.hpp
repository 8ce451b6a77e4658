// ompds.hpp -- header-only C++ adapter with the reference's class shapes
// (omplab::TeamRuntime / RtResult / RuntimeConfig / RuntimeEvent,
// proj/include/omplab/DeviceRuntime.h:26-119) over the C ABI in ompds.h.
//
// Drop-in for code written against omplab::TeamRuntime: same method names,
// argument meaning and error behaviour (RtResult with the reference's exact
// trap strings, no exceptions).  The protocol executes on the GPU: every call
// replays the team's call history through ompds_rt_replay, i.e. through the
// same __device__ state machine the sm_100a generic-mode kernels inline.
// Work functions are named by strings as in the reference; the device runtime
// stages integer ids (the order of successful prepares) and this adapter maps
// them back.
#ifndef OMPDS_HPP
#define OMPDS_HPP

#include "ompds.h"

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace ompds_cpp {

inline constexpr int DefaultPreallocEntries = OMPDS_DEFAULT_PREALLOC_ENTRIES;
inline constexpr int64_t SharedArgEntryBytes = OMPDS_SHARED_ARG_ENTRY_BYTES;
inline constexpr int64_t RuntimePrivateBytes = OMPDS_RUNTIME_PRIVATE_BYTES;

inline int64_t dynamicArgsBytes(int NArgs, int PreallocEntries = DefaultPreallocEntries) {
  return ompds_dynamic_args_bytes(NArgs, PreallocEntries);
}

struct RuntimeConfig {
  int PreallocEntries = DefaultPreallocEntries;
  bool FailDynamicAlloc = false;
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
  /// `PreallocBase` is reported for lists in the shared-memory window; lists
  /// that spill report a distinct non-zero global address per prepare.
  TeamRuntime(RuntimeConfig Config, uint64_t PreallocBase)
      : Config(Config), PreallocBase(PreallocBase) {}

  RtResult kernelInit(RtRole Role, int WorkerCount) {
    return run(OMPDS_OP_KERNEL_INIT, Role, WorkerCount).first;
  }
  RtResult prepareParallel(RtRole Role, const std::string &Fn, int64_t NArgs,
                           uint64_t &ArgsAddr) {
    auto R = run(OMPDS_OP_PREPARE_PARALLEL, Role, NArgs);
    if (R.first.Ok) {
      Fns.push_back(Fn);
      ArgsAddr = addr(R.second.addr_kind);
    }
    return R.first;
  }
  RtResult kernelParallel(RtRole Role, std::string &WfName, uint64_t &ArgsAddr,
                          bool &Participate) {
    auto R = run(OMPDS_OP_KERNEL_PARALLEL, Role, 0);
    if (R.first.Ok) {
      WfName = R.second.wf >= 0 ? Fns.at(R.second.wf) : std::string();
      ArgsAddr = addr(R.second.addr_kind);
      Participate = R.second.participate != 0;
    }
    return R.first;
  }
  RtResult endParallel(RtRole Role) { return run(OMPDS_OP_END_PARALLEL, Role, 0).first; }
  RtResult kernelDeinit(RtRole Role) { return run(OMPDS_OP_KERNEL_DEINIT, Role, 0).first; }

  int workerCount() const { return Summary.workers; }
  int64_t dynamicAllocs() const { return Summary.dynamic_allocs; }
  int64_t dynamicFrees() const { return Summary.dynamic_frees; }
  int64_t leakedBlocks() const { return Summary.leaked_blocks; }
  bool terminated() const { return Summary.terminated != 0; }
  std::vector<RuntimeEvent> events() const {
    std::vector<RuntimeEvent> Out;
    for (const ompds_event &E : Events)
      Out.push_back({static_cast<RuntimeEvent::Kind>(E.kind),
                     E.fn >= 0 && size_t(E.fn) < Fns.size() ? Fns[E.fn] : std::string(),
                     E.nargs, E.bytes});
    return Out;
  }

private:
  std::pair<RtResult, ompds_rt_result> run(int32_t Op, RtRole Role, int64_t Arg) {
    Calls.push_back({Op, Role == RtRole::Master ? OMPDS_ROLE_MASTER : OMPDS_ROLE_WORKER, Arg});
    std::vector<ompds_rt_result> Res(Calls.size());
    std::vector<ompds_event> Ev(4096);
    ompds_runtime_config C{Config.PreallocEntries, Config.FailDynamicAlloc ? 1 : 0};
    ompds_rt_summary S{};
    int32_t St = ompds_rt_replay(&C, Calls.data(), static_cast<int32_t>(Calls.size()),
                                 Res.data(), Ev.data(), static_cast<int32_t>(Ev.size()), &S);
    if (St != OMPDS_OK)
      throw std::runtime_error(std::string("ompds_rt_replay: ") + ompds_last_error());
    ompds_rt_result Last = Res.back();
    if (Last.status != OMPDS_OK) {
      Calls.pop_back(); // a trap leaves the runtime state untouched
      return {RtResult::trap(ompds_trap_reason(Last.status)), Last};
    }
    Summary = S;
    Ev.resize(static_cast<size_t>(S.n_events < 4096 ? S.n_events : 4096));
    Events = std::move(Ev);
    return {RtResult::ok(), Last};
  }
  uint64_t addr(int32_t Kind) const {
    if (Kind == OMPDS_ADDR_PREALLOC)
      return PreallocBase;
    if (Kind == OMPDS_ADDR_DYNAMIC)
      return 0x40000000ull + 0x100ull * Fns.size();
    return 0;
  }

  RuntimeConfig Config;
  uint64_t PreallocBase;
  std::vector<ompds_rt_call> Calls;
  std::vector<std::string> Fns;
  ompds_rt_summary Summary{};
  std::vector<ompds_event> Events;
};

} // namespace ompds_cpp

#endif // OMPDS_HPP
