// ompds_device.cuh -- sm_100a device runtime for implicit OpenMP data
// sharing in generic-mode target regions (arXiv 1711.10413), B200-native.
//
// What the reference models on the host (proj/src/DeviceRuntime.cpp and the
// team execution model of proj/src/Simulator.cpp) lives here as __device__
// code that generic-mode kernels inline:
//
//   * team runtime state machine (Uninitialized -> Idle -> Staged -> ... ->
//     Terminated) in the team's 49-byte runtime-private shared-memory span,
//     with the reference's exact trap semantics (DeviceRuntime.cpp:33-143);
//   * the shared-args list: 8*PreallocEntries bytes of shared memory right
//     after the depot, or a block of the team's global overflow slab when a
//     region captures more (DeviceRuntime.cpp:61-74, 108-121);
//   * named-barrier region handoff (bar.sync <id>, <count>) replacing the
//     simulator's "all live threads blocked" barrier (Simulator.cpp:481-499);
//     every lane of the reserved warp stays resident and arrives, because
//     exited threads never arrive at a hardware barrier;
//   * warp-aggregated fetch/retire (one shared-memory atomic per warp instead
//     of one per thread) and a warp-shuffle broadcast of the shared-variable
//     pointer list (get-shared-variables, Codegen.cpp:215-267);
//   * data-sharing stacks: per warp, a statically sized shared-memory slot
//     plus a global-memory overflow chain, managed in registers by the warp
//     that owns it (the master's kernel depot is its first frame,
//     Simulator.cpp:439-479, 651-669).
//
// Entry points keep the reference / LLVM runtime names as aliases:
//   __kmpc_kernel_init / _prepare_parallel / _parallel / _end_parallel /
//   _deinit, __kmpc_data_sharing_push_stack / _pop_stack,
//   __kmpc_get_shared_variables.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/ompds.h"

namespace ompds {

// The general (trap / event-log / global-list) paths of prepare and fetch
// are inlined: as calls they cost 3 % of config-4 bandwidth (the whole
// kernel's register allocation changes).  Overridable for experiments.
#ifndef OMPDS_GENERAL_INLINE
#define OMPDS_GENERAL_INLINE __forceinline__
#endif
constexpr int kWarp = 32;
constexpr uint32_t kBarHandoff = 1; // master <-> worker region handoff
constexpr uint32_t kBarRegion = 2;  // `omp barrier` among a region's workers

enum Phase : uint8_t { kUninit = 0, kIdle = 1, kStaged = 2, kTerminated = 3 };
enum Role : int { kMaster = OMPDS_ROLE_MASTER, kWorker = OMPDS_ROLE_WORKER };

// Byte offsets inside the runtime-private span.  Exactly 49 bytes, the
// reference's RuntimePrivateBytes (DeviceRuntime.h:31), so the team region
// footprint is depot + 8*PreallocEntries + 49 as in Simulator.cpp:281-284.
// The phase shares a 32-bit word with the staged work function, next to
// nargs: a worker's fetch reads everything it needs with one 8-byte load,
// and staging is two stores.  Active and the staged region's retired count
// live in their own word, so the workers' bookkeeping atomics never touch a
// word another lane of the warp is reading.
struct Rt {
  static constexpr int kArgs = 0;      // u64 args list (generic address)
  static constexpr int kState = 8;     // u32 phase << 24 | work fn (24-bit
                                       //   two's complement, -1 = none)
  static constexpr int kPhase = 11;    // u8 phase = the state word's top byte
  static constexpr int kNArgs = 12;    // i32 staged nargs
  static constexpr int kActive = 16;   // u32 retired << 16 | Active
  static constexpr int kWorkers = 20;  // i32 Workers
  static constexpr int kHeapTop = 24;  // u32 bytes in use in the global slab
  static constexpr int kDynAllocs = 28;// u32
  static constexpr int kDynFrees = 32; // u32
  static constexpr int kTrap = 36;     // i32 first trap code
  static constexpr int kDynBytes = 40; // u32 dynamic args bytes allocated
  static constexpr int kEvents = 44;   // u32 events logged
  static constexpr int kSpare = 48;    // u8 unused
  static constexpr int kBytes = 49;
  static constexpr uint32_t kActiveMask = 0xffffu;
  static constexpr int kRetiredShift = 16;
  static constexpr int kPhaseShift = 24;
  static constexpr uint32_t kFnMask = 0xffffffu;
};
// Work-function ids are 24-bit: [0, 2^23) (-1 = none).
constexpr int32_t kMaxWorkFn = (1 << 23) - 1;
__host__ __device__ constexpr uint32_t state_word(uint8_t phase, int32_t fn) {
  return (uint32_t(phase) << Rt::kPhaseShift) | (uint32_t(fn) & Rt::kFnMask);
}
__host__ __device__ constexpr int32_t state_fn(uint32_t w) {
  return static_cast<int32_t>(w << 8) >> 8; // sign-extend the low 24 bits
}
static_assert(Rt::kBytes == OMPDS_RUNTIME_PRIVATE_BYTES, "rt span");

__host__ __device__ constexpr int64_t round_up(int64_t v, int64_t a) {
  return (v + a - 1) / a * a;
}

// Dynamic shared memory of one team: [depot | window | rt].
__host__ __device__ constexpr int64_t team_region_bytes(int64_t depot,
                                                        int prealloc) {
  return depot + int64_t(prealloc) * OMPDS_SHARED_ARG_ENTRY_BYTES +
         OMPDS_RUNTIME_PRIVATE_BYTES;
}

//===----------------------------------------------------------------------===//
// Low-level primitives
//===----------------------------------------------------------------------===//

// Named barrier: the non-.aligned `barrier.sync` -- each thread arrives
// individually, so master and worker warps may reach the handoff barrier
// from different instructions and after divergent code.  `.aligned`
// (`bar.sync`) requires every participating thread of the CTA to execute
// the same instruction; at the master's and the workers' different call
// sites that is undefined behaviour (compute-sanitizer synccheck reports it),
// and a two-warp ping-pong measures both forms at 16 cycles per barrier
// (tools/micro_lat.cu).
__device__ __forceinline__ void bar_sync(uint32_t id, uint32_t count) {
  asm volatile("barrier.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// Not volatile: the lane id is invariant, so the compiler may hoist the
// (long-latency) S2R out of the region loops.
__device__ __forceinline__ uint32_t lane_id() {
  uint32_t l;
  asm("mov.u32 %0, %%laneid;" : "=r"(l));
  return l;
}

// Device time for the event trace (ns since an arbitrary epoch).
__device__ __forceinline__ int64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return static_cast<int64_t>(t);
}

//===----------------------------------------------------------------------===//
// Team context
//===----------------------------------------------------------------------===//

struct TeamCtx {
  unsigned char *region;   // team region in shared memory (generic address)
  int64_t depot_cap;       // master data-sharing slot bytes at region[0..)
  void **window;           // the preallocated shared-args list
  unsigned char *rt;       // runtime-private span
  unsigned char *slab;     // team's global overflow slab (args lists + frames)
  uint32_t slab_bytes;
  int32_t prealloc;        // PreallocEntries
  int32_t fail_dyn;        // FailDynamicAlloc
  ompds_event *events;     // per-team event log (nullptr: off)
  int32_t max_events;
  int32_t list_malloc;     // args lists past the window: 1 device malloc, 0 slab
  uint32_t rt_s;           // shared-window addresses of rt / window (computed
  uint32_t window_s;       // once: no address conversion on the region path)

  template <class T> __device__ __forceinline__ T &at(int off) const {
    return *reinterpret_cast<T *>(rt + off);
  }
  __device__ __forceinline__ uint8_t &phase() const { return at<uint8_t>(Rt::kPhase); }
  // The word at kActive: low 16 bits = Active (fetched - retired), high 16
  // bits = participants retired from the staged region (warp path).
  __device__ __forceinline__ uint32_t &active_word() const { return at<uint32_t>(Rt::kActive); }
  __device__ __forceinline__ int32_t active() const {
    return static_cast<int32_t>(active_word() & Rt::kActiveMask);
  }
  __device__ __forceinline__ void *&args() const { return at<void *>(Rt::kArgs); }
  __device__ __forceinline__ int32_t work_fn() const {
    return state_fn(at<uint32_t>(Rt::kState));
  }
  __device__ __forceinline__ void set_work_fn(int32_t fn) const {
    uint32_t &w = at<uint32_t>(Rt::kState);
    w = (w & ~Rt::kFnMask) | (uint32_t(fn) & Rt::kFnMask);
  }
  __device__ __forceinline__ int32_t &nargs() const { return at<int32_t>(Rt::kNArgs); }

  __device__ __forceinline__ bool args_dynamic() const {
    void *a = args();
    return a != nullptr && a != static_cast<void *>(window);
  }

  // Records the first trap of the team (Simulator's R.Trapped semantics).
  __device__ __forceinline__ int32_t trap(int32_t code) const {
    atomicCAS(&at<int32_t>(Rt::kTrap), 0, code);
    return code;
  }

  __device__ __forceinline__ void log(int32_t kind, int32_t fn, int64_t nargs,
                                      int64_t bytes) const {
    if (!events)
      return;
    uint32_t i = atomicAdd(&at<uint32_t>(Rt::kEvents), 1u);
    if (static_cast<int32_t>(i) < max_events)
      events[i] = ompds_event{kind, fn, nargs, bytes, globaltimer_ns()};
  }
  // Reserves `n` consecutive event slots, returns the first (or -1 if off).
  __device__ __forceinline__ int64_t log_reserve(uint32_t n) const {
    if (!events)
      return -1;
    return atomicAdd(&at<uint32_t>(Rt::kEvents), n);
  }
  __device__ __forceinline__ void log_at(int64_t i, int32_t kind, int32_t fn,
                                         int64_t nargs, int64_t bytes) const {
    if (i >= 0 && i < max_events)
      events[i] = ompds_event{kind, fn, nargs, bytes, globaltimer_ns()};
  }

  // LIFO allocator over the team's global slab.  The reference heap never
  // reuses memory (Simulator.cpp:150-162); ours is a stack because at most
  // one args list per team level is live (the phase machine forbids a new
  // prepare while a region is in flight).
  __device__ __forceinline__ void *slab_alloc(int64_t bytes) const {
    uint32_t &top = at<uint32_t>(Rt::kHeapTop);
    int64_t need = round_up(bytes, 16);
    if (slab == nullptr || top + need > slab_bytes)
      return nullptr;
    void *p = slab + top;
    top += static_cast<uint32_t>(need);
    return p;
  }
  __device__ __forceinline__ void slab_free(void *p) const {
    at<uint32_t>(Rt::kHeapTop) =
        static_cast<uint32_t>(static_cast<unsigned char *>(p) - slab);
  }
  // An args list that does not fit the window: the team slab (default), or
  // -- OMPDS_LIST_MALLOC, the paper's back-up scheme -- device malloc, freed
  // by the last retirement.
  __device__ __forceinline__ void *list_alloc(int64_t bytes) const {
    if (list_malloc)
      return malloc(static_cast<size_t>(bytes));
    return slab_alloc(bytes);
  }
  __device__ __forceinline__ void list_free(void *p) const {
    if (list_malloc)
      free(p);
    else
      slab_free(p);
  }
};

// Carves the team region out of dynamic shared memory and zero-initialises
// the runtime span (the simulator zero-fills team memory, Simulator.cpp:286).
__device__ __forceinline__ TeamCtx make_team(unsigned char *smem,
                                             int64_t depot_cap, int prealloc,
                                             int fail_dyn, unsigned char *slab,
                                             uint32_t slab_bytes,
                                             ompds_event *events,
                                             int max_events,
                                             int list_malloc = 0) {
  TeamCtx t;
  t.region = smem;
  t.depot_cap = depot_cap;
  t.window = reinterpret_cast<void **>(smem + depot_cap);
  t.rt = smem + depot_cap + int64_t(prealloc) * OMPDS_SHARED_ARG_ENTRY_BYTES;
  t.slab = slab;
  t.slab_bytes = slab_bytes;
  t.prealloc = prealloc;
  t.fail_dyn = fail_dyn;
  t.events = events;
  t.max_events = max_events;
  t.list_malloc = list_malloc;
  t.rt_s = static_cast<uint32_t>(__cvta_generic_to_shared(t.rt));
  t.window_s = static_cast<uint32_t>(__cvta_generic_to_shared(t.window));
  return t;
}

// Team state snapshots: every load issued in one asm block, so the
// compiler cannot sink a later load below a branch on an earlier one (one
// shared-memory round trip instead of a chain).
struct PrepareState {
  uint32_t phase;
  int32_t active;
};
__device__ __forceinline__ PrepareState load_prepare_state(const TeamCtx &t) {
  uint32_t sw, aw;
  asm volatile("ld.shared.u32 %0, [%2+8];\n\t"
               "ld.shared.u32 %1, [%2+16];"
               : "=r"(sw), "=r"(aw)
               : "r"(t.rt_s)
               : "memory");
  static_assert(Rt::kState == 8 && Rt::kActive == 16, "rt layout");
  return PrepareState{sw >> Rt::kPhaseShift, static_cast<int32_t>(aw & Rt::kActiveMask)};
}
// The fast path of prepare_parallel reads only the phase: the protocol
// keeps Idle => Active == 0 (Active rises only while a region is Staged, and
// the retirement that brings it back to 0 is the one that returns the team
// to Idle -- DeviceRuntime.cpp:81-128), so "Idle" already implies "no region
// in flight"; the general path loads Active too and checks both in the
// reference's order.
__device__ __forceinline__ uint32_t load_phase(const TeamCtx &t) {
  uint32_t sw;
  asm volatile("ld.shared.u32 %0, [%1+8];" : "=r"(sw) : "r"(t.rt_s) : "memory");
  static_assert(Rt::kState == 8, "rt layout");
  return sw >> Rt::kPhaseShift;
}
struct StagedState {
  uint32_t phase; // the state word's top byte (uint32: one compare, no byte sign-extension)
  int32_t fn;
  int32_t nargs;
  void **args; // the staged list (loaded only when the caller needs it)
  void *win;   // this lane's window entry (prefetch), or nullptr
};
// `win_off`: shared address of this lane's window entry, 0 = none.  kArgs:
// also load the list pointer (a list past the window is possible); without
// it the list is the window (the lean instantiation's guarantee).
template <bool kArgs = true>
__device__ __forceinline__ StagedState load_staged_state(const TeamCtx &t,
                                                         uint32_t win_off) {
  const uint32_t rt = t.rt_s;
  uint32_t sw, na;
  unsigned long long args = 0, win = 0;
  static_assert(Rt::kArgs == 0 && Rt::kState == 8 && Rt::kNArgs == 12, "rt layout");
  if (kArgs && win_off)
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%5+8];\n\t"
                 "ld.shared.u64 %2, [%5];\n\t"
                 "ld.shared.u64 %3, [%4];"
                 : "=r"(sw), "=r"(na), "=l"(args), "=l"(win)
                 : "r"(win_off), "r"(rt)
                 : "memory");
  else if (kArgs)
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%3+8];\n\t"
                 "ld.shared.u64 %2, [%3];"
                 : "=r"(sw), "=r"(na), "=l"(args)
                 : "r"(rt)
                 : "memory");
  else if (win_off)
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%4+8];\n\t"
                 "ld.shared.u64 %2, [%3];"
                 : "=r"(sw), "=r"(na), "=l"(win)
                 : "r"(win_off), "r"(rt)
                 : "memory");
  else
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2+8];"
                 : "=r"(sw), "=r"(na)
                 : "r"(rt)
                 : "memory");
  void **list = kArgs ? reinterpret_cast<void **>(args) : t.window;
  return StagedState{sw >> Rt::kPhaseShift, state_fn(sw),
                     static_cast<int32_t>(na), list, reinterpret_cast<void *>(win)};
}

//===----------------------------------------------------------------------===//
// Team runtime protocol -- single-caller semantics, identical to
// omplab::TeamRuntime (DeviceRuntime.cpp:33-143), trap order included.
//===----------------------------------------------------------------------===//

__device__ inline int32_t kernel_init(const TeamCtx &t, int role,
                                      int32_t workers) {
  if (role != kMaster)
    return OMPDS_TRAP_INIT_FROM_WORKER;
  if (t.phase() != kUninit)
    return OMPDS_TRAP_INIT_TWICE;
  if (workers <= 0)
    return OMPDS_TRAP_INIT_NO_WORKERS;
  t.phase() = kIdle;
  t.at<int32_t>(Rt::kWorkers) = workers;
  t.log(OMPDS_EV_INIT, -1, workers, 0);
  return OMPDS_OK;
}

// The phase checks of prepareParallel in the reference's order
// (DeviceRuntime.cpp:46-60), as a pure function of the team state so a warp
// can evaluate them on broadcast loads.
__device__ __forceinline__ int32_t prepare_check(uint32_t ph, int32_t active,
                                                 int64_t nargs) {
  if (ph == kUninit)
    return OMPDS_TRAP_PREPARE_BEFORE_INIT;
  if (ph == kTerminated)
    return OMPDS_TRAP_PREPARE_AFTER_DEINIT;
  if (ph == kStaged || active > 0)
    return OMPDS_TRAP_PREPARE_IN_FLIGHT;
  if (nargs < 0)
    return OMPDS_TRAP_NEGATIVE_NARGS;
  return OMPDS_OK;
}

// Placement decision of the shared-args list (DeviceRuntime.cpp:61-74):
// the preallocated window when nargs <= PreallocEntries, else a block of the
// team's global slab (nullptr: shared-args-alloc-failed).
__device__ __forceinline__ void **alloc_args_list(const TeamCtx &t, int32_t fn,
                                                  int64_t nargs) {
  if (nargs <= t.prealloc) {
    t.log(OMPDS_EV_PREPARE_PREALLOC, fn, nargs, 0);
    return t.window;
  }
  const int64_t bytes = nargs * OMPDS_SHARED_ARG_ENTRY_BYTES;
  void *p = t.fail_dyn ? nullptr : t.list_alloc(bytes);
  if (p == nullptr)
    return nullptr;
  t.at<uint32_t>(Rt::kDynAllocs) += 1;
  t.at<uint32_t>(Rt::kDynBytes) += static_cast<uint32_t>(bytes);
  t.log(OMPDS_EV_PREPARE_DYNAMIC, fn, nargs, bytes);
  return static_cast<void **>(p);
}

// Stages the region: Idle -> Staged.
__device__ __forceinline__ void stage_region(const TeamCtx &t, int32_t fn,
                                             int64_t nargs, void **list) {
  t.args() = list;
  t.nargs() = static_cast<int32_t>(nargs);
  t.at<uint32_t>(Rt::kState) = state_word(kStaged, fn);
}

// __kmpc_kernel_prepare_parallel / begin-sharing-variables: stages work
// function `fn` and returns the list the master fills with nargs pointers.
__device__ inline int32_t prepare_parallel(const TeamCtx &t, int role,
                                           int32_t fn, int64_t nargs,
                                           void ***out) {
  if (role != kMaster)
    return OMPDS_TRAP_PREPARE_FROM_WORKER;
  const PrepareState st = load_prepare_state(t);
  const int32_t s = prepare_check(st.phase, st.active, nargs);
  if (s)
    return s;
  void **list = alloc_args_list(t, fn, nargs);
  if (list == nullptr)
    return OMPDS_TRAP_ARGS_ALLOC_FAILED;
  stage_region(t, fn, nargs, list);
  *out = list;
  return OMPDS_OK;
}

// __kmpc_kernel_parallel: a worker fetches the staged region.
__device__ inline int32_t kernel_parallel(const TeamCtx &t, int role,
                                          int32_t *fn, void ***args,
                                          bool *participate) {
  if (role != kWorker)
    return OMPDS_TRAP_PARALLEL_FROM_MASTER;
  uint8_t ph = t.phase();
  if (ph == kTerminated) {
    *fn = -1;
    *args = nullptr;
    *participate = false;
    return OMPDS_OK;
  }
  if (ph != kStaged)
    return OMPDS_TRAP_PARALLEL_NOT_STAGED;
  *fn = t.work_fn();
  *args = static_cast<void **>(t.args());
  *participate = true;
  t.active_word() += 1;
  t.log(OMPDS_EV_FETCH, *fn, 0, 0);
  return OMPDS_OK;
}

__device__ __forceinline__ void retire_last(const TeamCtx &t) {
  if (t.args_dynamic()) {
    int64_t bytes = int64_t(t.nargs()) * OMPDS_SHARED_ARG_ENTRY_BYTES;
    t.list_free(t.args());
    t.at<uint32_t>(Rt::kDynFrees) += 1;
    t.log(OMPDS_EV_DYNAMIC_FREE, -1, 0, bytes);
  }
  t.at<uint32_t>(Rt::kState) = state_word(kIdle, -1);
  t.args() = nullptr;
  t.nargs() = 0;
  t.active_word() = 0;
}

// __kmpc_kernel_end_parallel: a worker retires; the last one frees the
// dynamic list and returns the team to Idle.
__device__ inline int32_t end_parallel(const TeamCtx &t, int role) {
  if (role != kWorker)
    return OMPDS_TRAP_END_FROM_MASTER;
  if (t.phase() != kStaged || t.active() <= 0)
    return OMPDS_TRAP_END_NOT_ACTIVE;
  t.active_word() -= 1;
  const int32_t rem = t.active();
  t.log(OMPDS_EV_RETIRE, -1, rem, 0);
  if (rem == 0)
    retire_last(t);
  return OMPDS_OK;
}

__device__ inline int32_t kernel_deinit(const TeamCtx &t, int role) {
  if (role != kMaster)
    return OMPDS_TRAP_DEINIT_FROM_WORKER;
  uint8_t ph = t.phase();
  if (ph == kUninit)
    return OMPDS_TRAP_DEINIT_BEFORE_INIT;
  if (ph == kStaged || t.active() > 0)
    return OMPDS_TRAP_DEINIT_IN_FLIGHT;
  if (ph == kTerminated)
    return OMPDS_TRAP_DEINIT_TWICE;
  t.phase() = kTerminated;
  t.log(OMPDS_EV_DEINIT, -1, 0, 0);
  return OMPDS_OK;
}

//===----------------------------------------------------------------------===//
// Warp-aggregated fetch / retire used by the generic-mode worker loop.  A
// warp call with m participating lanes is equivalent to m single calls in
// lane order: one shared-memory atomic per warp.
//===----------------------------------------------------------------------===//

struct Fetch {
  int32_t fn;        // -1: termination sentinel (wf == null)
  void **args;
  int32_t nargs;
  int32_t status;
  void *win;         // this lane's window entry, loaded speculatively
};

#ifndef OMPDS_PREFETCH_WINDOW
#define OMPDS_PREFETCH_WINDOW 1
#endif

// Participation of a worker warp's lanes (mine = tid < W).  It does not
// change between regions, so the worker loop computes it once instead of a
// ballot per fetch and per retire.
struct WarpMask {
  uint32_t ballot;  // participating lanes
  uint32_t n;       // their count
  uint32_t leader;  // lowest participating lane (does the warp's bookkeeping)
  bool is_leader;
  bool sole;        // this warp holds all W participants (W = the launch's
                    // thread_limit, which kernel_init records as Workers)
  // Also loop-invariant for a team, so hoisted with the mask (of(t, mine)):
  bool no_events;   // no event log: the fetch/retire fast paths apply
  uint32_t win_off; // shared address of this lane's window entry (0: none)
  __device__ __forceinline__ static WarpMask of(bool mine) {
    WarpMask m;
    m.ballot = __ballot_sync(0xffffffffu, mine);
    m.n = __popc(m.ballot);
    m.leader = m.ballot ? __ffs(m.ballot) - 1 : 0;
    m.is_leader = m.ballot != 0 && lane_id() == m.leader;
    m.sole = false;
    m.no_events = false; // general paths only (still correct)
    m.win_off = 0;
    return m;
  }
  __device__ __forceinline__ static WarpMask of(const TeamCtx &t, bool mine, int32_t workers) {
    WarpMask m = of(mine);
    m.sole = m.n == static_cast<uint32_t>(workers);
    m.no_events = t.events == nullptr;
#if OMPDS_PREFETCH_WINDOW
    if (static_cast<int32_t>(lane_id()) < t.prealloc)
      m.win_off = t.window_s + 8u * lane_id();
#endif
    return m;
  }
};

// Branch-free bookkeeping: shared-memory updates predicated on `p` (the
// warp stays converged; no reconvergence barrier around a leader-only block).
__device__ __forceinline__ void red_add_if(uint32_t saddr, uint32_t v, bool p) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t"
               "@q red.shared.add.u32 [%0], %1;\n\t}" ::"r"(saddr), "r"(v),
               "r"(static_cast<uint32_t>(p))
               : "memory");
}
// retire of a region whose list is the window: args = null, state = Idle
// with work_fn -1, nargs = 0, Active and retired 0 (retire_last's window
// case).
__device__ __forceinline__ void retire_window_if(const TeamCtx &t, bool p) {
  const uint32_t rt = t.rt_s;
  static_assert(Rt::kArgs == 0 && Rt::kState == 8 && Rt::kNArgs == 12 && Rt::kActive == 16,
                "rt layout");
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %1, 0;\n\t"
               "@q st.shared.u64 [%0], %2;\n\t"
               "@q st.shared.v2.u32 [%0+8], {%3, %4};\n\t"
               "@q st.shared.u32 [%0+16], %4;\n\t}" ::"r"(rt),
               "r"(static_cast<uint32_t>(p)), "l"(0ull), "r"(state_word(kIdle, -1)), "r"(0u)
               : "memory");
}
// staging of a region (stage_region's stores), predicated on `p`: two stores
// (Active and retired are already 0 -- prepare requires an idle team).
__device__ __forceinline__ void stage_region_if(const TeamCtx &t, int32_t fn,
                                                int32_t nargs, void **list, bool p) {
  const uint32_t rt = t.rt_s;
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %1, 0;\n\t"
               "@q st.shared.u64 [%0], %2;\n\t"
               "@q st.shared.v2.u32 [%0+8], {%3, %4};\n\t}" ::"r"(rt),
               "r"(static_cast<uint32_t>(p)),
               "l"(reinterpret_cast<unsigned long long>(list)),
               "r"(state_word(kStaged, fn)), "r"(static_cast<uint32_t>(nargs))
               : "memory");
}

// The lean instantiation's staging: only {state, work_fn} and nargs (its
// lists are always the window, which the workers address directly, and
// Active is never counted), predicated on `p`: one store.
__device__ __forceinline__ void stage_state_if(const TeamCtx &t, int32_t fn, int32_t nargs,
                                               bool p) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %1, 0;\n\t"
               "@q st.shared.v2.u32 [%0+8], {%2, %3};\n\t}" ::"r"(t.rt_s),
               "r"(static_cast<uint32_t>(p)), "r"(state_word(kStaged, fn)),
               "r"(static_cast<uint32_t>(nargs))
               : "memory");
}

// Without an event log nothing observes a region's Active / retired counts
// between its fetch and its join (the log is what records the workers'
// fetch and retire order), so the master completes every such region at the
// join -- freeing a heap list, returning the team to Idle -- and the
// workers keep no count: their fetch is the state load and a branch, their
// retirement nothing.  With an event log the workers retire as the
// reference does.  0 keeps the worker-side accounting everywhere.
#ifndef OMPDS_LEAN_JOIN_COMPLETES
#define OMPDS_LEAN_JOIN_COMPLETES 1
#endif
constexpr bool kLeanJoinCompletes = OMPDS_LEAN_JOIN_COMPLETES != 0;

// All 32 lanes of a worker warp call this after the release barrier.
// `mine` = this lane is a requested worker (tid < W); `m` = WarpMask::of(mine).
// Fetch from an already loaded team state (the loop issues the loads right
// after the release barrier).  `fast` is the common case -- a staged region
// and no event log -- decided by the caller.
__device__ __forceinline__ Fetch fetch_from(const StagedState &st) {
  Fetch f;
  f.win = st.win;
  f.status = OMPDS_OK;
  f.fn = st.fn;
  f.args = st.args;
  f.nargs = st.nargs;
  return f;
}
__device__ __forceinline__ bool fetch_is_fast(const StagedState &st,
                                              const WarpMask &m) {
  return st.phase == uint32_t(kStaged) && m.no_events;
}
// The fast fetch's bookkeeping, branch-free: Active += n by the warp's
// leader -- a plain store when this warp holds every participant (Active is
// 0 between regions and no other warp fetches), otherwise one
// fire-and-forget shared atomic.  The Active word is not one the fetch
// reads, so no lane of the warp can observe the update early.
__device__ __forceinline__ void fetch_account_fast(const TeamCtx &t,
                                                   const StagedState &,
                                                   const WarpMask &m) {
  asm volatile("{\n\t.reg .pred qs, qm;\n\t"
               "setp.ne.u32 qs, %2, 0;\n\t"
               "setp.ne.u32 qm, %3, 0;\n\t"
               "@qs st.shared.u32 [%0], %1;\n\t"
               "@qm red.shared.add.u32 [%0], %1;\n\t}" ::"r"(t.rt_s + Rt::kActive),
               "r"(m.n), "r"(static_cast<uint32_t>(m.is_leader && m.sole)),
               "r"(static_cast<uint32_t>(m.is_leader && !m.sole))
               : "memory");
}
// Every other case of the reference's kernel_parallel for a warp:
// termination, a fetch with nothing staged (trap), and the event log.
__device__ OMPDS_GENERAL_INLINE Fetch fetch_general(const TeamCtx &t, const StagedState &st,
                                            const WarpMask &m, bool mine) {
  Fetch f = fetch_from(st);
  const uint32_t ph = st.phase;
  if (ph == kTerminated) {
    f.fn = -1;
    f.args = nullptr;
    f.nargs = 0;
    return f;
  }
  if (ph != kStaged) {
    f.status = mine ? t.trap(OMPDS_TRAP_PARALLEL_NOT_STAGED) : OMPDS_OK;
    f.fn = -1;
    return f;
  }
  if (m.n == 0)
    return f;
  if (!t.events) { // staged, no log, reached through a general mask
    if (!kLeanJoinCompletes)
      fetch_account_fast(t, st, m);
    return f;
  }
  // staged, event log on
  int64_t ev = -1;
  if (m.is_leader) {
    atomicAdd(&t.active_word(), m.n);
    ev = t.log_reserve(m.n);
  }
  ev = __shfl_sync(0xffffffffu, ev, m.leader);
  const uint32_t lane = lane_id();
  if (mine && ev >= 0)
    t.log_at(ev + __popc(m.ballot & ((1u << lane) - 1u)), OMPDS_EV_FETCH, f.fn,
             0, 0);
  return f;
}

__device__ __forceinline__ Fetch begin_parallel_warp(const TeamCtx &t,
                                                     const WarpMask &m,
                                                     bool mine) {
  // Lane j's entry of the preallocated window (m.win_off) is loaded
  // alongside the team state (no dependency on the staged list pointer):
  // when the region's list is the window, get-shared-variables needs no
  // further load.
  const StagedState st = load_staged_state(t, m.win_off);
  if (__builtin_expect(fetch_is_fast(st, m), 1)) {
    fetch_account_fast(t, st, m);
    return fetch_from(st);
  }
  return fetch_general(t, st, m, mine);
}
__device__ __forceinline__ Fetch begin_parallel_warp(const TeamCtx &t,
                                                     bool mine) {
  return begin_parallel_warp(t, WarpMask::of(t, mine, t.at<int32_t>(Rt::kWorkers)), mine);
}

// What a worker warp needs to retire the region it fetched, packed in one
// register so nothing else stays live across the region body: bit 0 = this
// lane is the warp's leader, bit 1 = the warp holds all W participants,
// bit 2 = the list is the window (nothing to free), bit 3 = no event log,
// bits 8.. = participants.
__device__ __forceinline__ uint32_t retire_plan(const TeamCtx &t,
                                                const WarpMask &m,
                                                const Fetch &f) {
  // the list is the window iff nargs <= PreallocEntries (the placement law
  // of prepare_parallel, DeviceRuntime.cpp:61-74): a 32-bit compare
  return (m.n << 8) | (m.is_leader ? 1u : 0u) | (m.sole ? 2u : 0u) |
         (f.nargs <= t.prealloc ? 4u : 0u) | (m.no_events ? 8u : 0u);
}

// All 32 lanes of a worker warp call this when the region body is done.
// On the GPU a fast warp can retire before a slow warp has fetched, so
// "Active dropped to 0" would be premature; the last participant is instead
// the one whose retirement brings the region's retired count to W (every
// worker participates in every staged region, Codegen.cpp:403-513).  Under
// the reference's schedule (all fetches before any retire) both rules agree.
__device__ __forceinline__ void end_parallel_warp(const TeamCtx &t,
                                                  uint32_t plan) {
  const bool leader = plan & 1u;
  const uint32_t n = plan >> 8;
  if (__builtin_expect((plan & 12u) == 12u, 1)) { // window list, no event log
    if (plan & 2u) {
      // sole warp: it retires the last participant.  The __syncwarp orders
      // every lane's fetch reads before the leader's reset (lanes of one
      // warp are not implicitly ordered under independent thread scheduling).
      __syncwarp();
      retire_window_if(t, leader);
    } else {
      // Several worker warps, window list, no event log: each warp retires
      // its participants with one fire-and-forget atomic (retired += n,
      // Active -= n); the join barrier orders every retirement before the
      // master, which observes retired == W and completes the last
      // retirement (complete_region) -- no returning atomic on any worker.
      red_add_if(t.rt_s + Rt::kActive, (n << Rt::kRetiredShift) - n, leader);
    }
    return;
  }
  if (n == 0)
    return;
#ifndef OMPDS_SOLE_WARP_RETIRE
#define OMPDS_SOLE_WARP_RETIRE 1
#endif
#if OMPDS_SOLE_WARP_RETIRE
  // A warp holding all W participants retires the region's last one whatever
  // the order: no other warp touches the staged region, so its bookkeeping
  // needs no returning atomic (the leader's own fetch atomic precedes it in
  // program order).  Config 1 (W = 32) takes this path.
  if (plan & 2u) {
    if (t.events && leader) {
      const int64_t ev = t.log_reserve(n);
      for (uint32_t k = 0; k < n; ++k)
        t.log_at(ev + k, OMPDS_EV_RETIRE, -1, int64_t(n) - int64_t(k + 1), 0);
    }
    __syncwarp(); // every lane's fetch reads before the leader's reset
    if (plan & 4u)
      retire_window_if(t, leader);
    else if (leader)
      retire_last(t); // frees the global list
    return;
  }
#endif
  if (leader) {
    const uint32_t w = static_cast<uint32_t>(t.at<int32_t>(Rt::kWorkers));
    // retired += n (high half), Active -= n (low half; >= n: our own fetch).
    // acq_rel at CTA scope: every
    // participant's reads of the staged region happen-before the last
    // retiree's bookkeeping writes (retire_last).
    uint32_t old;
    asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], %2;"
                 : "=r"(old)
                 : "r"(t.rt_s + Rt::kActive),
                   "r"((n << Rt::kRetiredShift) - n)
                 : "memory");
    const uint32_t before = (old >> Rt::kRetiredShift) & Rt::kActiveMask;
    const uint32_t retired = before + n;
    if (t.events) {
      int64_t ev = t.log_reserve(n);
      for (uint32_t k = 0; k < n; ++k)
        t.log_at(ev + k, OMPDS_EV_RETIRE, -1, int64_t(w) - int64_t(before + k + 1), 0);
    }
    if (retired == w) // this warp retired the region's last participant
      retire_last(t);
  }
  // no __syncwarp: the join barrier that follows orders the leader's
  // shared-memory updates for every participant
}
// end_parallel_warp for a region whose list is the window and whose team
// keeps no event log (the lean instantiation: the launcher guarantees both).
__device__ __forceinline__ void end_parallel_window(const TeamCtx &t, uint32_t plan) {
  const bool leader = plan & 1u;
  const uint32_t n = plan >> 8;
  if (plan & 2u) {
    __syncwarp(); // every lane's fetch reads before the leader's reset
    retire_window_if(t, leader);
  } else {
    red_add_if(t.rt_s + Rt::kActive, (n << Rt::kRetiredShift) - n, leader);
  }
}
// Master warp, after the join barrier of a region staged with no event log
// (completes_at_join): every one of the W workers fetched it and arrived at
// the join after its body, and the join barrier orders all of their reads of
// the staged region before this point.  The master completes the region --
// the team returns to Idle (complete_region; a heap list is freed first,
// retire_last) -- without re-reading any count.  Logged regions are
// completed by their last retiring worker, in the reference's event order.
__device__ __forceinline__ bool completes_at_join(const TeamCtx &t, int32_t workers) {
  return (kLeanJoinCompletes || workers > kWarp) && t.events == nullptr;
}
__device__ __forceinline__ void complete_region(const TeamCtx &t, bool leader) {
  retire_window_if(t, leader);
  __syncwarp(); // every lane sees the reset in its next prepare checks
}

__device__ __forceinline__ void end_parallel_warp(const TeamCtx &t,
                                                  const WarpMask &m,
                                                  const Fetch &f) {
  end_parallel_warp(t, retire_plan(t, m, f));
}
__device__ __forceinline__ void end_parallel_warp(const TeamCtx &t, bool mine,
                                                  const Fetch &f) {
  end_parallel_warp(t, WarpMask::of(t, mine, t.at<int32_t>(Rt::kWorkers)), f);
}

//===----------------------------------------------------------------------===//
// get-shared-variables with a warp-shuffle broadcast.  Lane j < nargs loads
// entry j of the list (one coalesced 8-byte-per-lane load, from shared memory
// or the global overflow block); capture j is then a register shuffle away.
//===----------------------------------------------------------------------===//

struct SharedVars {
  void *mine;   // this lane's entry (lane j holds entry j)
  void **list;  // the list itself: entries past the first 32 are read here
  // Entry j of the list.  j < 32: a register shuffle (every lane of the warp
  // must call it, with the same j); j >= 32: a load from the list (shared
  // window or global block), since a shuffle source lane wraps modulo 32.
  __device__ __forceinline__ void *get(int j) const {
    if (j >= kWarp)
      return list[j];
    return reinterpret_cast<void *>(__shfl_sync(
        0xffffffffu, reinterpret_cast<unsigned long long>(mine), j));
  }
};

__device__ __forceinline__ SharedVars get_shared_variables(void **args,
                                                           int32_t nargs) {
  SharedVars v;
  const uint32_t lane = lane_id();
  v.mine = nullptr;
  v.list = args;
  if (args != nullptr && static_cast<int32_t>(lane) < nargs) {
    if (__isShared(args)) { // the preallocated window: a plain LDS
      const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(args));
      unsigned long long p;
      asm volatile("ld.shared.u64 %0, [%1];" : "=l"(p) : "r"(sa + 8u * lane));
      v.mine = reinterpret_cast<void *>(p);
    } else { // a global overflow block
      v.mine = args[lane];
    }
  }
  return v;
}

// get-shared-variables for a fetched region: the window entry was already
// loaded by begin_parallel_warp; a global list is read here.
__device__ __forceinline__ SharedVars get_shared_variables(const TeamCtx &t,
                                                           const Fetch &f) {
#if OMPDS_PREFETCH_WINDOW
  // the list is the window (placement law; a fetched region's list is never
  // null -- terminated or trapped fetches never reach get-shared-variables)
  if (f.nargs <= t.prealloc) {
    SharedVars v;
    v.mine = static_cast<int32_t>(lane_id()) < f.nargs ? f.win : nullptr;
    v.list = t.window;
    return v;
  }
#endif
  return get_shared_variables(f.args, f.nargs);
}

// Loads capture j's value through its pointer: lane j dereferences, then a
// shuffle broadcasts the value (T is 4 or 8 bytes).  A weak load suffices:
// the master's stores precede the release barrier, and bar.sync orders
// shared and global memory among the CTA's participating threads.
template <class T>
__device__ __forceinline__ T shared_value(const SharedVars &v, int j) {
  T x{};
  if (static_cast<int>(lane_id()) == j && v.mine)
    x = *static_cast<const T *>(v.mine);
  return __shfl_sync(0xffffffffu, x, j);
}

//===----------------------------------------------------------------------===//
// Data-sharing stack: one per warp, owned and managed in registers by that
// warp.  A statically sized slot in shared memory holds frames while they
// fit; once a push does not fit, frames continue on the warp's global-memory
// overflow chain until popped back (strict LIFO).  The master (1 lane)
// pushes DataSize; a worker warp pushes one DataSize frame per lane.
//===----------------------------------------------------------------------===//

struct Frame {
  unsigned char *base; // lane 0's frame (lane l: base + l*bytes_per_lane)
  int32_t offset;      // offset inside its segment, -1: none
  int32_t in_smem;     // 1: shared-memory slot, 0: global overflow chain
  int32_t status;
};

// Offsets and sizes are 32-bit (a slot is at most 227 KB, a chain slice is
// sized by the launcher): the push/pop bookkeeping is a handful of 32-bit
// register operations, no 64-bit arithmetic on the region's critical path.
struct DsStack {
  unsigned char *slot; // shared-memory slot (generic address)
  unsigned char *ovf;  // global overflow chain for this warp
  uint32_t slot_cap;
  uint32_t top;        // bytes used in the slot
  uint32_t ovf_cap;
  uint32_t ovf_top;    // bytes used on the chain
  int32_t depth;
  int32_t max_depth;
  uint32_t high_water; // max bytes in use (slot + chain)

  __device__ __forceinline__ void init(unsigned char *s, int64_t cap,
                                       unsigned char *o, int64_t ocap) {
    slot = s;
    slot_cap = static_cast<uint32_t>(cap < 0 ? 0 : cap > 0x7fffffff ? 0x7fffffff : cap);
    top = 0;
    ovf = o;
    ovf_cap = static_cast<uint32_t>(ocap < 0 ? 0 : ocap > 0x7fffffff ? 0x7fffffff : ocap);
    ovf_top = 0;
    depth = 0;
    max_depth = 0;
    high_water = 0;
  }

  // Frame bytes (rounded to 8), or 0xffffffff when the frame cannot fit
  // anywhere (over 2 GB, or negative).  Frame sizes are loop-invariant in
  // region code, so this is hoisted out of region loops.
  __device__ __forceinline__ static uint32_t frame_need(int64_t bytes_per_lane, int lanes) {
    const int64_t want = bytes_per_lane * lanes;
    return want < 0 || want > 0x7ffffff0 ? 0xffffffffu
                                         : (static_cast<uint32_t>(want) + 7u) & ~7u;
  }

  // __kmpc_data_sharing_push_stack(bytes_per_lane * lanes).  Branch-free:
  // the placement decision (slot while the chain is empty and the frame
  // fits, else the chain) and the bookkeeping are selects on 32-bit
  // registers, so the dependent chain from one push to the next is a few
  // integer instructions (profiles/: ompds_probe_overheads, bookkeeping mode).
  __device__ __forceinline__ Frame push(int64_t bytes_per_lane, int lanes) {
    return push_bytes(frame_need(bytes_per_lane, lanes));
  }
  __device__ __forceinline__ Frame push_bytes(uint32_t need) {
    const bool in_slot = (ovf_top == 0u) & (need <= slot_cap - top);
    const bool in_ovf = !in_slot & (ovf != nullptr) & (need <= ovf_cap - ovf_top);
    const bool ok = in_slot | in_ovf;
    const uint32_t off = in_slot ? top : ovf_top;
    Frame f;
    f.base = ok ? (in_slot ? slot : ovf) + off : nullptr;
    f.offset = ok ? static_cast<int32_t>(off) : -1;
    f.in_smem = in_slot;
    f.status = ok ? OMPDS_OK : OMPDS_TRAP_STACK_OVERFLOW;
    top += in_slot ? need : 0u;
    ovf_top += in_ovf ? need : 0u;
    depth += ok;
    max_depth = max(max_depth, depth);
    high_water = max(high_water, top + ovf_top);
    return f;
  }

  // __kmpc_data_sharing_pop_stack(frame): strict LIFO -- the frame must be
  // the top of its segment (and a slot frame can only be popped once the
  // chain is empty).  Branch-free like push.
  __device__ __forceinline__ int32_t pop(const Frame &f) {
    const uint32_t off = static_cast<uint32_t>(f.offset);
    const bool bad = (depth <= 0) | (f.offset < 0) |
                     (f.in_smem ? (ovf_top != 0u) | (off > top) : off > ovf_top);
    top = !bad && f.in_smem ? off : top;
    ovf_top = !bad && !f.in_smem ? off : ovf_top;
    depth -= !bad;
    return bad ? OMPDS_TRAP_STACK_UNDERFLOW : OMPDS_OK;
  }
};

//===----------------------------------------------------------------------===//
// Reference / LLVM-runtime entry-point names.  Like omplab::TeamRuntime
// (DeviceRuntime.h:81-119; one instance per team, calls serialised by the
// simulator, not thread-safe) these are single-caller: one thread of the team at a time, e.g. a code
// generator's master thread, or the protocol replay kernel.  Concurrent
// workers use the warp-level paths behind Master / Worker in
// ompds_generic.cuh (fetch_is_fast / fetch_account_fast / end_parallel_warp),
// which keep the same state, statistics and event log.
//===----------------------------------------------------------------------===//

__device__ __forceinline__ int32_t __kmpc_kernel_init(const TeamCtx &t,
                                                      int32_t workers) {
  return kernel_init(t, kMaster, workers);
}
__device__ __forceinline__ int32_t
__kmpc_kernel_prepare_parallel(const TeamCtx &t, int32_t fn, int64_t nargs,
                               void ***args) {
  return prepare_parallel(t, kMaster, fn, nargs, args);
}
__device__ __forceinline__ int32_t __kmpc_kernel_parallel(const TeamCtx &t,
                                                          int32_t *fn,
                                                          void ***args,
                                                          bool *p) {
  return kernel_parallel(t, kWorker, fn, args, p);
}
__device__ __forceinline__ int32_t __kmpc_kernel_end_parallel(const TeamCtx &t) {
  return end_parallel(t, kWorker);
}
__device__ __forceinline__ int32_t __kmpc_kernel_deinit(const TeamCtx &t) {
  return kernel_deinit(t, kMaster);
}
__device__ __forceinline__ SharedVars __kmpc_get_shared_variables(void **args,
                                                                  int32_t n) {
  return get_shared_variables(args, n);
}
__device__ __forceinline__ Frame
__kmpc_data_sharing_push_stack(DsStack &s, int64_t bytes, int lanes) {
  return s.push(bytes, lanes);
}
__device__ __forceinline__ int32_t __kmpc_data_sharing_pop_stack(DsStack &s,
                                                                 const Frame &f) {
  return s.pop(f);
}

} // namespace ompds
