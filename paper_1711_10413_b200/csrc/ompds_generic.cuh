// ompds_generic.cuh -- the generic-mode team kernel of the device runtime:
// master / worker state machine (proj/src/Codegen.cpp:316-513), the team
// region layout (proj/src/Simulator.cpp:281-292) and the host launch helper.
//
// A region program is a struct with
//   struct Args { ... };                              // kernel arguments
//   __device__ static void master(Master &, const Args &);   // sequential code
//   __device__ static void region(int32_t fn, const SharedVars &, Worker &,
//                                 const Args &);      // outlined region body
// master() runs on the reserved warp (lane 0 commits side effects) and calls
// Master::parallel / parallel_with for every parallel region; region() runs
// on every worker warp.  generic_mode_kernel<Prog> instantiates the team;
// launch_generic<Prog> launches it (csrc/ompds_kernels.cu holds the
// reference configs' programs; INTEGRATION.md shows a user-defined one).
#pragma once

#include "ompds_device.cuh"

#include <cuda_runtime.h>

#include <algorithm>
#include <map>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <type_traits>
#include <vector>

namespace ompds {

inline thread_local char g_last_error[512] = "";

inline int32_t cuda_fail(cudaError_t e, const char *what) {
  std::snprintf(g_last_error, sizeof(g_last_error), "%s: %s", what,
                cudaGetErrorString(e));
  return OMPDS_ERR_CUDA;
}
#define OMPDS_CUDA(call)                                                       \
  do {                                                                         \
    cudaError_t e_ = (call);                                                   \
    if (e_ != cudaSuccess)                                                     \
      return cuda_fail(e_, #call);                                             \
  } while (0)

//===----------------------------------------------------------------------===//
// Launch parameters shared by every generic-mode kernel.
//===----------------------------------------------------------------------===//

#ifndef OMPDS_GENERIC_LB_THREADS
#define OMPDS_GENERIC_LB_THREADS 1024 // any team up to 1024 threads ...
#endif
#ifndef OMPDS_GENERIC_LB_MIN
#define OMPDS_GENERIC_LB_MIN 1 // ... so at most 64 registers
#endif
// A program may opt into a second lean instantiation for the smallest teams
// (W <= 32: one worker warp + the master warp) with `static constexpr bool
// kSmallTeams = true;` -- bounded to 64 threads and 32 teams per SM, so
// ptxas fits it in 32 registers (config 1: no spills, 32 instead of 24
// teams per SM fit, +7 % regions/s).
// A program may ask the worker loop to load list entries 0..3 into every
// lane together with the team state (`static constexpr bool
// kPreloadEntries = true;`): its region then dereferences the captures it
// needs directly (broadcast loads), with no shuffle step on the chain.
template <class P, class = void> struct PreloadEntries : std::false_type {};
template <class P>
struct PreloadEntries<P, std::void_t<decltype(P::kPreloadEntries)>>
    : std::integral_constant<bool, P::kPreloadEntries> {};

template <class P, class = void> struct SmallTeams : std::false_type {};
template <class P>
struct SmallTeams<P, std::void_t<decltype(P::kSmallTeams)>>
    : std::integral_constant<bool, P::kSmallTeams> {};
constexpr int kSmallTeamThreads = 64;
constexpr int kSmallTeamsPerSM = 32;

constexpr int kMaxCaptures = 32;

// (kLeanJoinCompletes, ompds_device.cuh: without an event log the master
// completes every region at the join; the lean instantiation also keeps the
// phase in a register and defers the completion store.)

// kPreloadEntries: the list entries are loaded with ld.volatile so ptxas
// issues them with the team-state load, ahead of the phase test (plain loads
// are sunk past it, onto the chain).  0: plain loads.
#ifndef OMPDS_EARLY_ENTRIES
#define OMPDS_EARLY_ENTRIES 1
#endif
#if OMPDS_EARLY_ENTRIES
#define OMPDS_ENTRY_LD "ld.volatile.shared"
#else
#define OMPDS_ENTRY_LD "ld.shared"
#endif

// Region timeline (tools/timeline.cu only): clock64 stamps of the master's
// and worker warp 0's steps for the first OMPDS_TIMELINE regions of team 0.
#ifdef OMPDS_TIMELINE
__device__ long long g_timeline[OMPDS_TIMELINE][16];
__device__ __forceinline__ long long tl_clock() {
  long long c; // volatile + memory clobber: stays between the barriers
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c)::"memory");
  return c;
}
#define OMPDS_TL(r, k)                                                         \
  do {                                                                         \
    const long long c_ = tl_clock();                                           \
    if (blockIdx.x == 0 && (threadIdx.x & 31) == 0 && (r) < OMPDS_TIMELINE)    \
      g_timeline[(r)][(k)] = c_;                                               \
  } while (0)
#else
#define OMPDS_TL(r, k)                                                         \
  do {                                                                         \
  } while (0)
#endif

// Per-team %globaltimer stamps (tools/team_times.cu only): [0] kernel entry,
// [1] master before its first region, [2] before the first release, [3]
// after the first join, [4] at the end of the master, [5] after the
// prologue's zeroing barrier, [6] after kernel_init, for every team.
#ifdef OMPDS_TEAM_TIMES
__device__ long long g_team_times[OMPDS_TEAM_TIMES][8];
#define OMPDS_TT(k)                                                            \
  do {                                                                         \
    long long g_;                                                              \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_)::"memory");          \
    if ((threadIdx.x & 31) == 0 && blockIdx.x < OMPDS_TEAM_TIMES)              \
      g_team_times[blockIdx.x][(k)] = g_; /* a store only: no load latency */  \
  } while (0)
#else
#define OMPDS_TT(k)                                                            \
  do {                                                                         \
  } while (0)
#endif

struct TeamParams {
  int32_t workers;       // W
  int32_t prealloc;      // PreallocEntries
  int32_t fail_dyn;
  int32_t max_events;
  int64_t depot_cap;     // master data-sharing slot in smem (bytes, 8-aligned)
  int64_t total_shared;  // the layout's depot size (frame pushed by master)
  unsigned char *slabs;  // teams * slab_bytes of global memory
  uint32_t slab_bytes;
  int32_t n_caps;
  ompds_event *events;   // teams * max_events, or nullptr
  ompds_team_stats *stats;
  int64_t cap_off[kMaxCaptures]; // depot offsets of the captures (layout)
  int64_t aux_off;       // depot offset of the sequential loop counter (-1)
  int64_t warp_slot_bytes;       // per-warp data-sharing slot in smem
  unsigned char *warp_ovf;       // teams * worker_warps * warp_ovf_bytes
  int64_t warp_ovf_bytes;
  int32_t list_malloc;           // OMPDS_LIST_MALLOC
  int32_t first_team;            // omp_get_team_num() of CTA 0
  int32_t total_teams;           // omp_get_num_teams()
  int32_t *bar_arrivals;         // teams x (W+32) per-thread barrier arrivals, or null
};

// Depot accessors for the master's sequential code (see Master::with_depot).
struct SmemDepot {
  uint32_t base;        // shared-window address of the depot frame
  unsigned char *gbase; // the same frame as a generic pointer
  __device__ __forceinline__ void *ptr(int64_t off) const { return gbase + off; }
  template <class T> __device__ __forceinline__ T ld(int64_t off) const {
    static_assert(sizeof(T) == 4 || sizeof(T) == 8, "4/8-byte slots");
    if constexpr (sizeof(T) == 4) {
      uint32_t v;
      asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(base + uint32_t(off)) : "memory");
      return __builtin_bit_cast(T, v);
    } else {
      unsigned long long v;
      asm volatile("ld.shared.b64 %0, [%1];" : "=l"(v) : "r"(base + uint32_t(off)) : "memory");
      return __builtin_bit_cast(T, v);
    }
  }
  template <class T> __device__ __forceinline__ void st(int64_t off, T x) const {
    if constexpr (sizeof(T) == 4)
      asm volatile("st.shared.b32 [%0], %1;" ::"r"(base + uint32_t(off)),
                   "r"(__builtin_bit_cast(uint32_t, x)) : "memory");
    else
      asm volatile("st.shared.b64 [%0], %1;" ::"r"(base + uint32_t(off)),
                   "l"(__builtin_bit_cast(unsigned long long, x)) : "memory");
  }
};
struct GlobalDepot {
  unsigned char *gbase;
  __device__ __forceinline__ void *ptr(int64_t off) const { return gbase + off; }
  template <class T> __device__ __forceinline__ T ld(int64_t off) const {
    return *reinterpret_cast<const volatile T *>(gbase + off);
  }
  template <class T> __device__ __forceinline__ void st(int64_t off, T x) const {
    *reinterpret_cast<volatile T *>(gbase + off) = x;
  }
};

// Master-warp view of the sequential region.  Every lane runs it; lane 0
// (the master) commits side effects.
struct Master {
  TeamCtx t;
  const TeamParams *p;
  bool leader;
  bool lean;           // the launch's lean instantiation (a compile-time constant
                       // after inlining): no event log, every list fits the
                       // window -- the general prepare path is compiled out
  bool join_completes; // the master completes the region at the join:
                       // completes_at_join() -- every launch without an event
                       // log (kLeanJoinCompletes; else only several worker
                       // warps without one), so every lean launch
  int32_t fast_nargs;  // the fast prepare applies to nargs <= this: the
                       // window size without an event log, -1 with one
  uint32_t team_threads;
  int32_t trap = 0;
  int32_t barriers = 0;  // protocol barriers of the master (2 per region)
  int32_t regions = 0;
  DsStack ds;
  Frame depot;

  __device__ __forceinline__ int32_t sync_status(int32_t s) {
    s = __shfl_sync(0xffffffffu, s, 0);
    if (s && !trap) {
      trap = s;
      if (leader)
        t.trap(s);
    }
    return s;
  }

  __device__ __forceinline__ int32_t init() {
    int32_t s = 0;
    if (leader) {
      t.set_work_fn(-1); // the zeroed region's state word: no work function
      s = kernel_init(t, kMaster, p->workers);
    }
    __syncwarp(); // the master's init writes before any lane reads the state
    s = sync_status(s);
    OMPDS_TT(6);
    return s;
  }

  // The kernel frame group's depot is the first frame of the master's
  // data-sharing stack: the shared-memory slot when it fits, else the
  // team's global overflow chain (placement decision of config 2).
  __device__ __forceinline__ int32_t push_depot() {
    unsigned char *ovf = t.slab ? t.slab + (t.slab_bytes / 2) : nullptr;
    ds.init(t.region, p->depot_cap, ovf, t.slab_bytes / 2);
    depot = ds.push(p->total_shared, 1);
    if (depot.status == OMPDS_OK && !depot.in_smem) {
      // zero-fill like pushActivation (Simulator.cpp:453-456); smem was
      // zeroed in the prologue.
      for (int64_t i = lane_id() * 8; i < p->total_shared; i += 32 * 8)
        *reinterpret_cast<uint64_t *>(depot.base + i) = 0;
      __syncwarp();
    }
    return sync_status(depot.status);
  }

  __device__ __forceinline__ unsigned char *cap(int j) const {
    return depot.base + p->cap_off[j];
  }

  // Runs the sequential code `f(depot)` with a depot accessor that issues
  // shared-memory instructions (LDS/STS, 32-bit addresses) when the depot
  // frame is in the smem slot, generic ones when it is on the global chain.
  template <class F> __device__ __forceinline__ void with_depot(F &&f) {
    if (depot.in_smem)
      f(SmemDepot{static_cast<uint32_t>(__cvta_generic_to_shared(depot.base)),
                  depot.base});
    else
      f(GlobalDepot{depot.base});
  }

  // prepare_parallel + publish &capture_j into the list + release + join.
  // The captures are the layout's first kMaxCaptures depot slots
  // (TeamParams::cap_off); a region with more captures publishes its own
  // addresses through parallel_with.
  __device__ __forceinline__ int32_t parallel(int32_t fn, int32_t nargs) {
    if (nargs > kMaxCaptures)
      return sync_status(OMPDS_ERR_INVALID);
    return parallel_with(fn, nargs, [this](int j) -> void * { return cap(j); });
  }

  template <class AddrOf>
  __device__ __forceinline__ int32_t parallel_with(int32_t fn, int32_t nargs,
                                                   AddrOf addr_of) {
    OMPDS_TL(regions, 0);
    // The common case of prepare_parallel in one branch: every check passes,
    // the list fits the window and no event log is kept.  Everything else
    // (traps, a global list, events) takes parallel_general.
    // Idle implies Active == 0.  Lean: the team is Idle at every prepare
    // (the master is the phase's only writer and a region is complete at
    // its join; the word itself still shows the last region staged, see
    // below), so the phase is not read back.
    const bool lean_join = lean && kLeanJoinCompletes;
    const uint32_t phase = lean_join ? uint32_t(kIdle) : load_phase(t);
    if (__builtin_expect(phase == uint32_t(kIdle) && nargs >= 0 && nargs <= fast_nargs, 1)) {
      if (!lean_join)
        __syncwarp(); // every lane has read the state before the master stages
      OMPDS_TL(regions, 1);
      if (lean_join)
        stage_state_if(t, fn, nargs, leader); // lean: the list is the window
      else
        stage_region_if(t, fn, nargs, t.window, leader);
      const uint32_t sa = t.window_s;
      const int lane = static_cast<int>(lane_id());
      if (lane < nargs) // one predicated STS per lane for lists up to 32 entries
        asm volatile("st.shared.u64 [%0], %1;" ::"r"(sa + 8u * lane),
                     "l"(reinterpret_cast<unsigned long long>(addr_of(lane)))
                     : "memory");
      if (__builtin_expect(nargs > 32, 0)) // windows of more than 32 entries
        for (int j = lane + 32; j < nargs; j += 32)
          asm volatile("st.shared.u64 [%0], %1;" ::"r"(sa + 8u * j),
                       "l"(reinterpret_cast<unsigned long long>(addr_of(j)))
                       : "memory");
      OMPDS_TL(regions, 2);
      OMPDS_TT(2);
      bar_sync(kBarHandoff, team_threads); // release the workers
      OMPDS_TL(regions, 3);
      bar_sync(kBarHandoff, team_threads); // join
      OMPDS_TL(regions, 4);
      OMPDS_TT(3);
      // Lean: the region is complete at the join; the state word keeps the
      // staged fields until the next prepare overwrites them (no thread
      // reads it in between: workers read it only after a release, the
      // master only in kernel_deinit, which finish() precedes with the Idle
      // store).
      if (!lean_join && join_completes)
        complete_region(t, leader);
      barriers += 2;
      regions += 1;
      return OMPDS_OK;
    }
    if (lean) {
      if (lean_join) // Idle (see above): the word may still show the last region
        return parallel_refused(prepare_check(kIdle, 0, nargs));
      const PrepareState st = load_prepare_state(t);
      return parallel_refused(prepare_check(st.phase, st.active, nargs));
    }
    return parallel_general(fn, nargs, addr_of);
  }

  // Lean instantiation, a prepare the fast path does not cover: only a
  // protocol violation gets here (the launcher chose lean because no region
  // needs more than the window and nothing is logged).  The trap is recorded
  // and the handoff still runs, so the workers see an unstaged region.
  // (Inlined: a call would take the Master's address and move the whole
  // object to local memory for every region.)
  __device__ __forceinline__ int32_t parallel_refused(int32_t s) {
    if (s == OMPDS_OK)
      s = OMPDS_ERR_INVALID;
    sync_status(s);
    if (kLeanJoinCompletes)
      retire_window_if(t, leader); // the workers must not see the last region staged
    bar_sync(kBarHandoff, team_threads); // release the workers
    bar_sync(kBarHandoff, team_threads); // join
    barriers += 2;
    return trap;
  }

  template <class AddrOf>
  __device__ OMPDS_GENERAL_INLINE int32_t parallel_general(int32_t fn, int32_t nargs,
                                                   AddrOf addr_of) {
    void **list = nullptr;
    unsigned long long packed = 0;
    // Every lane evaluates prepare_parallel's phase checks on broadcast
    // loads, so the window case needs no shuffle from the master lane; only
    // a global list (nargs > PreallocEntries) is allocated by the master and
    // shuffled.  The __syncwarp orders every lane's reads before the
    // master's staging writes.
    {
      const PrepareState st = load_prepare_state(t);
      int32_t s = prepare_check(st.phase, st.active, nargs);
      list = t.window;
      if (s == OMPDS_OK && nargs > t.prealloc) {
        if (leader) {
          list = alloc_args_list(t, fn, nargs);
          packed = list ? reinterpret_cast<unsigned long long>(list)
                        : (static_cast<unsigned long long>(OMPDS_TRAP_ARGS_ALLOC_FAILED) |
                           (1ull << 63));
        }
        packed = __shfl_sync(0xffffffffu, packed, 0);
        if (packed >> 63)
          s = static_cast<int32_t>(packed & 0xffffffffu);
        list = reinterpret_cast<void **>(packed);
      } else if (s == OMPDS_OK && leader && t.events) {
        alloc_args_list(t, fn, nargs); // the window: logs PreparePrealloc
      }
      __syncwarp();
      OMPDS_TL(regions, 1);
      stage_region_if(t, fn, static_cast<int32_t>(nargs), list, leader && s == OMPDS_OK);
      if (__builtin_expect(s != OMPDS_OK, 0) && leader)
        t.trap(s); // the team's first trap, before any worker can record one
      packed = s ? (static_cast<unsigned long long>(s) | (1ull << 63))
                 : reinterpret_cast<unsigned long long>(list);
    }
    const bool ok = (packed >> 63) == 0;
    list = reinterpret_cast<void **>(packed);
    // The reserved warp publishes the pointer list lane-parallel (one
    // coalesced store per 32 entries) instead of nargs scalar stores.
    const int lane = static_cast<int>(lane_id());
    if (list == t.window) { // the smem window: STS, not generic stores
      const uint32_t sa = t.window_s;
      for (int j = lane; ok && j < nargs; j += 32)
        asm volatile("st.shared.u64 [%0], %1;" ::"r"(sa + 8u * j),
                     "l"(reinterpret_cast<unsigned long long>(addr_of(j)))
                     : "memory");
    } else {
      if (ok && lane < nargs)
        list[lane] = addr_of(lane);
      for (int j = lane + 32; ok && j < nargs; j += 32) // lists longer than a warp
        list[j] = addr_of(j);
    }
    // Released even when prepare trapped (keeps the handoff branch-free):
    // nothing is staged then, workers observe a non-Staged phase and skip.
    OMPDS_TL(regions, 2);
    bar_sync(kBarHandoff, team_threads); // release the workers
    OMPDS_TL(regions, 3);
    bar_sync(kBarHandoff, team_threads); // join
    OMPDS_TL(regions, 4);
    barriers += 2;
    if (ok && join_completes) {
      if (list == t.window) {
        complete_region(t, leader);
      } else { // the last retirement's work: free the heap list, Idle
        if (leader)
          retire_last(t);
        __syncwarp();
      }
    }
    if (__builtin_expect(!ok, 0)) {
      if (!trap)
        trap = static_cast<int32_t>(packed & 0xffffffffu);
      return trap;
    }
    regions += 1;
    return OMPDS_OK;
  }

  __device__ __forceinline__ void finish() {
    int32_t s = 0;
    if (lean && kLeanJoinCompletes && regions > 0)
      retire_window_if(t, leader); // the last region's completion (see parallel_with)
    if (leader)
      s = kernel_deinit(t, kMaster);
    sync_status(s);
    // SimStats::BarrierEntries for the reserved warp: the master (logical tid
    // W, lane 0) and the idle lanes (W+1.., lanes 1..31) each made this
    // lane's handoff arrivals -- the protocol's `barriers` plus the
    // termination release -- and no other barrier (they never reach a
    // region's `omp barrier`, id 2).
    if (p->bar_arrivals)
      p->bar_arrivals[size_t(blockIdx.x) * (p->workers + kWarp) + p->workers + lane_id()] =
          barriers + 1;
    if (leader && p->stats) {
      ompds_team_stats st{};
      st.trap = trap ? trap : t.at<int32_t>(Rt::kTrap);
      st.master_barriers = barriers;
      st.barrier_releases = barriers + 1;
      st.regions = regions;
      st.dynamic_alloc_bytes = t.at<uint32_t>(Rt::kDynBytes);
      st.dynamic_allocs = static_cast<int32_t>(t.at<uint32_t>(Rt::kDynAllocs));
      st.dynamic_frees = static_cast<int32_t>(t.at<uint32_t>(Rt::kDynFrees));
      st.depot_in_smem = depot.in_smem;
      st.depot_offset = depot.offset;
      st.n_events = static_cast<int32_t>(t.at<uint32_t>(Rt::kEvents));
      st.smem_bytes = team_region_bytes(p->depot_cap, p->prealloc);
      if (p->warp_slot_bytes > 0)
        st.smem_bytes = round_up(st.smem_bytes, 16) +
                        int64_t(team_threads / 32 - 1) * p->warp_slot_bytes;
      p->stats[blockIdx.x] = st;
    }
    __syncwarp();
    // Termination release: workers parked at await.work observe Terminated
    // (the null work function) and leave their loop.
    bar_sync(kBarHandoff, team_threads);
  }
};

// Worker-side context handed to region bodies.
struct Worker {
  int32_t wid;  // omp_get_thread_num
  bool mine;    // wid < W (padding lanes of the last worker warp idle)
  int32_t team;  // omp_get_team_num (first_team + CTA index)
  int32_t teams; // omp_get_num_teams (the whole grid, across shards)
  int32_t local_team;  // CTA index in this launch
  int32_t local_teams; // CTAs in this launch
  int32_t workers;
  int32_t warp;
  DsStack ds;   // this warp's data-sharing stack (nested regions)
  const TeamCtx *t;
  void **args;  // the fetched shared-args list
  int32_t nargs;
  int32_t region_index; // regions this warp ran before the current one
  uint32_t worker_threads; // 32 x worker warps (padding lanes included)
  // Entries 0..3 of the list, loaded by every lane together with the team
  // state when the program asks for them (kPreloadEntries) and the list is
  // the window (the lean instantiation); pre_ok says they are valid.
  void *pre[4];
  bool pre_ok = false;

  // `#pragma omp barrier` inside the region: every worker of the team (the
  // master warp is parked at the join and does not take part); all lanes of
  // every worker warp must arrive, padding lanes included.
  int32_t *arrivals;        // this lane's barrier arrival counter (or null)
  __device__ __forceinline__ void barrier() const {
    bar_sync(kBarRegion, worker_threads);
    if (arrivals)
      ++*arrivals;
  }

  // The warp's data-sharing stack for region code (__kmpc_data_sharing_
  // push_stack / _pop_stack, Simulator.cpp:439-479's activation frames):
  // one frame of `bytes_per_lane` bytes for each of the warp's 32 lanes,
  // lane l's part at f.base + l * bytes_per_lane -- in the warp's
  // shared-memory slot while it fits, else on its global overflow chain.
  // Warp-collective (every lane calls it, in the same order).
  __device__ __forceinline__ Frame push_frame(int64_t bytes_per_lane) {
    return ds.push(bytes_per_lane, kWarp);
  }
  __device__ __forceinline__ int32_t pop_frame(const Frame &f) { return ds.pop(f); }

  // A parallel region nested in this region's body (EXTENSION; the paper's
  // runtime-managed stack for nesting): serialized on each lane -- a team of
  // one, like the LLVM device runtime's __kmpc_serialized_parallel.  Each
  // lane's `nargs` capture addresses addr_of(j) are published in a list
  // frame on the warp's data-sharing stack (begin-sharing-variables; lane
  // l's list at base + 8*nargs*l), `body(NestedVars)` runs and reads them
  // back (get-shared-variables), then the list frame is popped.  The
  // encountering level's locals a nested region captures must themselves
  // live on the stack (push_frame) -- the globalization the frame pipeline
  // marks with the escape bit.  Warp-collective; returns 0 or
  // OMPDS_TRAP_STACK_OVERFLOW / _UNDERFLOW.
  struct NestedVars {
    void **list;
    int32_t nargs;
    __device__ __forceinline__ void *get(int j) const { return list[j]; }
  };
  template <class AddrOf, class Body>
  __device__ __forceinline__ int32_t parallel_serialized(int32_t nargs, AddrOf addr_of,
                                                         Body body) {
    Frame f{};
    f.offset = -1;
    void **list = nullptr;
    if (nargs > 0) {
      f = ds.push(int64_t(nargs) * 8, kWarp);
      if (f.status != OMPDS_OK)
        return f.status;
      list = reinterpret_cast<void **>(f.base) + size_t(lane_id()) * nargs;
      for (int32_t j = 0; j < nargs; ++j)
        list[j] = addr_of(j);
    }
    body(NestedVars{list, nargs});
    return nargs > 0 ? ds.pop(f) : OMPDS_OK;
  }
};

// kLean: the instantiation for launches with no event log, no allocation
// hook and no list past the window (decided on the host per launch): the
// general fetch / prepare / retire paths and the event-log bookkeeping are
// compiled out, which shortens the region's dependent chain and frees
// registers (more teams per SM).  Results and statistics are identical.
template <class Prog, bool kLean, bool kSmall = false>
__global__ void __launch_bounds__(kSmall ? kSmallTeamThreads : OMPDS_GENERIC_LB_THREADS,
                                  kSmall ? kSmallTeamsPerSM : OMPDS_GENERIC_LB_MIN)
    generic_mode_kernel(const __grid_constant__ TeamParams p,
                        const __grid_constant__ typename Prog::Args a) {
  extern __shared__ __align__(16) unsigned char smem[];
  if (threadIdx.x == 0)
    OMPDS_TT(0);
#ifndef OMPDS_WARM_PARAMS
#define OMPDS_WARM_PARAMS 1
#endif
#if OMPDS_WARM_PARAMS
  {
    // Touch every 8-byte word of the launch parameters at once, one per
    // thread: the SM's constant cache misses on them in parallel here
    // instead of one line at a time as the prologue, kernel_init and the
    // master's first prepare reach them.
    constexpr uint32_t kP = sizeof(TeamParams) / 8, kA = sizeof(typename Prog::Args) / 8;
    const uint32_t i = threadIdx.x;
    if (i < kP + kA) {
      const unsigned long long v =
          i < kP ? reinterpret_cast<const unsigned long long *>(&p)[i]
                 : reinterpret_cast<const unsigned long long *>(&a)[i - kP];
      asm volatile("" ::"l"(v));
    }
  }
#endif
  const uint32_t team_threads = blockDim.x;
  const int warp = threadIdx.x >> 5;
  const int worker_warps = static_cast<int>(team_threads >> 5) - 1;

  TeamCtx t = make_team(
      smem, p.depot_cap, p.prealloc, kLean ? 0 : p.fail_dyn,
      p.slabs ? p.slabs + size_t(blockIdx.x) * p.slab_bytes : nullptr,
      p.slab_bytes,
      !kLean && p.events ? p.events + size_t(blockIdx.x) * p.max_events : nullptr,
      kLean ? 0 : p.max_events, kLean ? 0 : p.list_malloc);
  // Prologue: zero the team region (Simulator.cpp:286), runtime span last.
  const int64_t region = team_region_bytes(p.depot_cap, p.prealloc);
  for (int64_t i = threadIdx.x; i < region; i += team_threads)
    smem[i] = 0;
  __syncthreads(); // (work_fn = -1 is set by the master's init: the workers
                   // read the state only after its first release)
  if (threadIdx.x == team_threads - 32)
    OMPDS_TT(5);

  if (warp < worker_warps) {
    Worker w;
    w.wid = threadIdx.x;
    w.mine = w.wid < p.workers;
    w.team = p.first_team + static_cast<int32_t>(blockIdx.x);
    w.teams = p.total_teams;
    w.local_team = blockIdx.x;
    w.local_teams = gridDim.x;
    w.worker_threads = static_cast<uint32_t>(worker_warps) * 32u;
    w.workers = p.workers;
    w.warp = warp;
    w.t = &t;
    w.args = nullptr;
    w.nargs = 0;
    // Per-warp data-sharing stack: a statically sized slot after the team
    // region, then this warp's slice of the global overflow chain.
    unsigned char *slot = smem + round_up(region, 16) + int64_t(warp) * p.warp_slot_bytes;
    unsigned char *ovf =
        p.warp_ovf ? p.warp_ovf + (size_t(blockIdx.x) * worker_warps + warp) * p.warp_ovf_bytes
                   : nullptr;
    w.ds.init(slot, p.warp_slot_bytes, ovf, p.warp_ovf ? p.warp_ovf_bytes : 0);
    // loop-invariant participation (Workers = the launch's W, which the
    // master's kernel_init records)
    const WarpMask wm = WarpMask::of(t, w.mine, p.workers);
    // barrier arrivals of this lane (SimStats::BarrierEntries), counted only
    // by the general instantiation when the launch asks for them
    int32_t arrivals = 0;
    const bool count = !kLean && p.bar_arrivals != nullptr;
    w.arrivals = count ? &arrivals : nullptr;
    // The worker loop, instantiated twice for programs that preload list
    // entries: with 16-byte loads of a 16-byte aligned window, or 8-byte
    // ones (a loop-invariant choice, made once, not per region).
    auto run = [&](auto w16_tag) {
      [[maybe_unused]] constexpr bool kW16 = decltype(w16_tag)::value;
      for (int32_t rr = 0;; ++rr) {
        bar_sync(kBarHandoff, team_threads); // await.work
        arrivals += count;
        OMPDS_TL(rr, 5);
        const StagedState st = load_staged_state<!kLean>(t, wm.win_off);
        if constexpr (kLean && PreloadEntries<Prog>::value) {
          // volatile: issued with the state load, ahead of the phase test
          // (ptxas sinks plain loads past it, onto the chain); two 16-byte
          // loads when the window is 16-byte aligned (the depot size decides)
          unsigned long long e0, e1, e2, e3;
          if constexpr (kW16)
            asm volatile(OMPDS_ENTRY_LD ".v2.u64 {%0, %1}, [%4];\n\t"
                         OMPDS_ENTRY_LD ".v2.u64 {%2, %3}, [%4+16];"
                         : "=l"(e0), "=l"(e1), "=l"(e2), "=l"(e3)
                         : "r"(t.window_s)
                         : "memory");
          else
            asm volatile(OMPDS_ENTRY_LD ".u64 %0, [%4];\n\t" // 8-byte aligned
                         OMPDS_ENTRY_LD ".u64 %1, [%4+8];\n\t"
                         OMPDS_ENTRY_LD ".u64 %2, [%4+16];\n\t"
                         OMPDS_ENTRY_LD ".u64 %3, [%4+24];"
                         : "=l"(e0), "=l"(e1), "=l"(e2), "=l"(e3)
                         : "r"(t.window_s)
                         : "memory");
          w.pre[0] = reinterpret_cast<void *>(e0);
          w.pre[1] = reinterpret_cast<void *>(e1);
          w.pre[2] = reinterpret_cast<void *>(e2);
          w.pre[3] = reinterpret_cast<void *>(e3);
          w.pre_ok = true;
        }
        Fetch f;
        if (__builtin_expect(fetch_is_fast(st, wm), 1)) {
          if constexpr (!kLeanJoinCompletes)
            fetch_account_fast(t, st, wm); // a staged region, no event log
          f = fetch_from(st);
        } else if constexpr (kLean) {
          if (st.phase == kTerminated)
            break; // termination sentinel (wf == null)
          if (w.mine) // the master's prepare trapped: nothing is staged
            t.trap(OMPDS_TRAP_PARALLEL_NOT_STAGED);
          bar_sync(kBarHandoff, team_threads);
          continue;
        } else {
          f = fetch_general(t, st, wm, w.mine);
          if (f.fn < 0) {
            if (f.status == OMPDS_OK)
              break; // termination sentinel (wf == null)
            bar_sync(kBarHandoff, team_threads); // trapped fetch: skip the region
            arrivals += count;
            continue;
          }
        }
        OMPDS_TL(rr, 6);
        w.args = f.args;
        w.nargs = f.nargs;
        w.region_index = rr;
        const uint32_t plan = retire_plan(t, wm, f);
        SharedVars sv = get_shared_variables(t, f);
        OMPDS_TL(rr, 7);
        Prog::region(f.fn, sv, w, a);
        OMPDS_TL(rr, 8);
        if constexpr (kLean) {
          if constexpr (!kLeanJoinCompletes)
            end_parallel_window(t, plan); // every list is the window, no log
          // else: the master completes the region at the join
        } else if (!kLeanJoinCompletes || !(plan & 8u)) {
          end_parallel_warp(t, plan); // with an event log: the workers retire
        }
        OMPDS_TL(rr, 9);
        bar_sync(kBarHandoff, team_threads); // barrier.parallel (join)
        arrivals += count;
        OMPDS_TL(rr, 10);
      }
    };
    if constexpr (kLean && PreloadEntries<Prog>::value) {
      if ((t.window_s & 15u) == 0)
        run(std::true_type{});
      else
        run(std::false_type{});
    } else {
      run(std::false_type{});
    }
    if (count && w.mine) // worker threads of the reference's team (tid < W)
      p.bar_arrivals[size_t(blockIdx.x) * (p.workers + kWarp) + w.wid] = arrivals;
  } else {
    Master m;
    m.t = t;
    m.p = &p;
    m.leader = lane_id() == 0;
    m.lean = kLean;
    m.join_completes = (kLean && kLeanJoinCompletes) || completes_at_join(t, p.workers);
    m.fast_nargs = t.events == nullptr ? t.prealloc : -1;
    m.team_threads = team_threads;
    if (m.init() == OMPDS_OK && m.push_depot() == OMPDS_OK) {
      OMPDS_TT(1);
      Prog::master(m, a);
    }
    OMPDS_TT(4);
    m.finish();
  }
}

//===----------------------------------------------------------------------===//
// Host side: workspace, layouts for the fixed configs, launch helper.
//===----------------------------------------------------------------------===//

// Library-owned global memory reused across launches, one set per (device,
// stream): buffer 0 holds the teams' overflow slabs (args lists, master
// depot overflow), buffer 1 the worker warps' data-sharing overflow chains,
// buffer 2 a region program's tables, buffer 3 the masters' local depot
// mirrors, buffer 4 the work counters of dynamically scheduled loops (zeroed
// when allocated; each launch leaves them zero again).  Launches on one
// stream run in order, so they can share a set;
// launches on different streams (or devices) get their own.
// A buffer that a larger launch supersedes is retired, not freed: a CUDA
// graph captured from an earlier launch on the stream keeps pointing at it,
// so it stays allocated until ompds_release_workspace (which therefore
// invalidates graphs captured from launches on that stream).  Buffers grow by
// at least 1.5x, so a stream retires O(log size) of them.
struct WsBuffers {
  static constexpr int kBuffers = 5;
  unsigned char *buf[kBuffers] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  size_t bytes[kBuffers] = {0, 0, 0, 0, 0};
  std::vector<unsigned char *> retired;
  // the region-program tables last copied into buf[2] (ompds_run_program
  // skips the copy when a launch stages the same bytes again, so launches
  // of a staged program can be captured into a CUDA graph)
  std::vector<unsigned char> staged;
  unsigned char *staged_at = nullptr;
};
struct Workspace {
  std::mutex mu;
  std::map<std::pair<int, void *>, WsBuffers> sets;
};
inline Workspace g_ws;

constexpr int kWorkCounters = 4;
inline int32_t ensure_buffer(int which, size_t bytes, unsigned char **out,
                             void *stream = nullptr) {
  std::lock_guard<std::mutex> lk(g_ws.mu);
  int dev = 0;
  OMPDS_CUDA(cudaGetDevice(&dev));
  WsBuffers &w = g_ws.sets[{dev, stream}];
  if (w.bytes[which] < bytes) {
    const size_t grow = std::max(bytes, w.bytes[which] + w.bytes[which] / 2);
    unsigned char *fresh = nullptr;
    OMPDS_CUDA(cudaMalloc(&fresh, grow));
    if (which == kWorkCounters) // launches rely on finding them zero
      OMPDS_CUDA(cudaMemset(fresh, 0, grow));
    if (w.buf[which]) // earlier launches (or captured graphs) may still use it
      w.retired.push_back(w.buf[which]);
    w.buf[which] = fresh;
    w.bytes[which] = grow;
  }
  *out = w.buf[which];
  return OMPDS_OK;
}

// Whether `tables` are already the contents of `dev` (buffer 2 of the
// stream's set); records them as such when not (the caller copies).
inline bool tables_staged(void *stream, const std::vector<unsigned char> &tables,
                          unsigned char *dev) {
  std::lock_guard<std::mutex> lk(g_ws.mu);
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess)
    return false;
  WsBuffers &w = g_ws.sets[{d, stream}];
  if (w.staged_at == dev && w.staged == tables)
    return true;
  w.staged = tables;
  w.staged_at = dev;
  return false;
}

inline int32_t release_workspace(void *stream) {
  std::lock_guard<std::mutex> lk(g_ws.mu);
  int dev = 0;
  OMPDS_CUDA(cudaGetDevice(&dev));
  auto it = g_ws.sets.find({dev, stream});
  if (it == g_ws.sets.end())
    return OMPDS_OK;
  OMPDS_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
  for (unsigned char *b : it->second.retired)
    OMPDS_CUDA(cudaFree(b));
  it->second.retired.clear();
  for (int k = 0; k < WsBuffers::kBuffers; ++k) {
    unsigned char *b = it->second.buf[k];
    it->second.buf[k] = nullptr;
    it->second.bytes[k] = 0;
    if (b)
      OMPDS_CUDA(cudaFree(b));
  }
  g_ws.sets.erase(it);
  return OMPDS_OK;
}

// Kernel frame group of a fixed config, in the reference's emission order:
// captured locals, then sequential loop counters, then __omp_worker's
// wf.addr / args.addr (Codegen.cpp:413-430, LoweringPasses.cpp:264-305).
struct FixedLayout {
  int64_t total_shared = 0;
  int64_t cap_off[kMaxCaptures] = {};
  int64_t aux_off = -1;
};

inline int32_t build_fixed_layout(const std::vector<int64_t> &cap_bytes,
                           int64_t aux_bytes, FixedLayout *out) {
  std::vector<ompds_frame_var> vars;
  for (int64_t b : cap_bytes)
    vars.push_back({0, 0, OMPDS_VAR_ESCAPES, -1, b, -1, -1});
  if (aux_bytes > 0)
    vars.push_back({0, 0, 0, -1, aux_bytes, -1, -1});
  vars.push_back({0, 1, OMPDS_VAR_PINNED, -1, 8, -1, -1}); // wf.addr
  vars.push_back({0, 1, OMPDS_VAR_PINNED, -1, 8, -1, -1}); // args.addr
  ompds_depot_layout lay{};
  ompds_depot_slot slots[kMaxCaptures + 4];
  int32_t owners[kMaxCaptures + 4];
  int32_t s = ompds_layout_build(vars.data(), static_cast<int32_t>(vars.size()),
                                 1, OMPDS_PIPELINE_DEFAULT, &lay, slots,
                                 kMaxCaptures + 4, owners, kMaxCaptures + 4);
  if (s)
    return s;
  out->total_shared = lay.total_shared;
  // Without merges every var owns its slot, in order.
  for (size_t j = 0; j < cap_bytes.size(); ++j)
    out->cap_off[j] = slots[j].offset;
  if (aux_bytes > 0)
    out->aux_off = slots[cap_bytes.size()].offset;
  return OMPDS_OK;
}

inline int32_t validate_launch(const ompds_launch *l) {
  if (!l || l->teams <= 0 || l->workers <= 0 || l->workers > 992 ||
      l->prealloc_entries < 0 || l->prealloc_entries > 4096 ||
      (l->list_allocator != OMPDS_LIST_SLAB && l->list_allocator != OMPDS_LIST_MALLOC) ||
      l->reserved0 != 0 || l->first_team < 0 || l->total_teams < 0 ||
      (l->total_teams > 0 && int64_t(l->first_team) + l->teams > l->total_teams) ||
      (l->total_teams == 0 && l->first_team != 0))
    return OMPDS_ERR_INVALID;
  return OMPDS_OK;
}

inline constexpr uint32_t kSlabBytes = 8192; // per team: args lists + depot overflow

// `n_caps`: the largest nargs any region of the program stages (the fixed
// configs' capture counts); `allow_lean = false` for programs whose regions
// are only known at run time (ProgramProg).
template <class Prog>
int32_t launch_generic(const ompds_launch *l, const FixedLayout &lay,
                       int32_t n_caps, const typename Prog::Args &args,
                       ompds_team_stats *stats, ompds_event *events,
                       int64_t warp_slot_bytes = 0, int64_t warp_ovf_bytes = 0,
                       bool allow_lean = true) {
  int32_t s = validate_launch(l);
  if (s)
    return s;
  TeamParams p{};
  p.workers = l->workers;
  p.prealloc = l->prealloc_entries;
  p.fail_dyn = l->fail_dynamic_alloc;
  p.max_events = l->log_events ? l->max_events : 0;
  p.total_shared = lay.total_shared;
  p.depot_cap = l->depot_capacity < 0 ? lay.total_shared
                                      : round_up(l->depot_capacity, 8);
  p.events = l->log_events ? events : nullptr;
  p.list_malloc = l->list_allocator == OMPDS_LIST_MALLOC;
  p.first_team = l->first_team;
  p.bar_arrivals = l->barrier_arrivals;
  p.total_teams = l->total_teams > 0 ? l->total_teams : l->teams;
  p.stats = stats;
  p.n_caps = n_caps;
  for (int j = 0; j < kMaxCaptures; ++j)
    p.cap_off[j] = lay.cap_off[j];
  p.aux_off = lay.aux_off;
  p.slab_bytes = std::max<uint32_t>(
      kSlabBytes, static_cast<uint32_t>(round_up(2 * lay.total_shared + 64, 256)));
  s = ensure_buffer(0, size_t(p.slab_bytes) * l->teams, &p.slabs, l->stream);
  if (s)
    return s;
  const int threads = static_cast<int>(round_up(l->workers, 32)) + 32;
  const int worker_warps = threads / 32 - 1;
  p.warp_slot_bytes = round_up(warp_slot_bytes, 16);
  p.warp_ovf_bytes = round_up(warp_ovf_bytes, 256);
  if (p.warp_ovf_bytes > 0) {
    s = ensure_buffer(1, size_t(p.warp_ovf_bytes) * worker_warps * l->teams, &p.warp_ovf,
                      l->stream);
    if (s)
      return s;
  }
  size_t smem = static_cast<size_t>(team_region_bytes(p.depot_cap, p.prealloc));
  if (p.warp_slot_bytes > 0)
    smem = static_cast<size_t>(round_up(int64_t(smem), 16) + worker_warps * p.warp_slot_bytes);
  if (smem > 227 * 1024)
    return OMPDS_ERR_INVALID;
  // the lean instantiation whenever nothing needs the general paths
  // (a program that preloads list entries 0..3 needs a window of >= 4
  // entries for them; smaller windows take the general instantiation)
  const bool lean = allow_lean && !l->log_events && !l->fail_dynamic_alloc &&
                    l->barrier_arrivals == nullptr &&
                    l->list_allocator == OMPDS_LIST_SLAB && n_caps <= l->prealloc_entries &&
                    (!PreloadEntries<Prog>::value || l->prealloc_entries >= 4);
  auto kern = lean ? generic_mode_kernel<Prog, true> : generic_mode_kernel<Prog, false>;
  if constexpr (SmallTeams<Prog>::value)
    if (lean && threads == kSmallTeamThreads)
      kern = generic_mode_kernel<Prog, true, true>;
  if (smem > 48 * 1024)
    OMPDS_CUDA(cudaFuncSetAttribute(kern,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(smem)));
  cudaStream_t st = static_cast<cudaStream_t>(l->stream);
  kern<<<l->teams, threads, smem, st>>>(p, args);
  OMPDS_CUDA(cudaGetLastError());
  return OMPDS_OK;
}


} // namespace ompds
