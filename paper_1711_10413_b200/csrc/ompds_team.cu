// ompds_team.cu -- the stateful per-team runtime handle of the C ABI
// (include/ompds.h "Team runtime handle"): omplab::TeamRuntime
// (proj/include/omplab/DeviceRuntime.h:81-119) as an opaque object whose
// state lives in device memory between calls.
//
// Each operation is one launch of a one-thread kernel that loads the team's
// shared-memory region (args window + 49-byte runtime span) from the
// handle's device state block into shared memory, runs the SAME __device__
// protocol function the generic-mode kernels inline (ompds_device.cuh:
// kernel_init / prepare_parallel / kernel_parallel / end_parallel /
// kernel_deinit), stores the region back and writes its outcome -- status,
// list placement, the events this call logged, the team counters -- into
// pinned, device-mapped host memory.  So a call costs O(1): one launch and
// one stream synchronisation, independent of the history.
//
// The caller's SharedArgsAllocator (DeviceRuntime.h:46-52) is a pair of host
// callbacks.  prepareParallel calls it exactly where the reference does
// (DeviceRuntime.cpp:61-74): after every phase check passed, only for lists
// past the window and only when FailDynamicAlloc is off -- a first launch
// evaluates the checks without changing the state, the host allocates, a
// second launch stages the region with the block the allocator returned.
// endParallel's last retirement hands the freed block back to the release
// callback (DeviceRuntime.cpp:108-121).  The device never dereferences a
// list address (the protocol only stages and compares it), so allocator
// addresses may be any non-zero integers, as in the reference's RecordingHeap.
#include "ompds_generic.cuh"

#include <new>
#include <vector>

namespace ompds {
namespace {

constexpr int kStepMaxEvents = 4;      // one call logs at most 2 events
constexpr uint64_t kWindowMark = 1;    // args == the window, in saved state

enum StepOp : int32_t { kStepPrepareCheck = 100 };

struct StepOut {
  int32_t status;
  int32_t addr_kind;     // OMPDS_ADDR_*
  int32_t wf;
  int32_t participate;
  uint64_t list;         // dynamic list address (addr_kind == DYNAMIC)
  int32_t need_alloc;    // prepare check: the list must come from the heap
  int32_t freed;         // end_parallel: the last retirement freed `freed_addr`
  int64_t need_bytes;
  uint64_t freed_addr;
  int32_t n_events;
  int32_t phase;
  ompds_rt_summary summary;
  ompds_event events[kStepMaxEvents];
};

__device__ __noinline__ void team_step(ompds_runtime_config cfg, int32_t op, int32_t role,
                                       int64_t arg, int32_t fn, uint64_t ext_list,
                                       int64_t ext_bytes, unsigned char *smem, StepOut *out);

// One protocol call against the team region saved in `state`
// (team_region_bytes(0, prealloc) bytes: window, then the runtime span).
__global__ void team_step_kernel(ompds_runtime_config cfg, int32_t op, int32_t role,
                                 int64_t arg, int32_t fn, uint64_t ext_list,
                                 int64_t ext_bytes, unsigned char *state, StepOut *out) {
  extern __shared__ __align__(16) unsigned char smem[];
  // The saved region moves between global and shared memory as 16-byte
  // vectors spread over the warp (one memory latency, not one per byte);
  // `state` and the dynamic shared memory are sized round_up(region, 16).
  const int64_t region = team_region_bytes(0, cfg.prealloc_entries);
  const int64_t nvec = (region + 15) / 16;
  for (int64_t i = threadIdx.x; i < nvec; i += blockDim.x)
    reinterpret_cast<uint4 *>(smem)[i] = reinterpret_cast<const uint4 *>(state)[i];
  __syncthreads();
  if (threadIdx.x == 0)
    team_step(cfg, op, role, arg, fn, ext_list, ext_bytes, smem, out);
  __syncthreads();
  for (int64_t i = threadIdx.x; i < nvec; i += blockDim.x)
    reinterpret_cast<uint4 *>(state)[i] = reinterpret_cast<const uint4 *>(smem)[i];
}

// The protocol call itself, on the region in shared memory (one thread).
__device__ __noinline__ void team_step(ompds_runtime_config cfg, int32_t op, int32_t role,
                                       int64_t arg, int32_t fn, uint64_t ext_list,
                                       int64_t ext_bytes, unsigned char *smem, StepOut *out) {
  ompds_event ev[kStepMaxEvents];
  // A dynamic list is the caller's block: the team "slab" is exactly that
  // block, so alloc_args_list returns it and the last retirement's
  // slab_free returns the slab to empty (no device code of its own).
  TeamCtx t = make_team(smem, 0, cfg.prealloc_entries, cfg.fail_dynamic_alloc,
                        reinterpret_cast<unsigned char *>(ext_list),
                        static_cast<uint32_t>(round_up(ext_bytes, 16)), ev, kStepMaxEvents);
  uint64_t &args_word = t.at<uint64_t>(Rt::kArgs);
  if (args_word == kWindowMark)
    args_word = reinterpret_cast<uint64_t>(t.window);
  // events of this call are numbered from 0; the running total is restored
  const uint32_t ev_total = t.at<uint32_t>(Rt::kEvents);
  t.at<uint32_t>(Rt::kEvents) = 0;
  t.at<uint32_t>(Rt::kHeapTop) = 0;
  const uint32_t frees_before = t.at<uint32_t>(Rt::kDynFrees);
  const uint64_t list_before = args_word;

  StepOut o{};
  o.wf = -1;
  int32_t s = OMPDS_ERR_INVALID;
  switch (op) {
  case OMPDS_OP_KERNEL_INIT:
    s = kernel_init(t, role, static_cast<int32_t>(arg));
    break;
  case kStepPrepareCheck: // prepareParallel up to the allocator call, no state change
    if (role != kMaster) {
      s = OMPDS_TRAP_PREPARE_FROM_WORKER;
    } else {
      const PrepareState st = load_prepare_state(t);
      s = prepare_check(st.phase, st.active, arg);
      if (s == OMPDS_OK && arg > t.prealloc && !t.fail_dyn) {
        o.need_alloc = 1;
        o.need_bytes = arg * OMPDS_SHARED_ARG_ENTRY_BYTES;
      }
    }
    break;
  case OMPDS_OP_PREPARE_PARALLEL: {
    void **list = nullptr;
    s = prepare_parallel(t, role, fn, arg, &list);
    if (s == OMPDS_OK) {
      o.addr_kind = list == t.window ? OMPDS_ADDR_PREALLOC : OMPDS_ADDR_DYNAMIC;
      o.list = reinterpret_cast<uint64_t>(list);
    }
    break;
  }
  case OMPDS_OP_KERNEL_PARALLEL: {
    int32_t wf = -1;
    void **args = nullptr;
    bool part = false;
    s = kernel_parallel(t, role, &wf, &args, &part);
    if (s == OMPDS_OK) {
      o.wf = wf;
      o.participate = part;
      o.addr_kind = args == nullptr ? OMPDS_ADDR_NULL
                    : args == t.window ? OMPDS_ADDR_PREALLOC
                                       : OMPDS_ADDR_DYNAMIC;
      o.list = reinterpret_cast<uint64_t>(args);
    }
    break;
  }
  case OMPDS_OP_END_PARALLEL:
    s = end_parallel(t, role);
    if (s == OMPDS_OK && t.at<uint32_t>(Rt::kDynFrees) != frees_before) {
      o.freed = 1;
      o.freed_addr = list_before;
    }
    break;
  case OMPDS_OP_KERNEL_DEINIT:
    s = kernel_deinit(t, role);
    break;
  }
  o.status = s;
  const uint32_t logged = t.at<uint32_t>(Rt::kEvents);
  o.n_events = static_cast<int32_t>(logged < kStepMaxEvents ? logged : kStepMaxEvents);
  for (int i = 0; i < o.n_events; ++i)
    o.events[i] = ev[i];
  t.at<uint32_t>(Rt::kEvents) = ev_total + logged;
  o.phase = t.phase();
  o.summary.workers = t.at<int32_t>(Rt::kWorkers);
  o.summary.terminated = t.phase() == kTerminated;
  o.summary.dynamic_allocs = t.at<uint32_t>(Rt::kDynAllocs);
  o.summary.dynamic_frees = t.at<uint32_t>(Rt::kDynFrees);
  o.summary.leaked_blocks = o.summary.dynamic_allocs - o.summary.dynamic_frees;
  o.summary.n_events = static_cast<int32_t>(ev_total + logged);
  if (args_word == reinterpret_cast<uint64_t>(t.window))
    args_word = kWindowMark; // smem addresses do not outlive the launch
  *out = o;
}

} // namespace
} // namespace ompds

using namespace ompds;

struct ompds_team {
  ompds_runtime_config cfg{};
  uint64_t prealloc_base = 0;
  ompds_alloc_fn alloc = nullptr;
  ompds_release_fn release = nullptr;
  void *user = nullptr;
  int device = 0;
  cudaStream_t stream = nullptr;
  unsigned char *state = nullptr; // device: the team region between calls
  StepOut *out = nullptr;         // pinned, mapped host memory
  StepOut *out_dev = nullptr;     // its device alias
  size_t region = 0;
  ompds_rt_summary summary{};
  std::vector<ompds_event> events;
};

namespace {

int32_t team_launch(ompds_team *h, int32_t op, int32_t role, int64_t arg, int32_t fn = -1,
                    uint64_t ext_list = 0, int64_t ext_bytes = 0) {
  int prev = 0;
  OMPDS_CUDA(cudaGetDevice(&prev));
  if (prev != h->device)
    OMPDS_CUDA(cudaSetDevice(h->device));
  team_step_kernel<<<1, 32, round_up(h->region, 16), h->stream>>>(h->cfg, op, role, arg, fn, ext_list,
                                                    ext_bytes, h->state, h->out_dev);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess)
    e = cudaStreamSynchronize(h->stream);
  if (prev != h->device)
    cudaSetDevice(prev);
  if (e != cudaSuccess)
    return cuda_fail(e, "ompds_team step");
  return OMPDS_OK;
}

// Records the outcome of a successful or trapped call (a trap leaves the
// state and the log untouched, as in the reference).
int32_t team_finish(ompds_team *h) {
  const StepOut &o = *h->out;
  if (o.status == OMPDS_OK) {
    for (int i = 0; i < o.n_events; ++i)
      h->events.push_back(o.events[i]);
    h->summary = o.summary;
  }
  return o.status;
}

bool valid(const ompds_team *h, int32_t role) {
  return h != nullptr && (role == OMPDS_ROLE_MASTER || role == OMPDS_ROLE_WORKER);
}

} // namespace

extern "C" {

int32_t ompds_team_create(const ompds_runtime_config *config, uint64_t prealloc_base,
                          ompds_alloc_fn alloc, ompds_release_fn release, void *user,
                          ompds_team **out) {
  if (!config || !out || config->prealloc_entries < 0 || config->prealloc_entries > 4096 ||
      (alloc == nullptr) != (release == nullptr))
    return OMPDS_ERR_INVALID;
  *out = nullptr;
  ompds_team *h = new (std::nothrow) ompds_team;
  if (!h)
    return OMPDS_ERR_INVALID;
  h->cfg = *config;
  h->prealloc_base = prealloc_base;
  h->alloc = alloc;
  h->release = release;
  h->user = user;
  h->region = static_cast<size_t>(team_region_bytes(0, config->prealloc_entries));
  cudaError_t e = cudaGetDevice(&h->device);
  if (e == cudaSuccess)
    e = cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess)
    e = cudaMalloc(&h->state, round_up(h->region, 16));
  if (e == cudaSuccess) // the simulator zero-fills team memory (Simulator.cpp:286)
    e = cudaMemset(h->state, 0, round_up(h->region, 16));
  if (e == cudaSuccess)
    e = cudaHostAlloc(reinterpret_cast<void **>(&h->out), sizeof(StepOut), cudaHostAllocMapped);
  if (e == cudaSuccess)
    e = cudaHostGetDevicePointer(reinterpret_cast<void **>(&h->out_dev), h->out, 0);
  if (e == cudaSuccess) { // Uninitialized, work_fn = -1, as generic kernels start
    const uint32_t none = state_word(kUninit, -1);
    e = cudaMemcpy(h->state + config->prealloc_entries * OMPDS_SHARED_ARG_ENTRY_BYTES +
                       Rt::kState,
                   &none, 4, cudaMemcpyHostToDevice);
  }
  if (e != cudaSuccess) {
    ompds_team_destroy(h);
    return cuda_fail(e, "ompds_team_create");
  }
  *out = h;
  return OMPDS_OK;
}

int32_t ompds_team_destroy(ompds_team *h) {
  if (!h)
    return OMPDS_OK;
  if (h->stream)
    cudaStreamSynchronize(h->stream);
  cudaFree(h->state);
  if (h->out)
    cudaFreeHost(h->out);
  if (h->stream)
    cudaStreamDestroy(h->stream);
  delete h;
  return OMPDS_OK;
}

int32_t ompds_team_kernel_init(ompds_team *h, int32_t role, int32_t workers) {
  if (!valid(h, role))
    return OMPDS_ERR_INVALID;
  if (int32_t s = team_launch(h, OMPDS_OP_KERNEL_INIT, role, workers))
    return s;
  return team_finish(h);
}

int32_t ompds_team_prepare_parallel(ompds_team *h, int32_t role, int32_t fn, int64_t nargs,
                                    uint64_t *args_addr) {
  if (!valid(h, role) || !args_addr || fn < 0 || fn > kMaxWorkFn)
    return OMPDS_ERR_INVALID;
  // A list that fits the window (or a FailDynamicAlloc team, whose heap is
  // never asked) needs no allocator call: one launch does the whole
  // prepare.  Otherwise a first launch runs the checks, then the heap is
  // asked, then the region is staged with its block.
  const bool may_alloc = nargs > h->cfg.prealloc_entries && !h->cfg.fail_dynamic_alloc;
  if (may_alloc) {
    if (int32_t s = team_launch(h, kStepPrepareCheck, role, nargs))
      return s;
    if (h->out->status != OMPDS_OK)
      return h->out->status;
  }
  uint64_t block = 0;
  int64_t bytes = 0;
  if (may_alloc && h->out->need_alloc) {
    bytes = h->out->need_bytes;
    block = h->alloc ? h->alloc(bytes, h->user) : 0;
    if (block == 0) // Heap.allocate returned 0 (DeviceRuntime.cpp:67-69)
      return OMPDS_TRAP_ARGS_ALLOC_FAILED;
  }
  if (int32_t s = team_launch(h, OMPDS_OP_PREPARE_PARALLEL, role, nargs, fn, block, bytes))
    return s;
  const int32_t s = team_finish(h);
  if (s == OMPDS_OK)
    *args_addr = h->out->addr_kind == OMPDS_ADDR_PREALLOC ? h->prealloc_base : h->out->list;
  return s;
}

int32_t ompds_team_kernel_parallel(ompds_team *h, int32_t role, int32_t *fn,
                                   uint64_t *args_addr, int32_t *participate) {
  if (!valid(h, role) || !fn || !args_addr || !participate)
    return OMPDS_ERR_INVALID;
  if (int32_t s = team_launch(h, OMPDS_OP_KERNEL_PARALLEL, role, 0))
    return s;
  const int32_t s = team_finish(h);
  if (s == OMPDS_OK) {
    const StepOut &o = *h->out;
    *fn = o.wf;
    *participate = o.participate;
    *args_addr = o.addr_kind == OMPDS_ADDR_PREALLOC ? h->prealloc_base
                 : o.addr_kind == OMPDS_ADDR_DYNAMIC ? o.list
                                                     : 0;
  }
  return s;
}

int32_t ompds_team_end_parallel(ompds_team *h, int32_t role) {
  if (!valid(h, role))
    return OMPDS_ERR_INVALID;
  if (int32_t s = team_launch(h, OMPDS_OP_END_PARALLEL, role, 0))
    return s;
  const int32_t s = team_finish(h);
  if (s == OMPDS_OK && h->out->freed && h->release) // Heap.release(ArgsAddr)
    h->release(h->out->freed_addr, h->user);
  return s;
}

int32_t ompds_team_kernel_deinit(ompds_team *h, int32_t role) {
  if (!valid(h, role))
    return OMPDS_ERR_INVALID;
  if (int32_t s = team_launch(h, OMPDS_OP_KERNEL_DEINIT, role, 0))
    return s;
  return team_finish(h);
}

int32_t ompds_team_summary(const ompds_team *h, ompds_rt_summary *out) {
  if (!h || !out)
    return OMPDS_ERR_INVALID;
  *out = h->summary;
  return OMPDS_OK;
}

int32_t ompds_team_events(const ompds_team *h, int32_t first, ompds_event *out,
                          int32_t max_events, int32_t *n_events) {
  if (!h || !n_events || first < 0 || max_events < 0 || (max_events > 0 && !out))
    return OMPDS_ERR_INVALID;
  const size_t n = h->events.size();
  *n_events = static_cast<int32_t>(n);
  size_t k = static_cast<size_t>(first);
  for (int32_t i = 0; k < n && i < max_events; ++i, ++k)
    out[i] = h->events[k];
  return k < n ? OMPDS_ERR_CAPACITY : OMPDS_OK;
}

} // extern "C"
