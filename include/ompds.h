/*
 * ompds.h -- C ABI of the B200-native implicit data-sharing runtime for
 * OpenMP generic-mode target regions (arXiv 1711.10413).
 *
 * This is the drop-in boundary for the hot path named by BASELINE.json's
 * north_star.  The reference (`omplab`, /root/reference/proj) exposes the path
 * as C++ classes; each entry point below names the reference interface it
 * replaces (file:line, relative to proj/).  Plain pointers and sizes only: no
 * C++ or torch types cross this boundary.  Every entry point returns an
 * `ompds_status` (0 = OK); runtime protocol traps return the trap code whose
 * exact reference string `ompds_trap_reason` yields.
 *
 * Compute entry points run on the GPU (sm_100a) and fail with
 * OMPDS_ERR_CUDA when no device is usable -- there is no CPU fallback.
 */
#ifndef OMPDS_H
#define OMPDS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------------------ */
/* Constants  (proj/include/omplab/DeviceRuntime.h:26-38)                    */
/* ------------------------------------------------------------------------ */
#define OMPDS_DEFAULT_PREALLOC_ENTRIES 20 /* DefaultPreallocEntries  :27 */
#define OMPDS_SHARED_ARG_ENTRY_BYTES 8    /* SharedArgEntryBytes     :29 */
#define OMPDS_RUNTIME_PRIVATE_BYTES 49    /* RuntimePrivateBytes     :31 */
#define OMPDS_RESERVED_WARP 32            /* Codegen.h:25 ReservedWarpSize */

/* ------------------------------------------------------------------------ */
/* Status / trap codes.  Codes 1..17 are the reference's RtResult trap      */
/* reasons (DeviceRuntime.cpp:33-143), strings via ompds_trap_reason().      */
/* ------------------------------------------------------------------------ */
typedef enum ompds_status {
  OMPDS_OK = 0,
  OMPDS_TRAP_INIT_FROM_WORKER = 1,
  OMPDS_TRAP_INIT_TWICE = 2,
  OMPDS_TRAP_INIT_NO_WORKERS = 3,
  OMPDS_TRAP_PREPARE_FROM_WORKER = 4,
  OMPDS_TRAP_PREPARE_BEFORE_INIT = 5,
  OMPDS_TRAP_PREPARE_AFTER_DEINIT = 6,
  OMPDS_TRAP_PREPARE_IN_FLIGHT = 7,
  OMPDS_TRAP_NEGATIVE_NARGS = 8,
  OMPDS_TRAP_ARGS_ALLOC_FAILED = 9,
  OMPDS_TRAP_PARALLEL_FROM_MASTER = 10,
  OMPDS_TRAP_PARALLEL_NOT_STAGED = 11,
  OMPDS_TRAP_END_FROM_MASTER = 12,
  OMPDS_TRAP_END_NOT_ACTIVE = 13,
  OMPDS_TRAP_DEINIT_FROM_WORKER = 14,
  OMPDS_TRAP_DEINIT_BEFORE_INIT = 15,
  OMPDS_TRAP_DEINIT_IN_FLIGHT = 16,
  OMPDS_TRAP_DEINIT_TWICE = 17,
  /* data-sharing stack (new; no reference counterpart) */
  OMPDS_TRAP_STACK_OVERFLOW = 18,  /* global overflow chain exhausted */
  OMPDS_TRAP_STACK_UNDERFLOW = 19, /* pop of a frame that is not the top */
  OMPDS_TRAP_OUT_OF_BOUNDS = 20,   /* region program: index outside its object
                                      (Simulator.cpp:313-377 "out-of-bounds") */
  OMPDS_TRAP_STEP_LIMIT = 21,      /* region program: a thread executed more
                                      than ompds_program.step_limit operations
                                      (Simulator.cpp:819-822, "step limit
                                      exceeded")                           */
  /* host-side errors */
  OMPDS_ERR_CUDA = 100,    /* no usable CUDA device / launch or copy failed */
  OMPDS_ERR_INVALID = 101, /* invalid argument */
  OMPDS_ERR_CAPACITY = 102 /* caller-provided output array too small */
} ompds_status;

/* Exact reference trap string for codes 1..17 ("" for OK). */
const char *ompds_trap_reason(int32_t code);
/* Last CUDA error text recorded by this library (thread-local). */
const char *ompds_last_error(void);
/* Library/ABI version, e.g. 0x00010000. */
uint32_t ompds_version(void);
/* Number of usable CUDA devices (0 when none). */
int32_t ompds_device_count(void);
/* Frees the library's device workspace (stack overflow chains, args-list
 * slabs, program tables) kept for `stream` (a cudaStream_t, NULL = the
 * default stream) on the current device, after waiting for the stream's
 * work.  Call it before destroying a stream the library launched on; the
 * next launch on a stream reallocates on demand.  Buffers a larger launch
 * superseded are kept until this call (CUDA graphs captured from earlier
 * launches still point at them), so it invalidates such graphs. */
int32_t ompds_release_workspace(void *stream);

/* ------------------------------------------------------------------------ */
/* Team runtime protocol: omplab::TeamRuntime  (DeviceRuntime.h:81-119)     */
/*                                                                          */
/* The five operations run on the GPU through the same __device__ code the */
/* generic-mode kernels inline (paper_1711_10413_b200/csrc/ompds_device.cuh).*/
/* A script of calls is replayed in order by one device thread against one */
/* team's shared-memory runtime state; every call's outcome is returned.   */
/* ------------------------------------------------------------------------ */
typedef struct ompds_runtime_config {  /* RuntimeConfig DeviceRuntime.h:40-43 */
  int32_t prealloc_entries;   /* PreallocEntries (default 20)              */
  int32_t fail_dynamic_alloc; /* FailDynamicAlloc test hook                */
} ompds_runtime_config;

enum { OMPDS_ROLE_MASTER = 0, OMPDS_ROLE_WORKER = 1 }; /* RtRole :54 */
enum {
  OMPDS_OP_KERNEL_INIT = 0,      /* TeamRuntime::kernelInit      cpp:33  */
  OMPDS_OP_PREPARE_PARALLEL = 1, /* TeamRuntime::prepareParallel cpp:46  */
  OMPDS_OP_KERNEL_PARALLEL = 2,  /* TeamRuntime::kernelParallel  cpp:81  */
  OMPDS_OP_END_PARALLEL = 3,     /* TeamRuntime::endParallel     cpp:102 */
  OMPDS_OP_KERNEL_DEINIT = 4     /* TeamRuntime::kernelDeinit    cpp:130 */
};
enum { /* where an args list lives */
  OMPDS_ADDR_NULL = 0,     /* termination sentinel (kernelParallel, cpp:87-92) */
  OMPDS_ADDR_PREALLOC = 1, /* the team's shared-memory window (PreallocBase)   */
  OMPDS_ADDR_DYNAMIC = 2   /* a global-memory block (Heap.allocate)            */
};

typedef struct ompds_rt_call {
  int32_t op;   /* OMPDS_OP_*                                   */
  int32_t role; /* OMPDS_ROLE_*                                 */
  int64_t arg;  /* workers for init, nargs for prepare_parallel */
} ompds_rt_call;

typedef struct ompds_rt_result {
  int32_t status;      /* 0 or trap code                               */
  int32_t addr_kind;   /* OMPDS_ADDR_* (prepare / kernel_parallel)     */
  int32_t wf;          /* staged work-function id, -1 = none (sentinel) */
  int32_t participate; /* kernel_parallel's Participate                */
  int64_t live_bytes;  /* bytes of the live dynamic block, else 0      */
  int64_t heap_live;   /* live dynamic blocks after the call           */
} ompds_rt_result;

enum { /* RuntimeEvent::Kind, DeviceRuntime.h:64-79 */
  OMPDS_EV_INIT = 0,
  OMPDS_EV_PREPARE_PREALLOC = 1,
  OMPDS_EV_PREPARE_DYNAMIC = 2,
  OMPDS_EV_FETCH = 3,
  OMPDS_EV_RETIRE = 4,
  OMPDS_EV_DYNAMIC_FREE = 5,
  OMPDS_EV_DEINIT = 6
};
typedef struct ompds_event {
  int32_t kind;  /* OMPDS_EV_*                                   */
  int32_t fn;    /* work-function id (-1 when not applicable)    */
  int64_t nargs; /* NArgs field: workers / nargs / remaining     */
  int64_t bytes; /* Bytes field                                  */
  int64_t t_ns;  /* device %globaltimer when logged (trace; the
                    reference's RuntimeEvent has no time)        */
} ompds_event;

typedef struct ompds_rt_summary { /* TeamRuntime accessors DeviceRuntime.h:97-102 */
  int32_t workers;
  int32_t terminated;
  int64_t dynamic_allocs;
  int64_t dynamic_frees;
  int64_t leaked_blocks;
  int32_t n_events; /* total events logged (may exceed max_events) */
  int32_t _pad;
} ompds_rt_summary;

int32_t ompds_rt_replay(const ompds_runtime_config *config,
                        const ompds_rt_call *calls, int32_t n_calls,
                        ompds_rt_result *results, ompds_event *events,
                        int32_t max_events, ompds_rt_summary *summary);

/* ------------------------------------------------------------------------ */
/* Team runtime handle: one omplab::TeamRuntime instance                   */
/* (DeviceRuntime.h:81-119, constructed per team at Simulator.cpp:290-292). */
/*                                                                          */
/* State lives on the device between calls; each call runs the same        */
/* __device__ protocol function the generic-mode kernels inline, O(1) per  */
/* call (one launch + one stream synchronisation).  Like the reference     */
/* class it is not thread-safe: one caller per handle.  Every operation    */
/* returns 0 or the reference trap code (1..17, ompds_trap_reason), or     */
/* OMPDS_ERR_*; a trap leaves the state, counters and event log unchanged. */
/* ------------------------------------------------------------------------ */
typedef struct ompds_team ompds_team; /* opaque */
/* SharedArgsAllocator (DeviceRuntime.h:46-52): allocate returns the block
 * address or 0 when the heap is exhausted; release gets back exactly the
 * address allocate returned.  The runtime only stores and compares list
 * addresses, so any non-zero integers are valid. */
typedef uint64_t (*ompds_alloc_fn)(int64_t bytes, void *user);
typedef void (*ompds_release_fn)(uint64_t addr, void *user);

/* TeamRuntime(RuntimeConfig, PreallocBase, SharedArgsAllocator&): `alloc`
 * and `release` both set or both NULL (NULL: every list past the window is
 * shared-args-alloc-failed).  Binds the handle to the current device. */
int32_t ompds_team_create(const ompds_runtime_config *config, uint64_t prealloc_base,
                          ompds_alloc_fn alloc, ompds_release_fn release, void *user,
                          ompds_team **out);
int32_t ompds_team_destroy(ompds_team *team);
/* TeamRuntime::kernelInit (DeviceRuntime.cpp:33-44) */
int32_t ompds_team_kernel_init(ompds_team *team, int32_t role, int32_t workers);
/* TeamRuntime::prepareParallel (:46-79); `fn` names the work function (an
 * id >= 0; the C++ adapter interns the reference's strings).  *args_addr =
 * prealloc_base for the window, else the allocator's block. */
int32_t ompds_team_prepare_parallel(ompds_team *team, int32_t role, int32_t fn,
                                    int64_t nargs, uint64_t *args_addr);
/* TeamRuntime::kernelParallel (:81-100); after deinit: *fn = -1,
 * *args_addr = 0, *participate = 0 (the termination sentinel). */
int32_t ompds_team_kernel_parallel(ompds_team *team, int32_t role, int32_t *fn,
                                   uint64_t *args_addr, int32_t *participate);
/* TeamRuntime::endParallel (:102-128); the last retirement of a region with
 * a heap list calls release(addr). */
int32_t ompds_team_end_parallel(ompds_team *team, int32_t role);
/* TeamRuntime::kernelDeinit (:130-143) */
int32_t ompds_team_kernel_deinit(ompds_team *team, int32_t role);
/* workerCount / dynamicAllocs / dynamicFrees / leakedBlocks / terminated */
int32_t ompds_team_summary(const ompds_team *team, ompds_rt_summary *out);
/* events(): copies events [first, first + max_events) of the log to `out`
 * and sets *n_events = the total logged so far (OMPDS_ERR_CAPACITY when
 * events past the copied ones remain; the handle keeps every event). */
int32_t ompds_team_events(const ompds_team *team, int32_t first, ompds_event *out,
                          int32_t max_events, int32_t *n_events);

/* Capacity law dynamicArgsBytes (DeviceRuntime.h:35-38). */
int64_t ompds_dynamic_args_bytes(int64_t nargs, int32_t prealloc_entries);

/* ------------------------------------------------------------------------ */
/* Frame-layout descriptors: DepotSlot / DepotLayout / FrameGroup           */
/* (IR.h:219-254) built by the reference's frame pipeline                   */
/* (LoweringPasses.cpp: buildDepots :264-305, lowerSharedFrames :345-380,   */
/*  colorStack :458-538, repackOffsets :556-593, audit :617-665).           */
/* ------------------------------------------------------------------------ */
enum { /* ompds_frame_var.flags */
  OMPDS_VAR_ESCAPES = 1u << 0, /* address stored as a value (captured):
                                  escapedAllocas, LoweringPasses.cpp:107-139 */
  OMPDS_VAR_PINNED = 1u << 1   /* frame value stored / passed to a call:
                                  never merged by coloring (:506-509)        */
};
enum { /* PipelineKind, LoweringPasses.h:43 */
  OMPDS_PIPELINE_DEFAULT = 0,
  OMPDS_PIPELINE_O0 = 1,
  OMPDS_PIPELINE_BAD_ORDER = 2
};

typedef struct ompds_frame_var { /* one alloca, in emission order */
  int32_t group;    /* frame group (0 = kernel + __omp_worker, then one per
                       outlined / wrapper function; LoweringPasses.cpp:270-280) */
  int32_t func;     /* member function within the group (coloring scope)  */
  uint32_t flags;   /* OMPDS_VAR_*                                        */
  int32_t def_pos;  /* position of the alloca in its function             */
  int64_t bytes;    /* allocation size before rounding                    */
  int32_t live_first; /* first / last position where the frame value      */
  int32_t live_last;  /* itself is an operand (-1: never)                 */
} ompds_frame_var;
/* Liveness is given in post-codegen instruction positions.  The builder
 * works in doubled coordinates (position p -> 2p) so that the address-space
 * cast the frame pipeline inserts right after an escaping alloca sits at
 * 2*def_pos+1 -- that cast is the escaping variable's only direct use when
 * coloring runs (LoweringPasses.cpp:212-258, 393-422). */

typedef struct ompds_depot_slot { /* DepotSlot IR.h:219-228 */
  int64_t offset;
  int64_t size;
  int32_t align;
  int32_t shared;      /* SharedResident                           */
  int32_t owner_begin; /* index into the owners array (var indices) */
  int32_t n_owners;
} ompds_depot_slot;

typedef struct ompds_depot_layout { /* DepotLayout IR.h:230-244 */
  int64_t total_local;
  int64_t total_shared; /* mirror of total_local */
  int32_t has_shared_depot;
  int32_t slot_begin; /* index into the slots array */
  int32_t n_slots;
  int32_t overlap_slot; /* findSharedLocalOverlap (IR.cpp:228-242), -1 none */
} ompds_depot_layout;

/* Runs the frame pipeline over `vars` (grouped by .group, n_groups groups).
 * Writes n_groups layouts, their slots and owner lists.  Returns
 * OMPDS_ERR_CAPACITY if max_slots / max_owners are too small. */
int32_t ompds_layout_build(const ompds_frame_var *vars, int32_t n_vars,
                           int32_t n_groups, int32_t pipeline,
                           ompds_depot_layout *layouts,
                           ompds_depot_slot *slots, int32_t max_slots,
                           int32_t *owners, int32_t max_owners);

/* ------------------------------------------------------------------------ */
/* Manifest JSON: the descriptor export of the reference compiler           */
/* (Compiler.cpp:112-155 manifestJson: nlohmann dump(2) + "\n").           */
/* ------------------------------------------------------------------------ */
typedef struct ompds_manifest {
  const char *kernel;               /* kernel function name ("" when none)  */
  int32_t teams;                    /* LaunchDefaults (IR.h:260-266)        */
  int32_t workers;
  int32_t prealloc_entries;
  int32_t has_layout;               /* 0: no kernel layout (empty depot)    */
  const ompds_depot_layout *layout; /* the kernel frame group's layout      */
  const ompds_depot_slot *slots;    /* the slots array of ompds_layout_build */
  const int32_t *owners;            /* its owners array (var indices)       */
  const char *const *var_names;     /* name of every var index              */
} ompds_manifest;

/* Writes the manifest text, byte-identical to the reference's, and a NUL.
 * *len = text length without the NUL; OMPDS_ERR_CAPACITY (with *len set)
 * when cap <= *len. */
int32_t ompds_manifest_write(const ompds_manifest *m, char *out, int64_t cap, int64_t *len);

typedef struct ompds_manifest_info {
  int64_t kernel;           /* offset of the kernel name in `names`         */
  int32_t teams;
  int32_t workers;
  int64_t total_local;
  int64_t total_shared;
  int32_t mirrored;
  int32_t prealloc_entries;
  int64_t stack_bytes;
  int64_t prealloc_bytes;
  int64_t runtime_bytes;
  int64_t shared_footprint;
  int32_t n_slots;
  int32_t n_owners;
} ompds_manifest_info;

/* Parses manifest JSON (any whitespace / key order).  Slots go to `slots`
 * (owner_begin / n_owners index `owner_names`, whose entries are offsets of
 * NUL-terminated names in `names`).  OMPDS_ERR_INVALID for malformed JSON,
 * a missing or mistyped field, or a manifest that breaks the reference's
 * laws: offsets are the prefix sums of the sizes, total_local = total_shared
 * = stack_bytes = the sum of the sizes, prealloc_bytes = 8 x
 * prealloc_entries, runtime_bytes = 49, shared_footprint = total_shared +
 * prealloc_bytes + runtime_bytes.  OMPDS_ERR_CAPACITY when an output array
 * is too small (info still filled). */
int32_t ompds_manifest_parse(const char *text, int64_t len, ompds_manifest_info *info,
                             ompds_depot_slot *slots, int32_t max_slots,
                             int64_t *owner_names, int32_t max_owners, char *names,
                             int64_t names_cap);

/* Per-team shared footprint: depot + prealloc window + runtime span
 * (Simulator.cpp:281-284, Occupancy.h:49-51). */
int64_t ompds_shared_footprint(int64_t total_shared, int32_t prealloc_entries);

/* ------------------------------------------------------------------------ */
/* Occupancy model (Occupancy.h / Occupancy.cpp:77-105) + a B200 row.       */
/* ------------------------------------------------------------------------ */
typedef struct ompds_gpu_spec { /* GpuSpec Occupancy.h:24-31 */
  int64_t shared_bytes_per_sm;
  int64_t registers_per_sm;
  int64_t max_blocks_per_sm;
  int32_t warp_size;
  int32_t max_regs_per_thread;
  int64_t max_threads_per_sm;      /* 0 = unlimited (reference model)      */
  int64_t reserved_smem_per_block; /* 0 in the reference model; 1 KB B200  */
  int32_t reg_alloc_unit;          /* registers per thread are allocated
                                      per warp in multiples of this: 8 on
                                      B200 (256 per warp, as ncu's
                                      occupancy_limit_registers counts);
                                      0 = exact (the reference model)     */
  int32_t reg_partitions;          /* the register file is split evenly over
                                      this many SM sub-partitions and a warp
                                      takes all its registers from one: 4 on
                                      B200 (16K registers per SMSP); 0 = one
                                      pool (the reference model)           */
} ompds_gpu_spec;

typedef struct ompds_occupancy { /* OccupancyResult Occupancy.h:62-68 */
  int64_t teams_by_regs;
  int64_t teams_by_smem;
  int64_t potential;
  int64_t actual;
  int64_t smem_used;
} ompds_occupancy;

/* name: "k40-16k", "k40-32k", "k40-48k", "p100" (Occupancy.cpp:14-22) or
 * "b200" (new). */
int32_t ompds_gpu_spec_get(const char *name, ompds_gpu_spec *out);
int32_t ompds_occupancy_for(const ompds_gpu_spec *gpu, int64_t footprint,
                            int32_t regs_per_thread, int32_t threads_per_team,
                            ompds_occupancy *out);
int64_t ompds_max_regs_for_teams(const ompds_gpu_spec *gpu, int64_t teams,
                                 int32_t threads_per_team);
int64_t ompds_max_shared_vars(const ompds_gpu_spec *gpu, int64_t teams);

/* ------------------------------------------------------------------------ */
/* Generic-mode target-region launches (the sm_100a hot path).              */
/*                                                                          */
/* Each launch runs `teams` CTAs of roundup32(workers)+32 threads: workers  */
/* [0,W), the master = first lane of the reserved last warp (Codegen.h:25-30,*/
/* Codegen.cpp:345-397).  Per team the CTA's dynamic shared memory is the   */
/* reference's team region [depot | 8*prealloc args window | 49 B runtime]  */
/* (Simulator.cpp:281-292).  The master stages every region through        */
/* prepare_parallel + named-barrier release/join; workers fetch it, read the */
/* shared-variable list (warp-shuffle broadcast) and retire it.             */
/* All pointers are DEVICE pointers unless the name says host.             */
/* ------------------------------------------------------------------------ */
typedef struct ompds_launch {
  int32_t teams;            /* CTAs                                       */
  int32_t workers;          /* W (thread_limit)                           */
  int32_t prealloc_entries; /* shared-args window entries (default 20)     */
  int32_t fail_dynamic_alloc;
  int64_t depot_capacity;   /* master data-sharing slot bytes in smem;
                               <0 = the layout's TotalShared (reference) */
  int32_t log_events;       /* record per-team runtime events             */
  int32_t max_events;       /* per-team event capacity when logging       */
  void *stream;             /* cudaStream_t (NULL = default stream)       */
  int32_t list_allocator;   /* where args lists past the window live:
                               OMPDS_LIST_SLAB (0, default) a per-team
                               global slab, LIFO; OMPDS_LIST_MALLOC (1)
                               device malloc/free per region -- the
                               paper's fallback (PAPER.md "back-up scheme") */
  int32_t first_team;       /* team range [first_team, first_team+teams)
                               of a grid of total_teams (0: total = teams):
                               omp_get_team_num() / omp_get_num_teams()
                               of the launched CTAs, so a team grid can be
                               sharded across GPUs by range             */
  int32_t total_teams;
  int32_t reserved0;        /* must be 0                                  */
  int32_t *barrier_arrivals; /* optional (NULL = off), device, teams x (W+32):
                               for every thread of the reference's team
                               (workers 0..W-1, the master W, the reserved
                               warp's idle lanes W+1..W+31) the hardware
                               barrier arrivals of the lane that plays it
                               (SimStats::BarrierEntries, Simulator.h:42-55;
                               see DESIGN.md for the idle lanes)          */
} ompds_launch;

#define OMPDS_LIST_SLAB 0
#define OMPDS_LIST_MALLOC 1

typedef struct ompds_team_stats { /* per team, written by the kernel */
  int32_t trap;                   /* first trap code, 0 = none            */
  int32_t master_barriers;        /* master handoff barrier entries (2/region) */
  int32_t barrier_releases;       /* handoff barrier releases (2R+1)      */
  int32_t regions;                /* regions staged                       */
  int64_t dynamic_alloc_bytes;
  int32_t dynamic_allocs;
  int32_t dynamic_frees;
  int32_t depot_in_smem;          /* 1 = master frame in the smem slot, 0 = global overflow */
  int32_t n_events;
  int64_t depot_offset;           /* frame offset inside its slot         */
  int64_t smem_bytes;             /* dynamic smem per CTA for this launch */
} ompds_team_stats;

/* Config 1: `regions` parallel regions in a sequential loop; the master
 * shares 4 scalars (c1,c2 int32 = 1,2; c3,c4 = 3,4 stored as `elem`) and
 * bumps c4 by 1 after every region; body a[team*W + tid] += c1+c2+c3+c4.
 * elem: 0 = int32 (reference analog, a is int32[teams*W]),
 *       1 = float64 (a is double[teams*W]; sum ((c1+c2) + c3) + c4 in fp64). */
int32_t ompds_run_regions(const ompds_launch *launch, int32_t elem,
                          int32_t regions, void *a,
                          ompds_team_stats *stats_dev, ompds_event *events_dev);

/* Config 2: a statically allocated shared array d[256] (depot slot
 * 256*sizeof(elem)), d[k] = 3k+1 staged by the master -- by
 * cp.async.bulk from `d_init` (device, 256 elems) when non-NULL, else by
 * the master's own loop -- then `parallel for i<n: a[i] += d[i & 255]`
 * on the cyclic schedule (AstLowering.cpp:429-462).
 * elem: 0 = int32, 1 = float64.  Pointers must be aligned to the element;
 * a 16-byte aligned `a` gets the vectorised body, any other the
 * element-wise one (same results). */
int32_t ompds_run_shared_array(const ompds_launch *launch, int32_t elem,
                               int64_t n, void *a, const void *d_init,
                               ompds_team_stats *stats_dev,
                               ompds_event *events_dev);

/* Config 4/5: streaming region with 8 implicitly shared scalars
 * c_k (k=1..8) on the cyclic schedule over elements [0, n):
 *   float64: y[i] = fma(c1, x[i], y[i]) + s,  s = ((((((c2+c3)+c4)+c5)+c6)+c7)+c8)
 *   int32  : y[i] = y[i] + (c1*x[i] + c2 + ... + c8)   (wrapping int32)
 * `coef` (host, 8 values of elem type) are the master's initial values.
 * x, y aligned to the element (may be NULL when n == 0: the region still
 * runs); both 16-byte aligned gets the vectorised body, otherwise the
 * element-wise one (same results). */
int32_t ompds_run_stream(const ompds_launch *launch, int32_t elem, int64_t n,
                         const void *x, void *y, const void *coef_host,
                         ompds_team_stats *stats_dev, ompds_event *events_dev);

/* Config 3: nested parallel regions, depth 3, serialized inner levels whose
 * captured locals live on per-warp data-sharing stacks: a statically sized
 * shared-memory slot of `warp_slot_bytes` per worker warp plus a
 * global-memory overflow chain (__kmpc_data_sharing_push_stack /
 * _pop_stack).  Program and semantics: DESIGN.md "config 3"; the reference
 * rejects nesting (DslParser.cpp:846-849), so the oracle restates it.
 * `warp_stats_dev` receives teams * ceil(W/32) records (may be NULL). */
typedef struct ompds_warp_stack_stats {
  int32_t frame_in_smem[2]; /* level-1 / level-2 frame: 1 smem slot, 0 chain */
  int64_t frame_offset[2];  /* offset inside that segment                  */
  int32_t status;           /* 0 or OMPDS_TRAP_STACK_*                       */
  int32_t max_depth;        /* deepest stack (frames)                         */
  int64_t high_water;       /* max bytes in use (slot + chain)               */
} ompds_warp_stack_stats;

int32_t ompds_run_nested(const ompds_launch *launch, int32_t elem,
                         int32_t regions, int64_t warp_slot_bytes,
                         int64_t warp_overflow_bytes, void *a,
                         ompds_team_stats *stats_dev,
                         ompds_warp_stack_stats *warp_stats_dev,
                         ompds_event *events_dev);

/* Region programs: the reference's kernel language (int32 scalars/arrays,
 * `parallel` / `parallel for`) lowered by paper_1711_10413_b200/program.py
 * to a stack bytecode that the generic-mode kernel interprets inside the
 * real protocol (master lane: sequential code; workers: region bodies).
 * Variables live where the frame layout puts them (space): 0 team depot
 * (shared slot), 1 the master's local depot mirror, 2 the worker's private
 * frame, 3 capture j of the current region (via get-shared-variables),
 * 4 mapped buffer.  All host arrays below are copied per launch.
 * Nested regions (EXTENSION; the reference rejects them): a PARALLEL in a
 * region body runs the child region serialized on the encountering thread
 * (omp_get_thread_num() 0, one thread), its capture list published on the
 * thread's data-sharing stack and read back with get-shared-variables; a
 * GLOBALIZE region's private frame lives on that stack too.  Each worker
 * lane has its own stack (1/32 of the warp's slot, then its slice of the
 * warp's overflow chain): lanes of a warp may nest divergently. */
typedef struct ompds_prog_var {
  int32_t space;  /* 0..4 as above                           */
  int32_t index;  /* byte offset (0..2), capture j, buffer k */
  int32_t count;  /* elements (int32) for bounds checks       */
  int32_t _pad;
} ompds_prog_var;
typedef struct ompds_prog_region {
  int32_t entry;      /* pc of the region body                              */
  int32_t n_captures; /* nargs of its prepare_parallel / nested list         */
  int32_t cap_begin;  /* into `captures` (var indices in the encountering
                         context: the master's, or the parent region's)      */
  int32_t parent;     /* -1: staged by the master; else the region whose body
                         encounters it (EXTENSION, nested: serialized on the
                         encountering thread); parent < index     */
  int32_t frame_bytes;/* its private frame (outlined group TotalLocal)      */
  int32_t flags;      /* OMPDS_REGION_GLOBALIZE: the frame holds locals a
                         nested region captures, so each activation's frame
                         is pushed on the thread's data-sharing stack        */
} ompds_prog_region;
#define OMPDS_REGION_GLOBALIZE 1
typedef struct ompds_program {
  const int32_t *code;
  int64_t n_code;
  const ompds_prog_var *vars;
  int32_t n_vars;
  int32_t n_regions;
  const ompds_prog_region *regions;
  const int32_t *captures;
  int32_t n_captures;
  int32_t n_buffers;
  void *const *buffers; /* host array of DEVICE int32 buffer pointers */
  int64_t total_shared; /* kernel frame group depot (TotalShared)     */
  int64_t total_local;  /* its local mirror                            */
  int64_t priv_bytes;   /* largest outlined-function frame             */
  int64_t step_limit;   /* operations one thread (the master's sequential
                           code, or one worker's region body) may execute
                           before the team traps OMPDS_TRAP_STEP_LIMIT;
                           <= 0: 20,000,000 (SimOptions::StepLimit's
                           default, Simulator.h:37)                     */
  int64_t stack_slot_bytes;     /* per worker warp: shared-memory slot of the
                                   lanes' data-sharing stacks (1/32 each);
                                   0 when no region nests or globalizes  */
  int64_t stack_overflow_bytes; /* per worker warp: global overflow chain  */
} ompds_program;

/* Checks a program without a GPU (ompds_run_program runs the same check
 * first): opcodes and operands in range, jump targets on instruction
 * boundaries, one stack depth in [0, 32] at every reachable instruction (0 at
 * PARALLEL), no falling off the end, and only variables the executing side
 * addresses (master: depot, local mirror, buffers; region bodies: private
 * frame, captures below the region's nargs, buffers), inside their frames.
 * OMPDS_OK or OMPDS_ERR_INVALID. */
int32_t ompds_program_verify(const ompds_program *prog);

/* Runs a verified program (asynchronous on launch->stream; the descriptor
 * and its arrays may be freed when the call returns).  The tables are copied
 * to the stream's workspace only when they differ from the last ones staged
 * there, so after one eager launch the same program (same tables and
 * buffers) can be captured into a CUDA graph. */
int32_t ompds_run_program(const ompds_launch *launch, const ompds_program *prog,
                          ompds_team_stats *stats_dev, ompds_event *events_dev);

/* The same region end to end from HOST buffers (pinned recommended): copies
 * x,y in, runs, copies y out, on `launch->stream`; synchronises. */
int32_t ompds_run_stream_host(const ompds_launch *launch, int32_t elem,
                              int64_t n, const void *x_host, void *y_host,
                              const void *coef_host, void *x_dev_scratch,
                              void *y_dev_scratch);

/* Counter-based inputs: out[i] = U[-1,1) from splitmix64(seed + first + i)
 * (float64), or (splitmix64(..) % 201) - 100 (int32). */
int32_t ompds_fill_uniform(int32_t elem, void *out, int64_t n, uint64_t seed,
                           int64_t first, void *stream);
/* Order-independent checksum: sum of the elements' bit patterns mod 2^64
 * (float64: 64-bit patterns; int32: sign-extended values).  Writes 8 bytes
 * to `out_dev` (device). */
int32_t ompds_checksum(int32_t elem, const void *data, int64_t n,
                       uint64_t *out_dev, void *stream);

/* Cost of the runtime's building blocks on one SM (north_star: "push/pop +
 * handoff overhead"), measured by one 2-warp CTA with clock64 and
 * %globaltimer.  Inputs (0 = default): iterations; frame_bytes per lane
 * (4..256, multiple of 4; 40 = config 3's level-1 frame); lanes (1..32);
 * max_depth (1..4, default 2 = config 3's two frames per worker warp);
 * seed; frame_bytes * lanes * max_depth <= 8192, the probe's smem slot).
 * Iteration i pushes d_i in [1, max_depth] frames (a hash of i and
 * seed: a run-time depth pattern), stores and loads one word per lane in
 * each and pops them.  Outputs, in cycles per iteration:
 *   smem_baseline / slot        the same accesses at fixed shared addresses /
 *                               through push+pop with frames in the smem slot;
 *   global_baseline / chain     fixed global addresses / push+pop with every
 *                               frame on the global overflow chain;
 *   bookkeeping(_baseline)      push+pop with no frame access (the
 *                               bookkeeping's dependent chain) / without;
 *   handoff                     release + join named barriers, master warp <->
 *                               one worker warp, nothing staged.
 * Cost per push+pop pair = (mode - its baseline) / (pairs / iterations). */
typedef struct ompds_overhead_probe {
  int32_t iterations;  /* in: [1, 1<<20]                          */
  int32_t frame_bytes; /* in                                       */
  int32_t lanes;       /* in                                       */
  int32_t max_depth;   /* in                                       */
  uint32_t seed;       /* in                                       */
  int32_t reserved0;
  double sm_clock_mhz; /* out: clock64 cycles per %globaltimer us  */
  double pairs;        /* out: push/pop pairs executed per mode    */
  double smem_baseline_cycles;
  double slot_cycles;
  double global_baseline_cycles;
  double chain_cycles;
  double bookkeeping_cycles;
  double bookkeeping_baseline_cycles;
  double handoff_cycles;
} ompds_overhead_probe; /* 96 bytes */

/* Runs the probe on the current device and `stream`; synchronises. */
int32_t ompds_probe_overheads(ompds_overhead_probe *io, void *stream);

/* Dynamic smem bytes per CTA the launchers request for a team region with
 * depot `total_shared` (== ompds_shared_footprint for the reference layout). */
int64_t ompds_team_smem_bytes(int64_t depot_capacity, int32_t prealloc_entries);

#ifdef __cplusplus
}
#endif
#endif /* OMPDS_H */
