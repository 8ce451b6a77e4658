// ompds_host.cpp -- host half of the C ABI (include/ompds.h): trap strings,
// the frame-layout descriptor builder and the occupancy model.  No CUDA here;
// these are the compile-time / launch-planning parts of the path that the
// reference also runs on the host (proj/src/LoweringPasses.cpp,
// proj/src/Occupancy.cpp), restated from their published behaviour.
#include "../../include/ompds.h"

#include <algorithm>
#include <cstring>
#include <vector>

namespace {

// proj/src/DeviceRuntime.cpp:33-143, byte for byte.
const char *const kTrapStrings[] = {
    "",
    "protocol error: kernel_init from a worker thread",
    "protocol error: kernel_init called twice",
    "protocol error: kernel_init with no workers",
    "protocol error: prepare_parallel from a worker thread",
    "protocol error: prepare_parallel before init",
    "protocol error: prepare_parallel after deinit",
    "protocol error: prepare_parallel while a region is in flight",
    "protocol error: negative shared-args count",
    "shared-args-alloc-failed",
    "protocol error: kernel_parallel from the master thread",
    "protocol error: kernel_parallel with no staged region",
    "protocol error: end_parallel from the master thread",
    "protocol error: end_parallel with no active region",
    "protocol error: kernel_deinit from a worker thread",
    "protocol error: kernel_deinit before init",
    "protocol error: kernel_deinit while a region is in flight",
    "protocol error: kernel_deinit called twice",
    "data-sharing stack overflow",
    "data-sharing stack underflow",
    "out-of-bounds access",
    "step limit exceeded", // Simulator.cpp:820
};

int64_t roundUp8(int64_t n) { return (n + 7) & ~int64_t(7); }

// Working state of one depot slot while the pipeline runs.
struct Slot {
  int64_t size = 0;
  int32_t align = 8;
  bool shared = false;
  std::vector<int32_t> owners; // var indices; empty = dropped by repacking
};

struct Group {
  std::vector<Slot> slots;
  std::vector<int32_t> slot_var; // slot -> defining var
};

// lower-shared-frames (LoweringPasses.cpp:345-380): slots of escaping
// variables become shared-resident.  Coloring may have merged other owners
// into such a slot; they are dragged along (the hazard the audit catches).
void lowerShared(Group &g, const ompds_frame_var *vars) {
  for (Slot &s : g.slots)
    for (int32_t v : s.owners)
      if (vars[v].flags & OMPDS_VAR_ESCAPES)
        s.shared = true;
}

// color-stack (LoweringPasses.cpp:458-538), per member function, restated
// as first-fit interval packing.  Each candidate slot (local, unpinned, with
// a live interval) is visited in slot order and joins the earliest packing
// group -- led by an earlier candidate -- whose hull (the span from the
// first to the last use of everything packed into it so far) it does not
// touch; otherwise it starts a group of its own.  Packing a slot into a
// group keeps the larger size and alignment and widens the group's hull.
// This is the reference's leader-by-leader scan seen from the other side:
// when slot b is visited, every earlier leader's hull holds exactly the
// slots before b that the reference would have merged into it by then, and
// b lands in the first leader that the reference's scan would give it to.
// Slots with no use are left alone (repacking drops the empty ones).
void colorStack(Group &g, const ompds_frame_var *vars) {
  struct Span {
    int64_t lo, hi; // doubled positions, inclusive
  };
  struct Packing {
    int32_t leader; // slot receiving the packed owners
    Span hull;
  };
  std::vector<int32_t> funcs; // member functions, first-appearance order
  for (int32_t v : g.slot_var)
    if (std::find(funcs.begin(), funcs.end(), vars[v].func) == funcs.end())
      funcs.push_back(vars[v].func);
  for (int32_t fn : funcs) {
    int32_t in_func = 0;
    for (int32_t v : g.slot_var)
      in_func += vars[v].func == fn;
    if (in_func < 2)
      continue; // a single frame index: nothing to color (SlotOfValue.size() < 2)
    std::vector<Packing> packs;
    for (size_t si = 0; si < g.slot_var.size(); ++si) {
      const ompds_frame_var &v = vars[g.slot_var[si]];
      Slot &slot = g.slots[si];
      if (v.func != fn || slot.shared)
        continue;
      // the span of the frame value's uses; an escaping alloca's only direct
      // use is the address-space cast right after it (doubled 2*def+1)
      Span use{-1, -1};
      bool pinned = false;
      if (v.flags & OMPDS_VAR_ESCAPES) {
        if (v.def_pos >= 0)
          use = {2 * int64_t(v.def_pos) + 1, 2 * int64_t(v.def_pos) + 1};
      } else {
        pinned = (v.flags & OMPDS_VAR_PINNED) != 0;
        if (v.live_first >= 0)
          use = {2 * int64_t(v.live_first), 2 * int64_t(v.live_last)};
      }
      if (pinned || use.lo < 0)
        continue; // never packed, never a leader
      Packing *home = nullptr;
      for (Packing &pk : packs)
        if (use.hi < pk.hull.lo || pk.hull.hi < use.lo) {
          home = &pk;
          break;
        }
      if (!home) {
        packs.push_back({static_cast<int32_t>(si), use});
        continue;
      }
      Slot &lead = g.slots[static_cast<size_t>(home->leader)];
      lead.size = std::max(lead.size, slot.size);
      lead.align = std::max(lead.align, slot.align);
      lead.owners.insert(lead.owners.end(), slot.owners.begin(), slot.owners.end());
      slot.owners.clear();
      home->hull = {std::min(home->hull.lo, use.lo), std::max(home->hull.hi, use.hi)};
    }
  }
}

} // namespace

extern "C" {

const char *ompds_trap_reason(int32_t code) {
  if (code < 0 ||
      code >= static_cast<int32_t>(sizeof(kTrapStrings) / sizeof(kTrapStrings[0])))
    return code == OMPDS_ERR_CUDA       ? "cuda error"
           : code == OMPDS_ERR_INVALID  ? "invalid argument"
           : code == OMPDS_ERR_CAPACITY ? "output capacity exceeded"
                                        : "unknown status";
  return kTrapStrings[code];
}

uint32_t ompds_version(void) { return 0x00010000u; }

int64_t ompds_dynamic_args_bytes(int64_t nargs, int32_t prealloc_entries) {
  return nargs <= prealloc_entries ? 0 : nargs * OMPDS_SHARED_ARG_ENTRY_BYTES;
}

int64_t ompds_shared_footprint(int64_t total_shared, int32_t prealloc_entries) {
  return total_shared + int64_t(prealloc_entries) * OMPDS_SHARED_ARG_ENTRY_BYTES +
         OMPDS_RUNTIME_PRIVATE_BYTES;
}

int32_t ompds_layout_build(const ompds_frame_var *vars, int32_t n_vars,
                           int32_t n_groups, int32_t pipeline,
                           ompds_depot_layout *layouts,
                           ompds_depot_slot *slots, int32_t max_slots,
                           int32_t *owners, int32_t max_owners) {
  if (n_vars < 0 || n_groups < 0 || (n_vars && !vars) ||
      (n_groups && !layouts) || pipeline < OMPDS_PIPELINE_DEFAULT ||
      pipeline > OMPDS_PIPELINE_BAD_ORDER)
    return OMPDS_ERR_INVALID;
  for (int32_t i = 0; i < n_vars; ++i)
    if (vars[i].group < 0 || vars[i].group >= n_groups || vars[i].bytes < 0)
      return OMPDS_ERR_INVALID;

  // build-depots (LoweringPasses.cpp:264-305): one slot per alloca in group
  // emission order, size roundUp8, align 8.
  std::vector<Group> groups(static_cast<size_t>(n_groups));
  for (int32_t i = 0; i < n_vars; ++i) {
    Group &g = groups[static_cast<size_t>(vars[i].group)];
    Slot s;
    s.size = roundUp8(vars[i].bytes);
    s.owners.push_back(i);
    g.slots.push_back(std::move(s));
    g.slot_var.push_back(i);
  }
  for (Group &g : groups) {
    switch (pipeline) {
    case OMPDS_PIPELINE_DEFAULT: // planFor(Default) :38-43
      lowerShared(g, vars);
      colorStack(g, vars);
      break;
    case OMPDS_PIPELINE_O0: // :44-48, no coloring
      lowerShared(g, vars);
      break;
    case OMPDS_PIPELINE_BAD_ORDER: // :49-54, coloring before lowering
      colorStack(g, vars);
      lowerShared(g, vars);
      break;
    }
  }

  // repack-offsets (:556-593): drop emptied slots, prefix-sum offsets,
  // TotalShared mirrors TotalLocal.
  int32_t ns = 0, no = 0;
  for (int32_t gi = 0; gi < n_groups; ++gi) {
    Group &g = groups[static_cast<size_t>(gi)];
    ompds_depot_layout &L = layouts[gi];
    std::memset(&L, 0, sizeof(L));
    L.slot_begin = ns;
    L.overlap_slot = -1;
    int64_t off = 0;
    for (const Slot &s : g.slots) {
      if (s.owners.empty())
        continue;
      if (ns >= max_slots || no + static_cast<int32_t>(s.owners.size()) > max_owners)
        return OMPDS_ERR_CAPACITY;
      ompds_depot_slot &o = slots[ns];
      o.offset = off;
      o.size = s.size;
      o.align = s.align;
      o.shared = s.shared ? 1 : 0;
      o.owner_begin = no;
      o.n_owners = static_cast<int32_t>(s.owners.size());
      for (int32_t v : s.owners)
        owners[no++] = v;
      // findSharedLocalOverlap (IR.cpp:228-242): a shared slot with >1 owner.
      if (s.shared && s.owners.size() > 1 && L.overlap_slot < 0)
        L.overlap_slot = L.n_slots;
      if (s.shared)
        L.has_shared_depot = 1;
      off += s.size;
      ++L.n_slots;
      ++ns;
    }
    L.total_local = off;
    L.total_shared = off;
  }
  return OMPDS_OK;
}

//===----------------------------------------------------------------------===//
// Occupancy (proj/src/Occupancy.cpp:14-105) plus a measured-B200 row.
//===----------------------------------------------------------------------===//

int32_t ompds_gpu_spec_get(const char *name, ompds_gpu_spec *out) {
  if (!name || !out)
    return OMPDS_ERR_INVALID;
  struct Row {
    const char *name;
    ompds_gpu_spec spec;
  };
  static const Row rows[] = {
      {"k40-16k", {16384, 65536, 16, 32, 255, 0, 0, 0, 0}},
      {"k40-32k", {32768, 65536, 16, 32, 255, 0, 0, 0, 0}},
      {"k40-48k", {49152, 65536, 16, 32, 255, 0, 0, 0, 0}},
      {"p100", {65536, 65536, 32, 32, 255, 0, 0, 0, 0}},
      // B200 (sm_100a): 228 KB smem per SM with 1 KB reserved per CTA,
      // 64K registers in 4 sub-partitions of 16K, allocated per warp in
      // units of 256 (8 per thread) from one sub-partition, 32 CTAs and
      // 2048 threads per SM.
      {"b200", {233472, 65536, 32, 32, 255, 2048, 1024, 8, 4}},
  };
  for (const Row &r : rows)
    if (std::strcmp(r.name, name) == 0) {
      *out = r.spec;
      return OMPDS_OK;
    }
  return OMPDS_ERR_INVALID;
}

// Teams of `threads` threads that fit the register file.  Reference model:
// registers_per_sm / (regs x threads).  With an allocation unit: per warp,
// regs rounded up to the unit; with sub-partitions: each warp takes its
// registers from one sub-partition, so whole warps are counted per
// sub-partition first (a 40-register 64-thread team: 16K / 1280 = 12 warps
// per SMSP, 48 per SM = 24 teams, not 65536 / 2560 = 25).
static int64_t ompds_teams_by_regs(const ompds_gpu_spec *g, int32_t regs, int32_t threads) {
  if (regs <= 0 || threads <= 0)
    return 0;
  if (g->reg_alloc_unit <= 0)
    return g->registers_per_sm / (int64_t(regs) * threads);
  const int64_t u = g->reg_alloc_unit;
  const int64_t per_warp = (int64_t(regs) + u - 1) / u * u * g->warp_size;
  const int64_t warps = (int64_t(threads) + g->warp_size - 1) / g->warp_size;
  const int64_t parts = g->reg_partitions > 0 ? g->reg_partitions : 1;
  const int64_t warps_per_sm = parts * ((g->registers_per_sm / parts) / per_warp);
  return warps_per_sm / warps;
}

int32_t ompds_occupancy_for(const ompds_gpu_spec *g, int64_t footprint,
                            int32_t regs, int32_t threads, ompds_occupancy *o) {
  if (!g || !o)
    return OMPDS_ERR_INVALID;
  o->teams_by_regs = ompds_teams_by_regs(g, regs, threads);
  const int64_t per_team_smem = footprint > 0 ? footprint + g->reserved_smem_per_block : 0;
  o->teams_by_smem = per_team_smem > 0 ? g->shared_bytes_per_sm / per_team_smem : 0;
  o->potential = std::min(o->teams_by_regs, g->max_blocks_per_sm);
  if (g->max_threads_per_sm > 0 && threads > 0)
    o->potential = std::min<int64_t>(o->potential, g->max_threads_per_sm / threads);
  o->actual = std::min(o->potential, o->teams_by_smem);
  o->smem_used = o->potential * footprint;
  return OMPDS_OK;
}

int64_t ompds_max_regs_for_teams(const ompds_gpu_spec *g, int64_t teams,
                                 int32_t threads) {
  if (!g)
    return 0;
  if (teams <= 0 || threads <= 0)
    return g->max_regs_per_thread;
  if (g->reg_alloc_unit > 0) { // the largest unit multiple that still fits
    int64_t r = g->max_regs_per_thread / g->reg_alloc_unit * g->reg_alloc_unit;
    while (r > 0 && ompds_teams_by_regs(g, static_cast<int32_t>(r), threads) < teams)
      r -= g->reg_alloc_unit;
    return r;
  }
  return std::min<int64_t>(g->registers_per_sm / (teams * threads),
                           g->max_regs_per_thread);
}

int64_t ompds_max_shared_vars(const ompds_gpu_spec *g, int64_t teams) {
  if (!g || teams <= 0)
    return 0;
  const int64_t budget = g->shared_bytes_per_sm / teams - g->reserved_smem_per_block;
  // scalars fixture with no variables (wf.addr + args.addr) + a loop counter
  const int64_t fixed =
      ompds_shared_footprint(16, OMPDS_DEFAULT_PREALLOC_ENTRIES) + 8;
  if (budget < fixed)
    return 0;
  return (budget - fixed) / 8;
}

} // extern "C"
