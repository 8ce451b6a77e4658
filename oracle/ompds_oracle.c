/*
 * ompds_oracle.c -- CPU oracle (TEST INFRASTRUCTURE ONLY; see ompds_oracle.h).
 *
 * Restates, in plain C, the reference semantics the sm_100a path must match.
 * Compiled with -ffp-contract=off so that fp64 rounding follows the written
 * operation order (the one explicit fma() is correctly rounded).
 */
#include "ompds_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ======================================================================== */
/* TeamRuntime  (proj/src/DeviceRuntime.cpp:33-143)                          */
/* ======================================================================== */

enum { PH_UNINIT, PH_IDLE, PH_STAGED, PH_TERM };

typedef struct {
  int32_t prealloc;
  int32_t fail;
  int phase;
  int32_t workers;
  int32_t work_fn;
  int32_t nargs;
  int dynamic; /* ArgsDynamic */
  int32_t active;
  int64_t allocs, frees;
  ompds_event *ev;
  int32_t max_ev, n_ev;
} Rt;

static void rt_log(Rt *t, int32_t kind, int32_t fn, int64_t nargs, int64_t bytes) {
  if (t->ev && t->n_ev < t->max_ev) {
    ompds_event e = {kind, fn, nargs, bytes, 0}; /* no device time on the CPU */
    t->ev[t->n_ev] = e;
  }
  t->n_ev++;
}

/* kernelInit :33-44 */
static int32_t rt_init(Rt *t, int32_t role, int64_t w) {
  if (role != OMPDS_ROLE_MASTER) return OMPDS_TRAP_INIT_FROM_WORKER;
  if (t->phase != PH_UNINIT) return OMPDS_TRAP_INIT_TWICE;
  if (w <= 0) return OMPDS_TRAP_INIT_NO_WORKERS;
  t->phase = PH_IDLE;
  t->workers = (int32_t)w;
  rt_log(t, OMPDS_EV_INIT, -1, w, 0);
  return 0;
}

/* prepareParallel :46-79 */
static int32_t rt_prepare(Rt *t, int32_t role, int32_t fn, int64_t nargs, int *kind,
                          int64_t *live) {
  if (role != OMPDS_ROLE_MASTER) return OMPDS_TRAP_PREPARE_FROM_WORKER;
  if (t->phase == PH_UNINIT) return OMPDS_TRAP_PREPARE_BEFORE_INIT;
  if (t->phase == PH_TERM) return OMPDS_TRAP_PREPARE_AFTER_DEINIT;
  if (t->phase == PH_STAGED || t->active > 0) return OMPDS_TRAP_PREPARE_IN_FLIGHT;
  if (nargs < 0) return OMPDS_TRAP_NEGATIVE_NARGS;
  if (nargs <= t->prealloc) {
    t->dynamic = 0;
    *kind = OMPDS_ADDR_PREALLOC;
    *live = 0;
    rt_log(t, OMPDS_EV_PREPARE_PREALLOC, fn, nargs, 0);
  } else {
    int64_t bytes = nargs * 8;
    if (t->fail) return OMPDS_TRAP_ARGS_ALLOC_FAILED; /* Heap returns 0 */
    t->dynamic = 1;
    t->allocs++;
    *kind = OMPDS_ADDR_DYNAMIC;
    *live = bytes;
    rt_log(t, OMPDS_EV_PREPARE_DYNAMIC, fn, nargs, bytes);
  }
  t->work_fn = fn;
  t->nargs = (int32_t)nargs;
  t->phase = PH_STAGED;
  return 0;
}

/* kernelParallel :81-100 */
static int32_t rt_parallel(Rt *t, int32_t role, int32_t *fn, int *kind, int *part) {
  if (role != OMPDS_ROLE_WORKER) return OMPDS_TRAP_PARALLEL_FROM_MASTER;
  if (t->phase == PH_TERM) {
    *fn = -1;
    *kind = OMPDS_ADDR_NULL;
    *part = 0;
    return 0;
  }
  if (t->phase != PH_STAGED) return OMPDS_TRAP_PARALLEL_NOT_STAGED;
  *fn = t->work_fn;
  *kind = t->dynamic ? OMPDS_ADDR_DYNAMIC : OMPDS_ADDR_PREALLOC;
  *part = 1;
  t->active++;
  rt_log(t, OMPDS_EV_FETCH, t->work_fn, 0, 0);
  return 0;
}

/* endParallel :102-128 */
static int32_t rt_end(Rt *t, int32_t role) {
  if (role != OMPDS_ROLE_WORKER) return OMPDS_TRAP_END_FROM_MASTER;
  if (t->phase != PH_STAGED || t->active <= 0) return OMPDS_TRAP_END_NOT_ACTIVE;
  t->active--;
  rt_log(t, OMPDS_EV_RETIRE, -1, t->active, 0);
  if (t->active == 0) {
    if (t->dynamic) {
      t->frees++;
      rt_log(t, OMPDS_EV_DYNAMIC_FREE, -1, 0, (int64_t)t->nargs * 8);
    }
    t->work_fn = -1;
    t->dynamic = 0;
    t->nargs = 0;
    t->phase = PH_IDLE;
  }
  return 0;
}

/* kernelDeinit :130-143 */
static int32_t rt_deinit(Rt *t, int32_t role) {
  if (role != OMPDS_ROLE_MASTER) return OMPDS_TRAP_DEINIT_FROM_WORKER;
  if (t->phase == PH_UNINIT) return OMPDS_TRAP_DEINIT_BEFORE_INIT;
  if (t->phase == PH_STAGED || t->active > 0) return OMPDS_TRAP_DEINIT_IN_FLIGHT;
  if (t->phase == PH_TERM) return OMPDS_TRAP_DEINIT_TWICE;
  t->phase = PH_TERM;
  rt_log(t, OMPDS_EV_DEINIT, -1, 0, 0);
  return 0;
}

int32_t orc_rt_replay(const ompds_runtime_config *cfg, const ompds_rt_call *calls,
                      int32_t n, ompds_rt_result *res, ompds_event *events,
                      int32_t max_events, ompds_rt_summary *sum) {
  Rt t;
  memset(&t, 0, sizeof(t));
  t.prealloc = cfg->prealloc_entries;
  t.fail = cfg->fail_dynamic_alloc;
  t.work_fn = -1;
  t.ev = events;
  t.max_ev = max_events;
  int32_t fn_seq = 0;
  for (int32_t i = 0; i < n; ++i) {
    ompds_rt_result r;
    memset(&r, 0, sizeof(r));
    r.wf = -1;
    int kind = 0, part = 0;
    int64_t live = 0;
    int32_t fn = -1;
    switch (calls[i].op) {
    case OMPDS_OP_KERNEL_INIT:
      r.status = rt_init(&t, calls[i].role, calls[i].arg);
      break;
    case OMPDS_OP_PREPARE_PARALLEL:
      r.status = rt_prepare(&t, calls[i].role, fn_seq, calls[i].arg, &kind, &live);
      if (!r.status) {
        fn_seq++;
        r.addr_kind = kind;
        r.live_bytes = live;
      }
      break;
    case OMPDS_OP_KERNEL_PARALLEL:
      r.status = rt_parallel(&t, calls[i].role, &fn, &kind, &part);
      if (!r.status) {
        r.wf = fn;
        r.addr_kind = kind;
        r.participate = part;
      }
      break;
    case OMPDS_OP_END_PARALLEL:
      r.status = rt_end(&t, calls[i].role);
      break;
    case OMPDS_OP_KERNEL_DEINIT:
      r.status = rt_deinit(&t, calls[i].role);
      break;
    default:
      r.status = OMPDS_ERR_INVALID;
    }
    r.heap_live = t.dynamic ? 1 : 0;
    res[i] = r;
  }
  memset(sum, 0, sizeof(*sum));
  sum->workers = t.workers;
  sum->terminated = t.phase == PH_TERM;
  sum->dynamic_allocs = t.allocs;
  sum->dynamic_frees = t.frees;
  sum->leaked_blocks = t.allocs - t.frees;
  sum->n_events = t.n_ev;
  return 0;
}

/* ======================================================================== */
/* Frame pipeline (proj/src/LoweringPasses.cpp)                              */
/* ======================================================================== */

typedef struct {
  int64_t size;
  int32_t align;
  int shared;
  int32_t *own; /* owner var indices */
  int32_t n_own;
  int32_t var;  /* defining var */
} OSlot;

static int64_t r8(int64_t n) { return (n + 7) & ~(int64_t)7; }

/* lowerSharedFrames :345-380 */
static void o_lower(OSlot *s, int32_t ns, const ompds_frame_var *v) {
  for (int32_t i = 0; i < ns; ++i)
    for (int32_t k = 0; k < s[i].n_own; ++k)
      if (v[s[i].own[k]].flags & OMPDS_VAR_ESCAPES) s[i].shared = 1;
}

/* colorStack / colorFunction :458-538 (positions doubled, see ompds.h) */
static void o_color(OSlot *s, int32_t ns, const ompds_frame_var *v) {
  int64_t *first = malloc(sizeof(int64_t) * (ns ? ns : 1));
  int64_t *last = malloc(sizeof(int64_t) * (ns ? ns : 1));
  int *pinned = malloc(sizeof(int) * (ns ? ns : 1));
  int32_t *ids = malloc(sizeof(int32_t) * (ns ? ns : 1));
  for (int32_t i = 0; i < ns; ++i) {
    const ompds_frame_var *x = &v[s[i].var];
    first[i] = last[i] = -1;
    pinned[i] = (x->flags & OMPDS_VAR_PINNED) != 0;
    if (x->flags & OMPDS_VAR_ESCAPES) {
      pinned[i] = 0;
      if (x->def_pos >= 0) first[i] = last[i] = 2 * (int64_t)x->def_pos + 1;
    } else if (x->live_first >= 0) {
      first[i] = 2 * (int64_t)x->live_first;
      last[i] = 2 * (int64_t)x->live_last;
    }
  }
  for (int32_t i = 0; i < ns; ++i) {
    /* one pass per member function, in first-appearance order */
    int32_t f = v[s[i].var].func;
    int seen = 0;
    for (int32_t j = 0; j < i; ++j)
      if (v[s[j].var].func == f) seen = 1;
    if (seen) continue;
    int32_t ni = 0;
    for (int32_t j = 0; j < ns; ++j)
      if (v[s[j].var].func == f) ids[ni++] = j;
    if (ni < 2) continue;
    for (int32_t a = 0; a < ni; ++a) {
      int32_t sa = ids[a];
      if (s[sa].shared || pinned[sa] || s[sa].n_own == 0) continue;
      for (int32_t b = a + 1; b < ni; ++b) {
        int32_t sb = ids[b];
        if (s[sb].n_own == 0 || s[sb].shared || pinned[sb]) continue;
        if (first[sb] < 0 || first[sa] < 0) continue;
        if (!(last[sa] < first[sb] || last[sb] < first[sa])) continue;
        if (s[sb].size > s[sa].size) s[sa].size = s[sb].size;
        if (s[sb].align > s[sa].align) s[sa].align = s[sb].align;
        for (int32_t k = 0; k < s[sb].n_own; ++k) s[sa].own[s[sa].n_own++] = s[sb].own[k];
        s[sb].n_own = 0;
        if (first[sb] < first[sa]) first[sa] = first[sb];
        if (last[sb] > last[sa]) last[sa] = last[sb];
      }
    }
  }
  free(first);
  free(last);
  free(pinned);
  free(ids);
}

int32_t orc_layout_build(const ompds_frame_var *vars, int32_t n_vars,
                         int32_t n_groups, int32_t pipeline,
                         ompds_depot_layout *layouts, ompds_depot_slot *slots,
                         int32_t max_slots, int32_t *owners, int32_t max_owners) {
  int32_t ns_out = 0, no_out = 0;
  int32_t *own_pool = malloc(sizeof(int32_t) * (size_t)(n_vars ? n_vars : 1) *
                             (size_t)(n_vars ? n_vars : 1));
  OSlot *s = malloc(sizeof(OSlot) * (n_vars ? n_vars : 1));
  for (int32_t g = 0; g < n_groups; ++g) {
    /* buildDepots :264-305 */
    int32_t ns = 0;
    for (int32_t i = 0; i < n_vars; ++i) {
      if (vars[i].group != g) continue;
      s[ns].size = r8(vars[i].bytes);
      s[ns].align = 8;
      s[ns].shared = 0;
      s[ns].own = own_pool + (size_t)ns * (size_t)n_vars;
      s[ns].own[0] = i;
      s[ns].n_own = 1;
      s[ns].var = i;
      ns++;
    }
    if (pipeline == OMPDS_PIPELINE_DEFAULT) {
      o_lower(s, ns, vars);
      o_color(s, ns, vars);
    } else if (pipeline == OMPDS_PIPELINE_O0) {
      o_lower(s, ns, vars);
    } else {
      o_color(s, ns, vars);
      o_lower(s, ns, vars);
    }
    /* repackOffsets :556-593 */
    ompds_depot_layout *L = &layouts[g];
    memset(L, 0, sizeof(*L));
    L->slot_begin = ns_out;
    L->overlap_slot = -1;
    int64_t off = 0;
    for (int32_t i = 0; i < ns; ++i) {
      if (s[i].n_own == 0) continue;
      if (ns_out >= max_slots || no_out + s[i].n_own > max_owners) {
        free(own_pool);
        free(s);
        return OMPDS_ERR_CAPACITY;
      }
      ompds_depot_slot *o = &slots[ns_out++];
      o->offset = off;
      o->size = s[i].size;
      o->align = s[i].align;
      o->shared = s[i].shared;
      o->owner_begin = no_out;
      o->n_owners = s[i].n_own;
      for (int32_t k = 0; k < s[i].n_own; ++k) owners[no_out++] = s[i].own[k];
      if (s[i].shared && s[i].n_own > 1 && L->overlap_slot < 0) L->overlap_slot = L->n_slots;
      if (s[i].shared) L->has_shared_depot = 1;
      off += s[i].size;
      L->n_slots++;
    }
    L->total_local = L->total_shared = off;
  }
  free(own_pool);
  free(s);
  return 0;
}

/* ======================================================================== */
/* Occupancy (proj/src/Occupancy.cpp:77-105)                                 */
/* ======================================================================== */

static int64_t mn(int64_t a, int64_t b) { return a < b ? a : b; }

/* Occupancy.cpp:77-88; B200 row (EXTENSION): registers per warp in
 * allocation units, each warp inside one register sub-partition. */
static int64_t o_teams_by_regs(const ompds_gpu_spec *g, int32_t regs, int32_t threads) {
  if (regs <= 0 || threads <= 0) return 0;
  if (g->reg_alloc_unit <= 0) return g->registers_per_sm / ((int64_t)regs * threads);
  int64_t u = g->reg_alloc_unit;
  int64_t warp_regs = (((int64_t)regs + u - 1) / u) * u * g->warp_size;
  int64_t warps = ((int64_t)threads + g->warp_size - 1) / g->warp_size;
  int64_t parts = g->reg_partitions > 0 ? g->reg_partitions : 1;
  int64_t per_part = (g->registers_per_sm / parts) / warp_regs;
  return parts * per_part / warps;
}

int32_t orc_occupancy_for(const ompds_gpu_spec *g, int64_t fp, int32_t regs,
                          int32_t threads, ompds_occupancy *o) {
  o->teams_by_regs = o_teams_by_regs(g, regs, threads);
  int64_t per = fp > 0 ? fp + g->reserved_smem_per_block : 0;
  o->teams_by_smem = per > 0 ? g->shared_bytes_per_sm / per : 0;
  o->potential = mn(o->teams_by_regs, g->max_blocks_per_sm);
  if (g->max_threads_per_sm > 0 && threads > 0)
    o->potential = mn(o->potential, g->max_threads_per_sm / threads);
  o->actual = mn(o->potential, o->teams_by_smem);
  o->smem_used = o->potential * fp;
  return 0;
}

int64_t orc_max_regs_for_teams(const ompds_gpu_spec *g, int64_t teams, int32_t threads) {
  if (teams <= 0 || threads <= 0) return g->max_regs_per_thread;
  if (g->reg_alloc_unit > 0) {
    int64_t r;
    for (r = g->max_regs_per_thread / g->reg_alloc_unit * g->reg_alloc_unit; r > 0;
         r -= g->reg_alloc_unit)
      if (o_teams_by_regs(g, (int32_t)r, threads) >= teams) break;
    return r;
  }
  return mn(g->registers_per_sm / (teams * threads), g->max_regs_per_thread);
}

int64_t orc_max_shared_vars(const ompds_gpu_spec *g, int64_t teams) {
  if (teams <= 0) return 0;
  int64_t budget = g->shared_bytes_per_sm / teams - g->reserved_smem_per_block;
  int64_t fixed = 16 + 160 + 49 + 8;
  if (budget < fixed) return 0;
  return (budget - fixed) / 8;
}

/* ======================================================================== */
/* Region semantics                                                          */
/* ======================================================================== */

uint64_t orc_splitmix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

void orc_fill(int32_t elem, void *out, int64_t n, uint64_t seed, int64_t first) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    uint64_t z = orc_splitmix64(seed + (uint64_t)(first + i));
    if (elem)
      ((double *)out)[i] = (double)(z >> 11) * 0x1p-52 - 1.0;
    else
      ((int32_t *)out)[i] = (int32_t)(z % 201) - 100;
  }
}

uint64_t orc_checksum(int32_t elem, const void *data, int64_t n) {
  uint64_t acc = 0;
#pragma omp parallel for reduction(+ : acc) schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    if (elem) {
      uint64_t b;
      memcpy(&b, (const double *)data + i, 8);
      acc += b;
    } else {
      acc += (uint64_t)(int64_t)((const int32_t *)data)[i];
    }
  }
  return acc;
}

static int32_t wrap_add(int32_t a, int32_t b) { return (int32_t)((uint32_t)a + (uint32_t)b); }
static int32_t wrap_mul(int32_t a, int32_t b) { return (int32_t)((uint32_t)a * (uint32_t)b); }

/* SequentialOracle.cpp:150-172 (bare parallel: every worker runs the body
 * once) inside the team's sequential loop; teams run independently
 * (execTeam :182-196). */
void orc_regions(int32_t elem, int32_t teams, int32_t workers, int32_t regions, void *a) {
  for (int32_t t = 0; t < teams; ++t) {
    int32_t c1 = 1, c2 = 2;
    if (elem) {
      double c3 = 3.0, c4 = 4.0;
      for (int32_t r = 0; r < regions; ++r) {
        for (int32_t w = 0; w < workers; ++w) {
          double sum = ((double)(c1 + c2) + c3) + c4;
          double *p = (double *)a + (int64_t)t * workers + w;
          *p = *p + sum;
        }
        c4 = c4 + 1.0;
      }
    } else {
      int32_t c3 = 3, c4 = 4;
      for (int32_t r = 0; r < regions; ++r) {
        for (int32_t w = 0; w < workers; ++w) {
          int32_t sum = wrap_add(wrap_add(wrap_add(c1, c2), c3), c4);
          int32_t *p = (int32_t *)a + (int64_t)t * workers + w;
          *p = wrap_add(*p, sum);
        }
        c4 = wrap_add(c4, 1);
      }
    }
  }
}

/* Master loop d[k] = 3k+1 then the parallel-for body; the cyclic schedule
 * (AstLowering.cpp:429-462) only permutes independent iterations. */
void orc_shared_array(int32_t elem, int64_t n, void *a) {
  if (elem) {
    double d[256];
    for (int k = 0; k < 256; ++k) d[k] = (double)(3 * k + 1);
    for (int64_t i = 0; i < n; ++i) ((double *)a)[i] = ((double *)a)[i] + d[i & 255];
  } else {
    int32_t d[256];
    for (int k = 0; k < 256; ++k) d[k] = 3 * k + 1;
    for (int64_t i = 0; i < n; ++i)
      ((int32_t *)a)[i] = wrap_add(((int32_t *)a)[i], d[i & 255]);
  }
}

void orc_stream(int32_t elem, int64_t n, const void *x, void *y, const void *coef,
                int32_t threads) {
#ifdef _OPENMP
  if (threads <= 0) threads = omp_get_max_threads();
#else
  (void)threads;
#endif
  if (elem) {
    const double *c = (const double *)coef;
    double s = c[1];
    for (int k = 2; k < 8; ++k) s = s + c[k];
    const double c1 = c[0];
    const double *xs = (const double *)x;
    double *ys = (double *)y;
#pragma omp parallel for schedule(static) num_threads(threads)
    for (int64_t i = 0; i < n; ++i) ys[i] = fma(c1, xs[i], ys[i]) + s;
  } else {
    const int32_t *c = (const int32_t *)coef;
    int32_t s = c[1];
    for (int k = 2; k < 8; ++k) s = wrap_add(s, c[k]);
    const int32_t c1 = c[0];
    const int32_t *xs = (const int32_t *)x;
    int32_t *ys = (int32_t *)y;
#pragma omp parallel for schedule(static) num_threads(threads)
    for (int64_t i = 0; i < n; ++i) ys[i] = wrap_add(ys[i], wrap_add(wrap_mul(c1, xs[i]), s));
  }
}

/* Config 4/5 checker over the element range [lo, hi) without materialising
 * x or y: each element is regenerated from the counter-based inputs
 * (orc_fill's formula), run through the region body once (orc_stream's
 * formula) and its bit pattern summed mod 2^64 (orc_checksum's), OpenMP over
 * `threads` (<= 0: all).  Equal to fill + stream + checksum of the range. */
uint64_t orc_stream_checksum(int32_t elem, int64_t lo, int64_t hi, uint64_t seed_x,
                             uint64_t seed_y, const void *coef, int32_t threads) {
#ifdef _OPENMP
  if (threads <= 0) threads = omp_get_max_threads();
#else
  (void)threads;
#endif
  uint64_t acc = 0;
  if (elem) {
    const double *c = (const double *)coef;
    double s = c[1];
    for (int k = 2; k < 8; ++k) s = s + c[k];
    const double c1 = c[0];
#pragma omp parallel for reduction(+ : acc) schedule(static) num_threads(threads)
    for (int64_t i = lo; i < hi; ++i) {
      const double x = (double)(orc_splitmix64(seed_x + (uint64_t)i) >> 11) * 0x1p-52 - 1.0;
      const double y = (double)(orc_splitmix64(seed_y + (uint64_t)i) >> 11) * 0x1p-52 - 1.0;
      const double r = fma(c1, x, y) + s;
      uint64_t b;
      memcpy(&b, &r, 8);
      acc += b;
    }
  } else {
    const int32_t *c = (const int32_t *)coef;
    int32_t s = c[1];
    for (int k = 2; k < 8; ++k) s = wrap_add(s, c[k]);
    const int32_t c1 = c[0];
#pragma omp parallel for reduction(+ : acc) schedule(static) num_threads(threads)
    for (int64_t i = lo; i < hi; ++i) {
      const int32_t x = (int32_t)(orc_splitmix64(seed_x + (uint64_t)i) % 201) - 100;
      const int32_t y = (int32_t)(orc_splitmix64(seed_y + (uint64_t)i) % 201) - 100;
      acc += (uint64_t)(int64_t)wrap_add(y, wrap_add(wrap_mul(c1, x), s));
    }
  }
  return acc;
}

void orc_nested(int32_t elem, int32_t teams, int32_t workers, int32_t regions, void *a) {
  for (int32_t t = 0; t < teams; ++t) {
    int32_t c = 1;
    for (int32_t r = 0; r < regions; ++r) {
      for (int32_t w = 0; w < workers; ++w) {
        int32_t e = wrap_add(w, c);
        if (elem) {
          double *p = (double *)a + (int64_t)t * workers + w;
          double v[4];
          double s = (double)(w % 8 + 1);
          for (int j = 0; j < 4; ++j) v[j] = s * (double)(j + 1);
          double f = (double)e + v[3];      /* L2 */
          *p = *p + (f + (double)c);        /* L3 */
          f = f * 2.0;
          v[0] = f;
          e = wrap_add(e, 1);
          *p = *p + (v[0] + (double)e);     /* back in L1 */
        } else {
          int32_t *p = (int32_t *)a + (int64_t)t * workers + w;
          int32_t v[4];
          int32_t s = w % 8 + 1;
          for (int j = 0; j < 4; ++j) v[j] = wrap_mul(s, j + 1);
          int32_t f = wrap_add(e, v[3]);
          *p = wrap_add(*p, wrap_add(f, c));
          f = wrap_mul(f, 2);
          v[0] = f;
          e = wrap_add(e, 1);
          *p = wrap_add(*p, wrap_add(v[0], e));
        }
      }
      c = wrap_add(c, 1);
    }
  }
}

int32_t orc_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ======================================================================== */
/* Data-sharing stack placement (EXTENSION)                                  */
/* ======================================================================== */

int32_t orc_ds_stack(int64_t slot_cap, int64_t ovf_cap, const int64_t *ops,
                     const int32_t *lanes, int32_t n, int32_t *in_smem,
                     int64_t *offset, int32_t *max_depth, int64_t *high_water) {
  int64_t top = 0, otop = 0, hw = 0;
  int32_t depth = 0, md = 0;
  /* frame stack for pops */
  int32_t *fs = malloc(sizeof(int32_t) * (n ? n : 1));
  int64_t *fo = malloc(sizeof(int64_t) * (n ? n : 1));
  int32_t status = 0;
  for (int32_t i = 0; i < n; ++i) {
    in_smem[i] = -1;
    offset[i] = -1;
    if (ops[i] > 0) {
      int64_t need = r8(ops[i] * lanes[i]);
      if (otop == 0 && top + need <= slot_cap) {
        in_smem[i] = 1;
        offset[i] = top;
        top += need;
      } else if (otop + need <= ovf_cap) {
        in_smem[i] = 0;
        offset[i] = otop;
        otop += need;
      } else {
        status = OMPDS_TRAP_STACK_OVERFLOW;
        break;
      }
      fs[depth] = in_smem[i];
      fo[depth] = offset[i];
      depth++;
      if (depth > md) md = depth;
      if (top + otop > hw) hw = top + otop;
    } else {
      if (depth == 0) {
        status = OMPDS_TRAP_STACK_UNDERFLOW;
        break;
      }
      depth--;
      if (fs[depth]) top = fo[depth];
      else otop = fo[depth];
    }
  }
  free(fs);
  free(fo);
  *max_depth = md;
  *high_water = hw;
  return status;
}
