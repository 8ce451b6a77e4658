// ref_golden.cpp -- TEST INFRASTRUCTURE ONLY.
//
// Links the unmodified reference library (omplab_core, compiled in place from
// /root/reference/proj/src by oracle/Makefile) and dumps golden vectors for
// the data-sharing hot path into tests/golden/*.json:
//
//   corpus.json     every proj/programs/*.ompk: AST (+sharing), frame layouts
//                   for the default / O0 / bad-order pipelines, the simulator's
//                   outputs, barrier/alloc statistics and per-team runtime
//                   event logs at several launches, and the sequential oracle's
//                   outputs (proj/src/Simulator.cpp, SequentialOracle.cpp).
//   generated.json  the reference's own race-free generator corpus
//                   (proj/tests/support/ProgramGen.cpp, seed 0x5eed01ab).
//   analogs.json    integer analogs of BASELINE.json configs 1/2/4 written in
//                   the reference DSL and run through the reference.
//   runtime.json    TeamRuntime call scripts (proj/tests/RuntimeTests.cpp
//                   scenarios + a seeded protocol fuzz) with every result.
//   occupancy.json  the reference occupancy model's tables and a grid of
//                   occupancyFor / maxSharedVars values (proj/src/Occupancy.cpp).
//
// The product never links or executes any of this; the repo's tests use the
// JSON to pin oracle/ompds_oracle.c and the CUDA path.
#include "omplab/Compiler.h"
#include "omplab/DeviceRuntime.h"
#include "omplab/LoweringPasses.h"
#include "omplab/Occupancy.h"
#include "omplab/SequentialOracle.h"
#include "omplab/Simulator.h"
#include "support/ProgramGen.h"

#include <json.hpp>

#include <cstdio>
#include <fstream>
#include <map>
#include <random>
#include <sstream>
#include <string>
#include <vector>

using namespace omplab;
using nlohmann::json;

static std::string readFile(const std::string &P) {
  std::ifstream In(P, std::ios::binary);
  if (!In) {
    std::fprintf(stderr, "cannot read %s\n", P.c_str());
    std::exit(2);
  }
  std::stringstream S;
  S << In.rdbuf();
  return S.str();
}

static json layoutsJson(const Module &M) {
  json Out = json::array();
  for (const FrameGroup &G : M.Groups) {
    const DepotLayout *L = M.layoutFor(G.Root);
    json J;
    J["root"] = G.Root;
    J["members"] = G.Members;
    json Slots = json::array();
    if (L) {
      for (const DepotSlot &S : L->Slots)
        Slots.push_back({{"offset", S.Offset},
                         {"size", S.Size},
                         {"align", S.Align},
                         {"shared", S.SharedResident},
                         {"owners", S.Owners}});
      J["total_local"] = L->TotalLocal;
      J["total_shared"] = L->TotalShared;
      J["has_shared_depot"] = L->HasSharedDepot;
      auto Ov = L->findSharedLocalOverlap();
      J["overlap"] = Ov ? json(*Ov) : json(nullptr);
    }
    J["slots"] = std::move(Slots);
    Out.push_back(std::move(J));
  }
  return Out;
}

static const char *eventKind(RuntimeEvent::Kind K) {
  switch (K) {
  case RuntimeEvent::Init: return "init";
  case RuntimeEvent::PreparePrealloc: return "prepare_prealloc";
  case RuntimeEvent::PrepareDynamic: return "prepare_dynamic";
  case RuntimeEvent::Fetch: return "fetch";
  case RuntimeEvent::Retire: return "retire";
  case RuntimeEvent::DynamicFree: return "dynamic_free";
  case RuntimeEvent::Deinit: return "deinit";
  }
  return "?";
}

static json eventsJson(const std::vector<RuntimeEvent> &Ev) {
  json A = json::array();
  for (const RuntimeEvent &E : Ev)
    A.push_back({eventKind(E.K), E.Fn, E.NArgs, E.Bytes});
  return A;
}

static json simJson(const Module &M, const SimOptions &O, bool WithEvents) {
  SimResult R = simulate(M, O);
  json J;
  J["ok"] = R.ok();
  J["trap"] = R.TrapReason;
  J["trap_team"] = R.TrapTeam;
  J["trap_thread"] = R.TrapThread;
  J["globals"] = R.FinalGlobals;
  J["steps"] = R.Stats.Steps;
  J["teams"] = R.Stats.Teams;
  J["launched_team_size"] = R.Stats.LaunchedTeamSize;
  J["barrier_releases"] = R.Stats.BarrierReleases;
  json Mb = json::array();
  json Idle = json::array();
  for (int T = 0; T < R.Stats.Teams; ++T) {
    Mb.push_back(R.Stats.masterBarrierEntries(T));
    int64_t IdleEntries = 0;
    if (T < (int)R.Stats.BarrierEntries.size())
      for (int Tid = R.Stats.RequestedWorkers + 1;
           Tid < R.Stats.LaunchedTeamSize; ++Tid)
        IdleEntries += R.Stats.BarrierEntries[T][Tid];
    Idle.push_back(IdleEntries);
  }
  J["master_barrier_entries"] = Mb;
  J["idle_lane_barrier_entries"] = Idle;
  // Worker barrier entries per team (tid 0), for the 2R+1 handoff count.
  json Wb = json::array();
  for (int T = 0; T < R.Stats.Teams; ++T)
    Wb.push_back(R.Stats.BarrierEntries.empty() || R.Stats.RequestedWorkers < 1
                     ? 0
                     : R.Stats.BarrierEntries[T][0]);
  J["worker0_barrier_entries"] = Wb;
  // SimStats::BarrierEntries[team][launched tid], every thread of every team
  J["barrier_entries"] = R.Stats.BarrierEntries;
  J["dynamic_alloc_bytes"] = R.Stats.DynamicAllocBytes;
  J["dynamic_allocs"] = R.Stats.DynamicAllocs;
  J["dynamic_frees"] = R.Stats.DynamicFrees;
  if (WithEvents) {
    json TE = json::array();
    for (const auto &Ev : R.TeamEvents)
      TE.push_back(eventsJson(Ev));
    J["team_events"] = std::move(TE);
  }
  return J;
}

/// The frame pipeline's input, read off the post-codegen module: every alloca
/// with its frame group (buildDepots grouping, LoweringPasses.cpp:270-280),
/// member function, byte size, escape flag (detectSharedVariables), and the
/// coloring liveness of its frame value (colorFunction, :470-509): the
/// instruction positions of its direct uses and whether it is stored as a
/// value or passed to a call.  Positions are per function, in order.
static json frameVarsJson(const Module &M) {
  auto Escaped = detectSharedVariables(M);
  std::vector<std::vector<const Function *>> Groups;
  const Function *K = M.kernel();
  Groups.push_back({K});
  if (const Function *W = M.findFunction(WorkerFnName))
    Groups.back().push_back(W);
  for (const auto &F : M.Functions)
    if (&F != K && F.Name != WorkerFnName)
      Groups.push_back({&F});
  json Out = json::array();
  for (size_t G = 0; G < Groups.size(); ++G) {
    for (size_t Fi = 0; Fi < Groups[G].size(); ++Fi) {
      const Function &F = *Groups[G][Fi];
      std::map<std::string, json> Vars;
      std::vector<std::string> Order;
      int Pos = 0;
      for (const auto &B : F.Blocks)
        for (const auto &I : B.Instrs) {
          if (I.Op == Opcode::Alloca) {
            json V;
            V["group"] = G;
            V["func"] = Fi;
            V["function"] = F.Name;
            V["name"] = I.Result;
            V["bytes"] = I.AllocaTy.sizeBytes();
            auto It = Escaped.find(F.Name);
            V["escapes"] = It != Escaped.end() && It->second.count(I.Result);
            V["pinned"] = false;
            V["def_pos"] = Pos;
            V["first"] = -1;
            V["last"] = -1;
            Vars[I.Result] = V;
            Order.push_back(I.Result);
          }
          for (size_t Oi = 0; Oi < I.Ops.size(); ++Oi) {
            const Value &Op = I.Ops[Oi];
            if (!Op.isTemp())
              continue;
            auto It = Vars.find(Op.Name);
            if (It == Vars.end())
              continue;
            json &V = It->second;
            if (V["first"].get<int>() < 0)
              V["first"] = Pos;
            V["last"] = Pos;
            if ((I.Op == Opcode::Store && Oi == 0) ||
                (I.Op == Opcode::Call && Oi >= 1))
              V["pinned"] = true;
          }
          ++Pos;
        }
      for (const auto &N : Order)
        Out.push_back(Vars[N]);
    }
  }
  return Out;
}

static json oracleJson(const ProgramAst &Ast, const OracleOptions &O) {
  OracleResult R = runSequentialOracle(Ast, O);
  json J;
  J["ok"] = R.ok();
  J["error"] = R.Error;
  J["globals"] = R.Globals;
  return J;
}

static json diagsJson(const DiagList &Ds) {
  json A = json::array();
  for (const Diagnostic &D : Ds)
    A.push_back({{"rule", D.Rule}, {"message", D.Message}});
  return A;
}

/// Compiles `Src` and records everything the hot path consumes or produces.
static json programJson(const std::string &Src, const std::string &Stem,
                        const std::vector<std::pair<int, int>> &Launches,
                        bool WithEvents,
                        const std::map<std::string, std::vector<int64_t>> &Ov =
                            {}) {
  json J;
  J["stem"] = Stem;
  J["source"] = Src;
  CompileOptions Opt;
  Opt.DumpAst = true;
  CompileResult C = compileSource(Src, Stem, Opt);
  J["compile_ok"] = C.Ok;
  J["diags"] = diagsJson(C.Diags);
  if (!C.Ok)
    return J;
  J["ast"] = json::parse(C.AstJson);
  J["kernel"] = C.Machine.kernel() ? C.Machine.kernel()->Name : "";
  J["layouts"] = layoutsJson(C.Machine);
  J["frame_vars"] = frameVarsJson(C.PostCodegen);
  J["manifest"] = json::parse(manifestJson(C.Machine, DefaultPreallocEntries));
  // the exact text (dump(2) + "\n") the reference writes, for byte-level parity
  J["manifest_text"] = manifestJson(C.Machine, DefaultPreallocEntries);
  {
    auto Det = detectSharedVariables(C.PostCodegen);
    json D = json::object();
    for (auto &[F, S] : Det)
      D[F] = std::vector<std::string>(S.begin(), S.end());
    J["detected_shared"] = D;
  }
  for (PipelineKind K : {PipelineKind::O0, PipelineKind::BadOrderDemo}) {
    PipelineResult P = runPipeline(C.PostCodegen, K);
    std::string Key = K == PipelineKind::O0 ? "layouts_o0" : "layouts_bad_order";
    J[Key] = P.ok() ? layoutsJson(P.M) : json(nullptr);
    if (K == PipelineKind::BadOrderDemo && P.ok()) {
      DiagList Audit = auditMachineModule(P.M);
      J["bad_order_audit"] = diagsJson(Audit);
      SimOptions SO;
      SO.ValidateLayout = false;
      SO.GlobalOverrides = Ov;
      J["bad_order_sim_unguarded"] = simJson(P.M, SO, false);
    }
  }
  json Runs = json::array();
  for (auto [T, W] : Launches) {
    SimOptions SO;
    SO.Teams = T;
    SO.Workers = W;
    SO.GlobalOverrides = Ov;
    OracleOptions OO;
    OO.Teams = T;
    OO.Workers = W;
    OO.GlobalOverrides = Ov;
    json R;
    R["teams"] = T;
    R["workers"] = W;
    R["sim"] = simJson(C.Machine, SO, WithEvents);
    R["oracle"] = oracleJson(*C.Ast, OO);
    Runs.push_back(std::move(R));
  }
  J["runs"] = std::move(Runs);
  return J;
}

//===----------------------------------------------------------------------===//
// Runtime scripts
//===----------------------------------------------------------------------===//

namespace {
class RecordingHeap : public SharedArgsAllocator {
public:
  uint64_t allocate(int64_t Bytes) override {
    uint64_t A = Next;
    Next += static_cast<uint64_t>(Bytes) + 64;
    Live[A] = Bytes;
    ++Allocs;
    return A;
  }
  void release(uint64_t A) override {
    Live.erase(A);
    ++Frees;
  }
  uint64_t Next = 0x1000;
  std::map<uint64_t, int64_t> Live;
  int Allocs = 0, Frees = 0;
};

constexpr uint64_t PreallocBase = 0x2000;

struct Call {
  int Op;     // 0 init, 1 prepare, 2 parallel, 3 end, 4 deinit
  int Role;   // 0 master, 1 worker
  int64_t Arg; // workers for init, nargs for prepare
};

json runScript(const std::string &Name, const std::vector<Call> &Calls,
               int PreallocEntries, bool FailDyn) {
  RecordingHeap Heap;
  RuntimeConfig Cfg;
  Cfg.PreallocEntries = PreallocEntries;
  Cfg.FailDynamicAlloc = FailDyn;
  TeamRuntime Rt(Cfg, PreallocBase, Heap);
  json J;
  J["name"] = Name;
  J["prealloc_entries"] = PreallocEntries;
  J["fail_dynamic_alloc"] = FailDyn;
  json Cs = json::array(), Rs = json::array();
  int FnSeq = 0;
  for (const Call &C : Calls) {
    Cs.push_back({C.Op, C.Role, C.Arg});
    RtRole Role = C.Role == 0 ? RtRole::Master : RtRole::Worker;
    RtResult R;
    json Out;
    switch (C.Op) {
    case 0:
      R = Rt.kernelInit(Role, static_cast<int>(C.Arg));
      break;
    case 1: {
      uint64_t Addr = 0xdead;
      std::string Fn = "region" + std::to_string(FnSeq);
      R = Rt.prepareParallel(Role, Fn, C.Arg, Addr);
      if (R.Ok) {
        ++FnSeq;
        Out["addr"] = Addr == PreallocBase ? "prealloc" : "dynamic";
        Out["live_bytes"] = Heap.Live.empty() ? 0 : Heap.Live.rbegin()->second;
      }
      break;
    }
    case 2: {
      std::string Wf = "stale";
      uint64_t Addr = 99;
      bool P = true;
      R = Rt.kernelParallel(Role, Wf, Addr, P);
      if (R.Ok) {
        Out["wf"] = Wf;
        Out["addr"] = Addr == 0 ? "null"
                      : Addr == PreallocBase ? "prealloc"
                                             : "dynamic";
        Out["participate"] = P;
      }
      break;
    }
    case 3:
      R = Rt.endParallel(Role);
      break;
    case 4:
      R = Rt.kernelDeinit(Role);
      break;
    }
    Out["ok"] = R.Ok;
    Out["trap"] = R.TrapReason;
    Out["heap_live"] = Heap.Live.size();
    Rs.push_back(std::move(Out));
  }
  J["calls"] = std::move(Cs);
  J["results"] = std::move(Rs);
  J["events"] = eventsJson(Rt.events());
  J["event_strings"] = json::array();
  for (const auto &E : Rt.events())
    J["event_strings"].push_back(E.str());
  J["workers"] = Rt.workerCount();
  J["dynamic_allocs"] = Rt.dynamicAllocs();
  J["dynamic_frees"] = Rt.dynamicFrees();
  J["leaked_blocks"] = Rt.leakedBlocks();
  J["terminated"] = Rt.terminated();
  return J;
}
} // namespace

static json runtimeGolden() {
  json Out = json::array();
  const int M = 0, W = 1;
  // proj/tests/RuntimeTests.cpp scenarios, as call scripts.
  Out.push_back(runScript("init_rules",
                          {{0, W, 8}, {0, M, 0}, {0, M, 8}, {0, M, 8}}, 20,
                          false));
  {
    std::vector<Call> C = {{0, M, 8}};
    for (int N : {0, 1, 19, 20}) {
      C.push_back({1, M, N});
      C.push_back({2, W, 0});
      C.push_back({3, W, 0});
    }
    Out.push_back(runScript("prealloc_window", C, 20, false));
  }
  {
    std::vector<Call> C = {{0, M, 8}};
    for (int N : {21, 32, 64, 128}) {
      C.push_back({1, M, N});
      C.push_back({2, W, 0});
      C.push_back({3, W, 0});
    }
    Out.push_back(runScript("heap_fallback", C, 20, false));
  }
  Out.push_back(runScript("window_boundary_4",
                          {{0, M, 8}, {1, M, 4}, {2, W, 0}, {3, W, 0},
                           {1, M, 5}},
                          4, false));
  Out.push_back(runScript("heap_failure", {{0, M, 8}, {1, M, 21}}, 20, true));
  Out.push_back(runScript("prepare_before_init", {{1, M, 1}}, 20, false));
  Out.push_back(runScript("worker_prepares", {{0, M, 8}, {1, W, 1}}, 20, false));
  Out.push_back(
      runScript("double_prepare", {{0, M, 8}, {1, M, 1}, {1, M, 1}}, 20, false));
  Out.push_back(runScript("prepare_while_active",
                          {{0, M, 8}, {1, M, 1}, {2, W, 0}, {1, M, 1}}, 20,
                          false));
  Out.push_back(runScript("fetch_nothing_staged", {{0, M, 8}, {2, W, 0}}, 20,
                          false));
  Out.push_back(
      runScript("master_fetches", {{0, M, 8}, {1, M, 1}, {2, M, 0}}, 20, false));
  Out.push_back(
      runScript("end_no_active", {{0, M, 8}, {3, W, 0}}, 20, false));
  Out.push_back(runScript("deinit_in_flight", {{0, M, 8}, {1, M, 1}, {4, M, 0}},
                          20, false));
  Out.push_back(
      runScript("double_deinit", {{0, M, 8}, {4, M, 0}, {4, M, 0}}, 20, false));
  Out.push_back(runScript("termination_sentinel", {{0, M, 8}, {4, M, 0}, {2, W, 0}},
                          20, false));
  Out.push_back(runScript("event_order",
                          {{0, M, 8}, {1, M, 21}, {2, W, 0}, {3, W, 0}, {4, M, 0}},
                          20, false));
  // Every remaining trap string at least once.
  Out.push_back(runScript("deinit_from_worker", {{0, M, 8}, {4, W, 0}}, 20, false));
  Out.push_back(runScript("deinit_before_init", {{4, M, 0}}, 20, false));
  Out.push_back(runScript("prepare_after_deinit", {{0, M, 8}, {4, M, 0}, {1, M, 2}},
                          20, false));
  Out.push_back(runScript("negative_nargs", {{0, M, 8}, {1, M, -1}}, 20, false));
  Out.push_back(runScript("end_from_master",
                          {{0, M, 8}, {1, M, 1}, {2, W, 0}, {3, M, 0}}, 20, false));
  Out.push_back(runScript("multi_worker_retire",
                          {{0, M, 4}, {1, M, 30}, {2, W, 0}, {2, W, 0}, {2, W, 0},
                           {2, W, 0}, {3, W, 0}, {3, W, 0}, {3, W, 0}, {3, W, 0},
                           {1, M, 3}, {2, W, 0}, {3, W, 0}, {4, M, 0}, {2, W, 0}},
                          20, false));
  // Byte law, proj/tests/RuntimeTests.cpp:235-252 (mt19937(1234), N in [0,128]).
  {
    std::mt19937 Rng(1234);
    std::uniform_int_distribution<int64_t> Dist(0, 128);
    for (int Round = 0; Round < 200; ++Round) {
      int64_t N = Dist(Rng);
      Out.push_back(runScript("byte_law_" + std::to_string(Round),
                              {{0, M, 8}, {1, M, N}}, 20, false));
    }
  }
  // Acceptance criterion 8's allocation law (AcceptanceMain.cpp:368-385:
  // mt19937(20260815), int N in [0,128], 400 rounds, workers 8).
  {
    std::mt19937 Rng(20260815);
    std::uniform_int_distribution<int> Dist(0, 128);
    for (int Round = 0; Round < 400; ++Round) {
      int N = Dist(Rng);
      Out.push_back(runScript("acceptance_law_" + std::to_string(Round),
                              {{0, M, 8}, {1, M, N}}, 20, false));
    }
  }
  // Seeded protocol fuzz: random roles, ops and counts, legal and not.
  {
    std::mt19937 Rng(0x5eed01ab);
    for (int S = 0; S < 400; ++S) {
      int Len = std::uniform_int_distribution<int>(1, 40)(Rng);
      int Pe = std::uniform_int_distribution<int>(0, 3)(Rng) == 0
                   ? std::uniform_int_distribution<int>(0, 24)(Rng)
                   : 20;
      bool Fail = std::uniform_int_distribution<int>(0, 9)(Rng) == 0;
      std::vector<Call> C;
      if (std::uniform_int_distribution<int>(0, 4)(Rng) != 0)
        C.push_back({0, M, std::uniform_int_distribution<int>(1, 64)(Rng)});
      for (int I = 0; I < Len; ++I) {
        int Op = std::uniform_int_distribution<int>(0, 9)(Rng);
        // Bias towards the legal cycle prepare -> parallel* -> end*.
        int OpMap[10] = {1, 1, 2, 2, 2, 3, 3, 3, 4, 0};
        int O = OpMap[Op];
        int Role = (O == 1 || O == 4 || O == 0) ? M : W;
        if (std::uniform_int_distribution<int>(0, 7)(Rng) == 0)
          Role = 1 - Role;
        int64_t Arg = 0;
        if (O == 0)
          Arg = std::uniform_int_distribution<int>(-1, 64)(Rng);
        if (O == 1)
          Arg = std::uniform_int_distribution<int>(-2, 80)(Rng);
        C.push_back({O, Role, Arg});
      }
      Out.push_back(runScript("fuzz_" + std::to_string(S), C, Pe, Fail));
    }
  }
  return Out;
}

static json occupancyGolden() {
  json J;
  J["footprint_scalars_csv"] = footprintScalarsCsv();
  J["footprint_arrays_csv"] = footprintArraysCsv();
  json Dev = json::object();
  for (const GpuSpec &G : knownGpus()) {
    json D;
    D["shared_bytes_per_sm"] = G.SharedBytesPerSM;
    D["registers_per_sm"] = G.RegistersPerSM;
    D["max_blocks_per_sm"] = G.MaxBlocksPerSM;
    D["occupancy_scalars_csv"] = occupancyScalarsCsv(G);
    D["occupancy_arrays_csv"] = occupancyArraysCsv(G);
    D["max_vars_csv"] = maxVarsCsv(G);
    json Grid = json::array();
    for (int64_t Fp : {0, 1, 49, 225, 233, 257, 289, 617, 1769, 2281, 5000,
                       20000, 70000})
      for (int Regs : {0, 16, 31, 36, 64, 136, 255})
        for (int Thr : {0, 64, 128, 256, 1024}) {
          OccupancyResult R = occupancyFor(G, Fp, Regs, Thr);
          Grid.push_back({Fp, Regs, Thr, R.TeamsByRegs, R.TeamsBySmem,
                          R.Potential, R.Actual, R.SmemUsed});
        }
    D["occupancy_grid"] = Grid;
    json Mv = json::array();
    for (int64_t T : {-1, 0, 1, 2, 3, 4, 7, 8, 12, 13, 14, 15, 16, 32, 100})
      Mv.push_back({T, maxSharedVars(G, T), maxRegsForTeams(G, T, 128)});
    D["max_shared_vars"] = Mv;
    Dev[G.Name] = D;
  }
  J["devices"] = Dev;
  json Sf = json::array();
  for (int N = 0; N <= 70; ++N)
    Sf.push_back({N, scalarsFixture(N).sharedFootprint(), dynamicArgsBytes(N)});
  J["scalars_fixture"] = Sf;
  json Af = json::array();
  for (int K = 0; K <= 6; ++K)
    Af.push_back({K, arraysFixture(K).sharedFootprint()});
  J["arrays_fixture"] = Af;
  return J;
}

// Counter-based integer inputs for the streaming analog: the same splitmix64
// as oracle/ompds_oracle.c, mapped to [-100, 100].
static uint64_t splitmix64(uint64_t Z) {
  Z += 0x9e3779b97f4a7c15ull;
  Z = (Z ^ (Z >> 30)) * 0xbf58476d1ce4e5b9ull;
  Z = (Z ^ (Z >> 27)) * 0x94d049bb133111ebull;
  return Z ^ (Z >> 31);
}

static json analogsGolden() {
  json Out = json::array();
  // Config 1 analog: 1 team x 32 workers, 4 shared scalars.
  {
    std::string S = "int a[32] = {0};\n\n#pragma omp target map(tofrom: a[:32])\n"
                    "{\n  #pragma omp teams num_teams(1) thread_limit(32)\n  {\n"
                    "    int c1 = 1;\n    int c2 = 2;\n    int c3 = 3;\n    int c4 = 4;\n"
                    "    #pragma omp parallel\n    {\n"
                    "      a[omp_get_thread_num()] += c1 + c2 + c3 + c4;\n    }\n  }\n}\n";
    Out.push_back(programJson(S, "cfg1_analog", {{1, 32}, {2, 32}, {1, 8}, {3, 64}},
                              true));
  }
  // Config 1 analog with the region inside a sequential loop (R regions, the
  // master mutating a capture between regions).
  {
    std::string S = "int a[32] = {0};\n\n#pragma omp target map(tofrom: a[:32])\n"
                    "{\n  #pragma omp teams num_teams(1) thread_limit(32)\n  {\n"
                    "    int c1 = 1;\n    int c2 = 2;\n    int c3 = 3;\n    int c4 = 4;\n"
                    "    for (int r = 0; r < 5; r++) {\n"
                    "      #pragma omp parallel\n      {\n"
                    "        a[omp_get_thread_num()] += c1 + c2 + c3 + c4;\n      }\n"
                    "      c4 += 1;\n    }\n  }\n}\n";
    Out.push_back(programJson(S, "cfg1_loop_analog", {{1, 32}, {2, 32}}, true));
  }
  // Config 2 analog: shared int d[256] filled by the master, parallel for.
  {
    std::string S = "int a[256] = {0};\n\n#pragma omp target map(tofrom: a[:256])\n"
                    "{\n  #pragma omp teams num_teams(4) thread_limit(96)\n  {\n"
                    "    int d[256] = {0};\n"
                    "    for (int k = 0; k < 256; k++) {\n      d[k] = 3 * k + 1;\n    }\n"
                    "    #pragma omp parallel for\n"
                    "    for (int i = 0; i < 256; i++) {\n      a[i] += d[i];\n    }\n"
                    "  }\n}\n";
    Out.push_back(programJson(S, "cfg2_analog", {{4, 96}, {1, 32}, {2, 8}}, true));
  }
  // Config 4 analog: streaming y[i] += c1*x[i] + c2 + ... + c8 with 8 captures.
  for (int N : {1024, 4096}) {
    std::ostringstream S;
    S << "int x[" << N << "] = {0};\nint y[" << N << "] = {0};\n\n"
      << "#pragma omp target map(to: x[:" << N << "]) map(tofrom: y[:" << N
      << "])\n{\n  #pragma omp teams num_teams(4) thread_limit(96)\n  {\n";
    for (int K = 1; K <= 8; ++K)
      S << "    int c" << K << " = " << K << ";\n";
    S << "    #pragma omp parallel for\n    for (int i = 0; i < " << N
      << "; i++) {\n      y[i] += c1 * x[i] + c2 + c3 + c4 + c5 + c6 + c7 + c8;\n"
      << "    }\n  }\n}\n";
    std::map<std::string, std::vector<int64_t>> Ov;
    std::vector<int64_t> X(N), Y(N);
    for (int I = 0; I < N; ++I) {
      X[I] = static_cast<int64_t>(splitmix64(0x5eed01abull + I) % 201) - 100;
      Y[I] = static_cast<int64_t>(splitmix64(0x5eed01acull + I) % 201) - 100;
    }
    Ov["x"] = X;
    Ov["y"] = Y;
    json P = programJson(S.str(), "cfg4_analog_" + std::to_string(N),
                         {{4, 96}, {2, 32}}, false, Ov);
    P["inputs"] = {{"x", X}, {"y", Y}};
    Out.push_back(std::move(P));
  }
  // Config 3: the reference rejects nested parallel regions at parse time.
  {
    std::string S = "int a[8] = {0};\n\n#pragma omp target map(tofrom: a[:8])\n"
                    "{\n  #pragma omp teams num_teams(1) thread_limit(8)\n  {\n"
                    "    int c = 1;\n    #pragma omp parallel\n    {\n"
                    "      int e = 2;\n      #pragma omp parallel\n      {\n"
                    "        a[omp_get_thread_num()] += c + e;\n      }\n    }\n  }\n}\n";
    Out.push_back(programJson(S, "cfg3_nested", {}, false));
  }
  return Out;
}

int main(int argc, char **argv) {
  if (argc < 3) {
    std::fprintf(stderr, "usage: ref_golden <proj dir> <out dir>\n");
    return 2;
  }
  std::string Proj = argv[1], OutDir = argv[2];
  const char *Stems[] = {"arrays_1",   "arrays_2",   "arrays_3",
                         "arrays_4",   "coloring_demo", "firstprivate",
                         "mixed_captures", "private_inner", "scalars_1",
                         "scalars_16", "scalars_2",  "scalars_32",
                         "scalars_4",  "scalars_64", "scalars_8",
                         "seq_only",   "shared_scalar", "two_regions"};
  json Corpus = json::array();
  for (const char *S : Stems) {
    std::string Src = readFile(Proj + "/programs/" + S + ".ompk");
    Corpus.push_back(programJson(
        Src, S, {{-1, -1}, {1, 8}, {2, 8}, {4, 8}, {1, 96}, {2, 96}, {4, 96}},
        true));
    std::fprintf(stderr, "corpus %s\n", S);
  }
  std::ofstream(OutDir + "/corpus.json") << Corpus.dump() << "\n";

  json Gen = json::array();
  auto G = generateCorpus(120, corpusSeed());
  for (const auto &P : G) {
    json J = programJson(P.Source, P.Name, {{P.Teams, P.Workers}}, true);
    J["gen_teams"] = P.Teams;
    J["gen_workers"] = P.Workers;
    Gen.push_back(std::move(J));
  }
  std::ofstream(OutDir + "/generated.json") << Gen.dump() << "\n";
  std::fprintf(stderr, "generated %zu\n", G.size());

  std::ofstream(OutDir + "/analogs.json") << analogsGolden().dump() << "\n";
  std::ofstream(OutDir + "/runtime.json") << runtimeGolden().dump() << "\n";
  std::ofstream(OutDir + "/occupancy.json") << occupancyGolden().dump() << "\n";
  return 0;
}
