// ref_shim.cpp -- TEST / BASELINE INFRASTRUCTURE ONLY.
//
// A C-ABI shim over the unmodified reference library (omplab_core) so that
// `bench.py --impl reference` can time the reference's own CPU path for the
// streaming region (BASELINE config 4) on the GPU box's host cores, where
// /root/reference does not exist (this .so is prebuilt here into oracle/_ref/).
//
// The reference language is integer-only (proj/docs/dsl.md:3-7), so the
// streaming body is its integer analog
//     y[i] += c1 * x[i] + c2 + ... + c8     (proj/programs style, 8 captures)
// compiled with compileSource (proj/src/Compiler.cpp:33-110) and executed by
// the reference's execution model `simulate` (proj/src/Simulator.cpp:853) or
// its sequential interpreter `runSequentialOracle`
// (proj/src/SequentialOracle.cpp:253).  Independent element chunks run on
// separate host threads (one reference instance per thread).
#include "omplab/Compiler.h"
#include "omplab/SequentialOracle.h"
#include "omplab/Simulator.h"

#include <chrono>
#include <sstream>
#include <string>
#include <vector>

using namespace omplab;

static std::string streamSource(int64_t N, int Teams, int Workers) {
  std::ostringstream S;
  S << "int x[" << N << "] = {0};\nint y[" << N << "] = {0};\n\n"
    << "#pragma omp target map(to: x[:" << N << "]) map(tofrom: y[:" << N
    << "])\n{\n  #pragma omp teams num_teams(" << Teams << ") thread_limit("
    << Workers << ")\n  {\n";
  for (int K = 1; K <= 8; ++K)
    S << "    int c" << K << " = " << K << ";\n";
  S << "    #pragma omp parallel for\n    for (int i = 0; i < " << N
    << "; i++) {\n      y[i] += c1 * x[i] + c2 + c3 + c4 + c5 + c6 + c7 + c8;\n"
    << "    }\n  }\n}\n";
  return S.str();
}

extern "C" {

/// Runs `nchunks` independent chunks of `chunk` elements each (x, y laid out
/// chunk-major, int64 values within int32 range).  mode 0 = simulator,
/// mode 1 = sequential oracle.  Returns 0 on success, else the index+1 of the
/// first failing chunk.  y is updated in place.
int omplab_ref_stream(int mode, int64_t chunk, int nchunks, int teams,
                      int workers, const int64_t *x, int64_t *y,
                      int nthreads) {
  CompileResult C = compileSource(streamSource(chunk, teams, workers),
                                  "stream_ref", {});
  if (!C.Ok)
    return -1;
  int Failed = 0;
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads)
  for (int K = 0; K < nchunks; ++K) {
    std::vector<int64_t> X(x + K * chunk, x + (K + 1) * chunk);
    std::vector<int64_t> Y(y + K * chunk, y + (K + 1) * chunk);
    std::map<std::string, std::vector<int64_t>> Ov{{"x", X}, {"y", Y}};
    std::vector<int64_t> Out;
    bool Ok = false;
    if (mode == 0) {
      SimOptions O;
      O.GlobalOverrides = Ov;
      O.StepLimit = int64_t(1) << 62;
      SimResult R = simulate(C.Machine, O);
      Ok = R.ok();
      if (Ok)
        Out = R.FinalGlobals["y"];
    } else {
      OracleOptions O;
      O.GlobalOverrides = Ov;
      O.StepLimit = int64_t(1) << 62;
      OracleResult R = runSequentialOracle(*C.Ast, O);
      Ok = R.ok();
      if (Ok)
        Out = R.Globals["y"];
    }
    if (!Ok || static_cast<int64_t>(Out.size()) != chunk) {
#pragma omp critical
      if (!Failed)
        Failed = K + 1;
      continue;
    }
    for (int64_t I = 0; I < chunk; ++I)
      y[K * chunk + I] = Out[I];
  }
  return Failed;
}

/// The config-1 analog through the reference simulator: one team of
/// `workers`, 4 shared scalars, `regions` parallel regions in a sequential
/// loop.  Returns seconds per region (wall), or a negative value on failure.
double omplab_ref_regions(int mode, int workers, int regions) {
  std::ostringstream S;
  S << "int a[" << workers << "] = {0};\n\n#pragma omp target map(tofrom: a[:"
    << workers << "])\n{\n  #pragma omp teams num_teams(1) thread_limit("
    << workers << ")\n  {\n    int c1 = 1;\n    int c2 = 2;\n    int c3 = 3;\n"
    << "    int c4 = 4;\n    for (int r = 0; r < " << regions << "; r++) {\n"
    << "      #pragma omp parallel\n      {\n"
    << "        a[omp_get_thread_num()] += c1 + c2 + c3 + c4;\n      }\n"
    << "    }\n  }\n}\n";
  CompileResult C = compileSource(S.str(), "regions_ref", {});
  if (!C.Ok)
    return -1.0;
  auto T0 = std::chrono::steady_clock::now();
  bool Ok;
  if (mode == 0) {
    SimOptions O;
    O.StepLimit = int64_t(1) << 62;
    Ok = simulate(C.Machine, O).ok();
  } else {
    OracleOptions O;
    O.StepLimit = int64_t(1) << 62;
    Ok = runSequentialOracle(*C.Ast, O).ok();
  }
  double Sec =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - T0)
          .count();
  return Ok ? Sec / regions : -2.0;
}
}
