// integration/executor_b200.cpp — the reference-side binding of the B200 path.
//
// Drop-in replacement for the reference's proj/src/executor.cpp and the
// run_once of proj/src/experiment.cpp:23-30: the same totsim::Executor class
// (proj/include/totsim/executor.hpp:43-62) and run_once signature
// (proj/include/totsim/experiment.hpp:27), implemented over the C ABI of
// include/spex.h, so reference code and tests that drive whole runs link
// against the device path unchanged. Errors come back as totsim::Error with the
// reference's Errc (status = Errc ordinal + 1, errors.hpp:9-28).
//
// Built by oracle/Makefile (target dropin) together with the reference's own
// tests/test_executor.cpp and its host-side modules (config, trace, tree, sim
// for the test's independent oracles) — executor.cpp and experiment.cpp are
// NOT linked: Executor and run_once resolve here.
#include <sstream>
#include <string>

#include "spex.h"
#include "totsim/errors.hpp"
#include "totsim/executor.hpp"
#include "totsim/experiment.hpp"
#include "totsim/trace.hpp"

namespace totsim {

namespace {

[[noreturn]] void raise(int rc) {
  const int ord = rc - 1;
  const Errc code = ord >= 0 && ord <= static_cast<int>(Errc::InvalidArgument) ? static_cast<Errc>(ord)
                                                                                : Errc::InvalidArgument;
  throw Error(code, std::string("spex: ") + spex_last_error());
}

std::string flags_csv(const SpexFlags& f) {
  std::string s;
  if (f.t1) s += "t1";
  if (f.t2) s += s.empty() ? "t2" : ",t2";
  if (f.t3) s += s.empty() ? "t3" : ",t3";
  return s;
}

}  // namespace

struct Executor::Impl {
  ExperimentConfig cfg;
  std::uint64_t seed;
  SpexFlags active;
  TraceWriter* trace;
  bool ran = false;

  RunTotals run() {
    if (ran) throw Error(Errc::InvalidArgument, "run() may be called once");  // executor.cpp:810
    ran = true;
    cfg.validate();  // executor.cpp:812 (the host config module)
    spex_executor* h = nullptr;
    const std::string cj = cfg.to_json().dump();
    if (int rc = spex_executor_create(cj.c_str(), seed, flags_csv(active).c_str(), 0, &h)) raise(rc);
    spex_totals t{};
    int rc = spex_executor_run(h, trace != nullptr, &t);
    if (rc == 0 && trace) {
      char* lines = nullptr;
      size_t n = 0;
      rc = spex_executor_log(h, &lines, &n);
      if (rc == 0) {
        std::istringstream in(std::string(lines, n));
        for (std::string l; std::getline(in, l);)
          if (!l.empty()) trace->emit(nlohmann::ordered_json::parse(l));
        trace->flush();
        spex_free(lines);
      }
    }
    spex_executor_destroy(h);
    if (rc) raise(rc);
    RunTotals out;
    out.makespan = t.makespan;
    out.generated_tokens = t.generated_tokens;
    out.committed_tokens = t.committed_tokens;
    out.reused_tokens = t.reused_tokens;
    out.wasted_tokens = t.wasted_tokens;
    out.queries = t.queries;
    out.correct_votes = t.correct_votes;
    out.early_terminated = t.early_terminated;
    for (int d = 1; d <= kMaxTrackedDistance; ++d) {
      out.hits[d] = t.hits[d];
      out.misses[d] = t.misses[d];
    }
    return out;
  }
};

Executor::Executor(const ExperimentConfig& cfg, std::uint64_t run_seed, const SpexFlags& active, TraceWriter* trace)
    : impl_(new Impl{cfg, run_seed, active, trace}) {}

Executor::~Executor() = default;

RunTotals Executor::run() { return impl_->run(); }

RunOutcome run_once(const ExperimentConfig& cfg, std::uint64_t seed, const SpexFlags& flags) {
  TraceWriter w = TraceWriter::to_memory();
  Executor ex(cfg, seed, flags, &w);
  RunOutcome out;
  out.totals = ex.run();
  out.log = w.lines();
  return out;
}

}  // namespace totsim
