// oracle/ref_split.cpp — TEST INFRASTRUCTURE ONLY (the checker, never the product).
//
// The split multi-GPU mode's oracle: W copies of the UNMODIFIED reference
// Executor (executor.cpp:809-851), one per host thread, each running query
// block [Q*r/W, Q*(r+1)/W) of one Q-query job on its own decode engine and
// clock, coupled only by the north_star's global budget exchange. Two
// reference functions are wrapped — the linker sees the reference's own
// definitions renamed by objcopy (oracle/Makefile `SPLIT_*`):
//
//   generate_workload (sim.cpp:171-198): a rank's executor asks for its
//       block's n queries; the wrapper generates the job's Q and returns the
//       block's slice, so every query keeps the seed (rng::mix(base, q + 1))
//       and golden label it has in the single-server run;
//   allocate_budgets (budget.cpp:45-96), called by scheduling_round
//       (executor.cpp:727-733) only when T2 is on, a candidate exists and
//       the rank has idle producer slots: the k-th call of every rank is one
//       exchange round. A rank posts (idle, its candidates' QueryStates) and
//       waits until every other rank has posted its k-th round or finished
//       its run; the allocation is the reference's allocate_budgets over the
//       concatenation in rank order with k_total = the sum of the posted
//       idle slots, and each rank takes its own candidates' grants.
//
// With W = 1 both wrappers are the identity, so the mode reduces to the
// reference's single-server run. The device implements the same exchange in
// the control kernel over peer memory (csrc/ctl_run.h `split_exchange`);
// tests/test_split_*.py compare the rank logs byte for byte.
#include <condition_variable>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "totsim/budget.hpp"
#include "totsim/config.hpp"
#include "totsim/errors.hpp"
#include "totsim/executor.hpp"
#include "totsim/sim.hpp"
#include "totsim/trace.hpp"

namespace totsim {
// the reference's definitions, renamed in copies of budget.o / sim.o
std::vector<int> allocate_budgets_orig(const std::vector<QueryState>& queries, int k_total, double tau,
                                       const HardwareProfile& hw);
std::vector<QueryProfile> generate_workload_orig(int n_queries, const WorkloadSpec& wl, std::uint64_t seed,
                                                 int max_depth);
}  // namespace totsim

using namespace totsim;

namespace {

struct Post {
  int idle = 0;
  std::vector<QueryState> states;
};

struct Group {
  int world = 1, q_job = 0;
  std::mutex mu;
  std::condition_variable cv;
  std::vector<long long> posted;  // rounds posted per rank
  std::vector<int> done;
  std::vector<Post> slot;         // [rank * 2 + round % 2]
  std::vector<long long> rounds;  // exchange rounds per rank (statistics)
};

thread_local Group* t_group = nullptr;
thread_local int t_rank = -1;
thread_local std::string t_err;

int block_lo(int q, int r, int w) { return static_cast<int>(static_cast<long long>(q) * r / w); }

char* dup_string(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.data(), s.size());
  p[s.size()] = 0;
  return p;
}

}  // namespace

namespace totsim {

std::vector<QueryProfile> generate_workload(int n_queries, const WorkloadSpec& wl, std::uint64_t seed,
                                            int max_depth) {
  if (!t_group) return generate_workload_orig(n_queries, wl, seed, max_depth);
  const int lo = block_lo(t_group->q_job, t_rank, t_group->world);
  std::vector<QueryProfile> all = generate_workload_orig(t_group->q_job, wl, seed, max_depth);
  return {all.begin() + lo, all.begin() + lo + n_queries};
}

std::vector<int> allocate_budgets(const std::vector<QueryState>& queries, int k_total, double tau,
                                  const HardwareProfile& hw) {
  if (!t_group) return allocate_budgets_orig(queries, k_total, tau, hw);
  Group& g = *t_group;
  const int me = t_rank;
  std::unique_lock<std::mutex> lk(g.mu);
  const long long k = ++g.posted[me];
  g.rounds[me] = k;
  Post& mine = g.slot[me * 2 + static_cast<int>(k & 1)];
  mine.idle = k_total;
  mine.states = queries;
  g.cv.notify_all();
  g.cv.wait(lk, [&] {
    for (int s = 0; s < g.world; ++s)
      if (g.posted[s] < k && !g.done[s]) return false;
    return true;
  });
  std::vector<QueryState> all;
  int total = 0, off = 0;
  for (int s = 0; s < g.world; ++s) {
    if (g.posted[s] < k) continue;  // finished before its k-th round
    const Post& p = g.slot[s * 2 + static_cast<int>(k & 1)];
    if (s == me) off = static_cast<int>(all.size());
    total += p.idle;
    all.insert(all.end(), p.states.begin(), p.states.end());
  }
  lk.unlock();
  const std::vector<int> grant = allocate_budgets_orig(all, total, tau, hw);
  return {grant.begin() + off, grant.begin() + off + static_cast<long>(queries.size())};
}

}  // namespace totsim

extern "C" {

const char* ref_split_last_error() { return t_err.c_str(); }

void ref_split_free(void* p) { std::free(p); }

/** One split job: `world` rank executors of the config's Q queries, seed
 *  `seed` (the job seed: every rank uses it), flags as in ref_run_log.
 *  out_logs[r] = rank r's event log (JSON lines), out_totals[r*24..] its
 *  totals (ref_driver.cpp layout), out_rounds[r] its exchange rounds.
 *  Returns 0 or the first failing rank's Errc ordinal + 1. */
int ref_split_run_log(const char* config_json, std::uint64_t seed, const char* flags_csv, int world, int trace,
                      char** out_logs, double* out_totals, long long* out_rounds) {
  ExperimentConfig cfg;
  SpexFlags fl;
  try {
    cfg = ExperimentConfig::from_json(nlohmann::ordered_json::parse(config_json));
    fl = flags_csv ? flags_from_string(flags_csv) : cfg.flags;
    if (world < 1 || world > cfg.n_queries) throw Error(Errc::InvalidArgument, "split: world must be in [1, n_queries]");
  } catch (const Error& e) {
    t_err = e.what();
    return static_cast<int>(e.code()) + 1;
  } catch (const std::exception& e) {
    t_err = e.what();
    return 100;
  }
  Group g;
  g.world = world;
  g.q_job = cfg.n_queries;
  g.posted.assign(world, 0);
  g.done.assign(world, 0);
  g.slot.resize(2 * world);
  g.rounds.assign(world, 0);
  std::vector<int> rc(world, 0);
  std::vector<std::string> err(world);
  std::vector<std::vector<std::string>> logs(world);
  std::vector<RunTotals> tot(world);
  std::vector<std::thread> th;
  for (int r = 0; r < world; ++r) {
    th.emplace_back([&, r] {
      t_group = &g;
      t_rank = r;
      try {
        ExperimentConfig c = cfg;
        c.n_queries = block_lo(g.q_job, r + 1, world) - block_lo(g.q_job, r, world);
        TraceWriter w = TraceWriter::to_memory();
        Executor ex(c, seed, fl, trace ? &w : nullptr);
        tot[r] = ex.run();
        logs[r] = w.lines();
      } catch (const Error& e) {
        rc[r] = static_cast<int>(e.code()) + 1;
        err[r] = e.what();
      } catch (const std::exception& e) {
        rc[r] = 100;
        err[r] = e.what();
      }
      {
        std::lock_guard<std::mutex> lk(g.mu);
        g.done[r] = 1;
      }
      g.cv.notify_all();
      t_group = nullptr;
    });
  }
  for (auto& t : th) t.join();
  for (int r = 0; r < world; ++r) {
    if (rc[r]) {
      t_err = "rank " + std::to_string(r) + ": " + err[r];
      return rc[r];
    }
  }
  for (int r = 0; r < world; ++r) {
    std::string s;
    for (const auto& line : logs[r]) {
      s += line;
      s += '\n';
    }
    out_logs[r] = dup_string(s);
    double* o = out_totals + 24 * r;
    const RunTotals& t = tot[r];
    o[0] = t.makespan;
    o[1] = static_cast<double>(t.generated_tokens);
    o[2] = static_cast<double>(t.committed_tokens);
    o[3] = static_cast<double>(t.reused_tokens);
    o[4] = static_cast<double>(t.wasted_tokens);
    o[5] = t.queries;
    o[6] = t.correct_votes;
    o[7] = t.early_terminated;
    for (int d = 1; d <= kMaxTrackedDistance; ++d) {
      o[7 + d] = static_cast<double>(t.hits[d]);
      o[15 + d] = static_cast<double>(t.misses[d]);
    }
    if (out_rounds) out_rounds[r] = g.rounds[r];
  }
  return 0;
}

}  // extern "C"
