// oracle/ref_driver.cpp — TEST INFRASTRUCTURE ONLY (the checker, never the product).
//
// A thin extern "C" driver around the UNMODIFIED reference simulator, compiled
// from /root/reference/proj/src/*.cpp by oracle/Makefile into oracle/_ref/.
// It is used by tests/ (golden-log generation, restatement pinning) and by
// bench.py's cpu_baseline / --impl reference legs. Nothing in the product
// path links or loads it.
//
// Entry points wrap the reference's own public API:
//   run_once            experiment.cpp:23-30
//   Executor::run       executor.cpp:809-851 (trace = nullptr for timing)
//   ucb_score           policy.cpp:25-30
//   rebase_widths       policy.cpp:65-118
//   allocate_budgets    budget.cpp:45-96
//   roofline_k_total    budget.cpp:23-39
//   RewardOracle::*     sim.cpp:106-169
//   unique_kv_tokens    sim.cpp:54-68
//   DecodeEngine        sim.cpp:204-384 (ref_engine_*, over SearchTrees built by ref_tree_*)
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "totsim/budget.hpp"
#include "totsim/config.hpp"
#include "totsim/executor.hpp"
#include "totsim/experiment.hpp"
#include "totsim/policy.hpp"
#include "totsim/rng.hpp"
#include "totsim/speculation.hpp"
#include "totsim/sim.hpp"
#include "totsim/termination.hpp"
#include "totsim/trace.hpp"
#include "totsim/tree.hpp"

using namespace totsim;

namespace {

thread_local std::string g_err;

char* dup_string(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.data(), s.size());
  p[s.size()] = 0;
  return p;
}

ExperimentConfig parse_cfg(const char* config_json) {
  return ExperimentConfig::from_json(nlohmann::ordered_json::parse(config_json));
}

void totals_out(const RunTotals& t, double* out) {
  // [makespan, generated, committed, reused, wasted, queries, correct, early,
  //  hits[1..8], misses[1..8]]
  out[0] = t.makespan;
  out[1] = static_cast<double>(t.generated_tokens);
  out[2] = static_cast<double>(t.committed_tokens);
  out[3] = static_cast<double>(t.reused_tokens);
  out[4] = static_cast<double>(t.wasted_tokens);
  out[5] = t.queries;
  out[6] = t.correct_votes;
  out[7] = t.early_terminated;
  for (int d = 1; d <= kMaxTrackedDistance; ++d) {
    out[7 + d] = static_cast<double>(t.hits[d]);
    out[15 + d] = static_cast<double>(t.misses[d]);
  }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_free(void* p) { std::free(p); }

/** Full run with the event log (run_once). Returns 0 or Errc ordinal + 1. */
int ref_run_log(const char* config_json, std::uint64_t seed, const char* flags_csv,
                char** out_log, double* out_totals) {
  try {
    ExperimentConfig cfg = parse_cfg(config_json);
    SpexFlags fl = flags_csv ? flags_from_string(flags_csv) : cfg.flags;
    RunOutcome out = run_once(cfg, seed, fl);
    std::string s;
    for (const auto& line : out.log) {
      s += line;
      s += '\n';
    }
    *out_log = dup_string(s);
    totals_out(out.totals, out_totals);
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    return static_cast<int>(e.code()) + 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 100;
  }
}

/** Timed runs: `reps` back-to-back Executor::run with or without tracing.
 *  Returns the total wall seconds through *secs. */
int ref_run_timed(const char* config_json, std::uint64_t seed, const char* flags_csv,
                  int with_trace, int reps, double* secs, double* out_totals) {
  try {
    ExperimentConfig cfg = parse_cfg(config_json);
    SpexFlags fl = flags_csv ? flags_from_string(flags_csv) : cfg.flags;
    auto t0 = std::chrono::steady_clock::now();
    RunTotals last;
    for (int r = 0; r < reps; ++r) {
      if (with_trace) {
        TraceWriter w = TraceWriter::to_memory();
        Executor ex(cfg, seed, fl, &w);
        last = ex.run();
      } else {
        Executor ex(cfg, seed, fl, nullptr);
        last = ex.run();
      }
    }
    auto t1 = std::chrono::steady_clock::now();
    *secs = std::chrono::duration<double>(t1 - t0).count();
    if (out_totals) totals_out(last, out_totals);
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    return static_cast<int>(e.code()) + 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 100;
  }
}

/** Parallel repetitions over OpenMP (run_experiment_full, experiment.cpp:50-134)
 *  as the reference's own multi-core mode. */
int ref_run_experiment(const char* config_json, double* secs, double* makespan,
                       double* speedup) {
  try {
    ExperimentConfig cfg = parse_cfg(config_json);
    auto t0 = std::chrono::steady_clock::now();
    ExperimentResult res = run_experiment_full(cfg);
    auto t1 = std::chrono::steady_clock::now();
    *secs = std::chrono::duration<double>(t1 - t0).count();
    *makespan = res.metrics.makespan;
    *speedup = res.metrics.speedup;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 100;
  }
}

/** run_experiment_full metrics as JSON (RunMetrics::to_json) — the oracle of
 *  the experiment harness (treatment + baseline pairs over repetitions). */
int ref_run_experiment_json(const char* config_json, char** out) {
  try {
    ExperimentConfig cfg = parse_cfg(config_json);
    ExperimentResult res = run_experiment_full(cfg);
    *out = dup_string(res.metrics.to_json().dump());
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    return static_cast<int>(e.code()) + 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 100;
  }
}

/** validate_trace over newline-separated JSON lines: report as JSON
 *  {ok, problems, generated, committed, reused, wasted, queries, makespan}. */
int ref_validate_trace(const char* lines_text, char** out) {
  try {
    std::vector<std::string> lines;
    std::string cur;
    for (const char* p = lines_text; *p; ++p) {
      if (*p == '\n') {
        if (!cur.empty()) lines.push_back(cur);
        cur.clear();
      } else {
        cur.push_back(*p);
      }
    }
    if (!cur.empty()) lines.push_back(cur);
    ReplayReport r = validate_trace(parse_trace_lines(lines));
    nlohmann::ordered_json j;
    j["ok"] = r.ok;
    j["problems"] = r.problems;
    j["generated"] = r.generated;
    j["committed"] = r.committed;
    j["reused"] = r.reused;
    j["wasted"] = r.wasted;
    j["queries"] = r.queries;
    j["makespan"] = r.makespan;
    *out = dup_string(j.dump());
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    return static_cast<int>(e.code()) + 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 100;
  }
}

/** Canonical config JSON (ExperimentConfig::to_json) after strict parsing. */
int ref_canonical_config(const char* config_json, char** out) {
  try {
    *out = dup_string(parse_cfg(config_json).to_json().dump());
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    return static_cast<int>(e.code()) + 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 100;
  }
}

// ---------------------------------------------------------------- pure KATs
double ref_ucb_score(double value, int cv, int pv, double c) { return ucb_score(value, cv, pv, c); }

int ref_rebase_widths(const double* rewards, int n, int budget, double temp, int sum_preserving,
                      int* out) {
  try {
    std::vector<double> r(rewards, rewards + n);
    auto w = rebase_widths(r, budget, temp,
                           sum_preserving ? WidthMode::SumPreserving : WidthMode::HalfAwayFromZero);
    for (int i = 0; i < n; ++i) out[i] = w[i];
    return 0;
  } catch (const Error& e) {
    return static_cast<int>(e.code()) + 1;
  }
}

int ref_allocate_budgets(const int* capacity, const double* hit_ema, const double* kv_bytes, int n,
                         int k_total, double tau, const double* hw6, int* out) {
  HardwareProfile hw;
  hw.weight_bytes = hw6[0];
  hw.mem_bandwidth = hw6[1];
  hw.peak_compute = hw6[2];
  hw.flops_per_token = hw6[3];
  hw.kv_bytes_per_token = hw6[4];
  hw.reward_latency = hw6[5];
  std::vector<QueryState> qs(n);
  for (int i = 0; i < n; ++i) {
    qs[i].query_id = i;
    qs[i].capacity = capacity[i];
    qs[i].hit_ema = hit_ema[i];
    qs[i].kv_bytes = kv_bytes[i];
  }
  auto g = allocate_budgets(qs, k_total, tau, hw);
  for (int i = 0; i < n; ++i) out[i] = g[i];
  return 0;
}

int ref_roofline_k_total(const double* hw6, int active, double avg_kv, int cap) {
  HardwareProfile hw;
  hw.weight_bytes = hw6[0];
  hw.mem_bandwidth = hw6[1];
  hw.peak_compute = hw6[2];
  hw.flops_per_token = hw6[3];
  hw.kv_bytes_per_token = hw6[4];
  hw.reward_latency = hw6[5];
  return roofline_k_total(hw, active, avg_kv, cap);
}

std::uint64_t ref_splitmix64(std::uint64_t x) { return rng::splitmix64(x); }
std::uint64_t ref_extend_hash(std::uint64_t h, int slot) { return rng::extend_hash(h, slot); }
double ref_uniform01(std::uint64_t h, std::uint64_t salt) { return rng::uniform01(h, salt); }
double ref_normal01(std::uint64_t h, std::uint64_t salt) { return rng::normal01(h, salt); }
double ref_log(double x) { return std::log(x); }
double ref_exp(double x) { return std::exp(x); }
double ref_cos(double x) { return std::cos(x); }

/** Default-workload token length for a child hash (RewardOracle::token_len). */
int ref_token_len(std::uint64_t child_hash) {
  WorkloadSpec wl;
  RewardOracle o(1, wl, 16);
  return o.token_len(child_hash);
}

/** Workload seeds: generate_workload (sim.cpp:171-198). out: seed, golden idx, probe depth. */
int ref_workload(int n, std::uint64_t seed, int max_depth, std::uint64_t* seeds, int* probe_depth) {
  WorkloadSpec wl;
  auto p = generate_workload(n, wl, seed, max_depth);
  for (int i = 0; i < n; ++i) {
    seeds[i] = p[i].seed;
    probe_depth[i] = p[i].probe_depth;
  }
  return 0;
}

/* transition_legal (tree.cpp:23-45) and SearchTree::prune_subtree
 * (tree.cpp:119-141) on a tree built from parents / statuses. */
int ref_transition_legal(int from, int to) {
  return transition_legal(static_cast<NodeStatus>(from), static_cast<NodeStatus>(to)) ? 1 : 0;
}
int ref_prune_subtree(const std::int32_t* parent, std::uint8_t* status, int n, std::uint32_t id, int* pruned) {
  try {
    SearchTree t(32, 1);
    for (int i = 1; i < n; ++i) t.add_node(static_cast<NodeId>(parent[i]), 10, false);
    for (int i = 0; i < n; ++i) t.node(static_cast<NodeId>(i)).status = static_cast<NodeStatus>(status[i]);
    *pruned = t.prune_subtree(id);
    for (int i = 0; i < n; ++i) status[i] = static_cast<std::uint8_t>(t.node(static_cast<NodeId>(i)).status);
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    return static_cast<int>(e.code()) + 1;
  }
}

/* dfs_speculative_select (speculation.cpp:182-218) on a tree built from plain
 * arrays (the layout of spex_speculation_dfs_plan). Returns 0 or Errc + 1. */
int ref_dfs_plan(const std::int32_t* parent, const std::uint8_t* status, const std::uint8_t* bits,
                 const double* reward, const std::int32_t* visits, const double* value, int n, int family,
                 double exploration_c, int width, const std::int32_t* depth_widths, int n_dw, int target_answers,
                 int k, std::uint32_t* out_node, std::int32_t* out_dist, int* n_out) {
  try {
    SearchTree t(32, 1);
    for (int i = 1; i < n; ++i) t.add_node(static_cast<NodeId>(parent[i]), 10, false);
    for (int i = 0; i < n; ++i) {
      ThoughtNode& d = t.node(static_cast<NodeId>(i));
      d.status = static_cast<NodeStatus>(status[i]);
      d.terminal = bits[i] & 1;
      d.gen_done = (bits[i] & 2) != 0;
      if (bits[i] & 4) d.reward = reward[i];
      d.visits = visits[i];
      d.value = value[i];
    }
    PolicyConfig cfg;
    cfg.family = static_cast<Family>(family);
    cfg.exploration_c = exploration_c;
    cfg.width = width;
    cfg.depth_widths.assign(depth_widths, depth_widths + n_dw);
    cfg.target_answers = target_answers;
    SpeculationLedger ledger;
    SpeculationPlan plan = dfs_speculative_select(t, ledger, k, cfg);
    *n_out = static_cast<int>(plan.targets.size());
    for (int i = 0; i < *n_out; ++i) {
      out_node[i] = plan.targets[i].node;
      out_dist[i] = plan.targets[i].predicted_distance;
    }
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    return static_cast<int>(e.code()) + 1;
  }
}

/* AnswerTally::should_terminate after recording answers (label index, weight)
 * as labels "a<idx>" (termination.cpp:7-48). */
int ref_should_terminate(const int* label, const double* weight, int n, int min_answers, double alpha) {
  AnswerTally t;
  for (int i = 0; i < n; ++i) t.record_answer("a" + std::to_string(label[i]), weight[i]);
  return t.should_terminate(min_answers, alpha) ? 1 : 0;
}

/* The reference DecodeEngine over reference SearchTrees (engine-handle parity tests). */
void* ref_tree_create(int prompt_tokens, std::uint64_t seed) { return new SearchTree(prompt_tokens, seed); }
void ref_tree_destroy(void* t) { delete static_cast<SearchTree*>(t); }
int ref_tree_add(void* t, std::uint32_t parent, int token_len) {
  try {
    return static_cast<int>(static_cast<SearchTree*>(t)->add_node(parent, token_len, false));
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}
void* ref_engine_create(const double* hw) {
  HardwareProfile h;
  h.weight_bytes = hw[0];
  h.mem_bandwidth = hw[1];
  h.peak_compute = hw[2];
  h.flops_per_token = hw[3];
  h.kv_bytes_per_token = hw[4];
  h.reward_latency = hw[5];
  return new DecodeEngine(h);
}
void ref_engine_destroy(void* e) { delete static_cast<DecodeEngine*>(e); }
int ref_engine_add_stream(void* e, int id, void* tree, std::uint32_t node, int tokens, double ready) {
  try {
    static_cast<DecodeEngine*>(e)->add_stream(id, static_cast<SearchTree*>(tree), node, tokens, ready);
    return 0;
  } catch (const Error& x) {
    g_err = x.what();
    return static_cast<int>(x.code()) + 1;
  }
}
int ref_engine_cancel(void* e, int id) { return static_cast<DecodeEngine*>(e)->cancel(id) ? 1 : 0; }
void ref_engine_drop(void* e, int id) { static_cast<DecodeEngine*>(e)->drop(id); }
double ref_engine_advance(void* e, double now, double limit, int* ids, int* tokens, int* cancelled, double* times,
                          int cap, int* n) {
  std::vector<DecodeEngine::Finished> out;
  const double r = static_cast<DecodeEngine*>(e)->advance(now, limit, out);
  *n = static_cast<int>(out.size());
  for (int i = 0; i < *n && i < cap; ++i) {
    ids[i] = out[i].id;
    tokens[i] = out[i].tokens_done;
    cancelled[i] = out[i].cancelled ? 1 : 0;
    times[i] = out[i].time;
  }
  return r;
}
int ref_engine_done_tokens(void* e, int id) { return static_cast<DecodeEngine*>(e)->done_tokens(id); }
int ref_engine_stream_count(void* e) { return static_cast<DecodeEngine*>(e)->stream_count(); }
int ref_engine_active_count(void* e) { return static_cast<DecodeEngine*>(e)->active_count(); }
double ref_engine_next_ready(void* e) { return static_cast<DecodeEngine*>(e)->next_ready(); }

}  // extern "C"

// ------------------------------------------------------------------ CLI
#ifdef REF_DRIVER_MAIN
int main(int argc, char** argv) {
  std::string config_path, flags, out;
  std::uint64_t seed = 0;
  bool have_seed = false, timed = false, no_trace = false;
  int reps = 1;
  for (int i = 1; i < argc; ++i) {
    std::string a = argv[i];
    auto next = [&]() { return std::string(argv[++i]); };
    if (a == "--config") config_path = next();
    else if (a == "--seed") { seed = std::stoull(next()); have_seed = true; }
    else if (a == "--flags") flags = next();
    else if (a == "--out") out = next();
    else if (a == "--time") timed = true;
    else if (a == "--no-trace") no_trace = true;
    else if (a == "--reps") reps = std::stoi(next());
  }
  std::ifstream in(config_path);
  std::stringstream ss;
  ss << in.rdbuf();
  ExperimentConfig cfg = ExperimentConfig::from_json(nlohmann::ordered_json::parse(ss.str()));
  if (!have_seed) seed = cfg.seed;
  const char* fcsv = flags.empty() ? nullptr : (flags == "baseline" ? "" : flags.c_str());
  SpexFlags fl = fcsv ? flags_from_string(fcsv) : cfg.flags;
  if (timed) {
    double secs = 0;
    double tot[24];
    ref_run_timed(ss.str().c_str(), seed, fcsv, !no_trace, reps, &secs, tot);
    std::cout << "{\"secs\": " << secs << ", \"reps\": " << reps << ", \"makespan\": " << tot[0]
              << ", \"queries\": " << tot[5] << "}\n";
    return 0;
  }
  RunOutcome o = run_once(cfg, seed, fl);
  std::ostream* os = &std::cout;
  std::ofstream f;
  if (!out.empty()) {
    f.open(out);
    os = &f;
  }
  for (const auto& l : o.log) *os << l << '\n';
  return 0;
}
#endif
