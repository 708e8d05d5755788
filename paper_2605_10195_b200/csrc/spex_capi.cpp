// spex_capi.cpp — host side of the C-ABI (include/spex.h).
//
// Parses and validates the experiment config exactly like
// ExperimentConfig::from_json/validate (proj/src/config.cpp:47-275), sizes the
// device arena, launches the persistent control kernel (ctl_kernel.cu) and
// serialises the binary event log with the same nlohmann::ordered_json dump
// the reference's TraceWriter uses (trace.cpp:32-36), so logs compare byte for
// byte.
//
// Built twice:
//   * product:  nvcc/g++ + ctl_kernel.cu -> libspex_b200.so (device path only)
//   * SPEX_EMU: g++ only -> build/emu/libspex_emu.so, a TEST-ONLY single-thread
//     emulation of the same control code used to check logic on a CPU box.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <sstream>
#include <thread>
#include <string>
#include <unordered_map>
#include <vector>

#include <json.hpp>

#include "../../include/spex.h"
#include "ctl_state.h"

#ifdef SPEX_EMU
#include "ctl_run.h"
#include "hook_tree.h"
#else
#include <cuda_runtime.h>

#include "model_host.h"
#endif

using nlohmann::ordered_json;
using namespace spex;

namespace {

thread_local std::string g_err;

struct SpexError {
  int code;
  std::string what;
};

[[noreturn]] void fail(int code, const std::string& msg) { throw SpexError{code, msg}; }

const char* errc_name(int code) {
  static const char* names[] = {"",
                                "UnknownParent",
                                "ParentPruned",
                                "NotSpeculative",
                                "UnknownNode",
                                "IllegalTransition",
                                "ZeroVisits",
                                "NoChildren",
                                "EmptyRewards",
                                "SearchComplete",
                                "NothingExpandable",
                                "UnknownSpeculation",
                                "NegativeWeight",
                                "EmptyTally",
                                "EmptyBatch",
                                "ConfigInvalid",
                                "IncompleteLog",
                                "IoFailure",
                                "InvalidArgument"};
  if (code >= 1 && code <= 18) return names[code];
  switch (code) {
    case ERR_CAP_NODES: return "CapacityNodes";
    case ERR_CAP_STREAMS: return "CapacityStreams";
    case ERR_CAP_LOG: return "CapacityLog";
    case ERR_CAP_STAGE: return "CapacityStage";
    case ERR_CAP_LABELS: return "CapacityLabels";
    case ERR_STALLED: return "NothingExpandable(stalled)";
    case ERR_CAP_KV: return "CapacityTreeKV";
    default: return "Internal";
  }
}

// ------------------------------------------------------------------ config
struct HostConfig {
  // mirrors ExperimentConfig (config.hpp:41-65)
  int family = kRstarDfs;
  double exploration_c = 1.0, balance_temperature = 1.0;
  int width = 4;
  std::vector<int> depth_widths;
  int target_answers = 10, max_depth = 16;
  double token_mu = 4.2485, token_sigma = 0.30;
  int token_min = 8, token_max = 400, shallow_min = 3;
  double shallow_p = 0.30;
  int shallow_max = 9, deep_min = 11;
  double deep_p = 0.25;
  int deep_max = 18;
  double skew = 0.0, golden_density = 0.55, reward_on = 0.8, reward_off = 0.3, noise_sigma = 0.0;
  double correct_base = 0.95, correct_slope = 0.07, correct_floor = 0.15;
  int answer_alphabet = 6, prompt_tokens = 32;
  double weight_bytes = 14e9, mem_bandwidth = 7e11, peak_compute = 1e14, flops_per_token = 14e9,
         kv_bytes_per_token = 0.0, reward_latency = 0.1;
  double tau = 2.0, ema_alpha = 0.2, initial_hit_ema = 0.5;
  double term_alpha = 0.5, min_frac = 0.6;
  int batch_size = 1, n_queries = 1, spec_k = 8, max_producers = 64;
  bool t1 = false, t2 = false, t3 = false;
  std::uint64_t seed = 1;
  int repetitions = 1;
};

const char* family_name(int f) {
  switch (f) {
    case kRstarDfs: return "rstar_dfs";
    case kRestHybrid: return "rest_hybrid";
    default: return "rebase_bfs";
  }
}

int family_from_name(const std::string& n) {
  if (n == "rstar_dfs") return kRstarDfs;
  if (n == "rest_hybrid") return kRestHybrid;
  if (n == "rebase_bfs") return kRebaseBfs;
  fail(ERR_CONFIG_INVALID, "unknown algorithm '" + n + "'");
}

// config.cpp:139-175
class SectionReader {
 public:
  SectionReader(const ordered_json& j, std::string name) : j_(j), name_(std::move(name)) {
    if (!j_.is_object()) fail(ERR_CONFIG_INVALID, name_ + ": expected an object");
  }
  template <typename T>
  void field(const char* key, T& out) {
    known_.push_back(key);
    auto it = j_.find(key);
    if (it == j_.end()) return;
    try {
      out = it->template get<T>();
    } catch (const ordered_json::exception&) {
      fail(ERR_CONFIG_INVALID, name_ + "." + key + ": wrong type");
    }
  }
  void finish() const {
    for (const auto& [key, value] : j_.items()) {
      (void)value;
      bool ok = false;
      for (const char* k : known_)
        if (key == k) ok = true;
      if (!ok) fail(ERR_CONFIG_INVALID, name_ + "." + key + ": unknown key");
    }
  }

 private:
  const ordered_json& j_;
  std::string name_;
  std::vector<const char*> known_;
};

void validate(const HostConfig& c) {
  auto bad = [](const std::string& w) { fail(ERR_CONFIG_INVALID, w); };
  // config.cpp:47-71
  if (c.exploration_c < 0.0) bad("policy.exploration_c: must be >= 0");
  if (c.balance_temperature <= 0.0) bad("policy.balance_temperature: must be > 0");
  if (c.width < 1) bad("policy.width: must be >= 1");
  for (int w : c.depth_widths)
    if (w < 1) bad("policy.depth_widths: entries must be >= 1");
  if (c.target_answers < 1) bad("policy.target_answers: must be >= 1");
  if (c.max_depth < 1) bad("policy.max_depth: must be >= 1");
  // sim.cpp:88-104
  if (c.token_min < 1 || c.token_max < c.token_min) bad("workload: bad token bounds");
  if (!(c.token_sigma >= 0.0) || !std::isfinite(c.token_mu)) bad("workload: bad token distribution");
  if (c.shallow_min < 1 || c.shallow_max < c.shallow_min) bad("workload: bad shallow depth range");
  if (c.deep_min <= c.shallow_max || c.deep_max < c.deep_min)
    bad("workload: deep range must sit above shallow range");
  if (c.shallow_p < 0.0 || c.shallow_p > 1.0 || c.deep_p < 0.0 || c.deep_p > 1.0)
    bad("workload: bad stop probability");
  if (c.skew < 0.0 || c.skew > 1.0) bad("workload: bad skew");
  if (c.golden_density < 0.0 || c.golden_density > 1.0) bad("workload: bad golden density");
  if (c.reward_on < 0.0 || c.reward_on > 1.0 || c.reward_off < 0.0 || c.reward_off > 1.0)
    bad("workload: rewards outside [0,1]");
  if (c.noise_sigma < 0.0) bad("workload: negative noise sigma");
  if (c.correct_base <= 0.0 || c.correct_base > 1.0 || c.correct_slope < 0.0 ||
      c.correct_floor < 0.0 || c.correct_floor > c.correct_base)
    bad("workload: bad correctness curve");
  if (c.answer_alphabet < 2) bad("workload: alphabet needs at least two labels");
  if (c.prompt_tokens < 0) bad("workload: negative prompt length");
  // budget.cpp:8-19
  auto pos = [&](double v, const char* n) {
    if (!(v > 0.0)) bad(std::string(n) + " must be positive");
  };
  pos(c.weight_bytes, "weight_bytes");
  pos(c.mem_bandwidth, "mem_bandwidth");
  pos(c.peak_compute, "peak_compute");
  pos(c.flops_per_token, "flops_per_token");
  if (c.kv_bytes_per_token < 0.0) bad("kv_bytes_per_token must be non-negative");
  if (c.reward_latency < 0.0) bad("reward_latency must be non-negative");
  if (c.tau < 0.0) bad("budget.tau: must be >= 0");
  if (c.ema_alpha <= 0.0 || c.ema_alpha > 1.0) bad("budget.ema_alpha: must be in (0,1]");
  if (c.initial_hit_ema < 0.0 || c.initial_hit_ema > 1.0) bad("budget.initial_hit_ema: must be in [0,1]");
  if (c.term_alpha < 0.0) bad("termination.alpha: must be >= 0");
  if (c.min_frac < 0.0 || c.min_frac > 1.0) bad("termination.min_frac: must be in [0,1]");
  if (c.batch_size < 1) bad("run.batch_size: must be >= 1");
  if (c.n_queries < 1) bad("run.n_queries: must be >= 1");
  if (c.spec_k < 0) bad("run.spec_k: must be >= 0");
  if (c.max_producers < 1) bad("run.max_producers: must be >= 1");
  if (c.repetitions < 1) bad("run.repetitions: must be >= 1");
  // device-path limits (capacity, not semantics)
  if (c.answer_alphabet > kMaxLabels) fail(ERR_CAP_LABELS, "answer_alphabet > 64 unsupported");
  if (c.spec_k > 64) fail(ERR_CAP_STAGE, "spec_k > 64 unsupported");
  if (static_cast<int>(c.depth_widths.size()) > kMaxDepthWidths)
    fail(ERR_CAP_STAGE, "more than 64 depth_widths unsupported");
}

// config.cpp:177-275
HostConfig parse_config(const std::string& text) {
  ordered_json j = ordered_json::parse(text, nullptr, false);
  if (j.is_discarded()) fail(ERR_CONFIG_INVALID, "config is not valid JSON");
  HostConfig c;
  if (!j.is_object()) fail(ERR_CONFIG_INVALID, "config: expected a JSON object");
  for (const auto& [key, value] : j.items()) {
    (void)value;
    if (key != "family" && key != "policy" && key != "workload" && key != "hardware" &&
        key != "budget" && key != "termination" && key != "run")
      fail(ERR_CONFIG_INVALID, key + ": unknown section");
  }
  if (j.contains("family")) {
    if (!j["family"].is_string()) fail(ERR_CONFIG_INVALID, "family: expected a string");
    c.family = family_from_name(j["family"].get<std::string>());
  }
  if (j.contains("policy")) {
    SectionReader s(j["policy"], "policy");
    s.field("exploration_c", c.exploration_c);
    s.field("balance_temperature", c.balance_temperature);
    s.field("width", c.width);
    s.field("depth_widths", c.depth_widths);
    s.field("target_answers", c.target_answers);
    s.field("max_depth", c.max_depth);
    s.finish();
  }
  if (j.contains("workload")) {
    SectionReader s(j["workload"], "workload");
    s.field("token_mu", c.token_mu);
    s.field("token_sigma", c.token_sigma);
    s.field("token_min", c.token_min);
    s.field("token_max", c.token_max);
    s.field("shallow_min", c.shallow_min);
    s.field("shallow_p", c.shallow_p);
    s.field("shallow_max", c.shallow_max);
    s.field("deep_min", c.deep_min);
    s.field("deep_p", c.deep_p);
    s.field("deep_max", c.deep_max);
    s.field("skew", c.skew);
    s.field("golden_density", c.golden_density);
    s.field("reward_on", c.reward_on);
    s.field("reward_off", c.reward_off);
    s.field("noise_sigma", c.noise_sigma);
    s.field("correct_base", c.correct_base);
    s.field("correct_slope", c.correct_slope);
    s.field("correct_floor", c.correct_floor);
    s.field("answer_alphabet", c.answer_alphabet);
    s.field("prompt_tokens", c.prompt_tokens);
    s.finish();
  }
  if (j.contains("hardware")) {
    SectionReader s(j["hardware"], "hardware");
    s.field("weight_bytes", c.weight_bytes);
    s.field("mem_bandwidth", c.mem_bandwidth);
    s.field("peak_compute", c.peak_compute);
    s.field("flops_per_token", c.flops_per_token);
    s.field("kv_bytes_per_token", c.kv_bytes_per_token);
    s.field("reward_latency", c.reward_latency);
    s.finish();
  }
  if (j.contains("budget")) {
    SectionReader s(j["budget"], "budget");
    s.field("tau", c.tau);
    s.field("ema_alpha", c.ema_alpha);
    s.field("initial_hit_ema", c.initial_hit_ema);
    s.finish();
  }
  if (j.contains("termination")) {
    SectionReader s(j["termination"], "termination");
    s.field("alpha", c.term_alpha);
    s.field("min_frac", c.min_frac);
    s.finish();
  }
  if (j.contains("run")) {
    SectionReader s(j["run"], "run");
    s.field("batch_size", c.batch_size);
    s.field("n_queries", c.n_queries);
    s.field("spec_k", c.spec_k);
    s.field("max_producers", c.max_producers);
    s.field("seed", c.seed);
    s.field("repetitions", c.repetitions);
    std::vector<std::string> fl;
    s.field("flags", fl);
    s.finish();
    if (j["run"].contains("flags")) {
      c.t1 = c.t2 = c.t3 = false;
      for (const std::string& n : fl) {
        if (n == "t1") c.t1 = true;
        else if (n == "t2") c.t2 = true;
        else if (n == "t3") c.t3 = true;
        else fail(ERR_CONFIG_INVALID, "run.flags: unknown flag " + n);
      }
    }
  }
  validate(c);
  return c;
}

void flags_from_csv(const std::string& csv, HostConfig& c) {
  c.t1 = c.t2 = c.t3 = false;
  std::stringstream ss(csv);
  std::string item;
  while (std::getline(ss, item, ',')) {
    if (item.empty()) continue;
    if (item == "t1") c.t1 = true;
    else if (item == "t2") c.t2 = true;
    else if (item == "t3") c.t3 = true;
    else fail(ERR_CONFIG_INVALID, "unknown flag: " + item);
  }
}

// config.cpp:73-137
ordered_json to_json(const HostConfig& c, bool t1, bool t2, bool t3) {
  ordered_json j;
  j["family"] = family_name(c.family);
  ordered_json p;
  p["exploration_c"] = c.exploration_c;
  p["balance_temperature"] = c.balance_temperature;
  p["width"] = c.width;
  p["depth_widths"] = c.depth_widths;
  p["target_answers"] = c.target_answers;
  p["max_depth"] = c.max_depth;
  j["policy"] = p;
  ordered_json w;
  w["token_mu"] = c.token_mu;
  w["token_sigma"] = c.token_sigma;
  w["token_min"] = c.token_min;
  w["token_max"] = c.token_max;
  w["shallow_min"] = c.shallow_min;
  w["shallow_p"] = c.shallow_p;
  w["shallow_max"] = c.shallow_max;
  w["deep_min"] = c.deep_min;
  w["deep_p"] = c.deep_p;
  w["deep_max"] = c.deep_max;
  w["skew"] = c.skew;
  w["golden_density"] = c.golden_density;
  w["reward_on"] = c.reward_on;
  w["reward_off"] = c.reward_off;
  w["noise_sigma"] = c.noise_sigma;
  w["correct_base"] = c.correct_base;
  w["correct_slope"] = c.correct_slope;
  w["correct_floor"] = c.correct_floor;
  w["answer_alphabet"] = c.answer_alphabet;
  w["prompt_tokens"] = c.prompt_tokens;
  j["workload"] = w;
  ordered_json h;
  h["weight_bytes"] = c.weight_bytes;
  h["mem_bandwidth"] = c.mem_bandwidth;
  h["peak_compute"] = c.peak_compute;
  h["flops_per_token"] = c.flops_per_token;
  h["kv_bytes_per_token"] = c.kv_bytes_per_token;
  h["reward_latency"] = c.reward_latency;
  j["hardware"] = h;
  ordered_json b;
  b["tau"] = c.tau;
  b["ema_alpha"] = c.ema_alpha;
  b["initial_hit_ema"] = c.initial_hit_ema;
  j["budget"] = b;
  ordered_json t;
  t["alpha"] = c.term_alpha;
  t["min_frac"] = c.min_frac;
  j["termination"] = t;
  ordered_json r;
  r["batch_size"] = c.batch_size;
  r["n_queries"] = c.n_queries;
  r["spec_k"] = c.spec_k;
  r["max_producers"] = c.max_producers;
  std::vector<std::string> fl;
  if (t1) fl.push_back("t1");
  if (t2) fl.push_back("t2");
  if (t3) fl.push_back("t3");
  r["flags"] = fl;
  r["seed"] = c.seed;
  r["repetitions"] = c.repetitions;
  j["run"] = r;
  return j;
}

// budget.cpp:23-39
int roofline_k_total(const HostConfig& c, int active, double avg_kv, int cap) {
  double compute_slope = c.flops_per_token / c.peak_compute;
  double memory_slope = avg_kv / c.mem_bandwidth;
  double weight_time = c.weight_bytes / c.mem_bandwidth;
  int b_star;
  if (compute_slope <= memory_slope) {
    b_star = cap;
  } else {
    double knee = std::ceil(weight_time / (compute_slope - memory_slope));
    b_star = knee < static_cast<double>(cap) ? static_cast<int>(knee) : cap;
  }
  return std::max(0, b_star - active);
}

std::vector<double>& log_table() {
  static std::vector<double> tab;
  static std::once_flag once;
  std::call_once(once, [] {
    tab.resize(1 << 16);
    tab[0] = -HUGE_VAL;
    for (size_t n = 1; n < tab.size(); ++n) tab[n] = std::log(static_cast<double>(n));
  });
  return tab;
}

// --------------------------------------------------------------- arena
struct Arena {
  std::vector<std::pair<void**, size_t>> parts;
  size_t total = 0;
  size_t hot = 0;  // bytes of the leading control-state region (L2 access-policy window)
  void mark_hot() { hot = total; }
  template <class T>
  void add(T*& p, size_t count) {
    parts.push_back({reinterpret_cast<void**>(&p), count * sizeof(T)});
    total += (count * sizeof(T) + 255) & ~size_t(255);
  }
  void carve(char* base) {
    size_t off = 0;
    for (auto& [pp, bytes] : parts) {
      *pp = base + off;
      off += (bytes + 255) & ~size_t(255);
    }
  }
};

}  // namespace

// ================================================================ executor
// Stepwise execution state (spex_frontier_step): the run's arena stays on the
// device (host memory in the emulation) between calls.
struct StepRun {
  Run R{};
  char* base = nullptr;
  Run* d_run = nullptr;
  double* d_tab = nullptr;
  std::vector<char> host_mem;  // emulation arena
  std::vector<int> sm;
  std::vector<double> smd;
  std::vector<long long> sml;
  std::vector<int> warp_off;
  long long sent = 0;  // records already returned
};

struct spex_executor {
  HostConfig hc;
  bool t1 = false, t2 = false, t3 = false;
  std::uint64_t run_seed = 0;
  int device = 0;
  bool ran = false;
  Run run{};  // host copy holding device pointers
  char* d_base = nullptr;
  Run* d_run = nullptr;
  GState* d_g = nullptr;
  double* d_logtab = nullptr;
  GState g{};
  std::vector<Rec> log;
  std::vector<QueryRun> qs;
  std::string cfg_dump;
  double device_ms = 0.0;
  int nthreads = 512;
  int record_sched = 0;
  int shard_lo = 0, shard_hi = -1;  // owned query range of the model work (-1: all)
  long long kv_pages_req = 0;       // tree-KV pool pages (0: sized from free HBM when a model is attached)
  long long kv_pt_cap = 0;          // page-table entries of the last run
  long long kv_pages = 0;           // pool pages of the last run
  int reward_prm = 0;               // reward source: 0 content oracle (reference), 1 PRM score
  std::vector<long long> finish_ns; // per-query device wall clock at query_done
  // split mode (spex_executor_set_split): rank / world of the job's query blocks
  int split_rank = 0, split_world = 1, split_qjob = 0;
  long long split_epoch = 0;
  std::vector<char*> split_boxes;   // the ranks' outboxes (device pointers; host memory in the emulation)
  int node_cap0 = 0;                // initial node capacity (0: 512 or SPEX_NODE_CAP)
  int split_emulate = 0;            // spex_executor_emulate_split: the other ranks run beside this one
  std::string cfg_text, flags_text; // as created (the emulated ranks' executors)
  char* emu_boxes = nullptr;        // the emulation's outboxes (device)
  std::unique_ptr<StepRun> step;    // stepwise execution in progress
#ifndef SPEX_EMU
  cudaStream_t stream = nullptr;
  cudaStream_t mstream = nullptr;
  bool with_model = false;
  std::vector<std::pair<const char*, double>> host_marks;  // SPEX_TIMING: host phase wall times
  ModelRunConfig mc;
  ModelRunResult mres;
  std::vector<DecodeOut> dec_out;
  std::vector<PrmOut> prm_out;
#endif
};

#ifndef SPEX_EMU
extern "C" int spex_launch_control(Run* d_run, int n_queries, int nthreads, cudaStream_t stream, float* ms);
extern "C" int spex_launch_control_async(Run* d_run, int n_queries, int nthreads, cudaStream_t stream, cudaEvent_t a,
                                         cudaEvent_t b);
extern "C" int spex_launch_control_batch_async(Run* d_runs, int n_runs, int n_queries, int nthreads,
                                               cudaStream_t stream, cudaEvent_t a, cudaEvent_t b);
extern "C" void spex_model_cache_clear();
extern "C" void spex_model_cache_release_mismatch(const ModelRunConfig* mc);
extern "C" long long spex_model_pool_slots(const ModelRunConfig* mc);
extern "C" void spex_model_prepare(const ModelRunConfig* mc, const ScheduleView* sv, cudaStream_t st);
#define CUDA_OK(x)                                                                  \
  do {                                                                              \
    cudaError_t e_ = (x);                                                           \
    if (e_ != cudaSuccess) fail(200, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)
#endif

namespace {

#ifndef SPEX_EMU
// The default stream-ordered pool returns freed memory to the driver at every
// synchronisation (release threshold 0): each search would unmap and remap its
// arena (measured: 0.1-1 s of host time per search). Keep it cached instead.
void keep_pool_memory(int device) {
  static std::mutex mu;
  static unsigned long long done = 0;
  std::lock_guard<std::mutex> lk(mu);
  if (device < 0 || device >= 64 || (done >> device) & 1ULL) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  cudaGetLastError();
  done |= 1ULL << device;
}

// Pinned, device-mapped host buffers for the streamed schedule, recycled
// across searches (cudaHostAlloc / cudaFreeHost cost milliseconds and may
// synchronise the device).
struct PinnedCache {
  std::mutex mu;
  std::vector<std::pair<void*, size_t>> free_list;
};
PinnedCache& pinned_cache() {
  static PinnedCache c;
  return c;
}
std::unordered_map<void*, size_t>& pinned_sizes() {
  static std::unordered_map<void*, size_t> m;
  return m;
}
void* pinned_acquire(size_t bytes) {
  PinnedCache& c = pinned_cache();
  {
    std::lock_guard<std::mutex> lk(c.mu);
    for (size_t i = 0; i < c.free_list.size(); ++i)
      if (c.free_list[i].second >= bytes) {
        void* p = c.free_list[i].first;
        c.free_list.erase(c.free_list.begin() + static_cast<long>(i));
        return p;
      }
  }
  void* p = nullptr;
  if (cudaHostAlloc(&p, bytes, cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess)
    fail(200, "cudaHostAlloc failed");
  std::lock_guard<std::mutex> lk(c.mu);
  pinned_sizes()[p] = bytes;
  return p;
}
void pinned_release(void* p) {
  PinnedCache& c = pinned_cache();
  std::lock_guard<std::mutex> lk(c.mu);
  c.free_list.push_back({p, pinned_sizes()[p]});
}
#endif

// split mode: query block [lo(r), lo(r + 1)) of rank r, its largest size and
// the outbox geometry (ctl_run.h split_exchange)
int split_block_lo(int q, int r, int w) { return static_cast<int>(static_cast<long long>(q) * r / w); }
int split_qmax(int q, int w) { return (q + w - 1) / w; }
long long split_slot_bytes(int qmax) { return (16 + 12LL * qmax + 15) / 16 * 16; }
long long split_outbox_bytes(int qmax) { return kXchHead + 2 * split_slot_bytes(qmax); }

void set_cfg(const spex_executor& ex, Cfg& c, int node_cap, int stream_cap, int log_cap,
             int stage_cap, int trace, int record_sched) {
  const HostConfig& h = ex.hc;
  std::memset(&c, 0, sizeof(c));
  c.family = h.family;
  c.exploration_c = h.exploration_c;
  c.balance_temperature = h.balance_temperature;
  c.width = h.width;
  c.n_depth_widths = static_cast<int>(h.depth_widths.size());
  for (int i = 0; i < c.n_depth_widths; ++i) c.depth_widths[i] = h.depth_widths[i];
  c.target_answers = h.target_answers;
  c.max_depth = h.max_depth;
  c.token_mu = h.token_mu;
  c.token_sigma = h.token_sigma;
  c.token_min = h.token_min;
  c.token_max = h.token_max;
  c.shallow_min = h.shallow_min;
  c.shallow_p = h.shallow_p;
  c.shallow_max = h.shallow_max;
  c.deep_min = h.deep_min;
  c.deep_p = h.deep_p;
  c.deep_max = h.deep_max;
  c.skew = h.skew;
  c.golden_density = h.golden_density;
  c.reward_on = h.reward_on;
  c.reward_off = h.reward_off;
  c.noise_sigma = h.noise_sigma;
  c.correct_base = h.correct_base;
  c.correct_slope = h.correct_slope;
  c.correct_floor = h.correct_floor;
  c.answer_alphabet = h.answer_alphabet;
  c.prompt_tokens = h.prompt_tokens;
  c.weight_bytes = h.weight_bytes;
  c.mem_bandwidth = h.mem_bandwidth;
  c.peak_compute = h.peak_compute;
  c.flops_per_token = h.flops_per_token;
  c.kv_bytes_per_token = h.kv_bytes_per_token;
  c.reward_latency = h.reward_latency;
  c.tau = h.tau;
  c.ema_alpha = h.ema_alpha;
  c.initial_hit_ema = h.initial_hit_ema;
  c.term_alpha = h.term_alpha;
  c.min_frac = h.min_frac;
  c.min_answers = static_cast<int>(std::ceil(h.min_frac * h.target_answers));  // config.cpp:43-45
  c.batch_size = h.batch_size;
  c.n_queries = h.n_queries;
  c.spec_k = h.spec_k;
  c.max_producers = h.max_producers;
  c.t1 = ex.t1;
  c.t2 = ex.t2;
  c.t3 = ex.t3;
  // executor.cpp:817-818
  c.producer_slots = std::max(1, std::min(h.max_producers, roofline_k_total(h, 0, 0.0, 1024)));
  c.run_seed = ex.run_seed;
  c.node_cap = node_cap;
  c.stream_cap = stream_cap;
  c.log_cap = log_cap;
  c.stage_cap = stage_cap;
  c.trace = trace;
  c.record_sched = record_sched;
  c.reward_prm = ex.reward_prm;
  c.shard_lo = std::min(ex.shard_lo, h.n_queries);
  c.shard_hi = ex.shard_hi < 0 ? h.n_queries : std::min(ex.shard_hi, h.n_queries);
  c.split_world = ex.split_world;
  c.split_rank = ex.split_rank;
  c.q_offset = ex.split_world > 1 ? split_block_lo(ex.split_qjob, ex.split_rank, ex.split_world) : 0;
  c.split_qmax = ex.split_world > 1 ? split_qmax(ex.split_qjob, ex.split_world) : 0;
  c.split_epoch = ex.split_epoch;
  c.xch_slot_bytes = split_slot_bytes(c.split_qmax);
  c.sched_cap = record_sched ? 4 * stream_cap + 1024 : 1;
  c.sched_rows_cap = record_sched ? 64 * stream_cap + 4096 : 1;
  // std::map<std::string,...> order of "a0".."a{n-1}" (termination.hpp:39)
  std::vector<std::pair<std::string, int>> names;
  for (int i = 0; i < h.answer_alphabet; ++i) names.push_back({"a" + std::to_string(i), i});
  std::sort(names.begin(), names.end());
  for (int r = 0; r < h.answer_alphabet; ++r) {
    c.lex_order[r] = names[r].second;
    c.lex_rank[names[r].second] = r;
  }
}

void layout(Arena& A, Run& R, int Q, int node_cap, int stream_cap, int log_cap, int slots,
            int stage_cap) {
  const size_t NN = static_cast<size_t>(Q) * node_cap;
  A.add(R.g, 1);
  A.add(R.n_parent, NN);
  A.add(R.n_depth, NN);
  A.add(R.n_slot, NN);
  A.add(R.n_tokens, NN);
  A.add(R.n_status, NN);
  A.add(R.n_flags, NN);
  A.add(R.n_reward, NN);
  A.add(R.n_value, NN);
  A.add(R.n_visits, NN);
  A.add(R.n_hash, NN);
  A.add(R.n_first_child, NN);
  A.add(R.n_last_child, NN);
  A.add(R.n_next_sib, NN);
  A.add(R.n_nchildren, NN);
  A.add(R.n_pred, NN);
  A.add(R.n_stream, NN);
  A.add(R.n_ready, NN);
  A.add(R.n_refc, NN);
  A.add(R.n_kvbase, NN);
  A.add(R.n_kvh, NN);
  A.add(R.qs, Q);
  A.add(R.q_tally, Q);
  A.add(R.q_finish_ns, Q);
  A.add(R.q_dirty, Q + 64);
  A.add(R.q_rest_stack, NN);
  A.add(R.q_layer, NN);
  A.add(R.q_cohort, NN);
  const size_t S = stream_cap;
  A.add(R.st_q, S);
  A.add(R.st_node, S);
  A.add(R.st_rem, S);
  A.add(R.st_done, S);
  A.add(R.st_state, S);
  A.add(R.st_cancel, S);
  A.add(R.st_ready, S);
  A.add(R.live, S);
  A.add(R.live_tmp, S);
  A.add(R.fins, S);
  A.add(R.fin_tokens, S);
  A.add(R.fin_cancel, S);
  A.add(R.ev_time, S);
  A.add(R.ev_q, S);
  A.add(R.ev_node, S);
  const size_t W = static_cast<size_t>(slots) * stage_cap;  // one staging slot per control thread
  A.add(R.stage_rec, W);
  A.add(R.stage_spawn, W);
  A.add(R.stage_push, W);
  const size_t IC = std::max<size_t>(S, Q) + 64;
  R.item_cap = static_cast<int>(IC);
  A.add(R.it_key, IC);
  A.add(R.it_warp, IC);
  A.add(R.it_rec_off, IC);
  A.add(R.it_rec_n, IC);
  A.add(R.it_spawn_off, IC);
  A.add(R.it_spawn_n, IC);
  A.add(R.it_push_off, IC);
  A.add(R.it_push_n, IC);
  A.add(R.it_fin, IC);
  A.add(R.it_sdelta, IC);
  A.add(R.it_tok, IC);
  A.add(R.it_scan_e, IC);
  A.add(R.fin_scored, IC);
  A.add(R.it_scan_a, IC);
  A.add(R.it_scan_b, IC);
  A.add(R.it_scan_c, IC);
  A.add(R.it_scan_d, IC);
  const size_t SS = static_cast<size_t>(slots) * (node_cap + 64);
  A.add(R.sp_visits, SS);
  A.add(R.sp_value, SS);
  A.add(R.sp_nchild, SS);
  A.add(R.sp_stack, SS);
  A.add(R.sp_dbl, 3 * SS);
  A.add(R.sp_int, 3 * SS);
  // allocation scratch: in split mode it holds every rank's candidates
  const size_t QA = static_cast<size_t>(std::max(Q, R.cfg.split_qmax * R.cfg.split_world)) + 64;
  A.add(R.al_cand, Q + 64);
  A.add(R.al_score, QA);
  A.add(R.al_w, QA);
  A.add(R.al_out, QA);
  A.add(R.al_rank, QA);
  A.add(R.al_order, QA);
  A.mark_hot();  // everything above is touched every consumer iteration; below: log and model schedule
  A.add(R.log, static_cast<size_t>(log_cap));
  A.add(R.sched_kind, static_cast<size_t>(R.cfg.sched_cap));
  A.add(R.sched_steps, static_cast<size_t>(R.cfg.sched_cap));
  A.add(R.sched_off, static_cast<size_t>(R.cfg.sched_cap));
  A.add(R.sched_n, static_cast<size_t>(R.cfg.sched_cap));
  A.add(R.srow_sid, static_cast<size_t>(R.cfg.sched_rows_cap));
  A.add(R.srow_pos0, static_cast<size_t>(R.cfg.sched_rows_cap));
  A.add(R.sched_u, static_cast<size_t>(R.cfg.sched_cap));
  A.add(R.srow_rstart, static_cast<size_t>(R.cfg.sched_rows_cap));
  A.add(R.srow_tstart, static_cast<size_t>(R.cfg.sched_rows_cap));
  if (R.cfg.record_sched) A.add(R.pub_e, static_cast<size_t>(R.cfg.sched_cap));
  if (R.cfg.reward_prm) {
    A.add(R.n_score, NN);
    A.add(R.n_prm_e, NN);
    A.add(R.prm_done, static_cast<size_t>(R.cfg.sched_cap));
  }
}

std::string label_str(int idx) { return idx < 0 ? std::string() : "a" + std::to_string(idx); }

// TraceWriter::emit (trace.cpp:32-36) with the executor's field order
// (executor.cpp:134-155,179-186,214-221,244-250,288-292,318-325,346-354,381-403,421-426)
void serialize_header(const spex_executor& ex, std::string& out) {
  ordered_json j;
  j["t"] = 0.0;
  j["ev"] = "run_begin";
  j["seed"] = ex.run_seed;
  j["config"] = ordered_json::parse(ex.cfg_dump);
  out += j.dump();
  out += '\n';
}

void serialize_record(const Rec& r, std::string& out) {
  ordered_json j;
  j["t"] = r.t;
  switch (r.kind) {
    case EV_ADMIT:
      j["ev"] = "admit";
      j["q"] = r.q;
      j["seed"] = static_cast<std::uint64_t>(r.y);
      break;
    case EV_NODE:
      j["ev"] = "node";
      j["q"] = r.q;
      j["node"] = r.node;
      j["parent"] = static_cast<std::uint32_t>(r.a);
      j["slot"] = r.b;
      j["spec"] = (r.flags & RF_SPEC) != 0;
      j["tokens"] = r.c;
      j["terminal"] = (r.flags & RF_TERMINAL) != 0;
      break;
    case EV_REQ:
      j["ev"] = "req";
      j["q"] = r.q;
      j["node"] = r.node;
      j["stream"] = r.a;
      j["spec"] = (r.flags & RF_SPEC) != 0;
      j["dist"] = r.b;
      break;
    case EV_DONE:
      j["ev"] = "done";
      j["q"] = r.q;
      j["node"] = r.node;
      j["stream"] = r.a;
      j["tokens"] = r.b;
      j["cancelled"] = (r.flags & RF_CANCELLED) != 0;
      j["stale"] = (r.flags & RF_STALE) != 0;
      break;
    case EV_REWARD:
      j["ev"] = "reward";
      j["q"] = r.q;
      j["node"] = r.node;
      j["r"] = r.x;
      break;
    case EV_PROMOTE:
      j["ev"] = "promote";
      j["q"] = r.q;
      j["node"] = r.node;
      j["ready"] = static_cast<long long>(r.y);
      j["dist"] = r.a;
      break;
    case EV_PRUNE:
      j["ev"] = "prune";
      j["q"] = r.q;
      j["node"] = r.node;
      j["count"] = r.a;
      break;
    case EV_ANSWER:
      j["ev"] = "answer";
      j["q"] = r.q;
      j["node"] = r.node;
      j["label"] = label_str(r.a);
      j["weight"] = r.x;
      j["correct"] = (r.flags & RF_CORRECT) != 0;
      break;
    case EV_TERMINATE:
      j["ev"] = "terminate";
      j["q"] = r.q;
      j["label"] = label_str(r.a);
      j["answers"] = r.b;
      break;
    case EV_QUERY_DONE:
      j["ev"] = "query_done";
      j["q"] = r.q;
      j["label"] = label_str(r.a);
      j["correct"] = (r.flags & RF_CORRECT) != 0;
      j["answers"] = r.b;
      j["early"] = (r.flags & RF_EARLY) != 0;
      break;
    default:
      j["ev"] = "?";
      break;
  }
  out += j.dump();
  out += '\n';
}

void serialize_footer(const spex_executor& ex, std::string& out) {
  long long gen = 0, com = 0, reu = 0, was = 0;
  for (const QueryRun& q : ex.qs) {
    gen += q.generated;
    com += q.committed;
    reu += q.reused;
    was += q.wasted;
  }
  ordered_json j;
  j["t"] = ex.g.makespan;
  j["ev"] = "run_end";
  j["makespan"] = ex.g.makespan;
  j["generated"] = gen;
  j["committed"] = com;
  j["reused"] = reu;
  j["wasted"] = was;
  j["queries"] = ex.g.finished_count;
  out += j.dump();
  out += '\n';
}

void serialize(const spex_executor& ex, std::string& out) {
  out.clear();
  out.reserve(ex.log.size() * 96 + 4096);
  serialize_header(ex, out);
  for (const Rec& r : ex.log) serialize_record(r, out);
  serialize_footer(ex, out);
}

void fill_totals(const spex_executor& ex, spex_totals* t) {
  std::memset(t, 0, sizeof(*t));
  t->makespan = ex.g.makespan;
  for (const QueryRun& q : ex.qs) {
    if (!q.admitted) continue;
    t->generated_tokens += q.generated;
    t->committed_tokens += q.committed;
    t->reused_tokens += q.reused;
    t->wasted_tokens += q.wasted;
    for (int d = 1; d <= SPEX_MAX_TRACKED; ++d) {
      t->hits[d] += q.hits[d];
      t->misses[d] += q.misses[d];
    }
    if (q.finished) {
      t->queries += 1;
      t->correct_votes += q.correct;
      t->early_terminated += q.early;
    }
  }
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const SpexError& e) {
    g_err = std::string(errc_name(e.code)) + ": " + e.what;
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return ERR_INTERNAL;
  }
}

// ---------------------------------------------------------- stepwise execution
void step_release(spex_executor& ex) {
  if (!ex.step) return;
#ifndef SPEX_EMU
  if (ex.step->base) cudaFree(ex.step->base);
  if (ex.step->d_run) cudaFree(ex.step->d_run);
  if (ex.step->d_tab) cudaFree(ex.step->d_tab);
#endif
  ex.step.reset();
}

// Set up the run's arena (trace on) for stepwise execution.
void step_begin(spex_executor& ex) {
  const int Q = ex.hc.n_queries;
  int node_cap = 512;
  if (const char* e = std::getenv("SPEX_NODE_CAP")) node_cap = std::max(16, std::atoi(e));
  if (ex.node_cap0 > 0) node_cap = ex.node_cap0;
  const long long sc = static_cast<long long>(Q) * (node_cap - 1) + 64;
  const long long lc = static_cast<long long>(Q) * node_cap * 6 + 64;
  if (sc > (1LL << 30) || lc > (1LL << 31) - 1) fail(ERR_CAP_STREAMS, "stepwise run too large");
  const int stage_cap = std::max(512, node_cap);
  auto st = std::make_unique<StepRun>();
  Run& R = st->R;
  ex.record_sched = 0;
  set_cfg(ex, R.cfg, node_cap, static_cast<int>(sc), static_cast<int>(lc), stage_cap, 1, 0);
  Arena A;
  layout(A, R, Q, node_cap, static_cast<int>(sc), static_cast<int>(lc), ex.nthreads, stage_cap);
  R.nwarps = ex.nthreads / 32;
  std::vector<double>& tab = log_table();
  R.log_tab_n = static_cast<int>(tab.size());
#ifdef SPEX_EMU
  st->host_mem.assign(A.total + 256, 0);
  char* base = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(st->host_mem.data()) + 255) & ~uintptr_t(255));
  A.carve(base);
  R.log_tab = tab.data();
  for (int q = 0; q < Q; ++q) R.qs[q].plan_empty_version = 0xffffffffu;
  st->sm.assign(2048, 0);
  st->smd.assign(64, 0.0);
  st->sml.assign(64, 0);
  st->warp_off.assign(3 * 64, 0);
#else
  CUDA_OK(cudaSetDevice(ex.device));
  if (!ex.stream) CUDA_OK(cudaStreamCreateWithFlags(&ex.stream, cudaStreamNonBlocking));
  CUDA_OK(cudaMalloc(reinterpret_cast<void**>(&st->base), A.total + 256));
  CUDA_OK(cudaMemsetAsync(st->base, 0, A.total + 256, ex.stream));
  A.carve(st->base);
  CUDA_OK(cudaMalloc(reinterpret_cast<void**>(&st->d_tab), tab.size() * sizeof(double)));
  CUDA_OK(cudaMemcpyAsync(st->d_tab, tab.data(), tab.size() * sizeof(double), cudaMemcpyHostToDevice, ex.stream));
  R.log_tab = st->d_tab;
  CUDA_OK(cudaMalloc(reinterpret_cast<void**>(&st->d_run), sizeof(Run)));
  CUDA_OK(cudaMemcpyAsync(st->d_run, &R, sizeof(Run), cudaMemcpyHostToDevice, ex.stream));
  CUDA_OK(cudaStreamSynchronize(ex.stream));
#endif
  ex.step = std::move(st);
  ex.log.clear();
}

// Run up to `iters` consumer-loop iterations (0: to the end), then bring the
// run scalars and the new records back.
void step_run(spex_executor& ex, long long iters) {
  StepRun& st = *ex.step;
  Run& R = st.R;
  const int Q = ex.hc.n_queries;
#ifdef SPEX_EMU
  R.g->step_iters = iters;
  HostExec hx;
  hx.sm = st.sm.data();
  hx.smd = st.smd.data();
  hx.sml = st.sml.data();
  run_loop(&R, hx, st.warp_off.data());
  ex.g = *R.g;
  const long long n0 = static_cast<long long>(ex.log.size());
  for (long long i = n0; i < ex.g.log_n; ++i) ex.log.push_back(R.log[i]);
  if (ex.g.phase == 2 || ex.g.error) ex.qs.assign(R.qs, R.qs + Q);
#else
  CUDA_OK(cudaMemcpyAsync(reinterpret_cast<char*>(R.g) + offsetof(GState, step_iters), &iters, sizeof(iters),
                          cudaMemcpyHostToDevice, ex.stream));
  cudaEvent_t ca, cb;
  cudaEventCreate(&ca);
  cudaEventCreate(&cb);
  const int lr = spex_launch_control_async(st.d_run, Q, ex.nthreads, ex.stream, ca, cb);
  if (lr != 0) fail(200, std::string("control kernel launch failed: ") + cudaGetErrorString(static_cast<cudaError_t>(lr)));
  CUDA_OK(cudaEventSynchronize(cb));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, ca, cb);
  cudaEventDestroy(ca);
  cudaEventDestroy(cb);
  ex.device_ms += ms;
  CUDA_OK(cudaMemcpyAsync(&ex.g, R.g, sizeof(GState), cudaMemcpyDeviceToHost, ex.stream));
  CUDA_OK(cudaStreamSynchronize(ex.stream));
  const long long n0 = static_cast<long long>(ex.log.size());
  if (ex.g.log_n > n0) {
    ex.log.resize(ex.g.log_n);
    CUDA_OK(cudaMemcpyAsync(ex.log.data() + n0, R.log + n0, sizeof(Rec) * (ex.g.log_n - n0), cudaMemcpyDeviceToHost,
                            ex.stream));
  }
  if (ex.g.phase == 2 || ex.g.error) {
    ex.qs.resize(Q);
    CUDA_OK(cudaMemcpyAsync(ex.qs.data(), R.qs, sizeof(QueryRun) * Q, cudaMemcpyDeviceToHost, ex.stream));
  }
  CUDA_OK(cudaStreamSynchronize(ex.stream));
#endif
}

// Paged tree-KV store of one run (ctl_state.h kKvPage): `pages` physical
// pages, root prompts static in the first Q * pp, the page table sized for
// every page handed out over the run (ex.kv_pt_cap grows on overflow).
void kv_configure(spex_executor& ex, Cfg& c, long long pages) {
  const int Q = ex.hc.n_queries;
  const long long pp = kv_pages_of(ex.hc.prompt_tokens);
  if (pages > INT32_MAX) pages = INT32_MAX;
  if (pages < static_cast<long long>(Q) * pp + kv_pages_of(ex.hc.token_max))
    fail(ERR_CAP_KV, "tree KV pool of " + std::to_string(pages) + " pages cannot hold the " + std::to_string(Q) +
                         " root prompts and one thought");
  if (ex.kv_pt_cap < static_cast<long long>(Q) * pp + std::max(4 * pages, 1LL << 20))
    ex.kv_pt_cap = static_cast<long long>(Q) * pp + std::max(4 * pages, 1LL << 20);
  c.kv_pages = static_cast<int>(pages);
  c.kv_pp_root = static_cast<int>(pp);
  c.kv_pt_cap = ex.kv_pt_cap;
  ex.kv_pages = pages;
}

// The policy / PRM models, their tree-KV pools and row buffers are one
// process-wide cache (model_host.cpp g_cache, with the K1 claim-order and L2
// policy settings): model-attached runs of distinct executors take turns on
// it. Control-only runs (no model) stay fully concurrent, as the reference's
// independent Executors are (experiment.cpp:61-78).
std::mutex g_model_mu;

#ifndef SPEX_EMU
struct GroupLaunch;
void group_launch(GroupLaunch& G, std::vector<spex_executor*>& exs, int device, int trace, int node_cap,
                  const std::vector<char*>* ext);
int group_finish(GroupLaunch& G, std::vector<spex_executor*>& exs, int trace, float* ms_out);
GroupLaunch* group_new();
void group_delete(GroupLaunch* G);
#endif

void run_executor(spex_executor& ex, int trace) {
  const HostConfig& h = ex.hc;
#ifndef SPEX_EMU
  std::unique_lock<std::mutex> model_lock(g_model_mu, std::defer_lock);
  if (ex.with_model) model_lock.lock();
#endif
#ifndef SPEX_EMU
  if (ex.reward_prm && (!ex.with_model || !ex.mc.with_prm))
    fail(ERR_INVALID_ARGUMENT, "PRM rewards need a model with a PRM (spex_executor_set_model)");
  if (ex.reward_prm && (ex.shard_lo > 0 || (ex.shard_hi >= 0 && ex.shard_hi < h.n_queries)))
    fail(ERR_INVALID_ARGUMENT, "PRM rewards need every query's PRM on this executor (no shard)");
  if (ex.reward_prm && std::getenv("SPEX_SEQUENTIAL"))
    fail(ERR_INVALID_ARGUMENT, "PRM rewards need the streamed forward (SPEX_SEQUENTIAL is set)");
#else
  if (ex.reward_prm) fail(ERR_INVALID_ARGUMENT, "PRM rewards need the CUDA build");
#endif
  const int Q = h.n_queries;
  int node_cap = 512;
  if (const char* e = std::getenv("SPEX_NODE_CAP")) node_cap = std::max(16, std::atoi(e));
  if (ex.node_cap0 > 0) node_cap = ex.node_cap0;
  for (int attempt = 0; attempt < 4; ++attempt) {
    const long long sc = static_cast<long long>(Q) * (node_cap - 1) + 64;
    if (sc > (1LL << 30)) fail(ERR_CAP_STREAMS, "stream table too large");
    const int stream_cap = static_cast<int>(sc);
    const long long lc = trace ? static_cast<long long>(Q) * node_cap * 6 + 64 : 64;
    if (lc > (1LL << 31) - 1) fail(ERR_CAP_LOG, "log too large");
    const int log_cap = static_cast<int>(lc);
    const int stage_cap = std::max(512, node_cap);  // records per thread slot per phase
    const int nwarps = ex.nthreads / 32;
    Run R{};
#ifndef SPEX_EMU
    ex.record_sched = ex.with_model ? 1 : 0;
#endif
    set_cfg(ex, R.cfg, node_cap, stream_cap, log_cap, stage_cap, trace, ex.record_sched);
    Arena A;
    layout(A, R, Q, node_cap, stream_cap, log_cap, ex.nthreads, stage_cap);
    R.nwarps = nwarps;
    std::vector<double>& tab = log_table();
    R.log_tab_n = static_cast<int>(tab.size());
#ifdef SPEX_EMU
    std::vector<char> mem(A.total + 256);
    char* base = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(mem.data()) + 255) & ~uintptr_t(255));
    std::memset(base, 0, A.total);
    A.carve(base);
    R.log_tab = tab.data();
    std::vector<int> kv_pt_h, kv_free_h;
    if (ex.kv_pages_req > 0) {
      kv_configure(ex, R.cfg, ex.kv_pages_req);
      kv_pt_h.assign(static_cast<size_t>(R.cfg.kv_pt_cap), -1);
      kv_free_h.assign(static_cast<size_t>(R.cfg.kv_pages), -1);
      R.kv_pt = kv_pt_h.data();
      R.kv_free = kv_free_h.data();
    }
    R.qs[0].admitted = 0;
    for (int q = 0; q < Q; ++q) R.qs[q].plan_empty_version = 0xffffffffu;
    R.xch = ex.split_world > 1 ? ex.split_boxes.data() : nullptr;
    std::vector<int> sm(2048);
    std::vector<double> smd(64);
    std::vector<i64> sml(64);
    std::vector<int> warp_off(3 * 64, 0);
    HostExec hx;
    hx.sm = sm.data();
    hx.smd = smd.data();
    hx.sml = sml.data();
    auto t0 = std::chrono::steady_clock::now();
    run_loop(&R, hx, warp_off.data());
    auto t1 = std::chrono::steady_clock::now();
    ex.device_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
    ex.g = *R.g;
    if (R.cfg.kv_pages > 0 && ex.g.error == 0) {
      // page-store self-check (tests): at the end every thought page is back
      // in the free ring exactly once and nothing else is
      const i64 root = static_cast<i64>(Q) * R.cfg.kv_pp_root;
      const i64 ring = ex.g.kv_free_tail - ex.g.kv_free_head;
      std::vector<char> seen(static_cast<size_t>(ex.g.kv_bump), 0);
      bool ok = ex.g.kv_live == root && ring == ex.g.kv_bump - root;
      for (i64 k = 0; ok && k < ring; ++k) {
        const int p = R.kv_free[(ex.g.kv_free_head + k) % R.cfg.kv_pages];
        ok = p >= root && p < ex.g.kv_bump && !seen[p];
        if (ok) seen[p] = 1;
      }
      if (!ok) fail(ERR_INTERNAL, "tree-KV page store inconsistent at the end of the run");
    }
    ex.qs.assign(R.qs, R.qs + Q);
    if (trace) ex.log.assign(R.log, R.log + ex.g.log_n);
#else
    const auto tm0 = std::chrono::steady_clock::now();
    auto mark = [&](const char* nm) {
      ex.host_marks.emplace_back(nm, std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tm0).count());
    };
    CUDA_OK(cudaSetDevice(ex.device));
    // single-GPU split emulation: the other ranks' control runs beside this
    // one (CTAs of one launch), exchanging through outboxes on this device
    std::vector<spex_executor*> peers;
    GroupLaunch* peer_group = nullptr;
    auto launch_peers = [&] {
      if (!ex.split_emulate) return;
      for (int r = 0; r < ex.split_world; ++r) {
        if (r == ex.split_rank) continue;
        spex_executor* p = nullptr;
        std::vector<void*> bx(ex.split_boxes.begin(), ex.split_boxes.end());
        if (spex_executor_create(ex.cfg_text.c_str(), ex.run_seed, ex.flags_text.empty() ? nullptr : ex.flags_text.c_str(),
                                 ex.device, &p) ||
            (peers.push_back(p), spex_executor_set_split(p, r, ex.split_world, bx.data(), ex.split_epoch)))
          fail(ERR_INTERNAL, "split emulation: peer rank setup failed: " + g_err);
      }
      peer_group = group_new();
      try {
        group_launch(*peer_group, peers, ex.device, 0, node_cap, &ex.split_boxes);
      } catch (...) {  // nothing launched: drop the group so finish_peers has nothing to wait for
        group_delete(peer_group);
        peer_group = nullptr;
        throw;
      }
    };
    auto finish_peers = [&]() -> int {
      int e = 0;
      if (peer_group) {
        e = group_finish(*peer_group, peers, 0, nullptr);
        group_delete(peer_group);
        peer_group = nullptr;
      }
      for (auto* p : peers) spex_executor_destroy(p);
      peers.clear();
      return e;
    };
    int peer_err = 0;
    if (!ex.stream) CUDA_OK(cudaStreamCreateWithFlags(&ex.stream, cudaStreamNonBlocking));
    if (!ex.mstream) CUDA_OK(cudaStreamCreateWithFlags(&ex.mstream, cudaStreamNonBlocking));
    keep_pool_memory(ex.device);
    char* base = nullptr;
    // stream-ordered allocations: concurrent searches (one control CTA each)
    // never synchronise the device through cudaMalloc/cudaFree
    CUDA_OK(cudaMallocAsync(reinterpret_cast<void**>(&base), A.total + 256, ex.stream));
    CUDA_OK(cudaMemsetAsync(base, 0, A.total + 256, ex.stream));
    A.carve(base);
    // Keep the control state L2-resident while the forward streams tens of GB
    // of tree KV through HBM: the control CTA is latency-bound and its misses
    // otherwise queue behind the K1 traffic (window = the hot region only).
    if (!std::getenv("SPEX_NO_L2PERSIST")) {
      int max_win = 0, max_persist = 0;
      cudaDeviceGetAttribute(&max_win, cudaDevAttrMaxAccessPolicyWindowSize, ex.device);
      cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, ex.device);
      if (max_win > 0 && max_persist > 0) {
        const size_t win = std::min<size_t>(A.hot, static_cast<size_t>(max_win));
        const size_t per = std::min<size_t>(win, static_cast<size_t>(max_persist));
        static size_t persist_set = 0;  // set once per process (may synchronize the device)
        if (persist_set < per) {
          cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, per);
          persist_set = per;
        }
        cudaStreamAttrValue av{};
        av.accessPolicyWindow.base_ptr = base;
        av.accessPolicyWindow.num_bytes = win;
        av.accessPolicyWindow.hitRatio = static_cast<float>(static_cast<double>(per) / static_cast<double>(win));
        av.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        av.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        cudaStreamSetAttribute(ex.stream, cudaStreamAttributeAccessPolicyWindow, &av);
        cudaGetLastError();
      }
      if (std::getenv("SPEX_TIMING"))
        std::fprintf(stderr, "[spex timing] arena %zu bytes, hot %zu, L2 window max %d, persist max %d\n", A.total,
                     A.hot, max_win, max_persist);
    }
    double* d_tab = nullptr;
    CUDA_OK(cudaMallocAsync(reinterpret_cast<void**>(&d_tab), tab.size() * sizeof(double), ex.stream));
    CUDA_OK(cudaMemcpyAsync(d_tab, tab.data(), tab.size() * sizeof(double), cudaMemcpyHostToDevice,
                            ex.stream));
    R.log_tab = d_tab;
    char** d_xch = nullptr;
    if (ex.split_world > 1) {
      CUDA_OK(cudaMallocAsync(reinterpret_cast<void**>(&d_xch), sizeof(char*) * ex.split_world, ex.stream));
      CUDA_OK(cudaMemcpyAsync(d_xch, ex.split_boxes.data(), sizeof(char*) * ex.split_world, cudaMemcpyHostToDevice,
                              ex.stream));
      R.xch = d_xch;
    }
    // streaming schedule: head + entries in pinned, device-mapped host memory
    const bool streaming = ex.with_model && !std::getenv("SPEX_SEQUENTIAL");
    PubHead* h_head = nullptr;
    PubEntry* h_ents = nullptr;
    if (streaming) {
      h_head = static_cast<PubHead*>(pinned_acquire(sizeof(PubHead)));
      h_ents = static_cast<PubEntry*>(pinned_acquire(sizeof(PubEntry) * R.cfg.sched_cap));
      std::memset(h_head, 0, sizeof(PubHead));
      CUDA_OK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&R.pub), h_head, 0));
      CUDA_OK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&R.pub_e), h_ents, 0));
    }
    int* d_kvpt = nullptr;
    int* d_kvfree = nullptr;
    if (ex.with_model) {
      // the pool: an explicit page count, else the resident cached pools or
      // 70% of free HBM (spex_model_pool_slots)
      const long long slots = ex.kv_pages_req > 0 ? ex.kv_pages_req * kKvPage : spex_model_pool_slots(&ex.mc);
      kv_configure(ex, R.cfg, slots / kKvPage);
      CUDA_OK(cudaMallocAsync(reinterpret_cast<void**>(&d_kvpt), sizeof(int) * R.cfg.kv_pt_cap, ex.stream));
      CUDA_OK(cudaMallocAsync(reinterpret_cast<void**>(&d_kvfree), sizeof(int) * R.cfg.kv_pages, ex.stream));
      R.kv_pt = d_kvpt;
      R.kv_free = d_kvfree;
      if (std::getenv("SPEX_TIMING"))
        std::fprintf(stderr, "[spex timing] tree KV pool: %d pages x %d tokens, page table %lld entries\n",
                     R.cfg.kv_pages, kKvPage, static_cast<long long>(R.cfg.kv_pt_cap));
    }
    mark("arena+pinned");
    Run* d_run = nullptr;
    CUDA_OK(cudaMallocAsync(reinterpret_cast<void**>(&d_run), sizeof(Run), ex.stream));
    CUDA_OK(cudaMemcpyAsync(d_run, &R, sizeof(Run), cudaMemcpyHostToDevice, ex.stream));
    auto cleanup = [&] {
      finish_peers();
      cudaFreeAsync(base, ex.stream);
      if (d_kvpt) cudaFreeAsync(d_kvpt, ex.stream);
      if (d_kvfree) cudaFreeAsync(d_kvfree, ex.stream);
      cudaFreeAsync(d_tab, ex.stream);
      if (d_xch) cudaFreeAsync(d_xch, ex.stream);
      cudaFreeAsync(d_run, ex.stream);
      cudaStreamSynchronize(ex.stream);
      if (h_head) pinned_release(h_head);
      if (h_ents) pinned_release(h_ents);
    };
    ScheduleView sv{};
    if (ex.with_model) {
      sv.tree.parent = R.n_parent;
      sv.tree.tokens = R.n_tokens;
      sv.tree.hash = R.n_hash;
      sv.tree.kvbase = R.n_kvbase;
      sv.tree.kv_pt = R.kv_pt;
      sv.tree.run_seed = R.cfg.run_seed;
      sv.node_score = R.cfg.reward_prm ? R.n_score : nullptr;
      sv.prm_done = R.cfg.reward_prm ? R.prm_done : nullptr;
      sv.tree.kv_pp_root = R.cfg.kv_pp_root;
      sv.tree.q_offset = R.cfg.q_offset;
      sv.tree.st_q = R.st_q;
      sv.tree.st_node = R.st_node;
      sv.tree.node_cap = node_cap;
      sv.tree.prompt_tokens = ex.hc.prompt_tokens;
      sv.n_queries = Q;
      sv.shard_lo = R.cfg.shard_lo;
      sv.shard_hi = R.cfg.shard_hi;
      sv.srow_sid = R.srow_sid;
      sv.srow_pos0 = R.srow_pos0;
      sv.srow_rstart = R.srow_rstart;
      sv.srow_tstart = R.srow_tstart;
      sv.max_decode_rows = 16384;
      sv.max_prm_rows = 1 << 17;
    }
    ModelRunConfig mc = ex.mc;
    void* d_rows = nullptr;
    void* d_scores = nullptr;
    auto alloc_outputs = [&](long long rows_cap) {
      if (!mc.record_outputs) return;
      mc.out_rows_cap = rows_cap;
      mc.out_scores_cap = static_cast<long long>(Q) * node_cap;
      CUDA_OK(cudaMalloc(&d_rows, std::max<long long>(mc.out_rows_cap, 1) * sizeof(DecodeOut)));
      CUDA_OK(cudaMalloc(&d_scores, std::max<long long>(mc.out_scores_cap, 1) * sizeof(PrmOut)));
      mc.out_rows = d_rows;
      mc.out_scores = d_scores;
    };
    cudaEvent_t ca, cb;
    cudaEventCreate(&ca);
    cudaEventCreate(&cb);
    bool model_done = false;
    ex.mres = ModelRunResult{};
    sv.kv_slots = static_cast<long long>(R.cfg.kv_pages) * kKvPage;
    if (ex.with_model) {
      // models, pools and row buffers exist before the control kernel starts
      // (nothing may synchronise the device while it waits on PRM scores)
      try {
        spex_model_prepare(&mc, &sv, ex.mstream);
      } catch (const std::exception& e) {
        cleanup();
        fail(201, std::string("model forward: ") + e.what());
      }
    }
    if (streaming) {
      CUDA_OK(cudaStreamSynchronize(ex.stream));
      sv.pub_head = h_head;
      sv.pub_entries = h_ents;
      alloc_outputs(static_cast<long long>(Q) * node_cap * 64);
      mark("pre-launch");
      try {
        launch_peers();
      } catch (...) {
        cleanup();
        throw;
      }
      int lr = spex_launch_control_async(d_run, Q, ex.nthreads, ex.stream, ca, cb);
      if (lr != 0) {
        cleanup();
        fail(200, std::string("control kernel launch failed: ") + cudaGetErrorString(static_cast<cudaError_t>(lr)));
      }
      try {
        run_model_schedule(mc, sv, &ex.mres, ex.mstream);
        model_done = true;
        mark("model-stream-done");
      } catch (const std::exception& e) {
        cudaDeviceSynchronize();  // the forward's streams (policy + PRM) and the control kernel
        cudaFree(d_rows);
        cudaFree(d_scores);
        cleanup();
        fail(201, std::string("model forward: ") + e.what());
      }
    } else {
      try {
        launch_peers();
      } catch (...) {
        cleanup();
        throw;
      }
      int lr = spex_launch_control_async(d_run, Q, ex.nthreads, ex.stream, ca, cb);
      if (lr != 0) {
        cleanup();
        fail(200, std::string("control kernel launch failed: ") + cudaGetErrorString(static_cast<cudaError_t>(lr)));
      }
    }
    CUDA_OK(cudaEventSynchronize(cb));
    peer_err = finish_peers();
    mark("control-done");
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ca, cb);
    ex.device_ms = ms;
    CUDA_OK(cudaMemcpyAsync(&ex.g, R.g, sizeof(GState), cudaMemcpyDeviceToHost, ex.stream));
    CUDA_OK(cudaStreamSynchronize(ex.stream));
    if (ex.with_model && ex.g.error == 0 && !model_done) {
      // sequential replay over the finished schedule
      std::vector<PubEntry> ents(ex.g.n_sched);
      if (!ents.empty())
        CUDA_OK(cudaMemcpy(ents.data(), streaming ? static_cast<void*>(h_ents) : static_cast<void*>(R.pub_e),
                           ents.size() * sizeof(PubEntry), streaming ? cudaMemcpyHostToHost : cudaMemcpyDeviceToHost));
      sv.pub_head = nullptr;
      sv.pub_entries = nullptr;
      sv.entries_host = ents.data();
      sv.n_entries = static_cast<int>(ents.size());
      if (!d_rows) alloc_outputs(ex.g.decode_rows);
      try {
        run_model_schedule(mc, sv, &ex.mres, ex.mstream);
      } catch (const std::exception& e) {
        cudaFree(d_rows);
        cudaFree(d_scores);
        cleanup();
        fail(201, std::string("model forward: ") + e.what());
      }
    }
    if (ex.with_model) {
      ex.mres.control_ms = ms;
      ex.mres.streamed = model_done ? 1 : 0;
      cudaEvent_t me;
      cudaEventCreate(&me);
      cudaEventRecord(me, ex.mstream);
      cudaEventSynchronize(me);
      float sm = 0.f;
      cudaEventElapsedTime(&sm, ca, me);
      ex.mres.step_ms = sm > ms ? sm : ms;
      cudaEventDestroy(me);
    }
    cudaEventDestroy(ca);
    cudaEventDestroy(cb);
    ex.qs.resize(Q);
    CUDA_OK(cudaMemcpyAsync(ex.qs.data(), R.qs, sizeof(QueryRun) * Q, cudaMemcpyDeviceToHost, ex.stream));
    ex.finish_ns.resize(Q);
    CUDA_OK(cudaMemcpyAsync(ex.finish_ns.data(), R.q_finish_ns, sizeof(long long) * Q, cudaMemcpyDeviceToHost,
                            ex.stream));
    CUDA_OK(cudaStreamSynchronize(ex.stream));
    if (trace && ex.g.log_n > 0) {
      ex.log.resize(ex.g.log_n);
      CUDA_OK(cudaMemcpyAsync(ex.log.data(), R.log, sizeof(Rec) * ex.g.log_n, cudaMemcpyDeviceToHost,
                              ex.stream));
      CUDA_OK(cudaStreamSynchronize(ex.stream));
    }
    if (mc.record_outputs && ex.with_model) {
      ex.dec_out.resize(ex.mres.out_rows);
      ex.prm_out.resize(ex.mres.out_scores);
      if (!ex.dec_out.empty())
        CUDA_OK(cudaMemcpy(ex.dec_out.data(), d_rows, ex.dec_out.size() * sizeof(DecodeOut), cudaMemcpyDeviceToHost));
      if (!ex.prm_out.empty())
        CUDA_OK(cudaMemcpy(ex.prm_out.data(), d_scores, ex.prm_out.size() * sizeof(PrmOut), cudaMemcpyDeviceToHost));
    }
    cudaFree(d_rows);
    cudaFree(d_scores);
    cleanup();
    mark("cleanup");
    if (std::getenv("SPEX_TIMING")) {
      for (auto& m : ex.host_marks) std::fprintf(stderr, "[spex timing] %-20s %10.2f ms\n", m.first, m.second);
    }
#endif
#ifndef SPEX_EMU
    if (ex.split_emulate) {
      const bool cap = ex.g.error == ERR_CAP_NODES || ex.g.error == ERR_CAP_STAGE || peer_err == ERR_CAP_NODES ||
                       peer_err == ERR_CAP_STAGE;
      if (cap) {
        node_cap *= 2;  // every rank reruns, a new epoch on the same outboxes
        ex.split_epoch += 1;
        ex.log.clear();
        continue;
      }
      if (peer_err) fail(peer_err, "split emulation: a peer rank failed");
    }
#endif
    if (ex.split_world > 1 && (ex.g.error == ERR_CAP_NODES || ex.g.error == ERR_CAP_STAGE)) {
      // a rank cannot rerun alone (its budget rounds pair with the others'):
      // every rank reruns, with a new epoch and this capacity (spex_split_run,
      // split.run_split_rank)
      ex.node_cap0 = node_cap * 2;
      fail(ex.g.error, "split rank " + std::to_string(ex.split_rank) + ": node capacity " +
                           std::to_string(node_cap) + " exhausted; rerun every rank with SPEX_NODE_CAP=" +
                           std::to_string(node_cap * 2) + " (a new epoch)");
    }
    if (ex.g.error == ERR_CAP_NODES || ex.g.error == ERR_CAP_STAGE) {
      node_cap *= 2;  // capacity, not semantics: rerun with a larger arena
      ex.log.clear();
      continue;
    }
    if (ex.g.error == ERR_CAP_KV && ex.g.error_node == 1u) {
      ex.kv_pt_cap *= 4;  // page table full: rerun with a larger one
      ex.log.clear();
      continue;
    }
    if (ex.g.error == ERR_CAP_KV)
      fail(ERR_CAP_KV, "tree KV pool exhausted: the live thoughts need more than " + std::to_string(ex.kv_pages) +
                           " pages of " + std::to_string(kKvPage) + " tokens (peak " + std::to_string(ex.g.kv_peak) +
                           " pages live); set a larger pool with spex_executor_set_kv_pages or shard the queries");
    if (ex.g.error != 0 && std::getenv("SPEX_DEBUG")) {
      std::string dump;
      serialize(ex, dump);
      std::fprintf(stderr, "%s", dump.c_str());
    }
    if (ex.g.error != 0)
      fail(ex.g.error, "device control error at query " + std::to_string(ex.g.error_q) + " node " +
                           std::to_string(static_cast<int>(ex.g.error_node)));
    return;
  }
  fail(ERR_CAP_NODES, "node capacity exhausted");
}

#ifndef SPEX_EMU
// Many independent searches (same config, different seeds) in ONE launch of the
// control kernel: CTA b runs search b (the device analog of the reference's
// OpenMP loop over repetitions, experiment.cpp:61-78). Control only (no model,
// no trace). Returns false if any search needs a larger arena; the caller then
// runs those searches one by one.
bool run_batch_device(std::vector<spex_executor*>& exs, int device, cudaStream_t st, float* ms_out) {
  const int n = static_cast<int>(exs.size());
  CUDA_OK(cudaSetDevice(device));
  const HostConfig& h = exs[0]->hc;
  const int Q = h.n_queries;
  int node_cap = 512;
  if (const char* e = std::getenv("SPEX_NODE_CAP")) node_cap = std::max(16, std::atoi(e));
  const int stream_cap = static_cast<int>(static_cast<long long>(Q) * (node_cap - 1) + 64);
  const int stage_cap = std::max(512, node_cap);
  const int nthreads = exs[0]->nthreads, nwarps = nthreads / 32;
  std::vector<double>& tab = log_table();
  double* d_tab = nullptr;
  CUDA_OK(cudaMallocAsync(reinterpret_cast<void**>(&d_tab), tab.size() * sizeof(double), st));
  CUDA_OK(cudaMemcpyAsync(d_tab, tab.data(), tab.size() * sizeof(double), cudaMemcpyHostToDevice, st));
  std::vector<Run> runs(n);
  std::vector<Arena> arenas(n);
  for (int b = 0; b < n; ++b) {
    Run& R = runs[b];
    R = Run{};
    exs[b]->record_sched = 0;
    set_cfg(*exs[b], R.cfg, node_cap, stream_cap, 64, stage_cap, 0, 0);
    layout(arenas[b], R, Q, node_cap, stream_cap, 64, nthreads, stage_cap);
    R.nwarps = nwarps;
    R.log_tab_n = static_cast<int>(tab.size());
    R.log_tab = d_tab;
  }
  // one allocation and one memset for all searches (same config: same layout)
  const size_t per = (arenas[0].total + 255) & ~size_t(255);
  char* big = nullptr;
  CUDA_OK(cudaMallocAsync(reinterpret_cast<void**>(&big), per * n + 256, st));
  CUDA_OK(cudaMemsetAsync(big, 0, per * n + 256, st));
  for (int b = 0; b < n; ++b) arenas[b].carve(big + per * b);
  Run* d_runs = nullptr;
  CUDA_OK(cudaMallocAsync(reinterpret_cast<void**>(&d_runs), sizeof(Run) * n, st));
  CUDA_OK(cudaMemcpyAsync(d_runs, runs.data(), sizeof(Run) * n, cudaMemcpyHostToDevice, st));
  cudaEvent_t ca, cb;
  cudaEventCreate(&ca);
  cudaEventCreate(&cb);
  const int lr = spex_launch_control_batch_async(d_runs, n, Q, nthreads, st, ca, cb);
  if (lr != 0) fail(200, std::string("control kernel launch failed: ") + cudaGetErrorString(static_cast<cudaError_t>(lr)));
  CUDA_OK(cudaEventSynchronize(cb));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, ca, cb);
  cudaEventDestroy(ca);
  cudaEventDestroy(cb);
  if (ms_out) *ms_out = ms;
  bool ok = true;
  for (int b = 0; b < n; ++b) {
    spex_executor& ex = *exs[b];
    ex.qs.resize(Q);
    CUDA_OK(cudaMemcpyAsync(&ex.g, runs[b].g, sizeof(GState), cudaMemcpyDeviceToHost, st));
    CUDA_OK(cudaMemcpyAsync(ex.qs.data(), runs[b].qs, sizeof(QueryRun) * Q, cudaMemcpyDeviceToHost, st));
  }
  CUDA_OK(cudaStreamSynchronize(st));
  for (int b = 0; b < n; ++b) {
    spex_executor& ex = *exs[b];
    ex.device_ms = ms;
    ex.ran = true;
    if (ex.g.error != 0) {
      ok = false;
      ex.ran = false;
    }
  }
  cudaFreeAsync(big, st);
  cudaFreeAsync(d_runs, st);
  cudaFreeAsync(d_tab, st);
  cudaStreamSynchronize(st);
  return ok;
}

// The ranks of one split job on ONE device, CTA r = rank r of one launch of
// the control kernel (co-resident: the exchange spins on the other ranks).
// Control only; with the event logs when `trace`. The outboxes are `ext`
// (device pointers, [rank] per executor's split_rank) or W fresh ones in the
// launch's allocation. group_launch returns with the kernel running on its
// own stream; group_finish waits and returns the first rank error (0: all ran).
struct GroupLaunch {
  cudaStream_t st = nullptr;
  char* big = nullptr;
  Run* d_runs = nullptr;
  std::vector<Run> runs;
  cudaEvent_t ca = nullptr, cb = nullptr;
};

void group_launch(GroupLaunch& G, std::vector<spex_executor*>& exs, int device, int trace, int node_cap,
                  const std::vector<char*>* ext) {
  const int n = static_cast<int>(exs.size());
  const int world = exs[0]->split_world;
  CUDA_OK(cudaSetDevice(device));
  CUDA_OK(cudaStreamCreateWithFlags(&G.st, cudaStreamNonBlocking));
  cudaStream_t st = G.st;
  const int nthreads = exs[0]->nthreads, nwarps = nthreads / 32;
  std::vector<double>& tab = log_table();
  const long long box = world > 1 ? split_outbox_bytes(split_qmax(exs[0]->split_qjob, world)) : 0;
  G.runs.assign(n, Run{});
  std::vector<Arena> arenas(n);
  std::vector<size_t> at(n + 1, 0);
  int qmax = 0;
  for (int b = 0; b < n; ++b) {
    Run& R = G.runs[b];
    spex_executor& ex = *exs[b];
    const int Q = ex.hc.n_queries;
    qmax = std::max(qmax, Q);
    const int stream_cap = static_cast<int>(static_cast<long long>(Q) * (node_cap - 1) + 64);
    const long long lc = trace ? static_cast<long long>(Q) * node_cap * 6 + 64 : 64;
    if (lc > (1LL << 31) - 1) fail(ERR_CAP_LOG, "log too large");
    ex.record_sched = 0;
    set_cfg(ex, R.cfg, node_cap, stream_cap, static_cast<int>(lc), std::max(512, node_cap), trace, 0);
    layout(arenas[b], R, Q, node_cap, stream_cap, static_cast<int>(lc), nthreads, std::max(512, node_cap));
    R.nwarps = nwarps;
    R.log_tab_n = static_cast<int>(tab.size());
    at[b + 1] = at[b] + ((arenas[b].total + 255) & ~size_t(255));
  }
  const size_t tab_off = at[n];
  const size_t box_off = tab_off + ((tab.size() * sizeof(double) + 255) & ~size_t(255));
  const size_t ptr_off = box_off + (ext ? 0 : static_cast<size_t>(box) * world);
  const size_t total = ptr_off + sizeof(char*) * std::max(world, 1) + 256;
  CUDA_OK(cudaMallocAsync(reinterpret_cast<void**>(&G.big), total, st));
  CUDA_OK(cudaMemsetAsync(G.big, 0, total, st));
  CUDA_OK(cudaMemcpyAsync(G.big + tab_off, tab.data(), tab.size() * sizeof(double), cudaMemcpyHostToDevice, st));
  std::vector<char*> boxes(world);
  for (int r = 0; r < world; ++r) boxes[r] = ext ? (*ext)[r] : G.big + box_off + static_cast<size_t>(box) * r;
  if (world > 1)
    CUDA_OK(cudaMemcpyAsync(G.big + ptr_off, boxes.data(), sizeof(char*) * world, cudaMemcpyHostToDevice, st));
  for (int b = 0; b < n; ++b) {
    arenas[b].carve(G.big + at[b]);
    G.runs[b].log_tab = reinterpret_cast<double*>(G.big + tab_off);
    G.runs[b].xch = world > 1 ? reinterpret_cast<char**>(G.big + ptr_off) : nullptr;
  }
  CUDA_OK(cudaMallocAsync(reinterpret_cast<void**>(&G.d_runs), sizeof(Run) * n, st));
  CUDA_OK(cudaMemcpyAsync(G.d_runs, G.runs.data(), sizeof(Run) * n, cudaMemcpyHostToDevice, st));
  cudaEventCreate(&G.ca);
  cudaEventCreate(&G.cb);
  const int lr = spex_launch_control_batch_async(G.d_runs, n, qmax, nthreads, st, G.ca, G.cb);
  if (lr != 0) {
    cudaFreeAsync(G.big, st);
    cudaFreeAsync(G.d_runs, st);
    cudaStreamSynchronize(st);
    cudaStreamDestroy(st);
    cudaEventDestroy(G.ca);
    cudaEventDestroy(G.cb);
    G = GroupLaunch{};
    fail(200, std::string("control kernel launch failed: ") + cudaGetErrorString(static_cast<cudaError_t>(lr)));
  }
}

int group_finish(GroupLaunch& G, std::vector<spex_executor*>& exs, int trace, float* ms_out) {
  const int n = static_cast<int>(exs.size());
  cudaStream_t st = G.st;
  CUDA_OK(cudaEventSynchronize(G.cb));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, G.ca, G.cb);
  cudaEventDestroy(G.ca);
  cudaEventDestroy(G.cb);
  if (ms_out) *ms_out = ms;
  int err = 0;
  for (int b = 0; b < n; ++b) {
    spex_executor& ex = *exs[b];
    const int Q = ex.hc.n_queries;
    CUDA_OK(cudaMemcpyAsync(&ex.g, G.runs[b].g, sizeof(GState), cudaMemcpyDeviceToHost, st));
    ex.qs.resize(Q);
    CUDA_OK(cudaMemcpyAsync(ex.qs.data(), G.runs[b].qs, sizeof(QueryRun) * Q, cudaMemcpyDeviceToHost, st));
    CUDA_OK(cudaStreamSynchronize(st));
    if (trace && ex.g.log_n > 0) {
      ex.log.resize(ex.g.log_n);
      CUDA_OK(cudaMemcpyAsync(ex.log.data(), G.runs[b].log, sizeof(Rec) * ex.g.log_n, cudaMemcpyDeviceToHost, st));
    }
    ex.device_ms = ms;
    if (ex.g.error != 0 && err == 0) err = ex.g.error;
  }
  cudaFreeAsync(G.big, st);
  cudaFreeAsync(G.d_runs, st);
  cudaStreamSynchronize(st);
  cudaStreamDestroy(st);
  G = GroupLaunch{};
  return err;
}

GroupLaunch* group_new() { return new GroupLaunch(); }
void group_delete(GroupLaunch* G) { delete G; }

int run_group_device(std::vector<spex_executor*>& exs, int device, int trace, int node_cap, float* ms_out) {
  GroupLaunch G;
  group_launch(G, exs, device, trace, node_cap, nullptr);
  return group_finish(G, exs, trace, ms_out);
}
#endif

}  // namespace

extern "C" {

const char* spex_last_error(void) { return g_err.c_str(); }

int spex_run_batch(const char* config_json, const uint64_t* seeds, int n, const char* flags_csv, int device,
                   spex_totals* totals, double* device_ms) {
  return guarded([&] {
    if (n <= 0) fail(ERR_INVALID_ARGUMENT, "empty batch");
    std::vector<spex_executor*> exs;
    auto free_all = [&] {
      for (auto* e : exs) spex_executor_destroy(e);
    };
    for (int b = 0; b < n; ++b) {
      spex_executor* e = nullptr;
      const int rc = spex_executor_create(config_json, seeds[b], flags_csv, device, &e);
      if (rc) {
        free_all();
        fail(rc, g_err);
      }
      exs.push_back(e);
    }
#ifndef SPEX_EMU
    cudaStream_t st = nullptr;
    CUDA_OK(cudaSetDevice(device));
    CUDA_OK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    float ms = 0.f;
    try {
      run_batch_device(exs, device, st, &ms);
    } catch (...) {
      cudaStreamDestroy(st);
      free_all();
      throw;
    }
    cudaStreamDestroy(st);
    if (device_ms) *device_ms = ms;
#endif
    for (int b = 0; b < n; ++b) {
      if (!exs[b]->ran) {  // capacity: rerun alone (the single-run path grows its arena)
        exs[b]->g = GState{};
        run_executor(*exs[b], 0);
        exs[b]->ran = true;
      }
      if (totals) fill_totals(*exs[b], &totals[b]);
    }
    free_all();
  });
}

void spex_free(void* p) { std::free(p); }

int spex_device_ok(void) {
#ifdef SPEX_EMU
  return 0;
#else
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) return 0;
  cudaDeviceProp p{};
  if (cudaGetDeviceProperties(&p, 0) != cudaSuccess) return 0;
  return p.major == 10 ? 1 : 0;
#endif
}

int spex_canonical_config(const char* config_json, char** out_json) {
  return guarded([&] {
    HostConfig c = parse_config(config_json);
    std::string s = to_json(c, c.t1, c.t2, c.t3).dump();
    *out_json = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(*out_json, s.c_str(), s.size() + 1);
  });
}

int spex_executor_create(const char* config_json, uint64_t run_seed, const char* flags_csv,
                         int device, spex_executor** out) {
  return guarded([&] {
    auto ex = new spex_executor();
    try {
      ex->hc = parse_config(config_json);
      HostConfig tmp = ex->hc;
      if (flags_csv) flags_from_csv(flags_csv, tmp);
      ex->t1 = tmp.t1;
      ex->t2 = tmp.t2;
      ex->t3 = tmp.t3;
      ex->run_seed = run_seed;
      ex->device = device;
      ex->cfg_text = config_json;
      ex->flags_text = flags_csv ? flags_csv : "";
      ex->split_qjob = ex->hc.n_queries;
      ex->cfg_dump = to_json(ex->hc, ex->t1, ex->t2, ex->t3).dump();
      if (const char* e = std::getenv("SPEX_CTL_THREADS")) {
        const int t = std::atoi(e);  // same clamp as the launcher: slots must match threads
        ex->nthreads = (t < 64 || t > 512 || (t & 31)) ? 512 : t;
      }
    } catch (...) {
      delete ex;
      throw;
    }
    *out = ex;
  });
}

int spex_executor_run(spex_executor* ex, int trace, spex_totals* totals) {
  return guarded([&] {
    if (ex->ran) fail(ERR_INVALID_ARGUMENT, "run() may be called once");
    ex->ran = true;
    run_executor(*ex, trace);
    if (totals) fill_totals(*ex, totals);
  });
}

int spex_frontier_step(spex_executor* ex, long long iterations, int* done, char** events, size_t* events_len) {
  return guarded([&] {
    if (done) *done = 0;
    if (ex->ran && !ex->step) fail(ERR_INVALID_ARGUMENT, "frontier_step: the executor already ran");
#ifndef SPEX_EMU
    if (ex->with_model) fail(ERR_INVALID_ARGUMENT, "frontier_step: stepwise execution is control only (no model)");
#endif
    if (ex->split_world > 1) fail(ERR_INVALID_ARGUMENT, "frontier_step: not with a split rank");
    if (iterations < 0) fail(ERR_INVALID_ARGUMENT, "frontier_step: negative iteration count");
    const bool first = !ex->step;
    if (first) step_begin(*ex);
    const long long from = static_cast<long long>(ex->log.size());
    step_run(*ex, iterations);
    if (ex->g.error == ERR_CAP_NODES || ex->g.error == ERR_CAP_STAGE || ex->g.error == ERR_CAP_STREAMS) {
      step_release(*ex);
      ex->ran = true;
      fail(ex->g.error, "frontier_step: node capacity exhausted (a stepwise run cannot be replayed); "
                        "rerun with a larger SPEX_NODE_CAP");
    }
    if (ex->g.error) {
      step_release(*ex);
      ex->ran = true;
      fail(ex->g.error, "device control error at query " + std::to_string(ex->g.error_q) + " node " +
                            std::to_string(static_cast<int>(ex->g.error_node)));
    }
    std::string out;
    if (first) serialize_header(*ex, out);
    for (long long i = from; i < static_cast<long long>(ex->log.size()); ++i) serialize_record(ex->log[i], out);
    const bool finished = ex->g.phase == 2;
    if (finished) {
      serialize_footer(*ex, out);
      step_release(*ex);
      ex->ran = true;
      if (done) *done = 1;
    }
    if (events) {
      *events = static_cast<char*>(std::malloc(out.size() + 1));
      std::memcpy(*events, out.data(), out.size());
      (*events)[out.size()] = 0;
    }
    if (events_len) *events_len = out.size();
  });
}

int spex_executor_log(spex_executor* ex, char** out_lines, size_t* out_len) {
  return guarded([&] {
    std::string s;
    serialize(*ex, s);
    *out_lines = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(*out_lines, s.data(), s.size());
    (*out_lines)[s.size()] = 0;
    if (out_len) *out_len = s.size();
  });
}

int spex_executor_stats(spex_executor* ex, spex_stats* out) {
  return guarded([&] {
    std::memset(out, 0, sizeof(*out));
    out->iterations = ex->g.iterations;
    out->epochs = ex->g.epochs;
    out->reward_events = ex->g.reward_events;
    out->decode_steps = ex->g.decode_steps;
    out->decode_rows = ex->g.decode_rows;
    out->log_records = ex->g.log_n;
    long long nodes = 0;
    for (const QueryRun& q : ex->qs) nodes += q.nnodes;
    out->nodes = nodes;
    out->device_ms = ex->device_ms;
    if (std::getenv("SPEX_PHASES")) {
      static const char* nm[8] = {"engine", "fins", "reward", "follow_items", "sched", "total", "spec_items", "follow_commit"};
      for (int i = 0; i < 8; ++i) std::fprintf(stderr, "phase %s: %lld Mcyc\n", nm[i], ex->g.cyc[i] / 1000000);
    }
  });
}

int spex_executor_set_model(spex_executor* ex, const char* policy_shape, const char* prm_shape,
                            uint64_t weight_seed, int record_outputs) {
  return guarded([&] {
#ifdef SPEX_EMU
    (void)ex;
    (void)policy_shape;
    (void)prm_shape;
    (void)weight_seed;
    (void)record_outputs;
    fail(ERR_INVALID_ARGUMENT, "the model forward needs the CUDA build");
#else
    ex->mc.policy = shape_by_name(policy_shape);
    ex->mc.with_prm = prm_shape && *prm_shape;
    if (ex->mc.with_prm) ex->mc.prm = shape_by_name(prm_shape);
    ex->mc.seed = weight_seed;
    ex->mc.record_outputs = record_outputs != 0;
    ex->with_model = true;
#endif
  });
}

int spex_executor_set_shard(spex_executor* ex, int rank, int world) {
  return guarded([&] {
    if (world < 1 || rank < 0 || rank >= world) fail(ERR_INVALID_ARGUMENT, "set_shard: rank out of range");
    if (ex->ran) fail(ERR_INVALID_ARGUMENT, "set_shard: executor already ran");
    const long long Q = ex->hc.n_queries;
    ex->shard_lo = static_cast<int>(Q * rank / world);
    ex->shard_hi = static_cast<int>(Q * (rank + 1) / world);
  });
}

long long spex_split_outbox_bytes(int n_queries_job, int world) {
  if (world < 1 || world > kMaxSplit || n_queries_job < world) return -1;
  return split_outbox_bytes(split_qmax(n_queries_job, world));
}

int spex_executor_set_split(spex_executor* ex, int rank, int world, void* const* outboxes, long long epoch) {
  return guarded([&] {
    if (ex->ran) fail(ERR_INVALID_ARGUMENT, "set_split: executor already ran");
    if (world < 1 || world > kMaxSplit || rank < 0 || rank >= world)
      fail(ERR_INVALID_ARGUMENT, "set_split: need 0 <= rank < world <= " + std::to_string(kMaxSplit));
    if (ex->shard_lo != 0 || ex->shard_hi >= 0) fail(ERR_INVALID_ARGUMENT, "set_split: executor has a coupled shard");
    const int qjob = ex->split_world > 1 ? ex->split_qjob : ex->hc.n_queries;
    if (qjob < world) fail(ERR_INVALID_ARGUMENT, "set_split: fewer queries than ranks");
    if (world > 1 && (!outboxes || epoch < 1)) fail(ERR_INVALID_ARGUMENT, "set_split: need the outboxes and epoch >= 1");
    if (world > 1 && epoch >= (1LL << 31)) fail(ERR_INVALID_ARGUMENT, "set_split: epoch out of range");
    ex->split_rank = rank;
    ex->split_world = world;
    ex->split_qjob = qjob;
    ex->split_epoch = epoch;
    ex->split_boxes.clear();
    for (int r = 0; world > 1 && r < world; ++r) ex->split_boxes.push_back(static_cast<char*>(outboxes[r]));
    // the rank's executor is the reference Executor over its block (n_queries = block size)
    ex->hc.n_queries = split_block_lo(qjob, rank + 1, world) - split_block_lo(qjob, rank, world);
    ex->cfg_dump = to_json(ex->hc, ex->t1, ex->t2, ex->t3).dump();
  });
}

int spex_executor_emulate_split(spex_executor* ex, int rank, int world) {
  return guarded([&] {
#ifdef SPEX_EMU
    (void)ex;
    (void)rank;
    (void)world;
    fail(ERR_INVALID_ARGUMENT, "split emulation needs the CUDA build");
#else
    if (ex->ran) fail(ERR_INVALID_ARGUMENT, "emulate_split: executor already ran");
    const long long box = spex_split_outbox_bytes(ex->split_qjob, world);
    if (box < 0 || rank < 0 || rank >= world) fail(ERR_INVALID_ARGUMENT, "emulate_split: bad rank / world");
    if (world == 1) return;
    CUDA_OK(cudaSetDevice(ex->device));
    if (ex->emu_boxes) cudaFree(ex->emu_boxes);
    CUDA_OK(cudaMalloc(reinterpret_cast<void**>(&ex->emu_boxes), static_cast<size_t>(box) * world));
    CUDA_OK(cudaMemset(ex->emu_boxes, 0, static_cast<size_t>(box) * world));
    CUDA_OK(cudaDeviceSynchronize());
    std::vector<void*> bx(world);
    for (int r = 0; r < world; ++r) bx[r] = ex->emu_boxes + box * r;
    const int rc = spex_executor_set_split(ex, rank, world, bx.data(), 1);
    if (rc) fail(rc, g_err);
    ex->split_emulate = 1;
#endif
  });
}

int spex_split_run(const char* config_json, uint64_t seed, const char* flags_csv, int world, int device, int trace,
                   spex_executor** out) {
  return guarded([&] {
    if (world < 1 || world > kMaxSplit) fail(ERR_INVALID_ARGUMENT, "split_run: world out of range");
    int node_cap = 512;
    if (const char* e = std::getenv("SPEX_NODE_CAP")) node_cap = std::max(16, std::atoi(e));
    for (int attempt = 0;; ++attempt) {
      std::vector<spex_executor*> exs;
      auto free_all = [&] {
        for (auto* e : exs) spex_executor_destroy(e);
        exs.clear();
      };
      const HostConfig hc = parse_config(config_json);
      const long long box = world > 1 ? spex_split_outbox_bytes(hc.n_queries, world) : 0;
      if (box < 0) fail(ERR_INVALID_ARGUMENT, "split_run: fewer queries than ranks");
      std::vector<char> host_boxes(static_cast<size_t>(box) * world + 64, 0);
      std::vector<void*> boxes(world, nullptr);
      for (int r = 0; r < world; ++r) boxes[r] = host_boxes.data() + box * r;  // emulation; the device runner has its own
      for (int r = 0; r < world; ++r) {
        spex_executor* e = nullptr;
        int rc = spex_executor_create(config_json, seed, flags_csv, device, &e);
        if (!rc) {
          exs.push_back(e);
          rc = spex_executor_set_split(e, r, world, boxes.data(), 1);
        }
        if (rc) {
          const std::string m = g_err;
          free_all();
          fail(rc, m);
        }
        e->node_cap0 = node_cap;
      }
      int err = 0;
#ifdef SPEX_EMU
      std::vector<std::thread> th;
      std::vector<int> rc(world, 0);
      std::vector<std::string> msg(world);
      for (int r = 0; r < world; ++r)
        th.emplace_back([&, r] {
          try {
            run_executor(*exs[r], trace);
          } catch (const SpexError& e) {
            rc[r] = e.code;
            msg[r] = e.what;
          } catch (const std::exception& e) {
            rc[r] = ERR_INTERNAL;
            msg[r] = e.what();
          }
        });
      for (auto& t : th) t.join();
      for (int r = 0; r < world && !err; ++r)
        if (rc[r]) err = rc[r];
      std::string first_msg;
      for (int r = 0; r < world; ++r)
        if (rc[r] && first_msg.empty()) first_msg = msg[r];
#else
      float ms = 0.f;
      try {
        err = run_group_device(exs, device, trace, node_cap, &ms);
      } catch (...) {
        free_all();
        throw;
      }
      const std::string first_msg = "device control error";
#endif
      if ((err == ERR_CAP_NODES || err == ERR_CAP_STAGE) && attempt < 3) {
        free_all();
        node_cap *= 2;  // every rank reruns with the larger arena
        continue;
      }
      if (err) {
        free_all();
        fail(err, "split_run: " + first_msg);
      }
      for (int r = 0; r < world; ++r) {
        exs[r]->ran = true;
        out[r] = exs[r];
      }
      return;
    }
  });
}

#ifndef SPEX_EMU
int spex_split_outbox_alloc(int device, long long bytes, void** dptr, unsigned char* ipc_handle) {
  return guarded([&] {
    CUDA_OK(cudaSetDevice(device));
    void* p = nullptr;
    CUDA_OK(cudaMalloc(&p, static_cast<size_t>(bytes)));
    CUDA_OK(cudaMemset(p, 0, static_cast<size_t>(bytes)));
    CUDA_OK(cudaDeviceSynchronize());
    if (ipc_handle) {
      cudaIpcMemHandle_t h;
      CUDA_OK(cudaIpcGetMemHandle(&h, p));
      std::memcpy(ipc_handle, &h, sizeof(h));
    }
    *dptr = p;
  });
}

int spex_split_outbox_open(int device, const unsigned char* ipc_handle, void** dptr) {
  return guarded([&] {
    CUDA_OK(cudaSetDevice(device));
    cudaIpcMemHandle_t h;
    std::memcpy(&h, ipc_handle, sizeof(h));
    CUDA_OK(cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess));
  });
}

int spex_split_outbox_close(void* dptr) {
  return guarded([&] { CUDA_OK(cudaIpcCloseMemHandle(dptr)); });
}

int spex_split_outbox_free(void* dptr) {
  return guarded([&] { CUDA_OK(cudaFree(dptr)); });
}
#else
int spex_split_outbox_alloc(int, long long, void**, unsigned char*) {
  return guarded([&] { fail(ERR_INVALID_ARGUMENT, "outboxes need the CUDA build"); });
}
int spex_split_outbox_open(int, const unsigned char*, void**) {
  return guarded([&] { fail(ERR_INVALID_ARGUMENT, "outboxes need the CUDA build"); });
}
int spex_split_outbox_close(void*) { return 0; }
int spex_split_outbox_free(void*) { return 0; }
#endif

int spex_executor_split_stats(spex_executor* ex, long long* rounds, double* wait_ms) {
  return guarded([&] {
    if (rounds) *rounds = ex->g.xch_rounds;
    if (wait_ms) *wait_ms = ex->g.xch_wait_ns * 1e-6;
  });
}

int spex_executor_model_stats(spex_executor* ex, spex_model_stats* out) {
  return guarded([&] {
    std::memset(out, 0, sizeof(*out));
#ifndef SPEX_EMU
    const ModelRunResult& r = ex->mres;
    out->model_ms = r.model_ms;
    out->attn_ms = r.attn_ms;
    out->attn_launches = r.attn_launches;
    out->attn_alg_bytes = r.attn_alg_bytes;
    out->decode_rows = r.decode_rows;
    out->decode_steps = r.decode_steps;
    out->prefill_rows = r.prefill_rows;
    out->prm_rows = r.prm_rows;
    out->prm_thoughts = r.prm_thoughts;
    out->policy_flops = r.policy_flops;
    out->prm_flops = r.prm_flops;
    out->launches = r.launches;
    out->control_ms = r.control_ms;
    out->gemm_calls = r.gemm_calls;
    out->step_ms = r.step_ms;
    out->streamed = r.streamed;
#else
    (void)ex;
#endif
  });
}

int spex_executor_set_kv_pages(spex_executor* ex, long long pages) {
  return guarded([&] {
    if (pages < 0) fail(ERR_INVALID_ARGUMENT, "set_kv_pages: negative page count");
    if (ex->ran) fail(ERR_INVALID_ARGUMENT, "set_kv_pages: executor already ran");
    ex->kv_pages_req = pages;
  });
}

int spex_executor_kv_stats(spex_executor* ex, spex_kv_stats* out) {
  return guarded([&] {
    std::memset(out, 0, sizeof(*out));
    out->pages = ex->kv_pages;
    out->page_tokens = kKvPage;
    out->root_pages = ex->kv_pages > 0 ? static_cast<long long>(ex->hc.n_queries) * kv_pages_of(ex->hc.prompt_tokens) : 0;
    out->peak_pages = ex->g.kv_peak;
    out->freed_pages = ex->g.kv_freed;
    out->live_pages_end = ex->g.kv_live;
    out->allocated_pages = ex->g.kv_next;
    out->fresh_pages = ex->g.kv_bump;
    out->page_table_entries = ex->kv_pt_cap;
  });
}

int spex_executor_decode_outputs(spex_executor* ex, void* buf, long long cap, long long* n) {
  return guarded([&] {
#ifndef SPEX_EMU
    long long k = std::min<long long>(cap, static_cast<long long>(ex->dec_out.size()));
    if (buf && k > 0) std::memcpy(buf, ex->dec_out.data(), k * sizeof(DecodeOut));
    *n = static_cast<long long>(ex->dec_out.size());
#else
    (void)ex;
    (void)buf;
    (void)cap;
    *n = 0;
#endif
  });
}

int spex_executor_prm_outputs(spex_executor* ex, void* buf, long long cap, long long* n) {
  return guarded([&] {
#ifndef SPEX_EMU
    long long k = std::min<long long>(cap, static_cast<long long>(ex->prm_out.size()));
    if (buf && k > 0) std::memcpy(buf, ex->prm_out.data(), k * sizeof(PrmOut));
    *n = static_cast<long long>(ex->prm_out.size());
#else
    (void)ex;
    (void)buf;
    (void)cap;
    *n = 0;
#endif
  });
}

int spex_executor_set_reward_source(spex_executor* ex, int source) {
  return guarded([&] {
    if (source != 0 && source != 1) fail(ERR_INVALID_ARGUMENT, "set_reward_source: 0 (content oracle) or 1 (PRM)");
    if (ex->ran) fail(ERR_INVALID_ARGUMENT, "set_reward_source: executor already ran");
    ex->reward_prm = source;
  });
}

int spex_executor_query_wall_ms(spex_executor* ex, double* out, int cap, int* n, double* reward_wait_ms) {
  return guarded([&] {
    const int q = static_cast<int>(ex->finish_ns.size());
    for (int i = 0; i < q && i < cap; ++i)
      out[i] = ex->finish_ns[i] > 0 ? 1e-6 * static_cast<double>(ex->finish_ns[i] - ex->g.start_ns) : -1.0;
    *n = q;
    if (reward_wait_ms) *reward_wait_ms = 1e-6 * static_cast<double>(ex->g.reward_wait_ns);
  });
}

int spex_executor_query_finish(spex_executor* ex, double* out, int cap, int* n) {
  return guarded([&] {
    const int q = static_cast<int>(ex->qs.size());
    for (int i = 0; i < q && i < cap; ++i) out[i] = ex->qs[i].finish_time;
    *n = q;
  });
}

void spex_executor_destroy(spex_executor* ex) {
  if (ex) step_release(*ex);
#ifndef SPEX_EMU
  if (ex && ex->emu_boxes) cudaFree(ex->emu_boxes);
  if (ex && ex->stream) cudaStreamDestroy(ex->stream);
  if (ex && ex->mstream) cudaStreamDestroy(ex->mstream);
#endif
  delete ex;
}

int spex_run_once(const char* config_json, uint64_t seed, const char* flags_csv,
                  spex_totals* totals, char** out_lines) {
  spex_executor* ex = nullptr;
  int rc = spex_executor_create(config_json, seed, flags_csv, 0, &ex);
  if (rc) return rc;
  rc = spex_executor_run(ex, 1, totals);
  if (rc == 0 && out_lines) rc = spex_executor_log(ex, out_lines, nullptr);
  spex_executor_destroy(ex);
  return rc;
}

int spex_run(const char* config_json, uint64_t seed, const char* flags_csv, spex_trace_cb trace_cb, void* user,
             long long chunk, spex_totals* totals) {
  spex_executor* ex = nullptr;
  int rc = spex_executor_create(config_json, seed, flags_csv, 0, &ex);
  if (rc) return rc;
  for (int done = 0; !rc && !done;) {
    char* ev = nullptr;
    size_t n = 0;
    rc = spex_frontier_step(ex, chunk > 0 ? chunk : 4096, &done, &ev, &n);
    if (!rc && trace_cb) {
      // one callback per event-log line, as TraceWriter::emit (trace.cpp:32-36)
      for (size_t a = 0; a < n;) {
        size_t b = a;
        while (b < n && ev[b] != '\n') ++b;
        const char keep = ev[b < n ? b : n];
        if (b < n) ev[b] = 0;
        trace_cb(ev + a, b - a, user);
        if (b < n) ev[b] = keep;
        a = b + 1;
      }
    }
    std::free(ev);
  }
  if (!rc && totals) rc = guarded([&] { fill_totals(*ex, totals); });
  spex_executor_destroy(ex);
  return rc;
}

}  // extern "C"

#ifdef SPEX_EMU
// ---- the policy / budget hooks of spex_hooks.cu, evaluated on the host by
// the same control functions (test-only emulation library: single thread).
namespace {
int emu_alloc_scratch(std::vector<int>& sm, std::vector<double>& smd, std::vector<i64>& sml, HostExec& hx) {
  sm.assign(2048, 0);
  smd.assign(64, 0.0);
  sml.assign(64, 0);
  hx.sm = sm.data();
  hx.smd = smd.data();
  hx.sml = sml.data();
  return 0;
}
}  // namespace

extern "C" int spex_policy_ucb_score(const double* value, const int* child_visits, const int* parent_visits, int n,
                                     double exploration_c, double* out, int* status) {
  for (int i = 0; i < n; ++i) {
    status[i] = child_visits[i] <= 0 || parent_visits[i] <= 0 ? ERR_ZERO_VISITS : 0;
    out[i] = status[i] ? 0.0
                       : value[i] + exploration_c * std::sqrt(glibc::log(static_cast<double>(parent_visits[i])) /
                                                              child_visits[i]);
  }
  return 0;
}

extern "C" int spex_policy_ucb_select(const double* value, const int* visits, const int* pruned, const int* offsets,
                                      const int* parent_visits, int n_problems, double exploration_c, int* out,
                                      int* status) {
  for (int p = 0; p < n_problems; ++p) {
    out[p] = -1;
    status[p] = ERR_NO_CHILDREN;
    double best_score = 0.0;
    bool unvisited = false;
    for (int i = offsets[p]; i < offsets[p + 1] && !unvisited; ++i) {
      if (pruned[i]) continue;
      status[p] = 0;
      if (visits[i] == 0) {
        out[p] = i - offsets[p];
        unvisited = true;
      }
    }
    if (unvisited || status[p]) continue;
    for (int i = offsets[p]; i < offsets[p + 1]; ++i) {
      if (pruned[i]) continue;
      if (visits[i] <= 0 || parent_visits[p] <= 0) {
        out[p] = -1;
        status[p] = ERR_ZERO_VISITS;
        break;
      }
      const double s = value[i] + exploration_c * std::sqrt(glibc::log(static_cast<double>(parent_visits[p])) /
                                                            visits[i]);
      if (out[p] < 0 || s > best_score) {
        out[p] = i - offsets[p];
        best_score = s;
      }
    }
  }
  return 0;
}

extern "C" int spex_policy_rebase_widths(const double* rewards, const int* offsets, const int* budgets, int n_problems,
                                         double temperature, int sum_preserving, int* widths, int* status) {
  for (int p = 0; p < n_problems; ++p) {
    const int a = offsets[p], n = offsets[p + 1] - offsets[p];
    GState g{};
    Run R{};
    R.g = &g;
    std::vector<double> w(std::max(n, 1)), quota(std::max(n, 1));
    std::vector<int> order(std::max(n, 1));
    rebase_widths(&R, p, rewards + a, n, budgets[p], temperature, sum_preserving != 0, widths + a, w.data(),
                  quota.data(), order.data());
    status[p] = g.error;
  }
  return 0;
}

extern "C" int spex_budget_k_total(const double* hw4, int active_batch, double avg_kv_bytes, int cap, int* out) {
  HostConfig h;
  h.weight_bytes = hw4[0];
  h.mem_bandwidth = hw4[1];
  h.peak_compute = hw4[2];
  h.flops_per_token = hw4[3];
  *out = roofline_k_total(h, active_batch, avg_kv_bytes, cap);
  return 0;
}

extern "C" int spex_content_token_len(const uint64_t* child_hash, int n, const spex_workload* wl, int* out) {
  for (int i = 0; i < n; ++i)
    out[i] = lognormal_tokens(child_hash[i], kSaltTokens, wl->token_mu, wl->token_sigma, wl->token_min, wl->token_max);
  return 0;
}

extern "C" int spex_content_eval(const uint64_t* path_hash, const int* offsets, int n, uint64_t query_seed,
                                 int max_depth, const spex_workload* wl, int* terminal, double* reward, int* label) {
  for (int i = 0; i < n; ++i)
    content_eval(reinterpret_cast<const u64*>(path_hash) + offsets[i], offsets[i + 1] - offsets[i], query_seed,
                 max_depth, *wl, terminal + i, reward + i, label + i);
  return 0;
}

extern "C" int spex_tree_transition_legal(const uint8_t* from, const uint8_t* to, int n, uint8_t* out) {
  for (int i = 0; i < n; ++i) out[i] = transition_legal(from[i], to[i]) ? 1 : 0;
  return 0;
}

extern "C" int spex_tree_prune_subtree(const int32_t* parent, uint8_t* status, int n_nodes, uint32_t id, int* pruned) {
  *pruned = 0;
  HookTree t;
  if (!hook_tree_build_min(t, parent, status, n_nodes)) return ERR_INVALID_ARGUMENT;
  if (id >= static_cast<uint32_t>(n_nodes)) return ERR_UNKNOWN_NODE;
  std::vector<u32> stack(t.S);
  GState g{};
  Run R{};
  R.cfg = t.cfg;
  R.n_parent = t.parent.data();
  R.n_first_child = t.first_child.data();
  R.n_next_sib = t.next_sib.data();
  R.n_status = t.status.data();
  R.n_flags = t.flags.data();
  R.n_tokens = t.tokens.data();
  R.qs = &t.qr;
  R.g = &g;
  R.sp_stack = stack.data();
  QC x = make_qc(&R, 0, nullptr, 0);
  const int cnt = prune_subtree(x, id);
  if (g.error) return ERR_INTERNAL;
  for (int i = 0; i < n_nodes; ++i) status[i] = t.status[i];
  *pruned = cnt;
  return 0;
}

extern "C" int spex_speculation_dfs_plan(const int32_t* parent, const uint8_t* status, const uint8_t* bits,
                                         const double* reward, const int32_t* visits, const double* value,
                                         const int32_t* depth, int n_nodes, int terminal_answers, int family,
                                         double exploration_c, int width, const int32_t* depth_widths,
                                         int n_depth_widths, int target_answers, int k, uint32_t* out_node,
                                         int32_t* out_dist, int* n_out) {
  *n_out = 0;
  if (k < 0 || k > 64) return ERR_INVALID_ARGUMENT;
  HookTree t;
  if (!hook_tree_build(t, parent, status, bits, reward, visits, value, depth, n_nodes, terminal_answers, family,
                       exploration_c, width, depth_widths, n_depth_widths, target_answers, k))
    return ERR_INVALID_ARGUMENT;
  if (family == kRebaseBfs || k == 0) return 0;
  std::vector<int> spv(t.S), spn(t.S), spi(3 * t.S);
  std::vector<double> spval(t.S), spd(3 * t.S);
  std::vector<u32> sps(t.S);
  GState g{};
  Run R{};
  R.cfg = t.cfg;
  R.n_parent = t.parent.data();
  R.n_first_child = t.first_child.data();
  R.n_next_sib = t.next_sib.data();
  R.n_status = t.status.data();
  R.n_flags = t.flags.data();
  R.n_reward = t.reward.data();
  R.n_value = t.value.data();
  R.n_visits = t.visits.data();
  R.n_depth = t.depth.data();
  R.n_nchildren = t.nchildren.data();
  R.qs = &t.qr;
  R.g = &g;
  R.sp_visits = spv.data();
  R.sp_value = spval.data();
  R.sp_nchild = spn.data();
  R.sp_stack = sps.data();
  R.sp_dbl = spd.data();
  R.sp_int = spi.data();
  R.log_tab_n = 0;
  QC x = make_qc(&R, 0, nullptr, 0);
  const int n = dfs_plan(x, k, out_node, out_dist);
  if (g.error) return ERR_INTERNAL;
  *n_out = n;
  return 0;
}

extern "C" int spex_termination_should_terminate(const int* counts, const double* weights, const int* offsets,
                                                 const int* n_total, int n_tallies, int min_answers, double alpha,
                                                 int* out) {
  for (int t = 0; t < n_tallies; ++t) {
    const int b = offsets[t], m = offsets[t + 1] - b;
    int labels = 0;
    for (int r = 0; r < m; ++r) labels += counts[b + r] > 0;
    out[t] = tally_should_terminate(
                 n_total[t], labels, m,
                 [&](int r, int* c, double* x) {
                   *c = counts[b + r];
                   *x = weights[b + r];
                 },
                 min_answers, alpha)
                 ? 1
                 : 0;
  }
  return 0;
}

extern "C" int spex_engine_advance(const spex_engine_hw*, double, double, spex_engine_stream*, int*,
                                   spex_engine_stream*, int*, const int*, const int*, int, spex_engine_finished*, int,
                                   int*, double*) {
  g_err = "spex_engine_advance needs the CUDA build";
  return 200;
}

extern "C" int spex_budget_allocate(const int* capacity, const double* hit_ema, const double* kv_bytes, int n,
                                    int k_total, double tau, double weight_bytes, int* out) {
  for (int i = 0; i < n; ++i) out[i] = 0;
  if (n <= 0 || k_total <= 0) return 0;
  std::vector<double> score(n), w(n);
  std::vector<int> order(n);
  for (int i = 0; i < n; ++i) score[i] = capacity[i] * hit_ema[i] * (weight_bytes + kv_bytes[i]);
  std::vector<int> sm;
  std::vector<double> smd;
  std::vector<i64> sml;
  HostExec hx;
  emu_alloc_scratch(sm, smd, sml, hx);
  GState g{};
  allocate_block(hx, &g, n, k_total, tau, score.data(), capacity, w.data(), out, order.data());
  return 0;
}
#endif

// ============================================================ engine handle
// The decode engine as a handle (SURVEY.md §8b spex_engine_*): the stream
// tables live here, each step runs DecodeEngine::advance's epochs on the
// device (spex_engine_advance, csrc/spex_hooks.cu). A stream names its strict
// ancestors by caller keys (unique per (tree, node), e.g. tree << 32 | node)
// with their token lengths: the engine's unique-KV-token cost (sim.cpp:54-78)
// deduplicates by key, as the reference does by (tree pointer, node).
struct spex_engine {
  spex_engine_hw hw{};
  int device = 0;
  struct Stream {
    spex_engine_stream s{};
    uint32_t node = 0;
    std::vector<int> anc;  // key indices
  };
  std::vector<Stream> active, staged;
  std::unordered_map<uint64_t, int> key_index;
  std::vector<int> key_tokens;
};

extern "C" {

int spex_engine_create(const spex_engine_hw* hw, int device, spex_engine** out) {
  return guarded([&] {
    if (!hw || !out) fail(ERR_INVALID_ARGUMENT, "engine_create: null argument");
    auto* e = new spex_engine();
    e->hw = *hw;
    e->device = device;
    *out = e;
  });
}

void spex_engine_destroy(spex_engine* e) { delete e; }

int spex_engine_add_stream(spex_engine* e, int id, uint32_t node, int tokens, double ready, const uint64_t* anc_keys,
                           const int* anc_tokens, int n_anc) {
  return guarded([&] {
    if (tokens <= 0) fail(ERR_INVALID_ARGUMENT, "add_stream: non-positive token budget");  // sim.cpp:206
    if (n_anc < 0 || (n_anc > 0 && (!anc_keys || !anc_tokens))) fail(ERR_INVALID_ARGUMENT, "add_stream: ancestors");
    spex_engine::Stream st;
    st.s.id = id;
    st.s.remaining = tokens;
    st.s.ready = ready;
    st.node = node;
    for (int i = 0; i < n_anc; ++i) {
      auto it = e->key_index.emplace(anc_keys[i], static_cast<int>(e->key_tokens.size()));
      if (it.second) e->key_tokens.push_back(anc_tokens[i]);
      else e->key_tokens[it.first->second] = anc_tokens[i];
      st.anc.push_back(it.first->second);
    }
    e->staged.push_back(std::move(st));
  });
}

// DecodeEngine::cancel (sim.cpp:216-233): *started = its return value
int spex_engine_cancel(spex_engine* e, int id, int* started) {
  return guarded([&] {
    int r = 1;
    bool hit = false;
    for (auto& st : e->active)
      if (st.s.id == id && !st.s.cancelled) {
        st.s.cancelled = 1;
        st.s.remaining = 1;
        hit = true;
        break;
      }
    if (!hit)
      for (auto it = e->staged.begin(); it != e->staged.end(); ++it)
        if (it->s.id == id) {
          e->staged.erase(it);
          r = 0;
          break;
        }
    if (started) *started = r;
  });
}

int spex_engine_drop(spex_engine* e, int id) {  // DecodeEngine::drop (sim.cpp:235-249)
  return guarded([&] {
    for (auto* v : {&e->active, &e->staged})
      for (auto it = v->begin(); it != v->end(); ++it)
        if (it->s.id == id) {
          v->erase(it);
          return;
        }
  });
}

// DecodeEngine::advance (sim.cpp:305-384) on the handle's streams
int spex_engine_step(spex_engine* e, double now, double limit, spex_engine_finished* out, int cap, int* n_out,
                     double* reached) {
  return guarded([&] {
    const int na0 = static_cast<int>(e->active.size()), ns0 = static_cast<int>(e->staged.size());
    const int tot = std::max(na0 + ns0, 1);
    std::vector<spex_engine_stream> act(tot), stg(tot);
    std::vector<int> anc;
    std::unordered_map<int, const spex_engine::Stream*> by_id;
    auto pack = [&](const spex_engine::Stream& st) {
      spex_engine_stream s = st.s;
      s.anc_off = static_cast<int>(anc.size());
      s.anc_n = static_cast<int>(st.anc.size());
      anc.insert(anc.end(), st.anc.begin(), st.anc.end());
      by_id[st.s.id] = &st;
      return s;
    };
    int na = 0, ns = 0;
    for (const auto& st : e->active) act[na++] = pack(st);
    for (const auto& st : e->staged) stg[ns++] = pack(st);
    int nf = 0;
    double now_out = now;
#ifndef SPEX_EMU
    CUDA_OK(cudaSetDevice(e->device));
#endif
    const int rc = spex_engine_advance(&e->hw, now, limit, act.data(), &na, stg.data(), &ns, anc.data(),
                                       e->key_tokens.data(), static_cast<int>(e->key_tokens.size()), out, cap, &nf,
                                       &now_out);
    if (rc) fail(rc, std::string("engine_step: ") + g_err);
    auto unpack = [&](const spex_engine_stream& s) {
      spex_engine::Stream st = *by_id.at(s.id);
      st.s.remaining = s.remaining;
      st.s.done = s.done;
      st.s.cancelled = s.cancelled;
      return st;
    };
    std::vector<spex_engine::Stream> a2, s2;
    for (int i = 0; i < na; ++i) a2.push_back(unpack(act[i]));
    for (int i = 0; i < ns; ++i) s2.push_back(unpack(stg[i]));
    e->active = std::move(a2);
    e->staged = std::move(s2);
    if (n_out) *n_out = nf;
    if (reached) *reached = now_out;
  });
}

int spex_engine_done_tokens(const spex_engine* e, int id) {  // DecodeEngine::done_tokens (sim.cpp:251-257)
  for (const auto* v : {&e->active, &e->staged})
    for (const auto& st : *v)
      if (st.s.id == id) return st.s.done;
  return 0;
}

int spex_engine_stream_count(const spex_engine* e) { return static_cast<int>(e->active.size() + e->staged.size()); }
int spex_engine_active_count(const spex_engine* e) { return static_cast<int>(e->active.size()); }

double spex_engine_next_ready(const spex_engine* e) {  // DecodeEngine::next_ready (sim.cpp:259-263)
  double r = HUGE_VAL;
  for (const auto& st : e->staged) r = std::min(r, st.s.ready);
  return r;
}

}  // extern "C"

extern "C" int spex_score_batch(const char* prm_shape, uint64_t weight_seed, const int32_t* tokens,
                                const int64_t* offsets, int n, float* scores, int device) {
  return guarded([&] {
    if (n < 0 || (n > 0 && (!tokens || !offsets || !scores))) fail(ERR_INVALID_ARGUMENT, "score_batch: arguments");
#ifdef SPEX_EMU
    (void)prm_shape;
    (void)weight_seed;
    (void)device;
    fail(ERR_INVALID_ARGUMENT, "score_batch needs the CUDA build");
#else
    std::lock_guard<std::mutex> lk(g_model_mu);  // the forward's kernels share process-wide state
    try {
      prm_score_sequences(shape_by_name(prm_shape ? prm_shape : ""), weight_seed, tokens,
                          reinterpret_cast<const long long*>(offsets), n, scores, device);
    } catch (const SpexError&) {
      throw;
    } catch (const std::exception& e) {
      fail(ERR_INVALID_ARGUMENT, std::string("score_batch: ") + e.what());
    }
#endif
  });
}
