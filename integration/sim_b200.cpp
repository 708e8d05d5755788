// integration/sim_b200.cpp — the reference-side binding of the B200 content
// and expand seams (include/spex.h, csrc/spex_hooks.cu).
//
// Defines, with the reference's own signatures (proj/include/totsim/sim.hpp),
//
//   RewardOracle::token_len / is_terminal / reward / answer_label
//       (sim.hpp:121-136, sim.cpp:112-169) over spex_content_token_len /
//       spex_content_eval: the content draws the device search makes, with
//       glibc's exp / log / cos restated bit for bit;
//   DecodeEngine::advance (sim.hpp:191-196, sim.cpp:305-384) over
//       spex_engine_advance: the engine's epochs on the device, the stream
//       vectors shipped in and out and the unique-KV-token cost computed from
//       each active stream's ancestor keys.
//
// oracle/Makefile weakens exactly these symbols in a copy of the reference's
// sim.o (objcopy), so these definitions win and the rest of sim.cpp (SimClock,
// step_cost, generate_workload, the engine's bookkeeping) stays the
// reference's; the reference's unmodified tests/test_sim.cpp then runs the
// oracle and engine cases through the device (tests/test_dropin_gpu.py).
#include <map>
#include <string>
#include <utility>
#include <vector>

#include "spex.h"
#include "totsim/errors.hpp"
#include "totsim/sim.hpp"
#include "totsim/tree.hpp"

namespace totsim {

namespace {

spex_workload to_c(const WorkloadSpec& w) {
  spex_workload c{};
  c.token_mu = w.token_mu;
  c.token_sigma = w.token_sigma;
  c.token_min = w.token_min;
  c.token_max = w.token_max;
  c.shallow_min = w.shallow_min;
  c.shallow_max = w.shallow_max;
  c.shallow_p = w.shallow_p;
  c.deep_min = w.deep_min;
  c.deep_max = w.deep_max;
  c.deep_p = w.deep_p;
  c.skew = w.skew;
  c.golden_density = w.golden_density;
  c.reward_on = w.reward_on;
  c.reward_off = w.reward_off;
  c.noise_sigma = w.noise_sigma;
  c.correct_base = w.correct_base;
  c.correct_slope = w.correct_slope;
  c.correct_floor = w.correct_floor;
  c.answer_alphabet = w.answer_alphabet;
  c.prompt_tokens = w.prompt_tokens;
  return c;
}

void check(int rc, const char* what) {
  if (rc == 0) return;
  if (rc >= 1 && rc <= static_cast<int>(Errc::InvalidArgument) + 1) throw Error(static_cast<Errc>(rc - 1), what);
  throw Error(Errc::InvalidArgument, std::string(what) + ": device call failed");
}

// path hashes of `id`'s depth-1 ancestor .. itself (empty for the root)
std::vector<std::uint64_t> path_of(const SearchTree& tree, NodeId id) {
  std::vector<std::uint64_t> p;
  for (const ThoughtNode* n = &tree.node(id); n->depth > 0; n = &tree.node(n->parent)) p.push_back(n->path_hash);
  return {p.rbegin(), p.rend()};
}

struct Content {
  int terminal;
  double reward;
  int label;
};

Content eval(const SearchTree& tree, NodeId id, std::uint64_t seed, int max_depth, const WorkloadSpec& wl) {
  const std::vector<std::uint64_t> p = path_of(tree, id);
  const int off[2] = {0, static_cast<int>(p.size())};
  const spex_workload c = to_c(wl);
  Content r{};
  check(spex_content_eval(p.data(), off, 1, seed, max_depth, &c, &r.terminal, &r.reward, &r.label), "content");
  return r;
}

}  // namespace

int RewardOracle::token_len(std::uint64_t child_hash) const {
  const spex_workload c = to_c(wl_);
  int out = 0;
  check(spex_content_token_len(&child_hash, 1, &c, &out), "token_len");
  return out;
}

bool RewardOracle::is_terminal(const SearchTree& tree, NodeId id) const {
  return eval(tree, id, query_seed_, max_depth_, wl_).terminal != 0;
}

double RewardOracle::reward(const SearchTree& tree, NodeId id) const {
  return eval(tree, id, query_seed_, max_depth_, wl_).reward;
}

std::string RewardOracle::answer_label(const SearchTree& tree, NodeId id) const {
  return "a" + std::to_string(eval(tree, id, query_seed_, max_depth_, wl_).label);
}

double DecodeEngine::advance(double now, double limit, std::vector<Finished>& out) {
  // ship the stream vectors with each stream's strict ancestors as keys
  std::map<std::pair<const SearchTree*, NodeId>, int> keys;
  std::vector<int> anc_key, anc_tokens;
  std::map<int, const Stream*> by_id;
  auto pack = [&](const Stream& s) {
    spex_engine_stream e{};
    e.id = s.id;
    e.remaining = s.remaining;
    e.done = s.done;
    e.cancelled = s.cancelled ? 1 : 0;
    e.ready = s.ready;
    e.anc_off = static_cast<int>(anc_key.size());
    for (NodeId cur = s.tree->node(s.node).parent; cur != kNoNode; cur = s.tree->node(cur).parent) {
      auto it = keys.find({s.tree, cur});
      if (it == keys.end()) {
        it = keys.emplace(std::make_pair(s.tree, cur), static_cast<int>(anc_tokens.size())).first;
        anc_tokens.push_back(s.tree->node(cur).token_len);
      }
      anc_key.push_back(it->second);
    }
    e.anc_n = static_cast<int>(anc_key.size()) - e.anc_off;
    by_id[s.id] = &s;
    return e;
  };
  const int total = static_cast<int>(active_.size() + staged_.size());
  std::vector<spex_engine_stream> act(total > 0 ? total : 1), stg(total > 0 ? total : 1);
  int na = 0, ns = 0;
  for (const Stream& s : active_) act[na++] = pack(s);
  for (const Stream& s : staged_) stg[ns++] = pack(s);
  const spex_engine_hw hw{hw_.weight_bytes,    hw_.mem_bandwidth,      hw_.peak_compute,
                          hw_.flops_per_token, hw_.kv_bytes_per_token, hw_.reward_latency};
  std::vector<spex_engine_finished> fin(total > 0 ? total : 1);
  int nf = 0;
  double now_out = now;
  check(spex_engine_advance(&hw, now, limit, act.data(), &na, stg.data(), &ns, anc_key.data(), anc_tokens.data(),
                            static_cast<int>(anc_tokens.size()), fin.data(), static_cast<int>(fin.size()), &nf,
                            &now_out),
        "DecodeEngine::advance");
  auto unpack = [&](const spex_engine_stream& e) {
    Stream s = *by_id.at(e.id);
    s.remaining = e.remaining;
    s.done = e.done;
    s.cancelled = e.cancelled != 0;
    return s;
  };
  for (int i = 0; i < nf; ++i) {
    const Stream& s = *by_id.at(fin[i].id);
    out.push_back({fin[i].id, s.node, fin[i].tokens_done, fin[i].cancelled != 0, fin[i].time});
  }
  std::vector<Stream> new_act, new_stg;
  for (int i = 0; i < na; ++i) new_act.push_back(unpack(act[i]));
  for (int i = 0; i < ns; ++i) new_stg.push_back(unpack(stg[i]));
  active_ = std::move(new_act);
  staged_ = std::move(new_stg);
  dirty_ = true;
  return now_out;
}

}  // namespace totsim
