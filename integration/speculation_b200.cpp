// integration/speculation_b200.cpp — the reference-side binding of the B200
// speculation (T1) and termination (T3) hooks (include/spex.h).
//
//   dfs_speculative_select (speculation.hpp:95-139, speculation.cpp:182-218)
//       over spex_speculation_dfs_plan: the tree's nodes marshalled into the
//       control kernel's layout, Algorithm 1's simulated selections (descend /
//       simulate_next with phantom children on the visit overlay) run by the
//       control kernel's own dfs_plan on the device;
//   AnswerTally::should_terminate (termination.hpp:15-55, termination.cpp:30-48)
//       over spex_termination_should_terminate: the tally's labels in its own
//       std::map order, the control kernel's tally_should_terminate on the device;
//   bfs_speculative_allocate (speculation.hpp:95-139, speculation.cpp:220-238)
//       over spex_policy_rebase_widths: the reference's definition (sum-preserving
//       softmax widths over the finished entries, budget = their count) with the
//       widths computed by the control kernel's rebase_widths on the device.
//
// oracle/Makefile weakens exactly these symbols in copies of the reference's
// termination.o / speculation.o (objcopy), so these definitions win (the
// reference's simulate_next, verify_bfs_speculation, record_outcome stay); the
// reference's unmodified tests/test_termination.cpp and tests/test_speculation.cpp
// then run through the device (tests/test_dropin_gpu.py).
#include <string>
#include <utility>
#include <vector>

#include "spex.h"
#include "totsim/errors.hpp"
#include "totsim/speculation.hpp"
#include "totsim/termination.hpp"
#include "totsim/tree.hpp"

namespace totsim {

namespace {

void check(int rc, const char* what) {
  if (rc == 0) return;
  if (rc >= 1 && rc <= static_cast<int>(Errc::InvalidArgument) + 1) throw Error(static_cast<Errc>(rc - 1), what);
  throw Error(Errc::InvalidArgument, std::string(what) + ": device call failed");
}

}  // namespace

bool AnswerTally::should_terminate(int min_answers, double alpha) const {
  std::vector<int> counts;
  std::vector<double> weights;
  for (const auto& [label, agg] : by_label_) {  // std::map: the reference's label order
    (void)label;
    counts.push_back(agg.count);
    weights.push_back(agg.weight_sum);
  }
  const int off[2] = {0, static_cast<int>(counts.size())};
  const int n_total = n_total_;
  int out = 0;
  check(spex_termination_should_terminate(counts.data(), weights.data(), off, &n_total, 1, min_answers, alpha, &out),
        "should_terminate");
  return out != 0;
}

SpeculationPlan dfs_speculative_select(const SearchTree& tree, const SpeculationLedger& ledger, int k,
                                       const PolicyConfig& cfg) {
  (void)ledger;  // outstanding speculation is visible through node state (speculation.cpp:184)
  const int n = static_cast<int>(tree.size());
  std::vector<int32_t> parent(n), visits(n), depth(n);
  std::vector<uint8_t> status(n), bits(n);
  std::vector<double> reward(n), value(n);
  for (int i = 0; i < n; ++i) {
    const ThoughtNode& t = tree.node(static_cast<NodeId>(i));
    parent[i] = t.parent == kNoNode ? -1 : static_cast<int32_t>(t.parent);
    status[i] = static_cast<uint8_t>(t.status);
    bits[i] = static_cast<uint8_t>((t.terminal ? 1 : 0) | (t.gen_done ? 2 : 0) | (t.reward.has_value() ? 4 : 0));
    reward[i] = t.reward.value_or(0.0);
    visits[i] = t.visits;
    value[i] = t.value;
    depth[i] = t.depth;
  }
  const std::vector<int32_t> dw(cfg.depth_widths.begin(), cfg.depth_widths.end());
  std::vector<uint32_t> node(64);
  std::vector<int32_t> dist(64);
  int nt = 0;
  check(spex_speculation_dfs_plan(parent.data(), status.data(), bits.data(), reward.data(), visits.data(), value.data(),
                                  depth.data(), n, tree.terminal_answer_count(), static_cast<int>(cfg.family),
                                  cfg.exploration_c, cfg.width, dw.data(), static_cast<int>(dw.size()),
                                  cfg.target_answers, k, node.data(), dist.data(), &nt),
        "dfs_speculative_select");
  SpeculationPlan plan;
  for (int i = 0; i < nt; ++i) plan.targets.push_back(SpecTarget{node[i], dist[i]});
  return plan;
}

std::vector<std::pair<NodeId, int>> bfs_speculative_allocate(const std::vector<FrontierEntry>& frontier_status,
                                                             const PolicyConfig& cfg) {
  std::vector<NodeId> nodes;
  std::vector<double> rewards;
  for (const auto& e : frontier_status)
    if (e.finished) {
      nodes.push_back(e.node);
      rewards.push_back(e.reward);
    }
  std::vector<std::pair<NodeId, int>> out;
  if (nodes.empty()) return out;
  const int budget = static_cast<int>(nodes.size());
  const int off[2] = {0, budget};
  std::vector<int> widths(nodes.size(), 0);
  int status = 0;
  check(spex_policy_rebase_widths(rewards.data(), off, &budget, 1, cfg.balance_temperature, 1, widths.data(), &status),
        "bfs_speculative_allocate");
  check(status, "bfs_speculative_allocate");
  for (std::size_t i = 0; i < nodes.size(); ++i) out.emplace_back(nodes[i], widths[i]);
  return out;
}

}  // namespace totsim
