// integration/policy_b200.cpp — the reference-side binding of the B200
// policy and budget hooks (include/spex.h, csrc/spex_hooks.cu).
//
// Defines the reference's own free functions with their reference signatures
// over the C ABI, so reference code that calls them runs the device
// arithmetic the control kernel uses inside a search:
//
//   totsim::ucb_score        (policy.hpp:43-47,  policy.cpp:25-30)
//   totsim::ucb_select       (policy.hpp:49-55,  policy.cpp:32-51)
//   totsim::rebase_widths    (policy.hpp:63-70,  policy.cpp:65-118)
//   totsim::roofline_k_total (budget.hpp:37-42,  budget.cpp:23-39)
//   totsim::allocate_budgets (budget.hpp:47-55,  budget.cpp:45-96)
//
// oracle/Makefile links the reference's unmodified tests/test_policy.cpp and
// tests/test_budget.cpp against these definitions: it weakens exactly these
// symbols in copies of the reference's policy.o / budget.o (objcopy), so the
// strong definitions below win and every other function stays the
// reference's. Errors come back as totsim::Error with the reference's Errc.
#include <string>
#include <vector>

#include "spex.h"
#include "totsim/budget.hpp"
#include "totsim/errors.hpp"
#include "totsim/policy.hpp"
#include "totsim/tree.hpp"

namespace totsim {

namespace {

void check(int rc, const char* what) {
  if (rc == 0) return;
  if (rc >= 1 && rc <= static_cast<int>(Errc::InvalidArgument) + 1)
    throw Error(static_cast<Errc>(rc - 1), what);
  throw Error(Errc::InvalidArgument, std::string(what) + ": device call failed");
}

}  // namespace

double ucb_score(double value, int child_visits, int parent_visits, double exploration_c) {
  double out = 0.0;
  int status = 0;
  check(spex_policy_ucb_score(&value, &child_visits, &parent_visits, 1, exploration_c, &out, &status), "ucb_score");
  check(status, "ucb_score needs positive visit counts");
  return out;
}

NodeId ucb_select(const SearchTree& tree, NodeId id, double exploration_c) {
  const ThoughtNode& parent = tree.node(id);  // UnknownNode as in the reference
  const std::vector<NodeId>& kids = parent.children;
  std::vector<double> value(kids.size());
  std::vector<int> visits(kids.size()), pruned(kids.size());
  for (std::size_t i = 0; i < kids.size(); ++i) {
    const ThoughtNode& c = tree.node(kids[i]);
    value[i] = c.value;
    visits[i] = c.visits;
    pruned[i] = c.status == NodeStatus::Pruned ? 1 : 0;
  }
  const int off[2] = {0, static_cast<int>(kids.size())};
  const int pv = parent.visits;
  int pick = -1, status = 0;
  check(spex_policy_ucb_select(value.data(), visits.data(), pruned.data(), off, &pv, 1, exploration_c, &pick, &status),
        "ucb_select");
  check(status, ("node " + std::to_string(id)).c_str());
  return kids[static_cast<std::size_t>(pick)];
}

std::vector<int> rebase_widths(const std::vector<double>& rewards, int budget, double temperature, WidthMode mode) {
  if (rewards.empty()) throw Error(Errc::EmptyRewards, "rebase_widths");
  const int off[2] = {0, static_cast<int>(rewards.size())};
  std::vector<int> widths(rewards.size(), 0);
  int status = 0;
  check(spex_policy_rebase_widths(rewards.data(), off, &budget, 1, temperature,
                                  mode == WidthMode::SumPreserving ? 1 : 0, widths.data(), &status),
        "rebase_widths");
  check(status, "rebase_widths");
  return widths;
}

int roofline_k_total(const HardwareProfile& hw, int active_batch, double avg_kv_bytes, int cap) {
  const double hw4[4] = {hw.weight_bytes, hw.mem_bandwidth, hw.peak_compute, hw.flops_per_token};
  int out = 0;
  check(spex_budget_k_total(hw4, active_batch, avg_kv_bytes, cap, &out), "roofline_k_total");
  return out;
}

std::vector<int> allocate_budgets(const std::vector<QueryState>& queries, int k_total, double tau,
                                  const HardwareProfile& hw) {
  const std::size_t n = queries.size();
  std::vector<int> cap(n), out(n, 0);
  std::vector<double> ema(n), kv(n);
  for (std::size_t i = 0; i < n; ++i) {
    cap[i] = queries[i].capacity;
    ema[i] = queries[i].hit_ema;
    kv[i] = queries[i].kv_bytes;
  }
  check(spex_budget_allocate(cap.data(), ema.data(), kv.data(), static_cast<int>(n), k_total, tau, hw.weight_bytes,
                             out.data()),
        "allocate_budgets");
  return out;
}

}  // namespace totsim
