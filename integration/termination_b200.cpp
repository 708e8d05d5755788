// integration/termination_b200.cpp — the reference-side binding of the B200
// termination and BFS-speculation hooks (include/spex.h).
//
//   AnswerTally::should_terminate (termination.hpp:15-55, termination.cpp:30-48)
//       over spex_termination_should_terminate: the tally's labels in its own
//       std::map order, the control kernel's tally_should_terminate on the device;
//   bfs_speculative_allocate (speculation.hpp:95-139, speculation.cpp:220-238)
//       over spex_policy_rebase_widths: the reference's definition (sum-preserving
//       softmax widths over the finished entries, budget = their count) with the
//       widths computed by the control kernel's rebase_widths on the device.
//
// oracle/Makefile weakens exactly these symbols in copies of the reference's
// termination.o / speculation.o (objcopy), so these definitions win; the
// reference's unmodified tests/test_termination.cpp and tests/test_speculation.cpp
// then run through the device (tests/test_dropin_gpu.py).
#include <string>
#include <utility>
#include <vector>

#include "spex.h"
#include "totsim/errors.hpp"
#include "totsim/speculation.hpp"
#include "totsim/termination.hpp"

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
