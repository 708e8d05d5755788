// integration/tree_b200.cpp — the reference-side binding of the B200 tree
// maintenance hooks (include/spex.h).
//
//   transition_legal (tree.hpp:43, tree.cpp:23-45) over spex_tree_transition_legal;
//   SearchTree::prune_subtree (tree.hpp:104, tree.cpp:119-141) over
//       spex_tree_prune_subtree: the tombstone DFS run by the control kernel's
//       own prune_subtree on the tree's parents and statuses, the new statuses
//       written back and the frontier filtered as the reference does.
//
// oracle/Makefile weakens exactly these symbols in a copy of the reference's
// tree.o (objcopy), so these definitions win; the reference's unmodified
// tests/test_tree.cpp then runs through the device (tests/test_dropin_gpu.py).
#include <string>
#include <vector>

#include "spex.h"
#include "totsim/errors.hpp"
#include "totsim/tree.hpp"

namespace totsim {

namespace {

void check(int rc, const char* what) {
  if (rc == 0) return;
  if (rc >= 1 && rc <= static_cast<int>(Errc::InvalidArgument) + 1) throw Error(static_cast<Errc>(rc - 1), what);
  throw Error(Errc::InvalidArgument, std::string(what) + ": device call failed");
}

}  // namespace

bool transition_legal(NodeStatus from, NodeStatus to) {
  const uint8_t f = static_cast<uint8_t>(from), t = static_cast<uint8_t>(to);
  uint8_t out = 0;
  check(spex_tree_transition_legal(&f, &t, 1, &out), "transition_legal");
  return out != 0;
}

int SearchTree::prune_subtree(NodeId id) {
  check_known(id);  // UnknownNode, as the reference
  const int n = static_cast<int>(nodes_.size());
  std::vector<int32_t> parent(n);
  std::vector<uint8_t> status(n);
  for (int i = 0; i < n; ++i) {
    parent[i] = nodes_[i].parent == kNoNode ? -1 : static_cast<int32_t>(nodes_[i].parent);
    status[i] = static_cast<uint8_t>(nodes_[i].status);
  }
  int pruned = 0;
  check(spex_tree_prune_subtree(parent.data(), status.data(), n, id, &pruned), "prune_subtree");
  for (int i = 0; i < n; ++i) nodes_[i].status = static_cast<NodeStatus>(status[i]);
  if (pruned > 0 && !frontier_.empty()) {  // tree.cpp:132-138
    std::vector<NodeId> kept;
    kept.reserve(frontier_.size());
    for (NodeId f : frontier_)
      if (nodes_[f].status != NodeStatus::Pruned) kept.push_back(f);
    frontier_ = std::move(kept);
  }
  return pruned;
}

}  // namespace totsim
