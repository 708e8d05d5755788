// hook_tree.h — one query's search tree in the control kernel's SoA layout,
// built on the host from plain arrays, so a hook can run the control's own
// tree functions on it (spex_speculation_dfs_plan: dfs_plan, ctl_drivers.h).
// Host code only; included by spex_hooks.cu (device copies) and by the
// test-only emulation build of spex_capi.cpp (host pointers).
#pragma once

#include <cstdint>
#include <cstring>
#include <vector>

#include "ctl_state.h"

namespace spex {

struct HookTree {
  int n = 0, cap = 0, S = 0;
  std::vector<u32> parent, first_child, next_sib;
  std::vector<u8> status;
  std::vector<u16> flags;
  std::vector<double> reward, value;
  std::vector<int> visits, depth, nchildren, tokens;
  Cfg cfg{};
  QueryRun qr{};
};

// Returns false on malformed input (a parent not below its child, a status
// code out of range, too many depth widths).
inline bool hook_tree_build(HookTree& t, const int32_t* parent, const uint8_t* status, const uint8_t* bits,
                            const double* reward, const int32_t* visits, const double* value, const int32_t* depth,
                            int n, int terminal_answers, int family, double exploration_c, int width,
                            const int32_t* depth_widths, int n_dw, int target_answers, int k) {
  if (n < 1 || k < 0 || n_dw < 0 || n_dw > kMaxDepthWidths || family < 0 || family > 2) return false;
  t.n = n;
  t.cap = n + k + 64;
  t.S = t.cap + 64;
  t.parent.assign(t.cap, kNoNode);
  t.first_child.assign(t.cap, kNoNode);
  t.next_sib.assign(t.cap, kNoNode);
  t.status.assign(t.cap, 0);
  t.flags.assign(t.cap, 0);
  t.reward.assign(t.cap, 0.0);
  t.value.assign(t.cap, 0.0);
  t.visits.assign(t.cap, 0);
  t.depth.assign(t.cap, 0);
  t.nchildren.assign(t.cap, 0);
  t.tokens.assign(t.cap, 0);
  std::vector<u32> last(t.cap, kNoNode);
  for (int i = 0; i < n; ++i) {
    if (status[i] > kTerminalAnswer) return false;
    if (i == 0 ? parent[i] != -1 : (parent[i] < 0 || parent[i] >= i)) return false;
    t.status[i] = status[i];
    t.flags[i] = static_cast<u16>(((bits[i] & 1) ? NF_TERMINAL : 0) | ((bits[i] & 2) ? NF_GEN_DONE : 0) |
                                  ((bits[i] & 4) ? NF_HAS_REWARD : 0));
    t.reward[i] = reward[i];
    t.value[i] = value[i];
    t.visits[i] = visits[i];
    t.depth[i] = depth[i];
    if (i > 0) {
      // children in NodeId order = the reference's slot order (add_node appends)
      const u32 p = static_cast<u32>(parent[i]);
      t.parent[i] = p;
      if (last[p] == kNoNode) t.first_child[p] = static_cast<u32>(i);
      else t.next_sib[last[p]] = static_cast<u32>(i);
      last[p] = static_cast<u32>(i);
      t.nchildren[p] += 1;
    }
  }
  std::memset(&t.cfg, 0, sizeof(t.cfg));
  t.cfg.family = family;
  t.cfg.exploration_c = exploration_c;
  t.cfg.width = width;
  t.cfg.n_depth_widths = n_dw;
  for (int i = 0; i < n_dw; ++i) t.cfg.depth_widths[i] = depth_widths[i];
  t.cfg.target_answers = target_answers;
  t.cfg.node_cap = t.cap;
  t.cfg.spec_k = k;
  std::memset(&t.qr, 0, sizeof(t.qr));
  t.qr.nnodes = n;
  t.qr.terminal_count = terminal_answers;
  return true;
}

// The tree alone (parents and statuses; the other node fields zero), for the
// tree-maintenance hooks (spex_tree_prune_subtree).
inline bool hook_tree_build_min(HookTree& t, const int32_t* parent, const uint8_t* status, int n) {
  std::vector<uint8_t> zb(n, 0);
  std::vector<double> zd(n, 0.0);
  std::vector<int32_t> zi(n, 0);
  return hook_tree_build(t, parent, status, zb.data(), zd.data(), zi.data(), zd.data(), zi.data(), n, 0, 0, 1.0, 1,
                         nullptr, 0, 1, 0);
}

}  // namespace spex
