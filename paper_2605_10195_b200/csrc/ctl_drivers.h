// ctl_drivers.h — event handlers, the three search-family drivers and
// speculative planning (one query per item; see ctl_core.h).
#pragma once

#include "ctl_core.h"

namespace spex {

SPEX_HD bool unpromoted_spec(u8 st) { return st == kSpeculative || st == kSpeculativeDone; }

// executor.cpp:450-463
SPEX_HD void dfs_on_done(const QC& x, u32 node) {
  QueryRun* qr = x.qr;
  if (node != qr->chain_tip) return;
  qr->chain_tip = kNoNode;
  if (has_fl(x, node, NF_TERMINAL)) {
    qr->rollout_active = 0;
    return;
  }
  u32 c = spawn_child(x, node, false, 0);
  qr->chain_tip = c;
}

// executor.cpp:366-411. `sid` already left the engine's active list.
SPEX_HDNI bool on_stream_done(const QC& x, int sid, int tokens_done, int cancelled) {
  Run* R = x.R;
  QueryRun* qr = x.qr;
  u32 node = R->st_node[sid];
  u32 ni = NI(x, node);
  R->n_stream[ni] = -1;
  qr->generated += tokens_done;
  if (R->n_status[ni] == kPruned) {
    qr->wasted += tokens_done;
    if (Rec* r = new_rec(x, EV_DONE, node)) {
      r->a = sid;
      r->b = tokens_done;
      r->flags = (cancelled ? RF_CANCELLED : 0) | RF_STALE;
    }
    return false;
  }
  set_fl(x, node, NF_GEN_DONE);
  qr->live_cache += R->n_tokens[ni];
  touch(x);
  if (Rec* r = new_rec(x, EV_DONE, node)) {
    r->a = sid;
    r->b = tokens_done;
  }
  if (R->n_status[ni] == kExpanding) {
    set_status(x, node, kAwaitingReward);
    qr->pending_rewards += 1;
  }
  Item* it = x.it;
  if (it->npsh >= it->psh_cap) {
    set_err(R, ERR_CAP_STAGE, x.q, node);
    return false;
  }
  it->psh[it->npsh++] = PushRec{x.q, node};
  if (x.c->family == kRstarDfs) dfs_on_done(x, node);
  return true;
}

// RewardOracle::reward (sim.cpp:146-152) realised by the PRM: the forward
// scores the thought in the schedule entry recorded at its completion and
// raises that entry's flag; the control waits for it (device only).
SPEX_HDNI double prm_reward(const QC& x, u32 node) {
  Run* R = x.R;
  const u32 ni = NI(x, node);
#if SPEX_DEVICE_PASS
  const int e = R->n_prm_e[ni];
  if (*reinterpret_cast<volatile int*>(&R->prm_done[e]) == 0) {
    const i64 t0 = spex_wall_ns();
    while (*reinterpret_cast<volatile int*>(&R->prm_done[e]) == 0) {
      __nanosleep(256);
      if (spex_wall_ns() - t0 > 120000000000LL) {  // watchdog: no score in 120 s (forward gone)
        set_err(R, ERR_STALLED, x.q, node);
        return 0.0;
      }
    }
    atomic_add_i64(&R->g->reward_wait_ns, spex_wall_ns() - t0);
  }
  __threadfence();
  const double s = static_cast<double>(*reinterpret_cast<volatile float*>(&R->n_score[ni]));
  return s < 0.0 ? 0.0 : (s > 1.0 ? 1.0 : s);
#else
  (void)R;
  (void)ni;
  set_err(x.R, ERR_INTERNAL, x.q, node);  // the host emulation has no PRM
  return 0.0;
#endif
}

// executor.cpp:413-444
SPEX_HDNI void on_reward(const QC& x, u32 node) {
  Run* R = x.R;
  QueryRun* qr = x.qr;
  u32 ni = NI(x, node);
  if (R->n_status[ni] == kPruned) return;
  double r;
  if (x.c->reward_prm && q_owned(*x.c, x.q)) {
    // the PRM's score of the thought (K4): wait for its schedule entry
    r = prm_reward(x, node);
  } else {
    r = oracle_reward(x, node);
  }
  R->n_reward[ni] = r;
  set_fl(x, node, NF_HAS_REWARD);
  touch(x);
  if (Rec* rec = new_rec(x, EV_REWARD, node)) rec->x = r;
  if (R->n_status[ni] == kSpeculative) {
    set_status(x, node, kSpeculativeDone);
    if (has_fl(x, node, NF_LEDGER_ACTIVE)) {
      clr_fl(x, node, NF_LEDGER_ACTIVE);
      qr->n_active_exp -= 1;
    }
    set_fl(x, node, NF_LEDGER_COMPLETED);
    return;
  }
  bool terminal = has_fl(x, node, NF_TERMINAL);
  set_status(x, node, terminal ? kTerminalAnswer : kCommitted);
  qr->pending_rewards -= 1;
  if (has_fl(x, node, NF_BATCH_PENDING)) {
    clr_fl(x, node, NF_BATCH_PENDING);
    qr->batch_pending -= 1;
  }
  if (has_fl(x, node, NF_COHORT_PENDING)) {
    clr_fl(x, node, NF_COHORT_PENDING);
    qr->cohort_pending -= 1;
  }
  if (x.c->family == kRstarDfs) backpropagate(x, node, r);
  if (terminal) record_answer_event(x, node, r);
}

// ------------------------------------------------------------ rollout chains
enum Rollout { kIssued, kEnded, kFinished };

// executor.cpp:467-525
SPEX_HDNI int dfs_one_rollout(const QC& x) {
  Run* R = x.R;
  QueryRun* qr = x.qr;
  u32 node = 0;
  for (;;) {
    if (R->g->error) return kFinished;
    u32 ni = NI(x, node);
    if (has_fl(x, node, NF_TERMINAL)) {
      double r = R->n_reward[ni];
      backpropagate(x, node, r);
      record_answer_event(x, node, r);
      return qr->finished ? kFinished : kEnded;
    }
    u32 pick = kNoNode;
    bool any = false;
    for (u32 c = R->n_first_child[ni]; c != kNoNode; c = R->n_next_sib[NI(x, c)]) {
      if (st_of(x, c) == kPruned) continue;
      any = true;
      if (R->n_visits[NI(x, c)] == 0) {
        pick = c;
        break;
      }
    }
    if (pick != kNoNode) {
      if (unpromoted_spec(st_of(x, pick))) {
        const bool mid_gen = !has_fl(x, pick, NF_GEN_DONE);
        const bool scored = has_fl(x, pick, NF_HAS_REWARD);
        do_promote(x, pick);
        if (mid_gen) {
          qr->chain_tip = pick;
          qr->rollout_active = 1;
          return kIssued;
        }
        if (scored) {
          double r = R->n_reward[NI(x, pick)];
          backpropagate(x, pick, r);
          if (has_fl(x, pick, NF_TERMINAL)) {
            record_answer_event(x, pick, r);
            return qr->finished ? kFinished : kEnded;
          }
        } else if (has_fl(x, pick, NF_TERMINAL)) {
          return kEnded;
        }
      }
      node = pick;
      continue;
    }
    if (R->n_nchildren[ni] < budget_at(*x.c, R->n_depth[ni])) {
      u32 c = spawn_child(x, node, false, 0);
      qr->chain_tip = c;
      qr->rollout_active = 1;
      return kIssued;
    }
    if (!any) {
      finish_query(x, false);
      return kFinished;
    }
    node = ucb_select(x, node);
    if (node == kNoNode) return kFinished;
  }
}

// executor.cpp:527-531
SPEX_HD void advance_dfs(const QC& x) {
  QueryRun* qr = x.qr;
  while (!qr->finished && !qr->rollout_active && qr->pending_rewards == 0 && !x.R->g->error) {
    if (dfs_one_rollout(x) != kEnded) break;
  }
}

// ------------------------------------------------------ batched best-first
// executor.cpp:537-581
SPEX_HDNI void advance_rest(const QC& x) {
  Run* R = x.R;
  QueryRun* qr = x.qr;
  while (!qr->finished && !R->g->error) {
    const u32 cur = qr->rest_cur;
    const u32 ci = NI(x, cur);
    const int width = budget_at(*x.c, R->n_depth[ci]);
    for (u32 c = R->n_first_child[ci]; c != kNoNode; c = R->n_next_sib[NI(x, c)]) {
      if (!unpromoted_spec(st_of(x, c))) continue;  // also skips pruned
      do_promote(x, c);
      u8 st = st_of(x, c);
      if (st == kExpanding || st == kAwaitingReward) {
        if (!has_fl(x, c, NF_BATCH_PENDING)) {
          set_fl(x, c, NF_BATCH_PENDING);
          qr->batch_pending += 1;
        }
      } else if (has_fl(x, c, NF_TERMINAL)) {
        record_answer_event(x, c, R->n_reward[NI(x, c)]);
        if (qr->finished) return;
      }
    }
    while (R->n_nchildren[ci] < width) {
      u32 c = spawn_child(x, cur, false, 0);
      if (c == kNoNode) return;
      set_fl(x, c, NF_BATCH_PENDING);
      qr->batch_pending += 1;
    }
    if (qr->batch_pending > 0) return;
    u32 best = kNoNode;
    for (u32 c = R->n_first_child[ci]; c != kNoNode; c = R->n_next_sib[NI(x, c)]) {
      if (st_of(x, c) == kPruned) continue;
      u32 cn = NI(x, c);
      if (has_fl(x, c, NF_TERMINAL) || R->n_visits[cn] > 0 || !has_fl(x, c, NF_HAS_REWARD)) continue;
      if (best == kNoNode || R->n_reward[cn] > R->n_reward[NI(x, best)]) best = c;
    }
    if (best != kNoNode) {
      backpropagate(x, best, R->n_reward[NI(x, best)]);
      R->q_rest_stack[x.base + qr->rest_sp++] = cur;
      qr->rest_cur = best;
      continue;
    }
    if (qr->rest_sp == 0) {
      finish_query(x, false);
      return;
    }
    qr->rest_cur = R->q_rest_stack[x.base + --qr->rest_sp];
  }
}

// ----------------------------------------------------- layered frontier (REBASE)
// executor.cpp:587-656
SPEX_HDNI void advance_layer(const QC& x) {
  Run* R = x.R;
  QueryRun* qr = x.qr;
  u32* layer = R->q_layer + x.base;
  u32* cohort = R->q_cohort + x.base;
  const int S = scratch_stride(*x.c);
  double* rewards = x.dbl;
  double* w = x.dbl + S;
  double* quota = x.dbl + 2 * S;
  int* widths = x.ints;
  int* order = x.ints + S;
  while (!qr->finished && !R->g->error) {
    if (qr->cohort_n > 0) {
      int m = 0;
      for (int i = 0; i < qr->cohort_n; ++i) {
        u32 c = cohort[i];
        if (st_of(x, c) == kCommitted && !has_fl(x, c, NF_TERMINAL)) layer[m++] = c;
      }
      qr->layer_n = m;
      qr->cohort_n = 0;
    }
    if (qr->layer_n == 0) {
      finish_query(x, false);
      return;
    }
    const int L = qr->layer_n;
    if (L == 1 && layer[0] == 0) {
      widths[0] = budget_at(*x.c, 1);
    } else {
      for (int i = 0; i < L; ++i) rewards[i] = R->n_reward[NI(x, layer[i])];
      int child_depth = R->n_depth[NI(x, layer[0])] + 1;
      if (!rebase_widths(R, x.q, rewards, L, budget_at(*x.c, child_depth),
                         x.c->balance_temperature, false, widths, w, quota, order))
        return;
    }
    for (int i = 0; i < L; ++i) {
      const u32 parent = layer[i];
      const int wd = widths[i];
      const u32 pi = NI(x, parent);
      for (u32 c = R->n_first_child[pi]; c != kNoNode; c = R->n_next_sib[NI(x, c)]) {
        if (!unpromoted_spec(st_of(x, c))) continue;
        if (R->n_slot[NI(x, c)] < wd) {
          const bool scored = has_fl(x, c, NF_HAS_REWARD);
          do_promote(x, c);
          cohort[qr->cohort_n++] = c;
          if (!scored && !has_fl(x, c, NF_COHORT_PENDING)) {
            set_fl(x, c, NF_COHORT_PENDING);
            qr->cohort_pending += 1;
          }
          if (st_of(x, c) == kTerminalAnswer) {
            record_answer_event(x, c, R->n_reward[NI(x, c)]);
            if (qr->finished) return;
          }
        } else {
          record_outcome(x, c, false, R->n_pred[NI(x, c)]);
          update_hit_rate(qr, false, x.c->ema_alpha);
          if (!has_fl(x, c, NF_GEN_DONE)) cancel_stream(x, c);
          int cnt = prune_subtree(x, c);
          if (Rec* r = new_rec(x, EV_PRUNE, c)) r->a = cnt;
        }
      }
      while (R->n_nchildren[pi] < wd) {
        u32 c = spawn_child(x, parent, false, 0);
        if (c == kNoNode) return;
        cohort[qr->cohort_n++] = c;
        set_fl(x, c, NF_COHORT_PENDING);
        qr->cohort_pending += 1;
      }
      kv_unpin(R, x.q, parent);  // an expanded layer gets no more children (executor.cpp:587-656)
    }
    qr->layer_n = 0;
    if (qr->cohort_pending > 0) return;
  }
}

// ======================================================= speculative planning
// TreeSnapshot over a private scratch tree (speculation.cpp:8-39,182-218):
// overlay visits/values for real nodes and up to `k` phantoms (ids >= nnodes).
struct Snap {
  const QC* x;
  int nreal;
  int nph;
  u32 ph_parent[64];
};

SPEX_HD u32 snap_parent(const Snap& s, u32 id) {
  if (static_cast<int>(id) < s.nreal) return s.x->R->n_parent[NI(*s.x, id)];
  return s.ph_parent[id - s.nreal];
}

SPEX_HD void snap_bump_path(Snap& s, u32 leaf) {
  for (u32 cur = leaf; cur != kNoNode; cur = snap_parent(s, cur)) s.x->sv[cur] += 1;
}

SPEX_HD void snap_backprop_path(Snap& s, u32 leaf, double reward) {
  for (u32 cur = leaf; cur != kNoNode; cur = snap_parent(s, cur)) {
    s.x->sv[cur] += 1;
    s.x->sval[cur] += (reward - s.x->sval[cur]) / s.x->sv[cur];
  }
}

enum PickKind { kGenerate, kUseSpec, kBlocked, kRevisit, kDeadEnd };

// Visit live children of `id` in slot order: real children, then phantoms.
// Phantoms are Speculative, not generated, unscored, non-terminal.
#define SNAP_FOR_CHILDREN(s, id, c, BODY)                                                  \
  do {                                                                                     \
    const QC& sx_ = *(s).x;                                                                \
    if (static_cast<int>(id) < (s).nreal) {                                                \
      for (u32 c = sx_.R->n_first_child[NI(sx_, id)]; c != kNoNode;                        \
           c = sx_.R->n_next_sib[NI(sx_, c)]) {                                            \
        if (sx_.R->n_status[NI(sx_, c)] == kPruned) continue;                              \
        BODY                                                                               \
      }                                                                                    \
    }                                                                                      \
    for (int p_ = 0; p_ < (s).nph; ++p_) {                                                 \
      if ((s).ph_parent[p_] != (id)) continue;                                             \
      u32 c = static_cast<u32>((s).nreal + p_);                                            \
      BODY                                                                                 \
    }                                                                                      \
  } while (0)

SPEX_HD bool snap_is_real(const Snap& s, u32 id) { return static_cast<int>(id) < s.nreal; }

// speculation.cpp:59-120
SPEX_HDNI int descend(Snap& s, u32* out) {
  const QC& x = *s.x;
  Run* R = x.R;
  const Cfg& cfg = *x.c;
  u32 node = 0;
  for (int steps = 0; steps < 4 * cfg.node_cap + 64; ++steps) {
    // phantoms are never terminal and never generated
    if (!snap_is_real(s, node)) {
      *out = node;
      return kBlocked;
    }
    u32 ni = NI(x, node);
    if (has_fl(x, node, NF_TERMINAL)) {
      *out = node;
      return kRevisit;
    }
    if (!has_fl(x, node, NF_GEN_DONE)) {
      *out = node;
      return kBlocked;
    }
    const int slots_used = x.snch[node];
    if (cfg.family == kRestHybrid) {
      if (slots_used < budget_at(cfg, R->n_depth[ni])) {
        *out = node;
        return kGenerate;
      }
      bool any = false;
      u32 use = kNoNode;
      SNAP_FOR_CHILDREN(s, node, c, {
        any = true;
        if (use == kNoNode && x.sv[c] == 0) {
          bool up = snap_is_real(s, c) ? unpromoted_spec(R->n_status[NI(x, c)]) : true;
          if (up) use = c;
        }
      });
      if (!any) {
        *out = node;
        return kDeadEnd;
      }
      if (use != kNoNode) {
        *out = use;
        return kUseSpec;
      }
      u32 best = kNoNode;
      SNAP_FOR_CHILDREN(s, node, c, {
        if (snap_is_real(s, c)) {
          u32 cn = NI(x, c);
          if (!(R->n_flags[cn] & NF_TERMINAL) && (R->n_flags[cn] & NF_HAS_REWARD)) {
            if (best == kNoNode || R->n_reward[cn] > R->n_reward[NI(x, best)]) best = c;
          }
        }
      });
      if (best == kNoNode) {
        *out = node;
        return kBlocked;
      }
      node = best;
      continue;
    }
    // DFS walk: unvisited first (slot order), then a fresh slot, then UCB.
    u32 unvisited = kNoNode;
    bool any = false;
    SNAP_FOR_CHILDREN(s, node, c, {
      any = true;
      if (unvisited == kNoNode && x.sv[c] == 0) unvisited = c;
    });
    if (unvisited != kNoNode) {
      bool up = snap_is_real(s, unvisited) ? unpromoted_spec(R->n_status[NI(x, unvisited)]) : true;
      if (up) {
        *out = unvisited;
        return kUseSpec;
      }
      node = unvisited;
      continue;
    }
    if (slots_used < budget_at(cfg, R->n_depth[ni])) {
      *out = node;
      return kGenerate;
    }
    if (!any) {
      *out = node;
      return kDeadEnd;
    }
    u32 best = kNoNode;
    double best_score = 0.0;
    const int pv = x.sv[node] > 1 ? x.sv[node] : 1;
    const double lpv = log_int(R, pv);
    SNAP_FOR_CHILDREN(s, node, c, {
      int cv = x.sv[c] > 1 ? x.sv[c] : 1;
      double sc = x.sval[c] + cfg.exploration_c * sqrt(lpv / cv);
      if (best == kNoNode || sc > best_score) {
        best = c;
        best_score = sc;
      }
    });
    node = best;
  }
  set_err(R, ERR_INTERNAL, x.q, node);
  *out = 0;
  return kDeadEnd;
}

// speculation.cpp:124-180. Returns kNoNode for NothingExpandable.
SPEX_HDNI u32 simulate_next(Snap& s, int* consumed) {
  const QC& x = *s.x;
  Run* R = x.R;
  u32 last_blocked = kNoNode;
  int blocked_repeats = 0;
  for (int guard = 0; guard < 4096; ++guard) {
    if (R->g->error) return kNoNode;
    u32 p = 0;
    int kind = descend(s, &p);
    switch (kind) {
      case kGenerate:
        return p;
      case kUseSpec: {
        bool real = snap_is_real(s, p);
        u16 f = real ? R->n_flags[NI(x, p)] : 0;
        if ((f & NF_GEN_DONE) && (f & NF_HAS_REWARD))
          snap_backprop_path(s, p, R->n_reward[NI(x, p)]);
        else
          snap_bump_path(s, p);
        if (f & NF_TERMINAL) *consumed += 1;
        break;
      }
      case kBlocked:
        if (p == 0) return kNoNode;
        blocked_repeats = (p == last_blocked) ? blocked_repeats + 1 : 0;
        last_blocked = p;
        if (blocked_repeats >= 8) return kNoNode;
        x.sv[p] += 1;
        *consumed += 1;
        break;
      case kRevisit:
      case kDeadEnd:
        if (p == 0) return kNoNode;
        snap_bump_path(s, p);
        *consumed += 1;
        break;
    }
  }
  return kNoNode;
}

// dfs_speculative_select (speculation.cpp:182-218): up to k targets (node,
// predicted distance) planned on the overlay; the live tree is not changed.
// Shared by dfs_speculate and the spex_speculation_dfs_plan hook.
SPEX_HDNI int dfs_plan(const QC& x, int k, u32* tnode, int* tdist) {
  Run* R = x.R;
  const int n = x.qr->nnodes;
  Snap s;
  s.x = &x;
  s.nreal = n;
  s.nph = 0;
  for (int id = 0; id < n; ++id) {
    u32 ni = NI(x, id);
    x.sv[id] = R->n_visits[ni];
    x.sval[id] = R->n_value[ni];
    x.snch[id] = R->n_nchildren[ni];
  }
  for (int id = 0; id < n; ++id) {
    u8 st = R->n_status[NI(x, id)];
    if (st == kExpanding || st == kAwaitingReward) snap_bump_path(s, static_cast<u32>(id));
  }
  int horizon = x.c->target_answers - x.qr->terminal_count;
  if (horizon < 1) horizon = 1;
  int ordinal = 0;
  int nt = 0;
  if (k > 64) k = 64;  // spec_k <= 64 is enforced at config time
  for (int t = 1; t <= k; ++t) {
    u32 node = simulate_next(s, &ordinal);
    if (node == kNoNode) break;
    if (ordinal >= horizon) break;
    ordinal += 1;
    tnode[nt] = node;
    tdist[nt] = ordinal;
    ++nt;
    // phantom in-flight child (scratch.add_node(x, 1, true)) + visit bump
    if (!snap_is_real(s, node) || R->n_status[NI(x, node)] == kPruned) {
      set_err(R, ERR_INTERNAL, x.q, node);
      break;
    }
    u32 ph = static_cast<u32>(n + s.nph);
    s.ph_parent[s.nph++] = node;
    x.sv[ph] = 0;
    x.sval[ph] = 0.0;
    x.snch[ph] = 0;
    x.snch[node] += 1;
    snap_bump_path(s, ph);
  }
  return nt;
}

// dfs_speculative_select fused with executor.cpp:699-702 (spawn each target).
// Returns the number of speculative children spawned.
SPEX_HDNI int dfs_speculate(const QC& x, int k) {
  u32 tnode[64];
  int tdist[64];
  const int nt = dfs_plan(x, k, tnode, tdist);
  for (int i = 0; i < nt; ++i) spawn_child(x, tnode[i], true, tdist[i]);
  return nt;
}

// executor.cpp:675-697 with bfs_speculative_allocate (speculation.cpp:220-238)
SPEX_HDNI int bfs_speculate(const QC& x, int k) {
  Run* R = x.R;
  QueryRun* qr = x.qr;
  const int S = scratch_stride(*x.c);
  const u32* cohort = R->q_cohort + x.base;
  u32* nodes = x.stack;  // finished entries
  double* rewards = x.dbl;
  double* w = x.dbl + S;
  double* quota = x.dbl + 2 * S;
  int* widths = x.ints;
  int* order = x.ints + S;
  int entries = 0, m = 0;
  for (int i = 0; i < qr->cohort_n; ++i) {
    u32 c = cohort[i];
    if (st_of(x, c) == kPruned || has_fl(x, c, NF_TERMINAL)) continue;
    ++entries;
    if (has_fl(x, c, NF_HAS_REWARD)) {
      nodes[m] = c;
      rewards[m] = R->n_reward[NI(x, c)];
      ++m;
    }
  }
  if (entries == 0 || m == 0) return 0;
  if (!rebase_widths(R, x.q, rewards, m, m, x.c->balance_temperature, true, widths, w, quota,
                     order))
    return 0;
  int left = k, spawned = 0;
  for (int i = 0; i < m; ++i) {
    const u32 parent = nodes[i];
    while (left > 0 && R->n_nchildren[NI(x, parent)] < widths[i]) {
      if (spawn_child(x, parent, true, 1) == kNoNode) return spawned;
      left -= 1;
      ++spawned;
    }
    if (left == 0) break;
  }
  return spawned;
}

// executor.cpp:674-703
SPEX_HD int issue_speculation(const QC& x, int k) {
  if (x.c->family == kRebaseBfs) return bfs_speculate(x, k);
  return dfs_speculate(x, k);
}

// executor.cpp:746-763 (per-query part)
SPEX_HD void followup(const QC& x) {
  QueryRun* qr = x.qr;
  if (!qr->admitted || qr->finished) return;
  switch (x.c->family) {
    case kRstarDfs:
      if (!qr->rollout_active && qr->pending_rewards == 0) advance_dfs(x);
      break;
    case kRestHybrid:
      if (qr->batch_pending == 0) advance_rest(x);
      break;
    default:
      if (qr->cohort_pending == 0) advance_layer(x);
      break;
  }
}

}  // namespace spex
