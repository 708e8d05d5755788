// ctl_core.h — per-query search control of one frontier-expansion step.
//
// One warp owns one query ("item") at a time; lane 0 runs the query's
// sequential state machine, exactly as the reference's single-writer consumer
// does for that query. Everything a query emits (event records, new decode
// streams, reward events, finish markers) is staged per item and placed into
// the global log / stream table / event FIFO by an order-preserving scan at
// commit time (ctl_run.h), which is what makes a parallel step reproduce the
// reference's sequential order exactly.
//
// Each function cites the reference code it restates.
#pragma once

#include "ctl_rng.h"
#include "ctl_state.h"

namespace spex {

// --------------------------------------------------------------------- item
struct Item {
  Rec* rec;
  int nrec, rec_cap;
  SpawnRec* spw;
  int nspw, spw_cap;
  PushRec* psh;
  int npsh, psh_cap;
  int sdelta;  // change of engine.stream_count() caused by this item
  int fin;     // the item's query finished
};

SPEX_HDNI void set_err(Run* R, int code, int q, u32 node) {
  GState* g = R->g;
#if SPEX_DEVICE_PASS
  if (atomicCAS(&g->error, 0, code) == 0) {
    g->error_q = q;
    g->error_node = node;
  }
#else
  if (g->error == 0) {
    g->error = code;
    g->error_q = q;
    g->error_node = node;
  }
#endif
}

SPEX_HD i64 atomic_add_i64(i64* p, i64 v) {
#if SPEX_DEVICE_PASS
  return static_cast<i64>(atomicAdd(reinterpret_cast<unsigned long long*>(p),
                                    static_cast<unsigned long long>(v)));
#else
  i64 o = *p;
  *p += v;
  return o;
#endif
}

SPEX_HD int atomic_add_int(int* p, int v) {
#if SPEX_DEVICE_PASS
  return atomicAdd(p, v);
#else
  int o = *p;
  *p += v;
  return o;
#endif
}

SPEX_HD i64 spex_clock() {
#if SPEX_DEVICE_PASS
  return static_cast<i64>(clock64());
#else
  return 0;
#endif
}

// Device wall clock in ns (globaltimer); 0 in the host emulation.
SPEX_HD i64 spex_wall_ns() {
#if SPEX_DEVICE_PASS
  u64 t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return static_cast<i64>(t);
#else
  return 0;
#endif
}

// ------------------------------------------------------- paged tree-KV store
// A thought's K/V rows live in pages of kKvPage tokens (ctl_state.h). Each
// node carries a hold count: its own pin (it may still get children: cleared
// when it is pruned, when its REBASE layer has been expanded, or when its
// query finishes; terminal thoughts never get one), one per child that still
// holds pages, and one while its decode stream is in the engine (released at
// the stream's completion, after the completion boundary's PRM batch is
// recorded, or when a staged stream is erased). The last release pushes the
// node's pages to the free ring and releases the parent's child hold.
//
// Reuse needs no fence against the forward, which lags behind the control:
// the policy and PRM forwards each run the schedule entries in order on one
// stream, a freed node is read only by entries recorded before it died, and
// the thought that reuses its pages writes them only in entries recorded
// after its spawn (tree.cpp:119-141 prune, executor.cpp:587-656 layers,
// executor.cpp:234-336 finish define when a thought can have no reader).
SPEX_HD bool kv_on(const Cfg& c, int q) { return c.kv_pages > 0 && q_owned(c, q); }

SPEX_HDNI void kv_release(Run* R, int q, u32 node) {
  const Cfg& c = R->cfg;
  const u32 b = static_cast<u32>(q) * static_cast<u32>(c.node_cap);
  while (node != kNoNode) {
    const int old = atomic_add_int(&R->n_kvh[b + node], -1);
    if (old > 1) return;
    if (old < 1) {
      set_err(R, ERR_INTERNAL, q, node);  // hold underflow
      return;
    }
    if (node == 0) return;  // root prompt pages are static
    const i64 pt = R->n_kvbase[b + node];
    if (pt >= 0) {
      const int np = kv_pages_of(R->n_tokens[b + node]);
      const i64 pos = atomic_add_i64(&R->g->kv_free_tail, np);
      for (int k = 0; k < np; ++k) R->kv_free[(pos + k) % c.kv_pages] = R->kv_pt[pt + k];
      atomic_add_i64(&R->g->kv_live, -np);
      atomic_add_i64(&R->g->kv_freed, np);
    }
    node = R->n_parent[b + node];
  }
}

// Drop the node's own pin (it can get no more children).
SPEX_HD void kv_unpin(Run* R, int q, u32 node) {
  const u32 i = static_cast<u32>(q) * static_cast<u32>(R->cfg.node_cap) + node;
  if (!kv_on(R->cfg, q) || !(R->n_flags[i] & NF_KV_SELF)) return;
  R->n_flags[i] &= static_cast<u16>(~NF_KV_SELF);
  kv_release(R, q, node);
}

struct QC {
  Run* R;
  int q;
  u32 base;  // q * node_cap
  QueryRun* qr;
  Item* it;
  const Cfg* c;
  // per-warp scratch (sized node_cap + 64)
  u32* stack;
  int* sv;       // overlay visits
  double* sval;  // overlay values
  int* snch;     // overlay child counts
  double* dbl;   // 3 * (node_cap + 64) doubles
  int* ints;     // 3 * (node_cap + 64) ints
};

SPEX_HD int scratch_stride(const Cfg& c) { return c.node_cap + 64; }

SPEX_HD QC make_qc(Run* R, int q, Item* it, int slot) {
  QC x;
  x.R = R;
  x.q = q;
  x.base = static_cast<u32>(q) * static_cast<u32>(R->cfg.node_cap);
  x.qr = &R->qs[q];
  x.it = it;
  x.c = &R->cfg;
  const int S = scratch_stride(R->cfg);
  x.stack = R->sp_stack + static_cast<i64>(slot) * S;
  x.sv = R->sp_visits + static_cast<i64>(slot) * S;
  x.sval = R->sp_value + static_cast<i64>(slot) * S;
  x.snch = R->sp_nchild + static_cast<i64>(slot) * S;
  x.dbl = R->sp_dbl + static_cast<i64>(slot) * 3 * S;
  x.ints = R->sp_int + static_cast<i64>(slot) * 3 * S;
  return x;
}

#define NI(x, id) ((x).base + (id))

SPEX_HD u8 st_of(const QC& x, u32 id) { return x.R->n_status[NI(x, id)]; }
SPEX_HD u16 fl_of(const QC& x, u32 id) { return x.R->n_flags[NI(x, id)]; }
SPEX_HD bool has_fl(const QC& x, u32 id, u16 f) { return (x.R->n_flags[NI(x, id)] & f) != 0; }
SPEX_HD void set_fl(const QC& x, u32 id, u16 f) { x.R->n_flags[NI(x, id)] |= f; }
SPEX_HD void clr_fl(const QC& x, u32 id, u16 f) { x.R->n_flags[NI(x, id)] &= static_cast<u16>(~f); }
SPEX_HD void touch(const QC& x) { x.qr->version += 1; }

SPEX_HDNI Rec* new_rec(const QC& x, u8 kind, u32 node) {
  if (!x.c->trace) return nullptr;
  Item* it = x.it;
  if (it->nrec >= it->rec_cap) {
    set_err(x.R, ERR_CAP_STAGE, x.q, node);
    return nullptr;
  }
  Rec* r = &it->rec[it->nrec++];
  r->t = x.R->g->now;
  r->x = 0.0;
  r->y = 0;
  r->q = x.q;
  r->node = node;
  r->a = r->b = r->c = 0;
  r->kind = kind;
  r->flags = 0;
  r->pad = 0;
  return r;
}

// ------------------------------------------------------------------ tree.cpp
// tree.cpp:23-45
SPEX_HD bool transition_legal(u8 from, u8 to) {
  if (to == kPruned) return from != kPruned;
  switch (from) {
    case kPendingExpansion: return to == kExpanding;
    case kExpanding: return to == kAwaitingReward;
    case kAwaitingReward: return to == kCommitted || to == kSpeculativeDone || to == kTerminalAnswer;
    case kSpeculative: return to == kSpeculativeDone || to == kExpanding || to == kAwaitingReward;
    case kSpeculativeDone: return to == kCommitted || to == kTerminalAnswer;
    default: return false;
  }
}

// tree.cpp:143-150 (+ incremental terminal_answer_count / live_cache_tokens)
SPEX_HD void set_status(const QC& x, u32 id, u8 to) {
  u8 from = st_of(x, id);
  if (!transition_legal(from, to)) {
    set_err(x.R, ERR_ILLEGAL_TRANSITION, x.q, id);
    return;
  }
  if (from == kTerminalAnswer) x.qr->terminal_count -= 1;
  if (to == kTerminalAnswer) x.qr->terminal_count += 1;
  x.R->n_status[NI(x, id)] = to;
  touch(x);
}

SPEX_HD bool counted_live(const QC& x, u32 id) {
  // executor.cpp:662-672: not pruned and (root or generated)
  return st_of(x, id) != kPruned && (id == 0 || has_fl(x, id, NF_GEN_DONE));
}

// tree.cpp:75-94
SPEX_HDNI u32 add_node(const QC& x, u32 parent, int token_len, bool spec) {
  Run* R = x.R;
  QueryRun* qr = x.qr;
  if (parent >= static_cast<u32>(qr->nnodes)) {
    set_err(R, ERR_UNKNOWN_PARENT, x.q, parent);
    return kNoNode;
  }
  if (st_of(x, parent) == kPruned) {
    set_err(R, ERR_PARENT_PRUNED, x.q, parent);
    return kNoNode;
  }
  if (token_len <= 0) {
    set_err(R, ERR_INVALID_ARGUMENT, x.q, parent);
    return kNoNode;
  }
  if (qr->nnodes >= x.c->node_cap) {
    set_err(R, ERR_CAP_NODES, x.q, parent);
    return kNoNode;
  }
  u32 id = static_cast<u32>(qr->nnodes++);
  u32 pi = NI(x, parent), ni = NI(x, id);
  int slot = R->n_nchildren[pi];
  R->n_parent[ni] = parent;
  R->n_depth[ni] = R->n_depth[pi] + 1;
  R->n_slot[ni] = slot;
  R->n_tokens[ni] = token_len;
  R->n_status[ni] = spec ? kSpeculative : kExpanding;
  const u64 h = extend_hash(R->n_hash[pi], slot);
  // the oracle's two path walks, memoised per node: id's path is golden iff
  // its parent's is and id's own draw passes (on_golden_path, sim.cpp:139-144);
  // "deep" is the draw of the depth-1 ancestor (deep_dominant, sim.cpp:118-123)
  const u16 pf = R->n_flags[pi];
  const bool golden = (pf & NF_GOLDEN_PATH) != 0 && uniform01(h, kSaltGolden) < x.c->golden_density;
  const bool deep = R->n_depth[pi] == 0 ? uniform01(h, kSaltDeep) < x.c->skew : (pf & NF_DEEP) != 0;
  R->n_flags[ni] =
      static_cast<u16>((spec ? NF_SPEC_ORIGIN : 0) | (golden ? NF_GOLDEN_PATH : 0) | (deep ? NF_DEEP : 0));
  R->n_reward[ni] = 0.0;
  R->n_value[ni] = 0.0;
  R->n_visits[ni] = 0;
  R->n_hash[ni] = h;
  R->n_first_child[ni] = kNoNode;
  R->n_last_child[ni] = kNoNode;
  R->n_next_sib[ni] = kNoNode;
  R->n_nchildren[ni] = 0;
  R->n_pred[ni] = 0;
  R->n_stream[ni] = -1;
  R->n_ready[ni] = 0;
  R->n_refc[ni] = 0;
  if (R->n_last_child[pi] == kNoNode)
    R->n_first_child[pi] = id;
  else
    R->n_next_sib[NI(x, R->n_last_child[pi])] = id;
  R->n_last_child[pi] = id;
  R->n_nchildren[pi] = slot + 1;
  touch(x);
  return id;
}

// tree.cpp:102-117
SPEX_HDNI void promote(const QC& x, u32 id) {
  u8 s = st_of(x, id);
  if (s != kSpeculative && s != kSpeculativeDone) {
    set_err(x.R, ERR_NOT_SPECULATIVE, x.q, id);
    return;
  }
  u8 to;
  if (s == kSpeculativeDone)
    to = has_fl(x, id, NF_TERMINAL) ? kTerminalAnswer : kCommitted;
  else if (has_fl(x, id, NF_GEN_DONE))
    to = kAwaitingReward;
  else
    to = kExpanding;
  set_status(x, id, to);
}

// tree.cpp:119-141 (iterative DFS; the frontier_ filter is unused by the executor)
SPEX_HDNI int prune_subtree(const QC& x, u32 id) {
  u32* stack = x.stack;
  Run* R = x.R;
  int pruned = 0;
  int sp = 0;
  stack[sp++] = id;
  while (sp > 0) {
    u32 cur = stack[--sp];
    u32 ci = NI(x, cur);
    if (R->n_status[ci] != kPruned) {
      if (counted_live(x, cur)) x.qr->live_cache -= R->n_tokens[ci];
      if (R->n_status[ci] == kTerminalAnswer) x.qr->terminal_count -= 1;
      R->n_status[ci] = kPruned;
      kv_unpin(R, x.q, cur);
      ++pruned;
    }
    // children are pushed in slot order and popped in reverse, as in the reference;
    // the count and the final state do not depend on the visiting order.
    for (u32 c = R->n_first_child[ci]; c != kNoNode; c = R->n_next_sib[NI(x, c)]) {
      if (sp >= x.c->node_cap) {
        set_err(R, ERR_INTERNAL, x.q, cur);
        return pruned;
      }
      stack[sp++] = c;
    }
  }
  touch(x);
  return pruned;
}

// ------------------------------------------------------- content oracle (sim.cpp)
// sim.cpp:112-115
SPEX_HDNI int oracle_token_len(const Cfg& c, u64 child_hash) {
  return lognormal_tokens(child_hash, kSaltTokens, c.token_mu, c.token_sigma, c.token_min,
                          c.token_max);
}

// sim.cpp:117-137
SPEX_HDNI bool oracle_is_terminal(const QC& x, u32 id) {
  Run* R = x.R;
  const Cfg& c = *x.c;
  int depth = R->n_depth[NI(x, id)];
  if (depth == 0) return false;
  const bool deep = (R->n_flags[NI(x, id)] & NF_DEEP) != 0;  // memoised by add_node
  int lo = deep ? c.deep_min : c.shallow_min;
  int hi = deep ? c.deep_max : c.shallow_max;
  double p = deep ? c.deep_p : c.shallow_p;
  if (hi > c.max_depth) hi = c.max_depth;
  if (depth >= hi) return true;
  if (depth < lo) return false;
  return uniform01(R->n_hash[NI(x, id)], kSaltTerminal) < p;
}

// sim.cpp:139-152
SPEX_HDNI double oracle_reward(const QC& x, u32 id) {
  Run* R = x.R;
  const Cfg& c = *x.c;
  // the reference walks id's path to the root testing each node's golden draw
  // (on_golden_path, sim.cpp:139-144); add_node memoised the walk in NF_GOLDEN_PATH
  const bool golden = (R->n_flags[NI(x, id)] & NF_GOLDEN_PATH) != 0;
  double r = golden ? c.reward_on : c.reward_off;
  if (c.noise_sigma > 0.0) r += c.noise_sigma * normal01(R->n_hash[NI(x, id)], kSaltNoise);
  if (r < 0.0) r = 0.0;
  if (1.0 < r) r = 1.0;
  return r;
}

// sim.cpp:154-169 (labels are indices; "a" + idx is formatted on the host)
SPEX_HD int golden_label_of(const Cfg& c, u64 query_seed) {
  return static_cast<int>(splitmix64(query_seed ^ kSaltLabel) %
                          static_cast<u64>(c.answer_alphabet));
}

SPEX_HDNI int oracle_answer_label(const QC& x, u32 id) {
  Run* R = x.R;
  const Cfg& c = *x.c;
  double p = c.correct_base - c.correct_slope * R->n_depth[NI(x, id)];
  if (p < c.correct_floor) p = c.correct_floor;
  else if (c.correct_base < p) p = c.correct_base;
  u64 h = R->n_hash[NI(x, id)];
  if (uniform01(h, kSaltCorrect) < p) return x.qr->golden;
  u64 alpha = static_cast<u64>(c.answer_alphabet);
  u64 gold = splitmix64(x.qr->seed ^ kSaltLabel) % alpha;
  u64 off = 1 + splitmix64(h ^ kSaltLabel) % (alpha - 1);
  return static_cast<int>((gold + off) % alpha);
}

// RewardOracle (sim.cpp:112-169) over a node given by its path hashes
// path[0..depth) (its depth-1 ancestor .. itself): terminality (depth windows
// by the depth-1 ancestor's draw), reward (golden path + clamped noise) and
// answer label. Shared by the spex_content_* hooks (device and emulation);
// the search itself memoises the same draws per node (add_node, oracle_*).
template <class W>
SPEX_HD void content_eval(const u64* path, int depth, u64 query_seed, int max_depth, const W& wl, int* terminal,
                          double* reward, int* label) {
  const u64 own = depth > 0 ? path[depth - 1] : splitmix64(query_seed);  // the root's hash (tree.cpp:57)
  // is_terminal (sim.cpp:127-139) with deep_dominant (:117-125)
  if (depth == 0) {
    *terminal = 0;
  } else {
    const bool deep = uniform01(path[0], kSaltDeep) < wl.skew;
    const int lo = deep ? wl.deep_min : wl.shallow_min;
    int hi = deep ? wl.deep_max : wl.shallow_max;
    const double p = deep ? wl.deep_p : wl.shallow_p;
    if (hi > max_depth) hi = max_depth;
    *terminal = depth >= hi ? 1 : depth < lo ? 0 : (uniform01(path[depth - 1], kSaltTerminal) < p ? 1 : 0);
  }
  // on_golden_path (:141-146) and reward (:148-154)
  bool golden = true;
  for (int i = depth - 1; i >= 0 && golden; --i) golden = uniform01(path[i], kSaltGolden) < wl.golden_density;
  double r = golden ? wl.reward_on : wl.reward_off;
  if (wl.noise_sigma > 0.0) r += wl.noise_sigma * normal01(own, kSaltNoise);
  *reward = r < 0.0 ? 0.0 : (r > 1.0 ? 1.0 : r);
  // answer_label (:162-169)
  double pc = wl.correct_base - wl.correct_slope * depth;
  if (pc < wl.correct_floor) pc = wl.correct_floor;
  else if (wl.correct_base < pc) pc = wl.correct_base;
  const u64 h = own;
  const u64 alpha = static_cast<u64>(wl.answer_alphabet);
  const u64 gold = splitmix64(query_seed ^ kSaltLabel) % alpha;
  if (uniform01(h, kSaltCorrect) < pc) {
    *label = static_cast<int>(gold);
  } else {
    const u64 off = 1 + splitmix64(h ^ kSaltLabel) % (alpha - 1);
    *label = static_cast<int>((gold + off) % alpha);
  }
}

// -------------------------------------------------------------- policy.cpp
SPEX_HD double log_int(const Run* R, int n) {
  if (n >= 1 && n < R->log_tab_n) return R->log_tab[n];
  return glibc::log(static_cast<double>(n));
}

// policy.cpp:25-30
SPEX_HD double ucb_score(const Run* R, double value, int cv, int pv, double c) {
  return value + c * sqrt(log_int(R, pv) / cv);
}

// policy.cpp:32-51
SPEX_HDNI u32 ucb_select(const QC& x, u32 id) {
  Run* R = x.R;
  u32 pi = NI(x, id);
  bool any = false;
  for (u32 c = R->n_first_child[pi]; c != kNoNode; c = R->n_next_sib[NI(x, c)]) {
    if (st_of(x, c) == kPruned) continue;
    any = true;
    if (R->n_visits[NI(x, c)] == 0) return c;
  }
  if (!any) {
    set_err(R, ERR_NO_CHILDREN, x.q, id);
    return kNoNode;
  }
  int pv = R->n_visits[pi];
  u32 best = kNoNode;
  double best_score = 0.0;
  for (u32 c = R->n_first_child[pi]; c != kNoNode; c = R->n_next_sib[NI(x, c)]) {
    if (st_of(x, c) == kPruned) continue;
    int cv = R->n_visits[NI(x, c)];
    if (cv <= 0 || pv <= 0) {
      set_err(R, ERR_ZERO_VISITS, x.q, id);
      return kNoNode;
    }
    double s = ucb_score(R, R->n_value[NI(x, c)], cv, pv, x.c->exploration_c);
    if (best == kNoNode || s > best_score) {
      best = c;
      best_score = s;
    }
  }
  return best;
}

// policy.cpp:53-63
SPEX_HDNI void backpropagate(const QC& x, u32 leaf, double reward) {
  Run* R = x.R;
  u8 s = st_of(x, leaf);
  if (s != kCommitted && s != kTerminalAnswer) {
    set_err(R, ERR_INVALID_ARGUMENT, x.q, leaf);
    return;
  }
  for (u32 cur = leaf; cur != kNoNode; cur = R->n_parent[NI(x, cur)]) {
    u32 ci = NI(x, cur);
    R->n_visits[ci] += 1;
    R->n_value[ci] += (reward - R->n_value[ci]) / R->n_visits[ci];
  }
  touch(x);
}

// policy.cpp:65-118. `w` and `quota` are scratch of length n.
SPEX_HDNI bool rebase_widths(Run* R, int q, const double* __restrict__ rewards, int n, int budget,
                           double temperature, bool sum_preserving, int* __restrict__ widths,
                           double* __restrict__ w, double* __restrict__ quota, int* __restrict__ order) {
  if (n <= 0) {
    set_err(R, ERR_EMPTY_REWARDS, q, kNoNode);
    return false;
  }
  if (budget < 0 || temperature <= 0.0) {
    set_err(R, ERR_INVALID_ARGUMENT, q, kNoNode);
    return false;
  }
  double rmax = rewards[0];
  for (int i = 1; i < n; ++i)
    if (rmax < rewards[i]) rmax = rewards[i];
  double total = 0.0;
  for (int i = 0; i < n; ++i) {
    w[i] = glibc::exp((rewards[i] - rmax) / temperature);
    total += w[i];
  }
  for (int i = 0; i < n; ++i) quota[i] = budget * w[i] / total;
  if (!sum_preserving) {
    bool all_zero = true;
    for (int i = 0; i < n; ++i) {
      widths[i] = static_cast<int>(round(quota[i]));
      if (widths[i] != 0) all_zero = false;
    }
    if (all_zero && budget > 0) {
      int best = 0;
      for (int i = 1; i < n; ++i)
        if (rewards[i] > rewards[best]) best = i;
      widths[best] = 1;
    }
    return true;
  }
  int assigned = 0;
  for (int i = 0; i < n; ++i) {
    widths[i] = static_cast<int>(floor(quota[i]));
    w[i] = quota[i] - widths[i];  // frac (w reused)
    assigned += widths[i];
  }
  int leftover = budget - assigned;
  if (leftover > 0) {
    // stable sort of indices by frac descending (insertion sort is stable)
    for (int i = 0; i < n; ++i) {
      int v = i;
      int j = i - 1;
      while (j >= 0 && w[order[j]] < w[v]) {
        order[j + 1] = order[j];
        --j;
      }
      order[j + 1] = v;
    }
    int k = 0;
    while (leftover > 0) {
      widths[order[k % n]] += 1;
      --leftover;
      ++k;
    }
  }
  return true;
}

// ------------------------------------------------------------- budget.cpp
// budget.cpp:98-100
SPEX_HD void update_hit_rate(QueryRun* qr, bool hit, double alpha) {
  qr->hit_ema = (1.0 - alpha) * qr->hit_ema + alpha * (hit ? 1.0 : 0.0);
}

// --------------------------------------------------------- speculation.cpp
// speculation.cpp:253-263 (histograms are kept clamped, executor.cpp:29,311-313)
SPEX_HDNI void record_outcome(const QC& x, u32 node, bool hit, int distance) {
  u16 f = fl_of(x, node);
  bool known = (f & (NF_LEDGER_ACTIVE | NF_LEDGER_COMPLETED | NF_HAS_PRED)) != 0;
  if (!known || (f & NF_LEDGER_RESOLVED)) {
    set_err(x.R, ERR_UNKNOWN_SPECULATION, x.q, node);
    return;
  }
  set_fl(x, node, NF_LEDGER_RESOLVED);
  if (f & NF_LEDGER_ACTIVE) {
    clr_fl(x, node, NF_LEDGER_ACTIVE);
    x.qr->n_active_exp -= 1;
  }
  clr_fl(x, node, NF_LEDGER_COMPLETED);
  int d = distance < 1 ? 1 : (distance > kMaxTracked ? kMaxTracked : distance);
  if (hit)
    x.qr->hits[d] += 1;
  else
    x.qr->misses[d] += 1;
  touch(x);
}

// --------------------------------------------------------- termination.cpp
// termination.cpp:7-13
SPEX_HD void tally_record(const QC& x, int label, double weight) {
  QueryRun* qr = x.qr;
  if (weight < 0.0) {
    set_err(x.R, ERR_NEGATIVE_WEIGHT, x.q, kNoNode);
    return;
  }
  QueryTally* ta = &x.R->q_tally[x.q];
  if (ta->count[label] == 0) qr->n_labels += 1;
  ta->count[label] += 1;
  ta->w[label] += weight;
  qr->n_answers += 1;
}

// termination.cpp:15-23 — labels iterate in std::map (lexicographic string) order
SPEX_HD int leading_label(const QC& x) {
  const QueryTally* ta = &x.R->q_tally[x.q];
  int best = -1;
  for (int r = 0; r < x.c->answer_alphabet; ++r) {
    int l = x.c->lex_order[r];
    if (ta->count[l] == 0) continue;
    if (best < 0 || ta->w[l] > ta->w[best]) best = l;
  }
  return best;
}

// AnswerTally::should_terminate (termination.cpp:30-48) over a tally whose
// n_slots label slots are visited in std::map (lexicographic) order; slot r's
// (answer count, weight sum) come from get(r, &count, &w), empty slots skipped.
// Shared by the control kernel and the spex_termination_should_terminate hook.
template <class F>
SPEX_HD bool tally_should_terminate(int n_total, int n_labels, int n_slots, F get, int min_answers, double alpha) {
  if (n_total < min_answers || n_labels == 0) return false;
  if (n_labels < 2) return true;
  int c1 = 0, c2 = 0;
  double w1 = 0.0, w2 = 0.0;
  bool has1 = false, has2 = false;
  for (int r = 0; r < n_slots; ++r) {
    int cnt;
    double w;
    get(r, &cnt, &w);
    if (cnt == 0) continue;
    if (!has1 || w > w1) {
      c2 = c1, w2 = w1, has2 = has1;
      c1 = cnt, w1 = w, has1 = true;
    } else if (!has2 || w > w2) {
      c2 = cnt, w2 = w, has2 = true;
    }
  }
  const double margin = w1 - w2;
  const double avg_second = c2 > 0 ? w2 / c2 : 0.0;
  return margin > alpha * avg_second;
}

SPEX_HDNI bool should_terminate(const QC& x, int min_answers, double alpha) {
  const QueryRun* qr = x.qr;
  const QueryTally* ta = &x.R->q_tally[x.q];
  const int* order = x.c->lex_order;
  return tally_should_terminate(
      qr->n_answers, qr->n_labels, x.c->answer_alphabet,
      [&](int r, int* cnt, double* w) {
        const int l = order[r];
        *cnt = ta->count[l];
        *w = ta->w[l];
      },
      min_answers, alpha);
}

// ============================================================ executor.cpp
// Streams created by this item carry local ordinals until commit.
SPEX_HD int stream_done_tokens(const QC& x, int sref) {
  if (sref >= 0) {
    // DecodeEngine::done_tokens (sim.cpp:251-257): 0 unless active/staged
    u8 s = x.R->st_state[sref];
    return (s == ST_ACTIVE || s == ST_STAGED) ? x.R->st_done[sref] : 0;
  }
  return 0;  // staged in this very step: nothing generated yet
}

// executor.cpp:124-164
SPEX_HDNI u32 spawn_child(const QC& x, u32 parent, bool spec, int dist) {
  Run* R = x.R;
  u32 pi = NI(x, parent);
  int slot = R->n_nchildren[pi];
  u64 child_hash = extend_hash(R->n_hash[pi], slot);
  int tokens = oracle_token_len(*x.c, child_hash);
  u32 id = add_node(x, parent, tokens, spec);
  if (id == kNoNode) return id;
  bool term = oracle_is_terminal(x, id);
  if (term) set_fl(x, id, NF_TERMINAL);
  R->n_kvbase[NI(x, id)] = -1;
  if (kv_on(*x.c, x.q)) {
    // own pin (non-terminal) + the stream's; the child holds its parent
    R->n_kvh[NI(x, id)] = term ? 1 : 2;
    if (!term) set_fl(x, id, NF_KV_SELF);
    atomic_add_int(&R->n_kvh[pi], 1);
  }
  if (Rec* r = new_rec(x, EV_NODE, id)) {
    r->a = static_cast<int>(parent);
    r->b = slot;
    r->c = tokens;
    r->flags = (spec ? RF_SPEC : 0) | (term ? RF_TERMINAL : 0);
  }
  Item* it = x.it;
  if (it->nspw >= it->spw_cap) {
    set_err(R, ERR_CAP_STAGE, x.q, id);
    return kNoNode;
  }
  int local = it->nspw++;
  it->spw[local] = SpawnRec{x.q, id, tokens, 0};
  if (Rec* r = new_rec(x, EV_REQ, id)) {
    r->a = local;
    r->b = dist;
    r->flags = (spec ? RF_SPEC : 0) | RF_LOCAL_SID;
  }
  R->n_stream[NI(x, id)] = -2 - local;
  it->sdelta += 1;
  if (spec) {
    set_fl(x, id, NF_LEDGER_ACTIVE | NF_HAS_PRED);
    x.qr->n_active_exp += 1;
    R->n_pred[NI(x, id)] = dist;
  }
  return id;
}

// executor.cpp:168-187
SPEX_HDNI void do_promote(const QC& x, u32 node) {
  Run* R = x.R;
  u32 ni = NI(x, node);
  if (!has_fl(x, node, NF_HAS_PRED)) {
    set_err(R, ERR_INTERNAL, x.q, node);  // predicted_distance.at() would throw
    return;
  }
  int dist = R->n_pred[ni];
  i64 ready;
  if (has_fl(x, node, NF_GEN_DONE)) {
    ready = R->n_tokens[ni];
  } else {
    int sref = R->n_stream[ni];
    if (sref == -1) {
      set_err(R, ERR_INTERNAL, x.q, node);  // stream_of.at() would throw
      return;
    }
    ready = stream_done_tokens(x, sref);
  }
  promote(x, node);
  R->n_ready[ni] = ready;
  set_fl(x, node, NF_HAS_READY);
  record_outcome(x, node, true, dist);
  update_hit_rate(x.qr, true, x.c->ema_alpha);
  if (st_of(x, node) == kAwaitingReward) x.qr->pending_rewards += 1;
  if (Rec* r = new_rec(x, EV_PROMOTE, node)) {
    r->y = static_cast<u64>(ready);
    r->a = dist;
  }
}

// executor.cpp:192-200 with DecodeEngine::cancel (sim.cpp:217-233)
SPEX_HDNI void cancel_stream(const QC& x, u32 node) {
  Run* R = x.R;
  u32 ni = NI(x, node);
  int sref = R->n_stream[ni];
  if (sref == -1) return;
  if (sref <= -2) {
    // staged in this step: erased with no completion record
    x.it->spw[-2 - sref].cancelled = 1;
    x.it->sdelta -= 1;
    R->n_stream[ni] = -1;
    if (kv_on(*x.c, x.q)) kv_release(R, x.q, node);  // the stream never ran
    return;
  }
  u8 s = R->st_state[sref];
  if (s == ST_ACTIVE) {
    if (!R->st_cancel[sref]) {
      R->st_cancel[sref] = 1;
      R->st_rem[sref] = 1;
    }
    return;  // stays mapped until its farewell completion
  }
  if (s == ST_STAGED) {
    R->st_state[sref] = ST_GONE;
    x.it->sdelta -= 1;
    R->n_stream[ni] = -1;
    if (kv_on(*x.c, x.q)) kv_release(R, x.q, node);  // erased before it started
  }
}

SPEX_HDNI void finish_query(const QC& x, bool early);

// executor.cpp:206-232
SPEX_HDNI void record_answer_event(const QC& x, u32 node, double r) {
  int label = oracle_answer_label(x, node);
  tally_record(x, label, r);
  x.qr->recorded += 1;
  if (Rec* rec = new_rec(x, EV_ANSWER, node)) {
    rec->a = label;
    rec->x = r;
    rec->flags = label == x.qr->golden ? RF_CORRECT : 0;
  }
  if (x.qr->recorded >= x.c->target_answers) {
    finish_query(x, false);
    return;
  }
  if (x.c->t3 && should_terminate(x, x.c->min_answers, x.c->term_alpha)) finish_query(x, true);
}

// executor.cpp:234-336 (the finished_count / admission / drain tail runs at commit)
SPEX_HDNI void finish_query(const QC& x, bool early) {
  Run* R = x.R;
  QueryRun* qr = x.qr;
  qr->finished = 1;
  qr->early = early ? 1 : 0;
  qr->finish_time = R->g->now;
  R->q_finish_ns[x.q] = spex_wall_ns();
  x.it->fin = 1;
  touch(x);
  if (early) {
    if (Rec* r = new_rec(x, EV_TERMINATE, kNoNode)) {
      r->a = leading_label(x);
      r->b = qr->recorded;
    }
  }
  const u32 n = static_cast<u32>(qr->nnodes);
  for (u32 id = 1; id < n; ++id) {
    switch (st_of(x, id)) {
      case kSpeculative:
        if (!has_fl(x, id, NF_GEN_DONE)) {
          qr->cancelled_inflight += 1;
          if (has_fl(x, id, NF_LEDGER_ACTIVE)) {
            clr_fl(x, id, NF_LEDGER_ACTIVE);
            qr->n_active_exp -= 1;
          }
          cancel_stream(x, id);
        } else {
          record_outcome(x, id, false, R->n_pred[NI(x, id)]);
          update_hit_rate(qr, false, x.c->ema_alpha);
        }
        break;
      case kSpeculativeDone:
        record_outcome(x, id, false, R->n_pred[NI(x, id)]);
        update_hit_rate(qr, false, x.c->ema_alpha);
        break;
      case kExpanding:
        cancel_stream(x, id);
        break;
      default:
        break;
    }
  }
  // tombstone everything outside the final answer set
  for (u32 id = 1; id < n; ++id) {
    u8 st = st_of(x, id);
    if (st == kCommitted || st == kTerminalAnswer || st == kPruned) continue;
    int cnt = prune_subtree(x, id);
    if (Rec* r = new_rec(x, EV_PRUNE, id)) r->a = cnt;
  }
  // the finished tree gets no more children: its thoughts' pages go as soon
  // as their streams and scoring are done
  for (u32 id = 0; id < n; ++id) kv_unpin(R, x.q, id);
  // conservation accounting
  for (u32 id = 1; id < n; ++id) {
    u32 ni = NI(x, id);
    u8 st = R->n_status[ni];
    if (st == kCommitted || st == kTerminalAnswer) {
      i64 ready = has_fl(x, id, NF_HAS_READY) ? R->n_ready[ni] : 0;
      qr->reused += ready;
      qr->committed += R->n_tokens[ni] - ready;
    } else if (has_fl(x, id, NF_GEN_DONE)) {
      qr->wasted += R->n_tokens[ni];
    }
  }
  int label = qr->n_answers > 0 ? leading_label(x) : -1;
  bool correct = label >= 0 && label == qr->golden;
  qr->correct = correct ? 1 : 0;
  if (Rec* r = new_rec(x, EV_QUERY_DONE, kNoNode)) {
    r->a = label;
    r->b = qr->recorded;
    r->flags = (correct ? RF_CORRECT : 0) | (early ? RF_EARLY : 0);
  }
}

}  // namespace spex
