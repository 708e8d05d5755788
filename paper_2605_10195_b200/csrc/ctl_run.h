// ctl_run.h — the frontier-expansion main loop (executor.cpp:785-807) as a
// sequence of block-parallel phases:
//
//   engine epoch   DecodeEngine::advance (sim.cpp:305-384): joins, roofline step
//                  cost from incrementally maintained prefix-shared KV tokens,
//                  bulk token advance, ordered completion list
//   completions    on_stream_done per finished stream (queries in parallel,
//                  streams of one query in rank rounds)
//   reward event   on_reward for the FIFO head
//   follow-ups     advance_dfs / advance_rest / advance_layer for every query
//                  whose state changed (consumer_step_followups, executor.cpp:746-763)
//   scheduling     capacity, T2 budget split (allocate_budgets, budget.cpp:45-96)
//                  and speculative planning (scheduling_round, executor.cpp:705-740)
//   commit         exclusive scans place every item's records, new streams and
//                  reward events in the reference's sequential order
//
// The template parameter EX is the execution context: DevExec (one CTA of the
// persistent kernel, ctl_kernel.cu) or HostExec (single thread, test-only
// emulation build).
#pragma once

#include "ctl_drivers.h"
#include "model.h"

namespace spex {

constexpr double kInf = HUGE_VAL;


// shared int scratch (ex.sm, 1032 ints): [0, nthr] slow scan, [0, nwarp) reductions,
// then disjoint regions for the fast scan, commit totals and query collection
constexpr int kSmScan = 560;     // 33 ints
constexpr int kSmCommit = 600;   // 8 ints
constexpr int kSmCollect = 640;  // 32 ints
enum { CY_ENGINE = 0, CY_FINS, CY_REWARD, CY_FOLLOW, CY_SCHED, CY_TOTAL, CY_ITEMS, CY_COMMIT };
#define SPEX_TIMED(ex, R, slot, stmt)                              \
  do {                                                             \
    i64 t0_ = (ex).tid == 0 ? spex_clock() : 0;                    \
    stmt;                                                          \
    if ((ex).tid == 0) (R)->g->cyc[slot] += spex_clock() - t0_;    \
  } while (0)

struct HostExec {
  int tid = 0, nthr = 1, warp = 0, nwarp = 1, lane = 0, lanes = 1;
  int* sm = nullptr;        // scan scratch (nthr + 2 ints)
  double* smd = nullptr;    // reduction scratch
  i64* sml = nullptr;
  void sync() {}
};

// ------------------------------------------------------------ block primitives
template <class EX>
SPEX_HDNI void ex_scan(EX& ex, int* a, int n, int* total) {
#if SPEX_DEVICE_PASS
  if (n <= ex.nthr) {
    // one element per thread: warp shuffle scans, warp totals in shared memory
    int* ws = ex.sm + kSmScan;
    const int v = ex.tid < n ? a[ex.tid] : 0;
    int incl = v;
    for (int off = 1; off < 32; off <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, off);
      if (ex.lane >= off) incl += y;
    }
    if (ex.lane == 31) ws[ex.warp] = incl;
    ex.sync();
    // every warp reduces the warp totals itself (lane w holds warp w's):
    // its exclusive offset and the grand total, no second barrier
    const int wv = ex.lane < ex.nwarp ? ws[ex.lane] : 0;
    int before = ex.lane < ex.warp ? wv : 0, all = wv;
    for (int off = 16; off > 0; off >>= 1) {
      before += __shfl_xor_sync(0xffffffffu, before, off);
      all += __shfl_xor_sync(0xffffffffu, all, off);
    }
    if (ex.tid < n) a[ex.tid] = before + incl - v;
    *total = all;
    ex.sync();
    return;
  }
  const int per = (n + ex.nthr - 1) / ex.nthr;
  const int lo = ex.tid * per;
  const int hi = lo + per < n ? lo + per : n;
  int s = 0;
  for (int i = lo; i < hi; ++i) s += a[i];
  ex.sm[ex.tid] = s;
  ex.sync();
  if (ex.warp == 0) {
    const int chunk = (ex.nthr + 31) / 32;
    const int b0 = ex.lane * chunk;
    int acc = 0;
    for (int j = 0; j < chunk; ++j)
      if (b0 + j < ex.nthr) acc += ex.sm[b0 + j];
    int incl = acc;
    for (int off = 1; off < 32; off <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, incl, off);
      if (ex.lane >= off) incl += y;
    }
    int run = incl - acc;
    for (int j = 0; j < chunk; ++j)
      if (b0 + j < ex.nthr) {
        int v = ex.sm[b0 + j];
        ex.sm[b0 + j] = run;
        run += v;
      }
    if (ex.lane == 31) ex.sm[ex.nthr] = incl;
  }
  ex.sync();
  int run = ex.sm[ex.tid];
  for (int i = lo; i < hi; ++i) {
    int v = a[i];
    a[i] = run;
    run += v;
  }
  *total = ex.sm[ex.nthr];
  ex.sync();
#else
  int run = 0;
  for (int i = 0; i < n; ++i) {
    int v = a[i];
    a[i] = run;
    run += v;
  }
  *total = run;
#endif
}

template <class EX>
SPEX_HDNI int ex_min_int(EX& ex, int v) {
#if SPEX_DEVICE_PASS
  for (int off = 16; off > 0; off >>= 1) {
    int y = __shfl_xor_sync(0xffffffffu, v, off);
    v = y < v ? y : v;
  }
  if (ex.lane == 0) ex.sm[ex.warp] = v;
  ex.sync();
  int r = ex.lane < ex.nwarp ? ex.sm[ex.lane] : ex.sm[0];
  for (int off = 16; off > 0; off >>= 1) {
    const int y = __shfl_xor_sync(0xffffffffu, r, off);
    r = y < r ? y : r;
  }
  ex.sync();
  return r;
#else
  return v;
#endif
}

template <class EX>
SPEX_HDNI i64 ex_sum_i64(EX& ex, i64 v) {
#if SPEX_DEVICE_PASS
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  if (ex.lane == 0) ex.sml[ex.warp] = v;
  ex.sync();
  i64 r = ex.lane < ex.nwarp ? ex.sml[ex.lane] : 0;
  for (int off = 16; off > 0; off >>= 1) r += __shfl_xor_sync(0xffffffffu, r, off);
  ex.sync();
  return r;
#else
  return v;
#endif
}

template <class EX>
SPEX_HDNI double ex_minmax_d(EX& ex, double v, bool want_max) {
#if SPEX_DEVICE_PASS
  for (int off = 16; off > 0; off >>= 1) {
    double y = __shfl_xor_sync(0xffffffffu, v, off);
    if (want_max ? (y > v) : (y < v)) v = y;
  }
  if (ex.lane == 0) ex.smd[ex.warp] = v;
  ex.sync();
  double r = ex.smd[0];
  for (int w = 1; w < ex.nwarp; ++w)
    if (want_max ? (ex.smd[w] > r) : (ex.smd[w] < r)) r = ex.smd[w];
  ex.sync();
  return r;
#else
  return v;
#endif
}

// --------------------------------------------------------------- engine math
// sim.cpp:277-289
SPEX_HD double eng_elapsed(const GState* g, int steps) {
  if (steps <= 0) return 0.0;
  double m = static_cast<double>(steps);
  if (g->mem_d_ <= 0.0) return m * (g->compute_ < g->mem_a_ ? g->mem_a_ : g->compute_);
  int i0 = 0;
  if (g->compute_ > g->mem_a_) {
    double cross = (g->compute_ - g->mem_a_) / g->mem_d_;
    int c = static_cast<int>(floor(cross)) + 1;
    i0 = steps < c ? steps : c;
  }
  double tail = static_cast<double>(steps - i0);
  return i0 * g->compute_ + tail * g->mem_a_ +
         g->mem_d_ * (static_cast<double>(i0) + m - 1.0) * tail / 2.0;
}

// sim.cpp:291-303
SPEX_HD int eng_steps_within(const GState* g, double budget, int max_steps) {
  if (budget < -kTimeEps || max_steps <= 0) return 0;
  if (eng_elapsed(g, max_steps) <= budget + kTimeEps) return max_steps;
  int lo = 0, hi = max_steps;
  while (hi - lo > 1) {
    int mid = lo + (hi - lo) / 2;
    if (eng_elapsed(g, mid) <= budget + kTimeEps)
      lo = mid;
    else
      hi = mid;
  }
  return lo;
}

// unique_kv_tokens bookkeeping (sim.cpp:54-68): a stream joining/leaving the
// active batch adds/removes its strict ancestors' token counts the first/last
// time an ancestor becomes/stops being shared by an active member.
SPEX_HD void kv_ancestors_adjust(Run* R, int sid, int delta) {
  const int q = R->st_q[sid];
  const u32 base = static_cast<u32>(q) * static_cast<u32>(R->cfg.node_cap);
  i64 acc = 0;
  for (u32 cur = R->n_parent[base + R->st_node[sid]]; cur != kNoNode;
       cur = R->n_parent[base + cur]) {
    int old = atomic_add_int(&R->n_refc[base + cur], delta);
    if (delta > 0 && old == 0) acc += R->n_tokens[base + cur];
    if (delta < 0 && old == 1) acc -= R->n_tokens[base + cur];
  }
  if (acc != 0) {
    atomic_add_i64(&R->g->u_anc, acc);
    if (q_owned(R->cfg, q)) atomic_add_i64(&R->g->u_anc_own, acc);
  }
}

// Publish schedule entry e to the host (all block writes before it become
// visible first: per-thread gpu fence, barrier, then the leader's system fence).
template <class EX>
SPEX_HDNI void publish_entry(Run* R, EX& ex, int e, int rows, int tiles) {
#if SPEX_DEVICE_PASS
  if (!R->pub_e) return;
  if (R->pub) __threadfence();
  ex.sync();
  if (ex.tid == 0) {
    PubEntry pe;
    pe.kind = R->sched_kind[e];
    pe.steps = R->sched_steps[e];
    pe.off = R->sched_off[e];
    pe.n = R->sched_n[e];
    pe.rows = rows;
    pe.tiles = tiles;
    pe.u0 = R->sched_u[e];
    pe.kv_next = R->g->kv_next;
    R->pub_e[e] = pe;
    if (R->pub) {
      __threadfence_system();
      *reinterpret_cast<volatile int*>(&R->pub->n_sched) = e + 1;
    }
  }
  ex.sync();
#else
  (void)R;
  (void)ex;
  (void)e;
  (void)rows;
  (void)tiles;
#endif
}

// Record one decode epoch of the model schedule: `steps` forward steps over
// the active streams (in active order) starting at their current positions.
template <class EX>
SPEX_HDNI void record_decode(Run* R, EX& ex, int steps) {
  GState* g = R->g;
  const int nreg = g->n_active_region;
  const bool sharded = R->cfg.shard_lo > 0 || R->cfg.shard_hi < R->cfg.n_queries;
  for (int i = ex.tid; i < nreg; i += ex.nthr) {
    const int sid = R->live[i];
    R->it_scan_b[i] = R->st_state[sid] == ST_ACTIVE && q_owned(R->cfg, R->st_q[sid]) ? 1 : 0;
  }
  ex.sync();
  int n = 0;
  ex_scan(ex, R->it_scan_b, nreg, &n);
  i64 own_done = 0;
  const int off = g->n_sched_rows;
  if (g->n_sched >= R->cfg.sched_cap || off + n > R->cfg.sched_rows_cap) {
    if (ex.tid == 0) set_err(R, ERR_CAP_STAGE, -1, kNoNode);
    ex.sync();
    return;
  }
  for (int i = ex.tid; i < nreg; i += ex.nthr) {
    int sid = R->live[i];
    if (R->st_state[sid] == ST_ACTIVE) {
      if (!q_owned(R->cfg, R->st_q[sid])) continue;
      R->srow_sid[off + R->it_scan_b[i]] = sid;
      R->srow_pos0[off + R->it_scan_b[i]] = R->st_done[sid];
      own_done += R->st_done[sid];
    }
  }
  if (sharded) own_done = ex_sum_i64(ex, own_done);
  if (ex.tid == 0) {
    const int e = g->n_sched++;
    R->sched_kind[e] = SCHED_DECODE;
    // U at epoch start (of the owned shard when sharded)
    R->sched_u[e] = sharded ? g->u_anc_own + own_done : g->u_anc + g->sum_done - static_cast<i64>(steps) * n;
    R->sched_steps[e] = steps;
    R->sched_off[e] = off;
    R->sched_n[e] = n;
    g->n_sched_rows = off + n;
  }
  ex.sync();
  publish_entry(R, ex, g->n_sched - 1, n, 0);
}

// DecodeEngine::advance (sim.cpp:305-384). On return g->engine_now holds the
// reached boundary and fins[0..nfins) the streams finishing there, in order.
template <class EX>
SPEX_HDNI void engine_advance(Run* R, EX& ex, double limit) {
  GState* g = R->g;
  const Cfg& c = R->cfg;
  // per-call scalars in GState scratch: s_limit = now, s_flag = mode
  if (ex.tid == 0) {
    g->s_limit = g->engine_now;
    g->nfins = 0;
  }
  ex.sync();
  for (int guard = 0;; ++guard) {
    // ---- joins at this boundary
    if (ex.tid == 0) {
      int j = g->n_active_region;
      const double now = g->s_limit;
      g->s_k_total = j;  // joined_lo
      while (j < g->n_live) {
        int sid = R->live[j];
        u8 s = R->st_state[sid];
        if (s == ST_GONE) {
          ++j;
          continue;
        }
        if (R->st_ready[sid] <= now + kTimeEps) {
          R->st_state[sid] = ST_ACTIVE;
          g->n_act += 1;
          g->n_staged -= 1;
          ++j;
        } else {
          break;
        }
      }
      g->s_leftover = j;  // joined_hi
      g->n_active_region = j;
    }
    ex.sync();
    for (int i = g->s_k_total + ex.tid; i < g->s_leftover; i += ex.nthr) {
      int sid = R->live[i];
      if (R->st_state[sid] == ST_ACTIVE) kv_ancestors_adjust(R, sid, +1);
    }
    ex.sync();
    if (ex.tid == 0) {
      g->s_flag = 0;  // 0 continue, 1 return
      if (g->n_act == 0) {
        if (g->n_staged == 0) {
          g->s_flag = 1;
          g->s_limit = limit;
        } else {
          double r = kInf;
          for (int j = g->n_active_region; j < g->n_live; ++j) {
            int sid = R->live[j];
            if (R->st_state[sid] == ST_STAGED) {
              r = R->st_ready[sid];
              break;
            }
          }
          if (r > limit + kTimeEps) {
            g->s_flag = 1;
            g->s_limit = limit;
          } else {
            g->s_limit = r;
            g->s_flag = 2;  // retry joins
          }
        }
      } else {
        // refresh_costs (sim.cpp:265-275): always recomputed (it is a pure
        // function of the active set, identical to the cached value when clean)
        const double B = static_cast<double>(g->n_act);
        const double U = static_cast<double>(g->u_anc + g->sum_done);
        g->compute_ = B * c.flops_per_token / c.peak_compute;
        double kv_bytes = c.kv_bytes_per_token * U;
        g->mem_a_ = (c.weight_bytes + kv_bytes) / c.mem_bandwidth;
        g->mem_d_ = c.kv_bytes_per_token * B / c.mem_bandwidth;
      }
    }
    ex.sync();
    if (g->s_flag == 1) break;
    if (g->s_flag == 2) continue;
    // ---- epoch length
    int mloc = 0x7fffffff;
    for (int i = ex.tid; i < g->n_active_region; i += ex.nthr) {
      int sid = R->live[i];
      if (R->st_state[sid] == ST_ACTIVE && R->st_rem[sid] < mloc) mloc = R->st_rem[sid];
    }
    int m_complete = ex_min_int(ex, mloc);
    if (ex.tid == 0) {
      const double now = g->s_limit;
      int m_limit = eng_steps_within(g, limit - now, m_complete);
      int target = m_complete;
      if (g->n_staged > 0) {
        double r = kInf;
        for (int j = g->n_active_region; j < g->n_live; ++j) {
          int sid = R->live[j];
          if (R->st_state[sid] == ST_STAGED) {
            r = R->st_ready[sid];
            break;
          }
        }
        int cap = m_complete < m_limit ? m_complete : m_limit;
        if (cap >= 1 && now + eng_elapsed(g, cap) >= r - kTimeEps) {
          int lo = 1, hi = cap;
          while (hi > lo) {
            int mid = lo + (hi - lo) / 2;
            if (now + eng_elapsed(g, mid) >= r - kTimeEps)
              hi = mid;
            else
              lo = mid + 1;
          }
          target = lo;
        }
      }
      if (target > m_limit) {
        g->s_k_total = m_limit;  // steps
        g->s_flag = 1;           // partial epoch: return after advancing
        if (m_limit > 0) g->s_limit = now + eng_elapsed(g, m_limit);
      } else {
        g->s_k_total = target;
        g->s_flag = 0;
        g->s_limit = now + eng_elapsed(g, target);
      }
      if (g->s_k_total > 0) {
        g->sum_done += static_cast<i64>(g->s_k_total) * g->n_act;
        g->decode_steps += g->s_k_total;
        g->decode_rows += static_cast<i64>(g->s_k_total) * g->n_act;
      }
    }
    ex.sync();
    const int steps = g->s_k_total;
    if (steps > 0 && c.record_sched) record_decode(R, ex, steps);
    if (steps > 0) {
      for (int i = ex.tid; i < g->n_active_region; i += ex.nthr) {
        int sid = R->live[i];
        if (R->st_state[sid] == ST_ACTIVE) {
          R->st_done[sid] += steps;
          R->st_rem[sid] -= steps;
        }
      }
    }
    ex.sync();
    if (g->s_flag == 1) break;
    // ---- full epoch: ordered completions, then compaction of the live list
    const int nreg = g->n_active_region;
    for (int i = ex.tid; i < nreg; i += ex.nthr) {
      int sid = R->live[i];
      R->it_scan_a[i] = (R->st_state[sid] == ST_ACTIVE && R->st_rem[sid] <= 0) ? 1 : 0;
    }
    ex.sync();
    int nf = 0;
    ex_scan(ex, R->it_scan_a, nreg, &nf);
    for (int i = ex.tid; i < nreg; i += ex.nthr) {
      int sid = R->live[i];
      if (R->st_state[sid] == ST_ACTIVE && R->st_rem[sid] <= 0) {
        int f = R->it_scan_a[i];
        R->fins[f] = sid;
        R->fin_tokens[f] = R->st_done[sid];
        R->fin_cancel[f] = R->st_cancel[sid];
        kv_ancestors_adjust(R, sid, -1);
        atomic_add_i64(&g->sum_done, -static_cast<i64>(R->st_done[sid]));
        R->st_state[sid] = ST_GONE;
      }
    }
    ex.sync();
    // compaction: keep ACTIVE and STAGED entries in order
    const int nl = g->n_live;
    for (int i = ex.tid; i < nl; i += ex.nthr) {
      u8 s = R->st_state[R->live[i]];
      R->it_scan_b[i] = (s == ST_ACTIVE || s == ST_STAGED) ? 1 : 0;
    }
    ex.sync();
    int kept = 0;
    ex_scan(ex, R->it_scan_b, nl, &kept);
    for (int i = ex.tid; i < nl; i += ex.nthr) {
      int sid = R->live[i];
      u8 s = R->st_state[sid];
      if (s == ST_ACTIVE || s == ST_STAGED) R->live_tmp[R->it_scan_b[i]] = sid;
    }
    ex.sync();
    for (int i = ex.tid; i < kept; i += ex.nthr) R->live[i] = R->live_tmp[i];
    if (ex.tid == 0) {
      g->nfins = nf;
      g->n_act -= nf;
      g->n_live = kept;
      g->n_active_region = g->n_act;  // ACTIVE entries form the prefix
      g->epochs += 1;
    }
    ex.sync();
    if (nf > 0) break;
    if (guard > (1 << 24)) {
      if (ex.tid == 0) set_err(R, ERR_STALLED, -1, kNoNode);
      ex.sync();
      break;
    }
  }
  if (ex.tid == 0) g->engine_now = g->s_limit;
  ex.sync();
}

// A query needs a follow-up pass: flag it and, on the flag's 0 -> 1 edge,
// push it on the dirty list so followups() need not scan every query record
// (the items of one phase own disjoint queries, so the edge test is race-free).
SPEX_HD void mark_followup(Run* R, int q) {
  QueryRun* qr = &R->qs[q];
  if (qr->need_followup) return;
  qr->need_followup = 1;
  R->q_dirty[atomic_add_int(&R->g->n_dirty, 1)] = q;
}

// --------------------------------------------------------------- admission
// executor.cpp:765-783 plus generate_workload seeds (sim.cpp:177-180)
SPEX_HDNI void admit_query(Run* R, int q, Rec* rec_slot) {
  const Cfg& c = R->cfg;
  QueryRun* qr = &R->qs[q];
  const u64 base = splitmix64(c.run_seed ^ kSaltQuery);
  const u64 seed = hash_mix(base, static_cast<u64>(q + c.q_offset) + 1);  // the job's query (split mode)
  // zero the query
  char* p = reinterpret_cast<char*>(qr);
  for (size_t i = 0; i < sizeof(QueryRun); ++i) p[i] = 0;
  qr->seed = seed;
  qr->golden = golden_label_of(c, seed);
  qr->hit_ema = c.initial_hit_ema;
  qr->admitted = 1;
  mark_followup(R, q);
  qr->nnodes = 1;
  qr->chain_tip = kNoNode;
  qr->rest_cur = 0;
  qr->live_cache = c.prompt_tokens;
  qr->plan_empty_version = 0xffffffffu;
  const u32 b = static_cast<u32>(q) * static_cast<u32>(c.node_cap);
  R->n_parent[b] = kNoNode;
  R->n_depth[b] = 0;
  R->n_slot[b] = 0;
  R->n_tokens[b] = c.prompt_tokens;
  R->n_status[b] = kCommitted;
  R->n_flags[b] = NF_GEN_DONE | NF_GOLDEN_PATH;  // the root's path is empty: golden
  R->n_reward[b] = 0.0;
  R->n_value[b] = 0.0;
  R->n_visits[b] = 0;
  R->n_hash[b] = splitmix64(seed);
  R->n_first_child[b] = kNoNode;
  R->n_last_child[b] = kNoNode;
  R->n_next_sib[b] = kNoNode;
  R->n_nchildren[b] = 0;
  R->n_pred[b] = 0;
  R->n_stream[b] = -1;
  R->n_ready[b] = 0;
  R->n_refc[b] = 0;
  R->n_kvbase[b] = -1;
  if (kv_on(c, q)) {
    // the root prompt's pages are static: query q owns pages [q*pp, (q+1)*pp)
    const i64 p0 = static_cast<i64>(q) * c.kv_pp_root;
    for (int k = 0; k < c.kv_pp_root; ++k) R->kv_pt[p0 + k] = static_cast<int>(p0 + k);
    R->n_kvbase[b] = p0;
    R->n_kvh[b] = 1;
    R->n_flags[b] |= NF_KV_SELF;
  }
  if (c.family == kRebaseBfs) {
    R->q_layer[b] = 0;
    qr->layer_n = 1;
  }
  if (rec_slot) {
    rec_slot->t = R->g->now;
    rec_slot->x = 0.0;
    rec_slot->y = seed;
    rec_slot->q = q;
    rec_slot->node = kNoNode;
    rec_slot->a = rec_slot->b = rec_slot->c = 0;
    rec_slot->kind = EV_ADMIT;
    rec_slot->flags = 0;
    rec_slot->pad = 0;
  }
}

// ------------------------------------------------------------------ items
enum ItemKind { IK_FIN = 0, IK_REWARD = 1, IK_FOLLOWUP = 2, IK_SPEC = 3 };

template <class EX>
SPEX_HDNI void process_items(Run* R, EX& ex, int n_items, int kind, int rank_filter,
                           int* warp_off) {
  GState* g = R->g;
  const Cfg& c = R->cfg;
  {
    // one item per thread: every thread is an independent sequential state
    // machine with its own staging slot and scratch (the items of a phase
    // touch disjoint queries). Items are dealt round-robin over the warps
    // first (item i -> warp i % nwarp, lane i / nwarp) so all warps share
    // the work and their memory latencies overlap.
    const int slot = ex.tid;
    int* off = warp_off + slot * 3;
    for (int i = ex.lane * ex.nwarp + ex.warp; i < n_items; i += ex.nthr) {
      if (kind == IK_FIN && R->it_scan_c[i] != rank_filter) continue;
      if (g->error) break;
      Item it;
      const i64 wb = static_cast<i64>(slot) * c.stage_cap;
      it.rec = R->stage_rec + wb + off[0];
      it.nrec = 0;
      it.rec_cap = c.stage_cap - off[0];
      it.spw = R->stage_spawn + wb + off[1];
      it.nspw = 0;
      it.spw_cap = c.stage_cap - off[1];
      it.psh = R->stage_push + wb + off[2];
      it.npsh = 0;
      it.psh_cap = c.stage_cap - off[2];
      it.sdelta = 0;
      it.fin = 0;
      int q;
      if (kind == IK_FIN) {
        int sid = R->fins[i];
        q = R->st_q[sid];
        QC x = make_qc(R, q, &it, slot);
        R->fin_scored[i] = on_stream_done(x, sid, R->fin_tokens[i], R->fin_cancel[i]) ? 1 : 0;
        mark_followup(R, q);
      } else if (kind == IK_REWARD) {
        q = R->it_key[i];
        QC x = make_qc(R, q, &it, slot);
        on_reward(x, R->ev_node[g->fifo_head - 1]);
        mark_followup(R, q);
      } else if (kind == IK_FOLLOWUP) {
        q = R->it_key[i];
        QC x = make_qc(R, q, &it, slot);
        followup(x);
      } else {
        q = R->it_key[i];
        QC x = make_qc(R, q, &it, slot);
        int k = R->qs[q].grant;
        int n = issue_speculation(x, k);
        if (n == 0) R->qs[q].plan_empty_version = R->qs[q].version;
      }
      R->it_rec_off[i] = static_cast<int>(wb) + off[0];
      R->it_rec_n[i] = it.nrec;
      R->it_spawn_off[i] = static_cast<int>(wb) + off[1];
      R->it_spawn_n[i] = it.nspw;
      R->it_push_off[i] = static_cast<int>(wb) + off[2];
      R->it_push_n[i] = it.npsh;
      R->it_fin[i] = it.fin;
      R->it_sdelta[i] = it.sdelta;
      {
        // tree-KV pages of the spawns that still hold them (a stream erased
        // in this very step frees a terminal thought before it has pages)
        int tk = 0;
        for (int j = 0; j < it.nspw; ++j) {
          SpawnRec& sp = it.spw[j];
          const u32 ni = static_cast<u32>(sp.q) * static_cast<u32>(c.node_cap) + sp.node;
          sp.kvp = kv_on(c, sp.q) && R->n_kvh[ni] > 0 ? kv_pages_of(sp.tokens) : 0;
          tk += sp.kvp;
        }
        R->it_tok[i] = tk;
      }
      off[0] += it.nrec;
      off[1] += it.nspw;
      off[2] += it.npsh;
    }
  }
  ex.sync();
}

template <class EX>
SPEX_HDNI void reset_warp_offsets(Run* R, EX& ex, int* warp_off) {
  for (int i = ex.tid; i < ex.nthr * 3; i += ex.nthr) warp_off[i] = 0;
  ex.sync();
}

// drain_remaining (executor.cpp:340-360), run by one thread
SPEX_HDNI void drain_remaining(Run* R) {
  GState* g = R->g;
  for (int j = 0; j < g->n_live; ++j) {
    int sid = R->live[j];
    u8 s = R->st_state[sid];
    if (s != ST_ACTIVE && s != ST_STAGED) continue;
    const int q = R->st_q[sid];
    const u32 node = R->st_node[sid];
    const int part = s == ST_ACTIVE ? R->st_done[sid] : 0;
    QueryRun* qr = &R->qs[q];
    qr->generated += part;
    qr->wasted += part;
    if (R->cfg.trace) {
      if (g->log_n >= R->cfg.log_cap) {
        set_err(R, ERR_CAP_LOG, q, node);
        return;
      }
      Rec* r = &R->log[g->log_n++];
      r->t = g->now;
      r->x = 0.0;
      r->y = 0;
      r->q = q;
      r->node = node;
      r->a = sid;
      r->b = part;
      r->c = 0;
      r->kind = EV_DONE;
      r->flags = RF_CANCELLED | RF_STALE;
      r->pad = 0;
    }
    R->st_state[sid] = ST_GONE;
    R->n_stream[static_cast<u32>(q) * static_cast<u32>(R->cfg.node_cap) + node] = -1;
    if (kv_on(R->cfg, q)) kv_release(R, q, node);
  }
  g->n_live = 0;
  g->n_active_region = 0;
  g->n_act = 0;
  g->n_staged = 0;
}

// Place the staged output of items [0, n) in item order.
template <class EX>
SPEX_HDNI void commit_items(Run* R, EX& ex, int n) {
  GState* g = R->g;
  const Cfg& c = R->cfg;
  const int Q = c.n_queries;
  // finish ranks -> admissions (finish j admits iff admitted0 + j < Q)
  const int ac0 = g->admitted_count;
  int nfin = 0, nrec = 0, nspw = 0, npsh = 0, ntok = 0;
#if SPEX_DEVICE_PASS
  if (n <= 32) {
    // all five scans in warp 0 with shuffles, one barrier to publish
    int* tot = ex.sm + kSmCommit;
    if (ex.warp == 0) {
      const int i = ex.lane;
      const bool in = i < n;
      auto xscan = [&](int v, int* t) {
        int incl = v;
        for (int off = 1; off < 32; off <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, incl, off);
          if (i >= off) incl += y;
        }
        *t = __shfl_sync(0xffffffffu, incl, 31);
        return incl - v;
      };
      int t0, t1, t2, t3, t4;
      const int f = in ? R->it_fin[i] : 0;
      const int fx = xscan(f, &t0);
      const int admit = (f && ac0 + fx < Q) ? 1 : 0;
      const int bx = xscan(in ? R->it_rec_n[i] + (c.trace ? admit : 0) : 0, &t1);
      const int cx = xscan(in ? R->it_spawn_n[i] : 0, &t2);
      const int dx = xscan(in ? R->it_push_n[i] : 0, &t3);
      const int ex_ = xscan(in ? R->it_tok[i] : 0, &t4);
      if (in) {
        R->it_scan_a[i] = fx;
        R->it_scan_b[i] = bx;
        R->it_scan_c[i] = cx;
        R->it_scan_d[i] = dx;
        R->it_scan_e[i] = ex_;
      }
      if (i == 0) {
        tot[0] = t0;
        tot[1] = t1;
        tot[2] = t2;
        tot[3] = t3;
        tot[4] = t4;
      }
    }
    ex.sync();
    nfin = tot[0];
    nrec = tot[1];
    nspw = tot[2];
    npsh = tot[3];
    ntok = tot[4];
  } else
#endif
  {
    for (int i = ex.tid; i < n; i += ex.nthr) R->it_scan_a[i] = R->it_fin[i];
    ex.sync();
    ex_scan(ex, R->it_scan_a, n, &nfin);
    for (int i = ex.tid; i < n; i += ex.nthr) {
      int admit = (R->it_fin[i] && ac0 + R->it_scan_a[i] < Q) ? 1 : 0;
      R->it_scan_b[i] = R->it_rec_n[i] + (c.trace ? admit : 0);
      R->it_scan_c[i] = R->it_spawn_n[i];
      R->it_scan_d[i] = R->it_push_n[i];
      R->it_scan_e[i] = R->it_tok[i];
    }
    ex.sync();
    ex_scan(ex, R->it_scan_b, n, &nrec);
    ex_scan(ex, R->it_scan_c, n, &nspw);
    ex_scan(ex, R->it_scan_d, n, &npsh);
    ex_scan(ex, R->it_scan_e, n, &ntok);
  }
  // tree-KV pages for this commit's spawns: page-table entries [kv0, kv0 + ntok)
  // take never-used pages first (consecutive: a thought stays one run of
  // pages), then pages from the free ring once the pool has been touched
  const i64 kv0 = g->kv_next;
  const i64 kv_room = c.kv_pages - g->kv_bump;
  const i64 kv_fresh = ntok < kv_room ? ntok : kv_room;
  const i64 kv_take = ntok - kv_fresh;
  if (ntok > 0 && (kv_take > g->kv_free_tail - g->kv_free_head || kv0 + ntok > c.kv_pt_cap)) {
    // error_node 1: the page table is full (the host retries with a larger
    // one); 0: the live thoughts exceed the pool
    if (ex.tid == 0) set_err(R, ERR_CAP_KV, -1, kv0 + ntok > c.kv_pt_cap ? 1u : 0u);
    ex.sync();
    return;
  }
  for (int k = ex.tid; k < ntok; k += ex.nthr)
    R->kv_pt[kv0 + k] = k < kv_fresh ? static_cast<int>(g->kv_bump + k)
                                     : R->kv_free[(g->kv_free_head + (k - kv_fresh)) % c.kv_pages];
  if (c.trace && g->log_n + nrec > c.log_cap) {
    if (ex.tid == 0) set_err(R, ERR_CAP_LOG, -1, kNoNode);
    ex.sync();
    return;
  }
  if (g->next_sid + nspw > c.stream_cap) {
    if (ex.tid == 0) set_err(R, ERR_CAP_STREAMS, -1, kNoNode);
    ex.sync();
    return;
  }
  const int log0 = g->log_n, sid0 = g->next_sid, live0 = g->n_live, fifo0 = g->fifo_tail;
  const double now = g->now;
  const double t_evt = now + c.reward_latency;
  // parallel placement: one warp per item, lanes over entries
  for (int i = ex.warp; i < n; i += ex.nwarp) {
    const int sbase = sid0 + R->it_scan_c[i];
    if (c.trace) {
      const int rb = log0 + R->it_scan_b[i];
      const Rec* src = R->stage_rec + R->it_rec_off[i];
      for (int j = ex.lane; j < R->it_rec_n[i]; j += ex.lanes) {
        Rec r = src[j];
        if (r.flags & RF_LOCAL_SID) {
          r.a = sbase + r.a;
          r.flags = static_cast<u8>(r.flags & ~RF_LOCAL_SID);
        }
        R->log[rb + j] = r;
      }
    }
    const SpawnRec* sp = R->stage_spawn + R->it_spawn_off[i];
    for (int j = ex.lane; j < R->it_spawn_n[i]; j += ex.lanes) {
      const int sid = sbase + j;
      const SpawnRec s = sp[j];
      R->st_q[sid] = s.q;
      R->st_node[sid] = s.node;
      R->st_rem[sid] = s.tokens;
      R->st_done[sid] = 0;
      R->st_cancel[sid] = 0;
      R->st_ready[sid] = now;
      R->st_state[sid] = s.cancelled ? ST_GONE : ST_STAGED;
      R->live[live0 + R->it_scan_c[i] + j] = sid;
      if (s.kvp > 0) {
        i64 kb = kv0 + R->it_scan_e[i];
        for (int k = 0; k < j; ++k) kb += sp[k].kvp;
        R->n_kvbase[static_cast<u32>(s.q) * static_cast<u32>(c.node_cap) + s.node] = kb;
      }
      if (!s.cancelled) {
        R->n_stream[static_cast<u32>(s.q) * static_cast<u32>(c.node_cap) + s.node] = sid;
      }
    }
    const PushRec* ps = R->stage_push + R->it_push_off[i];
    for (int j = ex.lane; j < R->it_push_n[i]; j += ex.lanes) {
      const int pos = fifo0 + R->it_scan_d[i] + j;
      R->ev_time[pos] = t_evt;
      R->ev_q[pos] = ps[j].q;
      R->ev_node[pos] = ps[j].node;
    }
    if (ex.lane == 0 && R->it_fin[i] && ac0 + R->it_scan_a[i] < Q) {
      const int qa = ac0 + R->it_scan_a[i];
      Rec* slot = c.trace ? &R->log[log0 + R->it_scan_b[i] + R->it_rec_n[i]] : nullptr;
      admit_query(R, qa, slot);
    }
  }
  int sd = 0;
  for (int i = ex.tid; i < n; i += ex.nthr) sd += R->it_sdelta[i];
  i64 sdelta = ex_sum_i64(ex, sd);
  if (ex.tid == 0) {
    g->log_n += c.trace ? nrec : 0;
    g->next_sid += nspw;
    g->n_live += nspw;
    g->n_staged += static_cast<int>(sdelta);
    g->fifo_tail += npsh;
    g->kv_next += ntok;
    g->kv_free_head += kv_take;
    g->kv_bump += kv_fresh;
    g->kv_live += ntok;
    if (g->kv_live > g->kv_peak) g->kv_peak = g->kv_live;
    int admits = Q - ac0 < nfin ? Q - ac0 : nfin;
    if (admits < 0) admits = 0;
    g->admitted_count += admits;
    g->finished_count += nfin;
    if (nfin > 0 && g->finished_count == Q) drain_remaining(R);
  }
  ex.sync();
}

// Build the list of queries with `pred` true, in query order, into it_key.
template <class EX, class Pred>
SPEX_HD int collect_queries(Run* R, EX& ex, Pred pred) {
  const int Q = R->cfg.n_queries;
#if SPEX_DEVICE_PASS
  // warp ballots + per-warp counts: two barriers per nthr queries, no global scratch
  int* wc = ex.sm + kSmCollect;
  int total = 0;
  for (int base = 0; base < Q; base += ex.nthr) {
    const int q = base + ex.tid;
    const bool p = q < Q && pred(q);
    const unsigned bal = __ballot_sync(0xffffffffu, p);
    if (ex.lane == 0) wc[ex.warp] = __popc(bal);
    ex.sync();
    const int cw = ex.lane < ex.nwarp ? wc[ex.lane] : 0;
    int before = ex.lane < ex.warp ? cw : 0, chunk = cw;
    for (int o = 16; o > 0; o >>= 1) {
      before += __shfl_xor_sync(0xffffffffu, before, o);
      chunk += __shfl_xor_sync(0xffffffffu, chunk, o);
    }
    const int off = total + before;
    if (p) R->it_key[off + __popc(bal & ((1u << ex.lane) - 1u))] = q;
    total += chunk;
    ex.sync();
  }
  return total;
#endif
  for (int q = ex.tid; q < Q; q += ex.nthr) R->it_scan_a[q] = pred(q) ? 1 : 0;
  ex.sync();
  int n = 0;
  ex_scan(ex, R->it_scan_a, Q, &n);
  for (int q = ex.tid; q < Q; q += ex.nthr)
    if (pred(q)) R->it_key[R->it_scan_a[q]] = q;
  ex.sync();
  return n;
}

// scheduling_round (executor.cpp:705-740) with allocate_budgets (budget.cpp:45-96)
// allocate_budgets (budget.cpp:45-96) over arrays, block-parallel: min-max
// normalised scores, exp(tau * norm) shares (left-fold sum), floors capped by
// capacity, then the flooring loss round-robin over a stable descending-score
// order to queries with spare capacity. Shared by scheduling_round and the
// spex_budget_allocate hook (spex_hooks.cu).
template <class EX>
SPEX_HDNI void allocate_block(EX& ex, GState* g, int n, int k_total, double tau, const double* score, const int* cap,
                              double* w, int* out, int* order) {
  double lo = kInf, hi = -kInf;
  for (int i = ex.tid; i < n; i += ex.nthr) {
    const double s = score[i];
    if (s < lo) lo = s;
    if (s > hi) hi = s;
  }
  lo = ex_minmax_d(ex, lo, false);
  hi = ex_minmax_d(ex, hi, true);
  for (int i = ex.tid; i < n; i += ex.nthr) {
    double norm = hi > lo ? (score[i] - lo) / (hi - lo) : 0.0;
    w[i] = glibc::exp(tau * norm);
  }
  ex.sync();
  if (ex.tid == 0) {
    double total = 0.0;
    for (int i = 0; i < n; ++i) total += w[i];
    g->s_total = total;
  }
  ex.sync();
  const double total = g->s_total;
  i64 fsum = 0;
  for (int i = ex.tid; i < n; i += ex.nthr) {
    int f = static_cast<int>(floor(k_total * w[i] / total));
    fsum += f;
    out[i] = cap[i] < f ? cap[i] : f;
  }
  const i64 floor_sum = ex_sum_i64(ex, fsum);
  const int leftover = k_total - static_cast<int>(floor_sum);
  if (leftover > 0) {
    // stable order by raw score, descending
    for (int i = ex.tid; i < n; i += ex.nthr) {
      const double si = score[i];
      int rank = 0;
      for (int j = 0; j < n; ++j) {
        const double sj = score[j];
        if (sj > si || (sj == si && j < i)) ++rank;
      }
      order[rank] = i;
    }
    ex.sync();
    if (ex.tid == 0) {
      int left = leftover;
      bool progress = true;
      while (left > 0 && progress) {
        progress = false;
        for (int r = 0; r < n; ++r) {
          if (left == 0) break;
          const int idx = order[r];
          if (out[idx] < cap[idx]) {
            out[idx] += 1;
            --left;
            progress = true;
          }
        }
      }
    }
    ex.sync();
  }
}

// ------------------------------------------------ split mode budget exchange
// north_star's multi-GPU data path: each rank owns a query block and runs its
// own engine; the only exchange is the T2 allocation's per-query gains. The
// k-th allocate_budgets call of every rank (executor.cpp:727-733: T2 on, a
// candidate, idle producer slots) is exchange round k: the rank posts its idle
// slots and its candidates' (score, capacity) to its outbox, waits until every
// other rank has posted round k or finished its run, and allocates over the
// concatenation in rank order with k_total = the posted idle slots' sum,
// keeping its own candidates' grants (oracle: oracle/ref_split.cpp, the
// reference's own executor in W threads). The outboxes live in each rank's HBM
// and are read by the others over NVLink (peer-mapped; on one GPU, one
// allocation); flags are epoch-tagged, so an outbox is never reset:
//   [0] u64 started = epoch   [8] u64 posted = epoch << 32 | round
//   [16] u64 done = epoch     [64 + (round & 1) * slot_bytes] slot:
//   int idle, int n, 8 pad, double score[qmax], int cap[qmax]
// A rank overwrites slot (k & 1) at round k + 2 only after every live rank
// posted round k + 1, i.e. finished reading round k; a run starts only after
// every rank started it, so no rank reads an earlier run's slots.
constexpr int kSmXch = 700;  // 3 * kMaxSplit ints of ex.sm

SPEX_HD u64 xch_load(const char* p) {
#if SPEX_DEVICE_PASS
  u64 v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
#else
  return __atomic_load_n(reinterpret_cast<const u64*>(p), __ATOMIC_ACQUIRE);
#endif
}

SPEX_HD void xch_store(char* p, u64 v) {
#if SPEX_DEVICE_PASS
  __threadfence_system();
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
#else
  __atomic_store_n(reinterpret_cast<u64*>(p), v, __ATOMIC_RELEASE);
#endif
}

SPEX_HD void xch_fence() {
#if SPEX_DEVICE_PASS
  __threadfence_system();
#else
  __atomic_thread_fence(__ATOMIC_SEQ_CST);
#endif
}

SPEX_HD void xch_pause() {
#if SPEX_DEVICE_PASS
  __nanosleep(128);
#else
  __builtin_ia32_pause();
#endif
}

// wait until `pred` holds; false after the 120 s watchdog (a rank gone)
template <class P>
SPEX_HD bool xch_wait(P pred) {
  const i64 t0 = spex_wall_ns();
  for (long long spin = 0; !pred(); ++spin) {
    xch_pause();
#if SPEX_DEVICE_PASS
    if ((spin & 1023) == 1023 && spex_wall_ns() - t0 > 120000000000LL) return false;
#else
    if (spin > (1LL << 36)) return false;
#endif
  }
  return true;
}

// run start: publish `started`, then wait until every rank started this run
template <class EX>
SPEX_HDNI void split_start(Run* R, EX& ex) {
  const Cfg& c = R->cfg;
  const u64 e = static_cast<u64>(c.split_epoch);
  if (ex.tid == 0) xch_store(R->xch[c.split_rank], e);
  ex.sync();
  for (int s = ex.tid; s < c.split_world; s += ex.nthr) {
    if (s == c.split_rank) continue;
    const char* p = R->xch[s];
    if (!xch_wait([&] { return xch_load(p) >= e; })) set_err(R, ERR_STALLED, -1, kNoNode);
  }
  ex.sync();
}

// run end: this rank takes part in no further round
template <class EX>
SPEX_HDNI void split_finish(Run* R, EX& ex) {
  const Cfg& c = R->cfg;
  if (ex.tid == 0) xch_store(R->xch[c.split_rank] + 16, static_cast<u64>(c.split_epoch));
  ex.sync();
}

// One exchange round over the local candidates' al_score / al_rank [0, n):
// on return al_score / al_rank [0, N) hold every posting rank's candidates in
// rank order; *k_total is the posted idle slots' sum, *my_off this rank's
// first candidate. Returns N.
template <class EX>
SPEX_HDNI int split_exchange(Run* R, EX& ex, int n, int idle, int* k_total, int* my_off) {
  GState* g = R->g;
  const Cfg& c = R->cfg;
  const int W = c.split_world, me = c.split_rank;
  const u64 e = static_cast<u64>(c.split_epoch);
  const i64 t0 = ex.tid == 0 ? spex_wall_ns() : 0;
  if (ex.tid == 0) g->xch_rounds += 1;
  ex.sync();
  const u64 k = static_cast<u64>(g->xch_rounds);
  auto slot_of = [&](int s) { return R->xch[s] + kXchHead + static_cast<i64>(k & 1) * c.xch_slot_bytes; };
  {
    char* slot = slot_of(me);
    double* sc = reinterpret_cast<double*>(slot + 16);
    int* cp = reinterpret_cast<int*>(sc + c.split_qmax);
    for (int i = ex.tid; i < n; i += ex.nthr) {
      sc[i] = R->al_score[i];
      cp[i] = R->al_rank[i];
    }
    if (ex.tid == 0) {
      reinterpret_cast<int*>(slot)[0] = idle;
      reinterpret_cast<int*>(slot)[1] = n;
    }
    xch_fence();
  }
  ex.sync();
  if (ex.tid == 0) xch_store(R->xch[me] + 8, (e << 32) | k);
  int* inc = ex.sm + kSmXch;          // [W] rank s posted round k
  int* off = inc + kMaxSplit;         // [W] its first candidate in the concatenation
  int* cnt = off + kMaxSplit;         // [W] its candidates
  for (int s = ex.tid; s < W; s += ex.nthr) {
    int in = 1;
    if (s != me) {
      const char* p = R->xch[s];
      auto posted = [&] {
        const u64 v = xch_load(p + 8);
        return (v >> 32) == e && (v & 0xffffffffULL) >= k;
      };
      const bool ok = xch_wait([&] { return posted() || xch_load(p + 16) == e; });
      if (!ok) set_err(R, ERR_STALLED, -1, kNoNode);
      in = ok && posted() ? 1 : 0;  // `done` is stored after the last post: re-read
    }
    inc[s] = in;
  }
  ex.sync();
  if (ex.tid == 0) {
    int N = 0, K = 0;
    for (int s = 0; s < W; ++s) {
      off[s] = N;
      cnt[s] = 0;
      if (!inc[s]) continue;
      const volatile int* h = reinterpret_cast<const volatile int*>(slot_of(s));
      cnt[s] = h[1];
      K += h[0];
      N += cnt[s];
    }
    g->s_k_total = K;
    g->s_n_items = N;
    g->xch_wait_ns += spex_wall_ns() - t0;
  }
  ex.sync();
  for (int s = 0; s < W; ++s) {
    if (!cnt[s]) continue;
    const volatile double* sc = reinterpret_cast<const volatile double*>(slot_of(s) + 16);
    const volatile int* cp = reinterpret_cast<const volatile int*>(sc + c.split_qmax);
    for (int i = ex.tid; i < cnt[s]; i += ex.nthr) {
      R->al_score[off[s] + i] = sc[i];
      R->al_rank[off[s] + i] = cp[i];
    }
  }
  *k_total = g->s_k_total;
  *my_off = off[me];
  const int N = g->s_n_items;
  ex.sync();
  return N;
}

template <class EX>
SPEX_HDNI void scheduling_round(Run* R, EX& ex, int* warp_off) {
  GState* g = R->g;
  const Cfg& c = R->cfg;
  if (!c.t1) return;
  // With T2 a round grants nothing while the producers are saturated
  // (executor.cpp:730-731, idle <= 0 returns); the per-query fields the
  // candidate scan writes are read only by this round, so skip it outright
  // (at Q = 4096 the scan of every query record is most of the control time).
  if (c.t2 && c.producer_slots - (g->n_act + g->n_staged) <= 0) return;
  const int Q = c.n_queries;
  for (int q = ex.tid; q < Q; q += ex.nthr) {
    QueryRun* qr = &R->qs[q];
    int cand = 0;
    if (qr->admitted && !qr->finished) {
      const int outstanding = qr->n_active_exp;
      const int cap = c.spec_k - outstanding;
      if (cap > 0) {
        cand = 1;
        qr->capacity = cap;
        qr->pending_specs = outstanding;
        if (c.t2) qr->kv_bytes = c.kv_bytes_per_token * static_cast<double>(qr->live_cache);
        qr->grant = cap;
      }
    }
    R->al_cand[q] = cand;
  }
  ex.sync();
  auto is_cand = [&](int q) { return R->al_cand[q] != 0; };
  const int n = collect_queries(R, ex, is_cand);
  if (n == 0) return;
  if (c.t2) {
    const int idle = c.producer_slots - (g->n_act + g->n_staged);
    if (idle <= 0) return;
    // scores (budget.cpp:41-43) and capacities of the candidates, then the split
    for (int i = ex.tid; i < n; i += ex.nthr) {
      const QueryRun* qr = &R->qs[R->it_key[i]];
      R->al_score[i] = qr->capacity * qr->hit_ema * (c.weight_bytes + qr->kv_bytes);
      R->al_rank[i] = qr->capacity;
    }
    ex.sync();
    int n_all = n, k_total = idle, my_off = 0;
    if (c.split_world > 1) n_all = split_exchange(R, ex, n, idle, &k_total, &my_off);
    allocate_block(ex, g, n_all, k_total, c.tau, R->al_score, R->al_rank, R->al_w, R->al_out, R->al_order);
    for (int i = ex.tid; i < n; i += ex.nthr) R->qs[R->it_key[i]].grant = R->al_out[my_off + i];
    ex.sync();
  }
  // issue: candidates with a grant and a plan that may be non-empty
  auto issue = [&](int q) {
    const QueryRun* qr = &R->qs[q];
    return R->al_cand[q] != 0 && qr->grant > 0 && qr->version != qr->plan_empty_version;
  };
  const int m = collect_queries(R, ex, issue);
  if (m == 0) return;
  reset_warp_offsets(R, ex, warp_off);
  SPEX_TIMED(ex, R, CY_ITEMS, process_items(R, ex, m, IK_SPEC, 0, warp_off));
  commit_items(R, ex, m);
}

// The queries needing a follow-up, ascending (item order = log order): from
// the dirty list when it is short (sorted by rank counting), else by a scan of
// every query record; the list is emptied either way.
template <class EX>
SPEX_HDNI int collect_dirty(Run* R, EX& ex) {
  GState* g = R->g;
  const int nd = g->n_dirty;
  auto need = [&](int q) {
    const QueryRun* qr = &R->qs[q];
    return qr->admitted && !qr->finished && qr->need_followup;
  };
  int n;
  if (nd > 512 || R->cfg.n_queries <= ex.nthr) {
    // a long list, or few enough queries for one ballot pass over all of them
    n = collect_queries(R, ex, need);
  } else {
    int* keep = R->it_scan_a;
    for (int i = ex.tid; i < nd; i += ex.nthr) keep[i] = need(R->q_dirty[i]) ? R->q_dirty[i] : -1;
    ex.sync();
    for (int i = ex.tid; i < nd; i += ex.nthr) {
      const int q = keep[i];
      if (q < 0) continue;
      int rank = 0;
      for (int j = 0; j < nd; ++j) rank += keep[j] >= 0 && keep[j] < q;
      R->it_key[rank] = q;
    }
    int m = 0;
    for (int i = ex.tid; i < nd; i += ex.nthr) m += keep[i] >= 0;
    n = static_cast<int>(ex_sum_i64(ex, m));
  }
  ex.sync();
  if (ex.tid == 0) g->n_dirty = 0;
  ex.sync();
  return n;
}

// consumer_step_followups (executor.cpp:746-763)
template <class EX>
SPEX_HDNI void followups(Run* R, EX& ex, int* warp_off) {
  for (int pass = 0; pass < 4; ++pass) {
    const int n = collect_dirty(R, ex);
    if (n == 0 || R->g->error) break;
    for (int i = ex.tid; i < n; i += ex.nthr) R->qs[R->it_key[i]].need_followup = 0;
    ex.sync();
    reset_warp_offsets(R, ex, warp_off);
    SPEX_TIMED(ex, R, CY_FOLLOW, process_items(R, ex, n, IK_FOLLOWUP, 0, warp_off));
    SPEX_TIMED(ex, R, CY_COMMIT, commit_items(R, ex, n));
  }
  if (!R->g->error) SPEX_TIMED(ex, R, CY_SCHED, scheduling_round(R, ex, warp_off));
}

// Completion phase: on_stream_done for fins in order (executor.cpp:794).
template <class EX>
SPEX_HDNI void completions(Run* R, EX& ex, int* warp_off) {
  GState* g = R->g;
  const int nf = g->nfins;
  // rank of each completion among those of the same query
  if (ex.tid == 0) {
    int maxr = 0;
    for (int f = 0; f < nf; ++f) R->qs[R->st_q[R->fins[f]]].grant = 0;
    for (int f = 0; f < nf; ++f) {
      QueryRun* qr = &R->qs[R->st_q[R->fins[f]]];
      R->it_scan_c[f] = qr->grant;
      qr->grant += 1;
      if (qr->grant > maxr) maxr = qr->grant;
    }
    g->s_flag = maxr;
  }
  ex.sync();
  const int rounds = g->s_flag;
  reset_warp_offsets(R, ex, warp_off);
  for (int r = 0; r < rounds; ++r) process_items(R, ex, nf, IK_FIN, r, warp_off);
  if (R->cfg.record_sched) {
    // reward batch of this boundary: the non-stale completions, in order
    // (owned query shard only: the other ranks score the rest)
    for (int f = ex.tid; f < nf; f += ex.nthr)
      R->it_scan_a[f] = R->fin_scored[f] && q_owned(R->cfg, R->st_q[R->fins[f]]) ? 1 : 0;
    ex.sync();
    const int e_prm = g->n_sched;  // this boundary's PRM entry (read before thread 0 bumps it)
    int ns = 0;
    ex_scan(ex, R->it_scan_a, nf, &ns);
    const int off = g->n_sched_rows;
    if (ns > 0 && (g->n_sched >= R->cfg.sched_cap || off + ns > R->cfg.sched_rows_cap)) {
      if (ex.tid == 0) set_err(R, ERR_CAP_STAGE, -1, kNoNode);
    } else if (ns > 0) {
      for (int f = ex.tid; f < nf; f += ex.nthr) {
        const int sc = R->fin_scored[f] && q_owned(R->cfg, R->st_q[R->fins[f]]);
        R->it_scan_b[f] = sc ? R->fin_tokens[f] : 0;
        R->it_scan_d[f] = sc ? (R->fin_tokens[f] + kTileRows - 1) / kTileRows : 0;
      }
      ex.sync();
      int nrows = 0, ntiles = 0;
      ex_scan(ex, R->it_scan_b, nf, &nrows);
      ex_scan(ex, R->it_scan_d, nf, &ntiles);
      for (int f = ex.tid; f < nf; f += ex.nthr)
        if (R->fin_scored[f] && q_owned(R->cfg, R->st_q[R->fins[f]])) {
          if (R->cfg.reward_prm)
            R->n_prm_e[static_cast<u32>(R->st_q[R->fins[f]]) * static_cast<u32>(R->cfg.node_cap) +
                       R->st_node[R->fins[f]]] = e_prm;
          const int k = off + R->it_scan_a[f];
          R->srow_sid[k] = R->fins[f];
          R->srow_pos0[k] = R->fin_tokens[f];
          R->srow_rstart[k] = R->it_scan_b[f];
          R->srow_tstart[k] = R->it_scan_d[f];
        }
      if (ex.tid == 0) {
        const int e = g->n_sched++;
        R->sched_kind[e] = SCHED_PRM;
        R->sched_u[e] = 0;
        R->sched_steps[e] = 0;
        R->sched_off[e] = off;
        R->sched_n[e] = ns;
        g->n_sched_rows = off + ns;
      }
      ex.sync();
      publish_entry(R, ex, g->n_sched - 1, nrows, ntiles);
    }
    ex.sync();
  }
  // the finished streams' own holds (after their PRM batch is recorded)
  if (R->cfg.kv_pages > 0) {
    for (int f = ex.tid; f < nf; f += ex.nthr) {
      const int q = R->st_q[R->fins[f]];
      if (kv_on(R->cfg, q)) kv_release(R, q, R->st_node[R->fins[f]]);
    }
    ex.sync();
  }
  commit_items(R, ex, nf);
}

// The whole run: admission of the first batch, then the consumer loop.
template <class EX>
SPEX_HD void run_loop(Run* R, EX& ex, int* warp_off) {
  GState* g = R->g;
  const Cfg& c = R->cfg;
  const int Q = c.n_queries;
  if (g->phase == 2) return;  // a finished run (stepwise execution called once more)
  const bool resume = g->phase == 1;
  if (!resume && c.split_world > 1) split_start(R, ex);
  if (!resume && ex.tid == 0) {
    const int first = c.batch_size < Q ? c.batch_size : Q;
    for (int q = 0; q < first; ++q) {
      Rec* slot = c.trace ? &R->log[g->log_n++] : nullptr;
      admit_query(R, q, slot);
    }
    g->admitted_count = first;
    const i64 root_pages = c.kv_pages > 0 ? static_cast<i64>(Q) * c.kv_pp_root : 0;
    g->kv_next = root_pages;
    g->kv_bump = root_pages;
    g->kv_live = root_pages;
    g->kv_peak = root_pages;
    g->start_ns = spex_wall_ns();
  }
  ex.sync();
  if (!resume) followups(R, ex, warp_off);
  // stepwise execution: at most step_iters consumer-loop iterations this launch
  const i64 budget = g->step_iters;
  i64 done_iters = 0;
  bool paused = false;
  for (;;) {
    ex.sync();
    if (g->error || g->finished_count >= Q) break;
    if (budget > 0 && done_iters >= budget) {
      paused = true;
      break;
    }
    ++done_iters;
    if (ex.tid == 0) g->iterations += 1;
    const double t_evt = g->fifo_head < g->fifo_tail ? R->ev_time[g->fifo_head] : kInf;
    if (g->n_act + g->n_staged > 0) {
      SPEX_TIMED(ex, R, CY_ENGINE, engine_advance(R, ex, t_evt));
      if (g->nfins > 0) {
        if (ex.tid == 0 && g->now < g->engine_now) g->now = g->engine_now;
        ex.sync();
        SPEX_TIMED(ex, R, CY_FINS, completions(R, ex, warp_off));
        followups(R, ex, warp_off);
        continue;
      }
    }
    // every thread reads the FIFO state before thread 0 pops it (a block-uniform
    // branch: without this barrier a slow thread could see the popped head)
    const bool fifo_empty = g->fifo_head >= g->fifo_tail;
    ex.sync();
    if (fifo_empty) {
      if (ex.tid == 0) set_err(R, ERR_STALLED, -1, kNoNode);
      ex.sync();
      break;
    }
    if (ex.tid == 0) {
      const int h = g->fifo_head++;
      const double et = R->ev_time[h];
      if (g->now < et) g->now = et;
      if (g->n_act + g->n_staged == 0 && g->engine_now < et) g->engine_now = et;
      R->it_key[0] = R->ev_q[h];
      g->reward_events += 1;
    }
    ex.sync();
    SPEX_TIMED(ex, R, CY_REWARD, {
      reset_warp_offsets(R, ex, warp_off);
      process_items(R, ex, 1, IK_REWARD, 0, warp_off);
      commit_items(R, ex, 1);
    });
    followups(R, ex, warp_off);
  }
  if (paused) {
    if (ex.tid == 0) g->phase = 1;
    ex.sync();
    return;
  }
  if (ex.tid == 0) {
    g->phase = 2;
    double ms = 0.0;
    for (int q = 0; q < Q; ++q)
      if (R->qs[q].finished && R->qs[q].finish_time > ms) ms = R->qs[q].finish_time;
    g->makespan = ms;
  }
  ex.sync();
  if (c.split_world > 1) split_finish(R, ex);
#if SPEX_DEVICE_PASS
  if (R->pub && ex.tid == 0) {
    __threadfence_system();
    *reinterpret_cast<volatile int*>(&R->pub->error) = g->error;
    *reinterpret_cast<volatile int*>(&R->pub->done) = 1;
  }
#endif
}

}  // namespace spex
