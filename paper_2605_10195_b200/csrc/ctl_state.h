// ctl_state.h — device-resident layout of one frontier-expansion run.
//
// Everything the reference keeps in std::vector<ThoughtNode>, std::map/set
// ledgers, the DecodeEngine stream vectors and the SimClock heap lives here as
// flat structure-of-arrays in HBM, indexed by (query, node) or stream id:
//
//   node arrays   [n_queries * node_cap]   tree.hpp:45-63 ThoughtNode fields,
//                                          children as a slot-ordered linked list,
//                                          ledger/batch/cohort set membership as bits
//   query array   [n_queries]              executor.cpp:63-94 QueryRun scalars
//   per-query u32 lists (rest stack, BFS layer/cohort) [n_queries * node_cap]
//   stream table  [stream_cap]             sim.hpp:201-209 DecodeEngine::Stream
//   live list     [stream_cap]             active_ ++ staged_ in stream-id order
//   event FIFO    [stream_cap]             SimClock (reward pushes are time-monotone,
//                                          so the heap degenerates to a FIFO)
//   event log     [log_cap] of Rec         trace.hpp:14-29 records, binary
#pragma once

#include "spex_hd.h"

namespace spex {

constexpr u32 kNoNode = 0xffffffffu;
constexpr int kMaxLabels = 64;
constexpr int kMaxDepthWidths = 64;
constexpr int kMaxTracked = 8;  // executor.hpp:16 kMaxTrackedDistance
constexpr double kTimeEps = 1e-9;  // sim.cpp:14

enum NodeStatus : u8 {
  kPendingExpansion = 0,
  kExpanding = 1,
  kAwaitingReward = 2,
  kCommitted = 3,
  kSpeculative = 4,
  kSpeculativeDone = 5,
  kPruned = 6,
  kTerminalAnswer = 7,
};

enum Family : int { kRstarDfs = 0, kRestHybrid = 1, kRebaseBfs = 2 };

// node flag bits
enum : u16 {
  NF_SPEC_ORIGIN = 1u << 0,
  NF_GEN_DONE = 1u << 1,
  NF_TERMINAL = 1u << 2,
  NF_HAS_REWARD = 1u << 3,
  NF_LEDGER_ACTIVE = 1u << 4,     // SpeculationLedger::active_expansions
  NF_LEDGER_COMPLETED = 1u << 5,  // completed_speculations
  NF_LEDGER_RESOLVED = 1u << 6,   // resolved
  NF_HAS_PRED = 1u << 7,          // predicted_distance
  NF_BATCH_PENDING = 1u << 8,     // QueryRun::batch_pending
  NF_COHORT_PENDING = 1u << 9,    // QueryRun::cohort_pending
  NF_HAS_READY = 1u << 10,        // ready_at_promote
  NF_GOLDEN_PATH = 1u << 11,      // every node on the path to the root passes the golden draw (oracle_reward)
  NF_DEEP = 1u << 12,             // the depth-1 ancestor's deep draw passed (oracle_is_terminal)
  NF_KV_SELF = 1u << 13,          // the node still holds its own tree-KV pin (may get children)
};

// Tree-KV pages: a thought's K/V rows live in pages of kKvPage tokens of the
// model's KV pools; a node's pages are listed in kv_pt[n_kvbase .. + pages).
constexpr int kKvPage = 16;
SPEX_HD int kv_pages_of(int tokens) { return (tokens + kKvPage - 1) / kKvPage; }

// stream states
enum : u8 { ST_NONE = 0, ST_STAGED = 1, ST_ACTIVE = 2, ST_GONE = 3 };

// event-log record kinds (trace.hpp:14-29)
enum : u8 {
  EV_ADMIT = 1,
  EV_NODE,
  EV_REQ,
  EV_DONE,
  EV_REWARD,
  EV_PROMOTE,
  EV_PRUNE,
  EV_ANSWER,
  EV_TERMINATE,
  EV_QUERY_DONE,
};
enum : u8 {
  RF_SPEC = 1,
  RF_TERMINAL = 2,
  RF_CANCELLED = 4,
  RF_STALE = 8,
  RF_CORRECT = 16,
  RF_EARLY = 32,
  RF_LOCAL_SID = 64,  // `a` holds an item-local spawn ordinal until commit
};

struct Rec {
  double t;
  double x;  // reward r / answer weight
  u64 y;     // admit seed / promote ready tokens
  int q;
  u32 node;
  int a, b, c;
  u8 kind, flags;
  u16 pad;
};
static_assert(sizeof(Rec) == 48, "Rec layout");

struct SpawnRec {
  int q;
  u32 node;
  int tokens;
  int cancelled;
  int kvp;  // tree-KV pages to allocate at commit (0: none)
};

struct PushRec {
  int q;
  u32 node;
};

// Error codes: 1 + totsim::Errc ordinal (errors.hpp:9-28), plus capacity errors.
enum : int {
  ERR_NONE = 0,
  ERR_UNKNOWN_PARENT = 1,
  ERR_PARENT_PRUNED = 2,
  ERR_NOT_SPECULATIVE = 3,
  ERR_UNKNOWN_NODE = 4,
  ERR_ILLEGAL_TRANSITION = 5,
  ERR_ZERO_VISITS = 6,
  ERR_NO_CHILDREN = 7,
  ERR_EMPTY_REWARDS = 8,
  ERR_SEARCH_COMPLETE = 9,
  ERR_NOTHING_EXPANDABLE = 10,
  ERR_UNKNOWN_SPECULATION = 11,
  ERR_NEGATIVE_WEIGHT = 12,
  ERR_EMPTY_TALLY = 13,
  ERR_EMPTY_BATCH = 14,
  ERR_CONFIG_INVALID = 15,
  ERR_INCOMPLETE_LOG = 16,
  ERR_IO_FAILURE = 17,
  ERR_INVALID_ARGUMENT = 18,
  ERR_CAP_NODES = 100,
  ERR_CAP_STREAMS = 101,
  ERR_CAP_LOG = 102,
  ERR_CAP_STAGE = 103,
  ERR_CAP_LABELS = 104,
  ERR_STALLED = 105,
  ERR_INTERNAL = 106,
  ERR_CAP_KV = 107,  // the live tree KV exceeds the pool (pages) or the page table
};

struct Cfg {
  // policy (policy.hpp:27-40)
  int family;
  double exploration_c;
  double balance_temperature;
  int width;
  int n_depth_widths;
  int depth_widths[kMaxDepthWidths];
  int target_answers;
  int max_depth;
  // workload (sim.hpp:82-108)
  double token_mu, token_sigma;
  int token_min, token_max;
  int shallow_min;
  double shallow_p;
  int shallow_max;
  int deep_min;
  double deep_p;
  int deep_max;
  double skew, golden_density, reward_on, reward_off, noise_sigma;
  double correct_base, correct_slope, correct_floor;
  int answer_alphabet, prompt_tokens;
  // hardware (budget.hpp:13-22)
  double weight_bytes, mem_bandwidth, peak_compute, flops_per_token, kv_bytes_per_token,
      reward_latency;
  // budget / termination (config.hpp:29-39)
  double tau, ema_alpha, initial_hit_ema;
  double term_alpha, min_frac;
  int min_answers;
  // run
  int batch_size, n_queries, spec_k, max_producers;
  int t1, t2, t3;
  int producer_slots;
  u64 run_seed;
  // capacities / options
  int node_cap;
  int stream_cap;
  int log_cap;
  int stage_cap;   // records per warp stage
  int trace;       // emit the event log
  int record_sched;    // record the decode/PRM schedule for the model forward
  int sched_cap;       // schedule entries
  int sched_rows_cap;  // schedule rows
  // Query shard whose model work this rank runs ([shard_lo, shard_hi)); the
  // search itself (every query) is replicated, so decisions are unaffected.
  int shard_lo, shard_hi;
  // Paged tree-KV store (0 pages: no model attached, no KV bookkeeping).
  int kv_pages;     // physical pages in the pools
  int kv_pp_root;   // pages of a root prompt (static: query q owns pages [q*pp, (q+1)*pp))
  i64 kv_pt_cap;    // page-table entries
  // Reward source: 0 = the content oracle (RewardOracle::reward, sim.cpp:146-152,
  // the reference); 1 = the PRM score of the thought (K4), awaited on device.
  int reward_prm;
  // Split multi-GPU mode: this run is rank split_rank of the
  // split_world query blocks of one job. Local query q is the job's query
  // q + q_offset (its seed and golden label), the decode engine and clock are
  // this rank's own, and T2 budget allocation is global through the ranks'
  // outboxes (ctl_run.h split_exchange). split_world = 1: the single server.
  int split_world, split_rank, q_offset, split_qmax;
  i64 split_epoch;     // run id tagging the outbox flags (>= 1)
  i64 xch_slot_bytes;  // bytes of one outbox slot
  int lex_rank[kMaxLabels];   // label index -> rank of "a<idx>" in std::map order
  int lex_order[kMaxLabels];  // rank -> label index
};

SPEX_HD bool q_owned(const Cfg& c, int q) { return q >= c.shard_lo && q < c.shard_hi; }

SPEX_HD int budget_at(const Cfg& c, int depth) {
  if (depth >= 0 && depth < c.n_depth_widths) return c.depth_widths[depth];
  return c.width;
}

// split mode outboxes (ctl_run.h split_exchange): header bytes, most ranks
constexpr int kXchHead = 64;
constexpr int kMaxSplit = 64;

struct QueryRun {
  u64 seed;
  double hit_ema, kv_bytes, finish_time;
  i64 live_cache;  // live_cache_tokens (executor.cpp:662-672), maintained incrementally
  i64 generated, committed, reused, wasted;
  int golden;
  int nnodes;
  int recorded;
  int pending_rewards;
  int admitted, finished, early, correct;
  int rollout_active;
  u32 chain_tip;
  u32 rest_cur;
  int rest_sp;
  int batch_pending;   // |batch_pending|
  int layer_n, cohort_n;
  int cohort_pending;  // |cohort_pending|
  int n_answers;       // AnswerTally::n_total_
  int n_labels;        // by_label_.size()
  int n_active_exp;    // |active_expansions|
  int cancelled_inflight;
  int terminal_count;  // terminal_answer_count()
  int capacity, pending_specs;
  u32 version, plan_empty_version;
  int need_followup;
  int grant;
  int hits[kMaxTracked + 1], misses[kMaxTracked + 1];
};

static_assert(sizeof(QueryRun) % 16 == 0, "QueryRun is staged to shared memory in 16-byte units");

// AnswerTally::by_label_ (termination.hpp:15-43), by label index; kept apart
// from QueryRun so the hot per-query records stay small (shared-memory resident
// in the control kernel).
struct QueryTally {
  int count[kMaxLabels];
  double w[kMaxLabels];
};

// Global scalars of one run (the executor's Impl scalars + engine scalars).
struct GState {
  double now, engine_now;
  double compute_, mem_a_, mem_d_;
  double makespan;
  i64 u_anc;     // sum over distinct (tree, strict ancestor of an active member) token_len
  i64 u_anc_own;  // the same over the owned query shard (model-work accounting only)
  i64 sum_done;  // sum of partial tokens over active members
  int next_sid;
  int finished_count, admitted_count;
  int log_n;
  int fifo_head, fifo_tail;
  int n_live, n_active_region, n_act, n_staged;
  int nfins;
  int error;
  int error_q;
  u32 error_node;
  int iterations, epochs, reward_events, decode_steps;
  // scratch scalars broadcast between phases
  int s_n_items, s_flag, s_k_total, s_leftover;
  double s_limit, s_total;
  i64 decode_rows;  // sum over decode steps of active rows (model work)
  i64 kv_next;      // next free page-table entry (bump: entries are never reused)
  i64 kv_bump;      // next never-used physical page
  i64 kv_free_head, kv_free_tail;  // FIFO ring of freed physical pages (kv_free)
  i64 kv_live, kv_peak, kv_freed;  // pages held by live thoughts (peak) and pages freed
  int n_sched, n_sched_rows;
  int n_dirty;    // queries pushed on q_dirty since the last follow-up pass
  int pad_dirty;
  i64 start_ns;   // device wall clock at the start of the run
  i64 reward_wait_ns;  // time the control spent waiting for PRM scores (reward_prm)
  // stepwise execution (spex_frontier_step): 0 not started, 1 admitted and
  // paused between calls, 2 finished; step_iters = consumer-loop iterations of
  // the next launch (0: run to the end)
  int phase, pad_phase;
  i64 step_iters;
  i64 xch_rounds;      // split mode: budget exchange rounds of this rank
  i64 xch_wait_ns;     // split mode: time spent waiting for the other ranks
  // device cycle counters per phase (thread 0's view)
  i64 cyc[8];
};

// Schedule entry published to the host (pinned, mapped) while the control
// kernel runs, so the model forward for it can start immediately.
struct PubEntry {
  int kind, steps, off, n, rows, tiles;
  i64 u0;
  i64 kv_next;
};

struct PubHead {
  int n_sched;
  int done;
  int error;
  int pad;
};

struct Run {
  Cfg cfg;
  GState* g;
  // node arrays
  u32* n_parent;
  int* n_depth;
  int* n_slot;
  int* n_tokens;
  u8* n_status;
  u16* n_flags;
  double* n_reward;
  double* n_value;
  int* n_visits;
  u64* n_hash;
  u32* n_first_child;
  u32* n_last_child;
  u32* n_next_sib;
  int* n_nchildren;
  int* n_pred;
  int* n_stream;  // stream_of: >=0 global sid, <= -2 item-local spawn (-2-k), -1 none
  i64* n_ready;
  int* n_refc;    // active-descendant count (unique_kv_tokens bookkeeping)
  i64* n_kvbase;  // first page-table entry of the node's thought (-1: no pages)
  int* n_kvh;     // tree-KV holds: own pin + live children + running stream; 0 frees the pages
  int* kv_pt;     // page table [kv_pt_cap]: physical page of each entry
  int* kv_free;   // freed physical pages, FIFO ring [kv_pages]
  // PRM-scored rewards (cfg.reward_prm): the forward writes each scored
  // thought's score and raises its schedule entry's flag
  float* n_score;  // [NN]
  int* n_prm_e;    // [NN] schedule entry that scores the node
  int* prm_done;   // [sched_cap]
  // per-query
  QueryRun* qs;
  QueryTally* q_tally;
  i64* q_finish_ns;  // device wall clock (globaltimer) at each query's query_done
  int* q_dirty;      // queries whose need_followup went 0 -> 1 (unordered; follow-up work list)
  u32* q_rest_stack;
  u32* q_layer;
  u32* q_cohort;
  // streams
  int* st_q;
  u32* st_node;
  int* st_rem;
  int* st_done;
  u8* st_state;
  u8* st_cancel;
  double* st_ready;
  int* live;      // [stream_cap]
  int* live_tmp;  // [stream_cap]
  int* fins;      // [stream_cap] sids finishing at the current boundary
  int* fin_tokens;
  int* fin_cancel;
  // event fifo
  double* ev_time;
  int* ev_q;
  u32* ev_node;
  // log
  Rec* log;
  // per-thread staging (nthreads * stage_cap)
  Rec* stage_rec;
  SpawnRec* stage_spawn;
  PushRec* stage_push;
  // per-item descriptors [item_cap]
  int* it_key;  // query or fin index
  int* it_warp;
  int* it_rec_off;
  int* it_rec_n;
  int* it_spawn_off;
  int* it_spawn_n;
  int* it_push_off;
  int* it_push_n;
  int* it_fin;     // query finished inside this item
  int* it_sdelta;  // stream_count delta
  int* it_tok;     // tokens spawned by the item (KV slots to allocate)
  int* it_scan_e;
  int* fin_scored; // completion was not stale: the thought goes to the PRM
  // schedule for the model forward
  int* sched_kind;
  int* sched_steps;
  int* sched_off;
  int* sched_n;
  int* srow_sid;
  int* srow_pos0;
  i64* sched_u;  // engine unique KV tokens at the start of a decode epoch
  int* srow_rstart;  // PRM entries: first row of each thought in the entry
  int* srow_tstart;  // PRM entries: first tile of each thought in the entry
  PubHead* pub;      // host-mapped (nullptr: no streaming)
  PubEntry* pub_e;
  int* it_scan_a;  // scan scratch
  int* it_scan_b;
  int* it_scan_c;
  int* it_scan_d;
  int item_cap;
  // per-thread speculation scratch (nthreads * (node_cap + 64))
  int* sp_visits;
  double* sp_value;
  int* sp_nchild;
  u32* sp_stack;  // prune / generic stack per warp
  double* sp_dbl;  // rebase / alloc scratch per warp (node_cap)
  int* sp_int;
  // block-level scratch for allocation [n_queries]
  int* al_cand;
  double* al_score;
  double* al_w;
  int* al_out;
  int* al_rank;
  int* al_order;
  // split mode: the ranks' outboxes (peer-mapped device pointers), [split_rank] own
  char* const* xch;
  // host-built glibc log table for integer arguments (UCB)
  const double* log_tab;
  int log_tab_n;
  int nwarps;
};

}  // namespace spex
