/*
 * spex.h — C-ABI drop-in boundary of the B200 frontier-expansion path.
 *
 * The reference (totsim, C++20) has no C ABI; its seams are the concrete C++
 * classes the executor owns. Each entry point below replaces
 * one of them and is what a reference-side binding would call:
 *
 *   spex_executor_create/run  <- totsim::Executor(cfg, seed, flags, trace) + run()
 *   spex_frontier_step        <- one main_loop iteration at a time (executor.cpp:785-807)
 *                                (proj/include/totsim/executor.hpp:50-58,
 *                                 proj/src/executor.cpp:809-860)
 *   spex_run                  <- Executor::run with a TraceWriter sink, events streamed
 *   spex_run_once             <- totsim::run_once (proj/include/totsim/experiment.hpp:27,
 *                                 proj/src/experiment.cpp:23-30)
 *   spex_canonical_config     <- ExperimentConfig::from_json + to_json
 *                                (proj/src/config.cpp:73-137,177-275)
 *   spex_totals               <- totsim::RunTotals (executor.hpp:20-33)
 *   spex_policy_ucb_score / ucb_select / rebase_widths
 *                             <- totsim::ucb_score / ucb_select / rebase_widths
 *                                (policy.hpp:43-70, policy.cpp:25-118)
 *   spex_budget_k_total / allocate
 *                             <- totsim::roofline_k_total / allocate_budgets
 *                                (budget.hpp:37-55, budget.cpp:23-96)
 *   spex_tree_transition_legal / prune_subtree
 *                             <- totsim::transition_legal, SearchTree::prune_subtree (tree.cpp:23-45,119-141)
 *   spex_speculation_dfs_plan <- totsim::dfs_speculative_select (speculation.cpp:182-218)
 *   spex_termination_should_terminate
 *                             <- totsim::AnswerTally::should_terminate (termination.cpp:30-48)
 *   spex_engine_advance       <- totsim::DecodeEngine::advance (sim.cpp:305-384)
 *   spex_engine_create / add_stream / cancel / drop / step / done_tokens ...
 *                             <- totsim::DecodeEngine as a handle (sim.hpp:165-220)
 *   spex_content_token_len / eval
 *                             <- RewardOracle::token_len / is_terminal / reward /
 *                                answer_label (sim.cpp:112-169)
 *   spex_score_batch          <- RewardOracle::reward realised by the PRM, standalone
 *   spex_executor_set_reward_source
 *                             <- RewardOracle::reward (sim.hpp:115-142), the
 *                                content oracle or the PRM's score (model mode)
 *
 * Conventions: plain pointers and sizes, no exceptions across the ABI, status
 * 0 = ok, otherwise totsim::Errc ordinal + 1 (errors.hpp:9-28) or >= 100 for
 * capacity/device failures. One CUDA stream per executor handle; distinct
 * handles may be driven from different threads (single writer per handle, as
 * executor.hpp:92-99 requires); runs with a model attached share the
 * process-wide model cache and take turns on a process lock. Memory returned
 * through char** is released with spex_free.
 */
#ifndef SPEX_H_
#define SPEX_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPEX_MAX_TRACKED 8 /* executor.hpp:16 kMaxTrackedDistance */

typedef struct spex_totals {
  double makespan;
  long long generated_tokens;
  long long committed_tokens;
  long long reused_tokens;
  long long wasted_tokens;
  long long hits[SPEX_MAX_TRACKED + 1];   /* index 1..8 */
  long long misses[SPEX_MAX_TRACKED + 1]; /* index 1..8 */
  int queries;
  int correct_votes;
  int early_terminated;
  int pad_;
} spex_totals;

typedef struct spex_stats {
  long long iterations;     /* consumer-loop iterations (main_loop) */
  long long epochs;         /* engine epochs that ended at a completion */
  long long reward_events;  /* reward events handled */
  long long decode_steps;   /* virtual decode steps run by the engine */
  long long decode_rows;    /* sum over decode steps of active streams */
  long long log_records;    /* binary event records produced */
  long long nodes;          /* thought nodes created */
  double device_ms;         /* CUDA-event time of the control kernel */
} spex_stats;

typedef struct spex_model_stats {
  double model_ms;        /* device time of the policy/PRM forward (CUDA events) */
  double attn_ms;         /* summed device time of the K1 tree-attention launches */
  long long attn_launches;
  double attn_alg_bytes;  /* algorithmic K1 bytes: unique KV tokens x bytes/token x layers */
  long long decode_rows;  /* policy rows (one token of one stream) */
  long long decode_steps;
  long long prefill_rows; /* root prompt rows (each model) */
  long long prm_rows;     /* PRM rows (tokens of scored thoughts) */
  long long prm_thoughts;
  double policy_flops;    /* 2 * projection params * rows */
  double prm_flops;
  long long launches;     /* kernels of this library launched by the forward (cuBLAS excluded) */
  long long gemm_calls;   /* cuBLAS GEMM calls */
  double control_ms;      /* control kernel device time (overlapped with the forward when streaming) */
  double step_ms;         /* device time of the whole search: control start -> last kernel (CUDA events) */
  int streamed;           /* 1: the forward ran concurrently with the control kernel */
  int pad_;
} spex_model_stats;

/* Paged tree-KV store of the last run (pages of page_tokens tokens in the
 * policy and PRM KV pools; the root prompts hold root_pages static pages). */
typedef struct spex_kv_stats {
  long long pages;             /* pool pages */
  long long page_tokens;       /* tokens per page (16) */
  long long root_pages;        /* static root-prompt pages */
  long long peak_pages;        /* most pages held by live thoughts at once */
  long long freed_pages;       /* pages returned to the free ring */
  long long live_pages_end;    /* pages still held at the end (roots + undrained) */
  long long allocated_pages;   /* page-table entries handed out (root + thought pages) */
  long long fresh_pages;       /* distinct pages ever touched (high-water mark of the pool) */
  long long page_table_entries;
} spex_kv_stats;

/* Per decode row-step shadow output (K3): argmax, logsumexp, logit sum. */
typedef struct spex_decode_out {
  int q;
  uint32_t node;
  int pos;
  int argmax;
  float lse;
  float logit_sum;
} spex_decode_out;

typedef struct spex_prm_out {
  int q;
  uint32_t node;
  float score;
  int pad_;
} spex_prm_out;

typedef struct spex_executor spex_executor;

/* Error text of the last failing call on this thread. */
const char* spex_last_error(void);
void spex_free(void* p);

/* 1 when the library was built for sm_100a and a CUDA device is usable. */
int spex_device_ok(void);

/* Strict config parse (unknown keys are errors) -> canonical JSON (to_json). */
int spex_canonical_config(const char* config_json, char** out_json);

/* Executor(cfg, run_seed, flags, trace). flags_csv: "t1,t2,t3" style, ""
 * for no flags, NULL to use the config's own run.flags. */
int spex_executor_create(const char* config_json, uint64_t run_seed, const char* flags_csv,
                         int device, spex_executor** out);
/* Run to completion (call once; a second call returns InvalidArgument + 1).
 * trace != 0 records the event log (trace.hpp:14-29) on the device. */
int spex_executor_run(spex_executor* ex, int trace, spex_totals* totals);
/* Stepwise execution, the fused device frontier step (SURVEY.md §8b
 * spex_frontier_step): each call runs up to `iterations` consumer-loop
 * iterations of the search on the device (executor.cpp:785-807: one engine
 * epoch with its completions and follow-ups, or one reward event; 0 = to the
 * end) and returns, the run's state staying on the device between calls.
 * `events` (spex_free) receives the event-log lines produced by this call (the
 * first call starts with run_begin, the last ends with run_end), so the
 * concatenation over calls is the run_once log byte for byte; *done = 1 after
 * the last. Control only (no model attached), not for split ranks; the
 * executor then counts as run (stats, log, totals). */
int spex_frontier_step(spex_executor* ex, long long iterations, int* done, char** events, size_t* events_len);
/* Event log of a traced run as JSON lines, byte-compatible with TraceWriter. */
int spex_executor_log(spex_executor* ex, char** out_lines, size_t* out_len);
int spex_executor_stats(spex_executor* ex, spex_stats* out);
/* Attach the policy/PRM forward (real decode of every scheduled row and PRM
 * scoring of every completed thought; shadow outputs in parity mode).
 * Shapes: "small_policy", "small_prm", "mid_policy", "mid_prm", "llama3_8b",
 * "prm_1p5b"; prm_shape "" disables the PRM. Call before spex_executor_run. */
int spex_executor_set_model(spex_executor* ex, const char* policy_shape, const char* prm_shape,
                            uint64_t weight_seed, int record_outputs);
/* Query-sharded model work across `world` GPUs, the search replicated: this
 * executor runs the policy/PRM forward only for queries
 * [Q*rank/world, Q*(rank+1)/world) while its control kernel still runs the
 * whole search, so every rank makes the reference's single-server decisions
 * (one virtual clock, global T2 budgets, executor.cpp:705-740) with no
 * exchange. Call before spex_executor_run. Replaces nothing in the reference
 * (one server); SURVEY.md §8e. */
int spex_executor_set_shard(spex_executor* ex, int rank, int world);

/* Split mode (north_star's multi-GPU data path): one job of Q
 * queries over `world` GPUs, rank r owning query block [Q*r/world,
 * Q*(r+1)/world) with its OWN decode engine, clock and tree KV. The only
 * exchange is T2's: the k-th allocate_budgets call of every rank
 * (executor.cpp:727-733) is one round in which each rank posts its idle
 * producer slots and its candidates' (score, capacity) to its outbox and the
 * allocation (budget.cpp:45-96) runs over every rank's candidates in rank
 * order with k_total = the ranks' idle slots summed. The control kernels
 * exchange through the outboxes directly (peer loads over NVLink), no host
 * round trip. world = 1 is the reference's single server.
 *
 *   spex_split_outbox_bytes   bytes of one rank's outbox (-1: bad arguments)
 *   spex_split_outbox_alloc   zeroed outbox on `device` + its CUDA IPC handle
 *                             (64 bytes) for the other ranks' processes
 *   spex_split_outbox_open    map another rank's outbox (peer access)
 *   spex_executor_set_split   this executor is rank `rank`: outboxes[world]
 *                             (device pointers, [rank] its own), `epoch` a run
 *                             id >= 1, the same on every rank and new for each
 *                             run (outboxes are never reset). The executor's
 *                             n_queries becomes its block's size.
 *   spex_split_run            every rank of one job on ONE device, as CTAs of
 *                             one control launch (tests; control only); fills
 *                             out[world] with executors that have run (logs,
 *                             totals, stats; destroy each).
 *   spex_executor_split_stats exchange rounds and the time spent waiting.
 *   spex_executor_emulate_split  one rank with its model, the others beside it
 *                             on the same device (per-rank timing on one GPU).
 * Oracle: oracle/ref_split.cpp (the reference's executor, one thread per rank,
 * coupled by the same exchange). */
long long spex_split_outbox_bytes(int n_queries_job, int world);
int spex_split_outbox_alloc(int device, long long bytes, void** dptr, unsigned char* ipc_handle);
int spex_split_outbox_open(int device, const unsigned char* ipc_handle, void** dptr);
int spex_split_outbox_close(void* dptr);
int spex_split_outbox_free(void* dptr);
int spex_executor_set_split(spex_executor* ex, int rank, int world, void* const* outboxes, long long epoch);
int spex_split_run(const char* config_json, uint64_t seed, const char* flags_csv, int world, int device, int trace,
                   spex_executor** out);
int spex_executor_split_stats(spex_executor* ex, long long* rounds, double* wait_ms);
/* Single-GPU emulation of one rank of a `world`-GPU split job: this executor
 * runs rank `rank` (with its model, if attached) while the other ranks'
 * control kernels run beside it on the same device (CTAs of one launch,
 * control only), exchanging through outboxes in this device's memory. The
 * exchange is timing-independent, so the rank's decisions, log and model work
 * are those of the multi-GPU run; its step time is the multi-GPU one up to the
 * world - 1 SMs the other ranks' control occupies. */
int spex_executor_emulate_split(spex_executor* ex, int rank, int world);
int spex_executor_model_stats(spex_executor* ex, spex_model_stats* out);
/* Tree-KV pool size in pages (0 = the default: the resident pools, else 70%
 * of free HBM). Pages of dead thoughts (pruned, REBASE layers expanded,
 * scored terminals, finished queries) are reused (no reference counterpart:
 * the reference holds no KV, SearchTree::prune_subtree tree.cpp:119-141 and
 * finish_query executor.cpp:234-336 define when a thought dies). The run fails
 * with CapacityTreeKV when the live thoughts exceed the pool. Call before
 * spex_executor_run; with the host emulation library it enables the page
 * bookkeeping without a model. */
int spex_executor_set_kv_pages(spex_executor* ex, long long pages);
int spex_executor_kv_stats(spex_executor* ex, spex_kv_stats* out);
/* Copies up to cap records; *n receives the total available. */
int spex_executor_decode_outputs(spex_executor* ex, void* buf, long long cap, long long* n);
int spex_executor_prm_outputs(spex_executor* ex, void* buf, long long cap, long long* n);
/* n independent searches of one config (seeds[0..n)) in ONE launch of the
 * control kernel, one CTA per search (the device analog of run_experiment_full's
 * OpenMP loop over repetitions, experiment.cpp:61-78); control only (no model,
 * no trace). totals[n]; device_ms = the launch's CUDA-event time. */
int spex_run_batch(const char* config_json, const uint64_t* seeds, int n, const char* flags_csv, int device,
                   spex_totals* totals, double* device_ms);

/* Reward source: 0 = the content oracle (RewardOracle::reward, sim.cpp:146-152;
 * the reference, event logs byte-compatible), 1 = the PRM score of the
 * thought (K4; "model mode"). With 1 the control kernel waits on device for
 * each scored thought's PRM batch before its reward event, so the search is
 * steered by the model; needs set_model with a PRM, no shard, the streamed
 * forward. Call before spex_executor_run. */
int spex_executor_set_reward_source(spex_executor* ex, int source);
/* Device wall-clock latency of each query (ms from the run's start to its
 * query_done; -1 if unfinished) and the total time the control kernel spent
 * waiting for PRM scores. */
int spex_executor_query_wall_ms(spex_executor* ex, double* out, int cap, int* n, double* reward_wait_ms);

/* Per-query virtual finish time (query_done.t; admission is at t = 0 when
 * batch_size = n_queries): the search latency of each query. */
int spex_executor_query_finish(spex_executor* ex, double* out, int cap, int* n);
void spex_executor_destroy(spex_executor* ex);

/* ---- policy and budget hooks (csrc/spex_hooks.cu): the reference's free
 * functions as batched device calls running the control kernel's own
 * arithmetic. Per-problem status: 0 ok, else Errc ordinal + 1. */
/* ucb_score (policy.hpp:43-47): n independent scores. */
int spex_policy_ucb_score(const double* value, const int* child_visits, const int* parent_visits, int n,
                          double exploration_c, double* out, int* status);
/* ucb_select (policy.hpp:49-55): problem p's children are entries
 * [offsets[p], offsets[p+1]) in NodeId order; out[p] = the chosen child's
 * index within its problem. */
int spex_policy_ucb_select(const double* value, const int* visits, const int* pruned, const int* offsets,
                           const int* parent_visits, int n_problems, double exploration_c, int* out, int* status);
/* rebase_widths (policy.hpp:63-70): problem p's rewards are entries
 * [offsets[p], offsets[p+1]); sum_preserving = WidthMode::SumPreserving. */
int spex_policy_rebase_widths(const double* rewards, const int* offsets, const int* budgets, int n_problems,
                              double temperature, int sum_preserving, int* widths, int* status);
/* roofline_k_total (budget.hpp:37-42); hw4 = {weight_bytes, mem_bandwidth,
 * peak_compute, flops_per_token}. */
int spex_budget_k_total(const double* hw4, int active_batch, double avg_kv_bytes, int cap, int* out);
/* allocate_budgets (budget.hpp:47-55) over n queries (capacity, hit_ema,
 * kv_bytes), query_score = capacity * hit_ema * (weight_bytes + kv_bytes). */
int spex_budget_allocate(const int* capacity, const double* hit_ema, const double* kv_bytes, int n, int k_total,
                         double tau, double weight_bytes, int* out);

/* ---- content hooks: RewardOracle (sim.hpp:115-142) evaluated on the device
 * with the search's own draws (glibc exp/log/cos restated bit for bit). */
typedef struct spex_workload { /* WorkloadSpec (sim.hpp:82-108) */
  double token_mu, token_sigma;
  int token_min, token_max;
  int shallow_min;
  int shallow_max;
  double shallow_p;
  int deep_min;
  int deep_max;
  double deep_p;
  double skew, golden_density, reward_on, reward_off, noise_sigma;
  double correct_base, correct_slope, correct_floor;
  int answer_alphabet, prompt_tokens;
} spex_workload;
/* token_len (sim.cpp:112-115) of n child path hashes. */
int spex_content_token_len(const uint64_t* child_hash, int n, const spex_workload* wl, int* out);
/* is_terminal / reward / answer_label (sim.cpp:117-169) of n nodes of one
 * query: node i's path is path_hash[offsets[i] .. offsets[i+1]) = the path
 * hashes of its depth-1 ancestor .. itself (empty: the root). Labels are the
 * index k of "a<k>". */
int spex_content_eval(const uint64_t* path_hash, const int* offsets, int n, uint64_t query_seed, int max_depth,
                      const spex_workload* wl, int* terminal, double* reward, int* label);

/* ---- expand seam: DecodeEngine::advance (sim.hpp:165-220, sim.cpp:305-384)
 * on the device. The engine's active and staged stream vectors go in and come
 * back out in the reference's order; each stream lists its strict ancestors
 * as entries [anc_off, anc_off + anc_n) of anc_key (one key per distinct
 * (tree, node), tokens in anc_tokens[key]) for the unique-KV-token cost.
 * Completions come back in active order (cap entries; CapacityStage when more). */
typedef struct spex_engine_hw { /* HardwareProfile (budget.hpp:13-22) */
  double weight_bytes, mem_bandwidth, peak_compute, flops_per_token, kv_bytes_per_token, reward_latency;
} spex_engine_hw;
typedef struct spex_engine_stream {
  int id, remaining, done, cancelled;
  double ready;
  int anc_off, anc_n;
} spex_engine_stream;
typedef struct spex_engine_finished {
  int id, tokens_done, cancelled, pad;
  double time;
} spex_engine_finished;
int spex_engine_advance(const spex_engine_hw* hw, double now, double limit, spex_engine_stream* active,
                        int* n_active, spex_engine_stream* staged, int* n_staged, const int* anc_key,
                        const int* anc_tokens, int n_keys, spex_engine_finished* out, int cap, int* n_out,
                        double* now_out);

/* Tree maintenance hooks (tree.hpp:43,104): transition_legal (tree.cpp:23-45)
 * for n (from, to) NodeStatus pairs, and SearchTree::prune_subtree
 * (tree.cpp:119-141) on one tree given by parents (parent[0] = -1, children in
 * NodeId order) and statuses — the statuses are updated in place, *pruned =
 * the nodes newly tombstoned; UnknownNode + 1 for an id outside the tree. The
 * control kernel's own transition_legal / prune_subtree. */
int spex_tree_transition_legal(const uint8_t* from, const uint8_t* to, int n, uint8_t* out);
int spex_tree_prune_subtree(const int32_t* parent, uint8_t* status, int n_nodes, uint32_t id, int* pruned);

/* T1 planning hook: dfs_speculative_select (speculation.hpp:95-139,
 * speculation.cpp:182-218) on one tree, on the device with the control
 * kernel's dfs_plan (Algorithm 1's simulated selections over a visit overlay
 * with phantom children). The tree: n_nodes nodes in NodeId order (children in
 * NodeId order, as add_node appends them), parent[0] = -1, status = the
 * NodeStatus ordinal, bits = terminal | gen_done << 1 | has_reward << 2, the
 * reward where present; the PolicyConfig fields; k <= 64. Writes up to k
 * targets (node, predicted distance); 0 targets for rebase_bfs (frontier
 * policies plan by allocation). */
int spex_speculation_dfs_plan(const int32_t* parent, const uint8_t* status, const uint8_t* bits, const double* reward,
                              const int32_t* visits, const double* value, const int32_t* depth, int n_nodes,
                              int terminal_answers, int family, double exploration_c, int width,
                              const int32_t* depth_widths, int n_depth_widths, int target_answers, int k,
                              uint32_t* out_node, int32_t* out_dist, int* n_out);

/* Termination hook: AnswerTally::should_terminate (termination.hpp:15-55,
 * termination.cpp:30-48) for n_tallies tallies, on the device with the
 * control kernel's own code. Tally t's labels are [offsets[t],
 * offsets[t + 1]) in the tally's label (std::map) order with their answer
 * counts and weight sums; n_total[t] its answer count; out[t] = 0/1. */
int spex_termination_should_terminate(const int* counts, const double* weights, const int* offsets,
                                      const int* n_total, int n_tallies, int min_answers, double alpha, int* out);

/* The decode engine as a handle (SURVEY.md §8b spex_engine_*; DecodeEngine,
 * sim.hpp:165-220): the stream tables on the host side of the handle, each
 * step's epochs on the device (the same code as spex_engine_advance). A stream
 * names its strict ancestors by caller keys, unique per (tree, node) — e.g.
 * tree << 32 | node — with their token lengths; the unique-KV-token cost
 * (sim.cpp:54-78) deduplicates by key as the reference does by (tree, node).
 *   spex_engine_create / destroy   DecodeEngine(hw)
 *   spex_engine_add_stream         add_stream(id, tree, node, tokens, ready)   sim.cpp:204-214
 *   spex_engine_cancel             cancel(id), *started = its return value      sim.cpp:216-233
 *   spex_engine_drop               drop(id)                                     sim.cpp:235-249
 *   spex_engine_step               advance(now, limit, out): finished streams
 *                                  in out[cap], *reached = the clock reached    sim.cpp:305-384
 *   spex_engine_done_tokens / stream_count / active_count / next_ready
 * Stream ids must be unique among the handle's streams (the reference looks
 * them up by id, first match). */
typedef struct spex_engine spex_engine;
int spex_engine_create(const spex_engine_hw* hw, int device, spex_engine** out);
void spex_engine_destroy(spex_engine* e);
int spex_engine_add_stream(spex_engine* e, int id, uint32_t node, int tokens, double ready, const uint64_t* anc_keys,
                           const int* anc_tokens, int n_anc);
int spex_engine_cancel(spex_engine* e, int id, int* started);
int spex_engine_drop(spex_engine* e, int id);
int spex_engine_step(spex_engine* e, double now, double limit, spex_engine_finished* out, int cap, int* n_out,
                     double* reached);
int spex_engine_done_tokens(const spex_engine* e, int id);
int spex_engine_stream_count(const spex_engine* e);
int spex_engine_active_count(const spex_engine* e);
double spex_engine_next_ready(const spex_engine* e);

/* PRM scoring of standalone token sequences (SURVEY.md §8b spex_score_batch;
 * the score hook RewardOracle::reward, sim.hpp:115-142, realised by the PRM):
 * sequence i is tokens[offsets[i], offsets[i + 1]), scores[i] the PRM's
 * value-head score (sigmoid) at its last token — the executor's PRM arithmetic
 * (K4 prefill tiles on the tensor cores) with the weights
 * spex_executor_set_model gives the PRM for the same weight_seed. Host buffers
 * in and out; InvalidArgument for an unknown shape, an empty sequence or a
 * token outside the vocabulary. */
int spex_score_batch(const char* prm_shape, uint64_t weight_seed, const int32_t* tokens, const int64_t* offsets,
                     int n, float* scores, int device);

/* spex_run (SURVEY.md §8b spex_run(config, seed, flags, trace_cb)): the whole
 * run stepped through spex_frontier_step `chunk` consumer-loop iterations at a
 * time (<= 0: 4096), each event-log line handed to trace_cb as it is produced
 * (line without its newline, its length, `user`); the lines are the run_once
 * log. trace_cb may be NULL. */
typedef void (*spex_trace_cb)(const char* line, size_t len, void* user);
int spex_run(const char* config_json, uint64_t seed, const char* flags_csv, spex_trace_cb trace_cb, void* user,
             long long chunk, spex_totals* totals);

/* run_once: traced run returning totals and the JSON-lines log. */
int spex_run_once(const char* config_json, uint64_t seed, const char* flags_csv,
                  spex_totals* totals, char** out_lines);

#ifdef __cplusplus
}
#endif

#endif /* SPEX_H_ */
