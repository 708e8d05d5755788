// model_host.h — host interface of the policy / PRM schedule replay.
#pragma once

#include <cuda_runtime.h>

#include <string>
#include <utility>
#include <cstdio>
#include <vector>

#include "ctl_state.h"
#include "model.h"

namespace spex {

struct ModelRunConfig {
  ModelShape policy;
  ModelShape prm;
  bool with_prm = true;
  unsigned long long seed = 1;
  bool time_attn = true;
  bool record_outputs = false;
  void* out_rows = nullptr;  // DecodeOut[out_rows_cap] (device)
  long long out_rows_cap = 0;
  void* out_scores = nullptr;  // PrmOut[out_scores_cap] (device)
  long long out_scores_cap = 0;
};

struct ScheduleView {
  TreeView tree;
  int n_queries;
  int shard_lo = 0, shard_hi = 0;  // owned query range [lo, hi): prompt prefill (the schedule arrives filtered)
  long long kv_slots;        // tree KV pool capacity (slots)
  int max_decode_rows;       // row-buffer capacity for decode steps (larger entries are chunked)
  int max_prm_rows;          // row-buffer capacity for one PRM batch
  // finished schedule (sequential mode)
  int n_entries = 0;
  const PubEntry* entries_host = nullptr;
  // live schedule (streaming mode; host-mapped, written by the control kernel)
  void* pub_head = nullptr;
  void* pub_entries = nullptr;
  const int* srow_sid;
  const int* srow_pos0;
  const int* srow_rstart;
  const int* srow_tstart;
  // PRM rewards (reward source 1): each scored thought's score at node_score[q*node_cap+node],
  // then prm_done[entry] = 1 (the control kernel waits on it)
  float* node_score = nullptr;
  int* prm_done = nullptr;
};

struct ModelRunResult {
  double model_ms = 0.0;
  double attn_ms = 0.0;
  long long attn_launches = 0;
  double attn_alg_bytes = 0.0;
  long long decode_rows = 0, decode_steps = 0, prefill_rows = 0, prm_rows = 0, prm_thoughts = 0;
  long long out_rows = 0, out_scores = 0;
  double policy_flops = 0.0, prm_flops = 0.0;
  int control_error = 0;
  double control_ms = 0.0;
  long long launches = 0;  // kernels of this library launched by the replay (cuBLAS excluded)
  long long gemm_calls = 0;
  double step_ms = 0.0;  // control start -> last of (control end, forward end), CUDA events
  int streamed = 0;      // 1: forward overlapped with the control kernel; 0: replayed after it
};

struct AttnTimer {
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;
  int n = 0;
  double total_ms = 0.0;
  int control_error = 0;
  double control_ms = 0.0;
  long long launches = 0;
  double cur_bytes = 0.0;       // algorithmic bytes of each launch of the current forward
  std::vector<double> bytes;    // per pending launch
  FILE* dump = nullptr;         // SPEX_ATTN_LOG: one line per launch (index, alg bytes, ms)
  void begin(cudaStream_t st);
  void end(cudaStream_t st);
  void flush();
  ~AttnTimer();
};

ModelShape shape_by_name(const std::string& name);
long long model_weight_params(const ModelShape& s, bool prm);
double model_matmul_flops_per_row(const ModelShape& s, bool prm);
void run_model_schedule(const ModelRunConfig& mc, const ScheduleView& sv, ModelRunResult* res, cudaStream_t st);
// PRM scores of standalone token sequences (spex_score_batch): sequence i is
// tokens[offsets[i], offsets[i + 1]); scores[i] = the value head at its last token.
void prm_score_sequences(const ModelShape& sh, uint64_t weight_seed, const int* tokens, const long long* offsets,
                         int n, float* scores, int device);

}  // namespace spex
