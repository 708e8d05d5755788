// spex_hooks.cu — the reference's policy and budget hooks as batched device
// calls over the C ABI (include/spex.h, SURVEY.md §8b "policy hooks"):
//
//   spex_policy_ucb_score      <- totsim::ucb_score        (policy.cpp:22-30)
//   spex_policy_ucb_select     <- totsim::ucb_select       (policy.cpp:32-51)
//   spex_policy_rebase_widths  <- totsim::rebase_widths    (policy.cpp:65-118)
//   spex_budget_k_total        <- totsim::roofline_k_total (budget.cpp:23-39)
//   spex_budget_allocate       <- totsim::allocate_budgets (budget.cpp:45-96)
//   spex_content_token_len     <- RewardOracle::token_len  (sim.cpp:112-115)
//   spex_content_eval          <- RewardOracle::is_terminal / reward / answer_label
//                                 (sim.cpp:117-169)
//   spex_engine_advance        <- DecodeEngine::advance    (sim.cpp:305-384)
//
// Each call runs the same device functions the control kernel runs inside a
// search (ctl_core.h, ctl_run.h allocate_block), so a reference-side binding
// (integration/policy_b200.cpp) that routes the reference's own calls here
// exercises exactly the in-search arithmetic; the reference's unit tests
// (tests/test_policy.cpp, test_budget.cpp) run against it on the GPU
// (tests/test_dropin_gpu.py). Batched forms take many independent problems
// per launch (one thread per problem; one block for an allocation).
// Status: 0 ok, else totsim::Errc ordinal + 1 per problem.
#include <cuda_runtime.h>

#include <cstring>
#include <mutex>
#include <vector>

#include "../../include/spex.h"
#include "ctl_run.h"
#include "hook_tree.h"

namespace spex {
namespace {

struct HookExec {
  int tid, nthr, warp, nwarp, lane, lanes;
  int* sm;
  double* smd;
  i64* sml;
  __device__ __forceinline__ void sync() { __syncthreads(); }
};

__device__ int err_of(const GState& g) { return g.error; }

// ucb_score (policy.cpp:22-30): throws ZeroVisits when either count is zero.
__global__ void ucb_score_kernel(const double* value, const int* cv, const int* pv, int n, double c, double* out,
                                 int* status) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (cv[i] <= 0 || pv[i] <= 0) {
    status[i] = ERR_ZERO_VISITS;
    out[i] = 0.0;
    return;
  }
  out[i] = value[i] + c * sqrt(glibc::log(static_cast<double>(pv[i])) / cv[i]);
  status[i] = 0;
}

// ucb_select (policy.cpp:32-51) over problem p's children [off[p], off[p+1]) in
// NodeId order: the first unvisited live child, else the strict-> argmax
// (lowest index on ties); pruned children are skipped.
__global__ void ucb_select_kernel(const double* value, const int* visits, const int* pruned, const int* off,
                                  const int* parent_visits, int n_prob, double c, int* out, int* status) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n_prob) return;
  const int a = off[p], b = off[p + 1];
  int any = 0;
  for (int i = a; i < b; ++i) {
    if (pruned[i]) continue;
    any = 1;
    if (visits[i] == 0) {
      out[p] = i - a;
      status[p] = 0;
      return;
    }
  }
  if (!any) {
    out[p] = -1;
    status[p] = ERR_NO_CHILDREN;
    return;
  }
  const int pv = parent_visits[p];
  int best = -1;
  double best_score = 0.0;
  for (int i = a; i < b; ++i) {
    if (pruned[i]) continue;
    if (visits[i] <= 0 || pv <= 0) {
      out[p] = -1;
      status[p] = ERR_ZERO_VISITS;
      return;
    }
    const double s = value[i] + c * sqrt(glibc::log(static_cast<double>(pv)) / visits[i]);
    if (best < 0 || s > best_score) {
      best = i - a;
      best_score = s;
    }
  }
  out[p] = best;
  status[p] = 0;
}

// rebase_widths (policy.cpp:65-118) per problem, through the control's own
// device function (ctl_core.h).
__global__ void rebase_widths_kernel(const double* rewards, const int* off, const int* budget, int n_prob,
                                     double temperature, int sum_preserving, int* widths, double* scratch_d,
                                     int* scratch_i, GState* gs, int* status) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n_prob) return;
  GState& g = gs[p];  // global: set_err reports through an atomic
  memset(&g, 0, sizeof(g));
  Run R;
  memset(&R, 0, sizeof(R));
  R.g = &g;
  const int a = off[p], n = off[p + 1] - off[p];
  rebase_widths(&R, p, rewards + a, n, budget[p], temperature, sum_preserving != 0, widths + a, scratch_d + 2 * a,
                scratch_d + 2 * a + n, scratch_i + a);
  status[p] = err_of(g);
}

// roofline_k_total (budget.cpp:23-39).
__global__ void k_total_kernel(double weight_bytes, double mem_bandwidth, double peak_compute, double flops_per_token,
                               int active, double avg_kv, int cap, int* out) {
  const double compute_slope = flops_per_token / peak_compute;
  const double memory_slope = avg_kv / mem_bandwidth;
  const double weight_time = weight_bytes / mem_bandwidth;
  int b_star;
  if (compute_slope <= memory_slope) {
    b_star = cap;
  } else {
    const double knee = ceil(weight_time / (compute_slope - memory_slope));
    b_star = knee < static_cast<double>(cap) ? static_cast<int>(knee) : cap;
  }
  const int k = b_star - active;
  *out = k > 0 ? k : 0;
}

// allocate_budgets (budget.cpp:45-96): one block, the control's allocate_block.
// AnswerTally::should_terminate per tally (the control kernel's tally_should_terminate)
__global__ void terminate_kernel(const int* count, const double* w, const int* off, const int* n_total, int n,
                                 int min_answers, double alpha, int* out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int b = off[t], m = off[t + 1] - b;
  int labels = 0;
  for (int r = 0; r < m; ++r) labels += count[b + r] > 0;
  out[t] = tally_should_terminate(
               n_total[t], labels, m,
               [&](int r, int* c, double* x) {
                 *c = count[b + r];
                 *x = w[b + r];
               },
               min_answers, alpha)
               ? 1
               : 0;
}

// dfs_speculative_select on one tree (the control kernel's dfs_plan)
__global__ void dfs_plan_kernel(Run* R, int k, u32* out_node, int* out_dist, int* n_out) {
  QC x = make_qc(R, 0, nullptr, 0);
  *n_out = dfs_plan(x, k, out_node, out_dist);
  if (R->g->error) *n_out = -1;
}

// SearchTree::prune_subtree on one tree (the control kernel's prune_subtree)
__global__ void prune_kernel(Run* R, u32 id, int* out) {
  QC x = make_qc(R, 0, nullptr, 0);
  *out = prune_subtree(x, id);
  if (R->g->error) *out = -1;
}

// transition_legal (tree.cpp:23-45) for n pairs
__global__ void transition_kernel(const u8* from, const u8* to, int n, u8* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = transition_legal(from[i], to[i]) ? 1 : 0;
}

__global__ void __launch_bounds__(256) allocate_kernel(const int* capacity, const double* hit_ema,
                                                       const double* kv_bytes, int n, int k_total, double tau,
                                                       double weight_bytes, double* score, double* w, int* out,
                                                       int* order) {
  __shared__ int sm[1024 + 8];
  __shared__ double smd[32];
  __shared__ long long sml[32];
  __shared__ GState g;
  HookExec ex{static_cast<int>(threadIdx.x), static_cast<int>(blockDim.x), static_cast<int>(threadIdx.x >> 5),
              static_cast<int>(blockDim.x >> 5), static_cast<int>(threadIdx.x & 31), 32, sm, smd, sml};
  for (int i = ex.tid; i < n; i += ex.nthr) score[i] = capacity[i] * hit_ema[i] * (weight_bytes + kv_bytes[i]);
  __syncthreads();
  allocate_block(ex, &g, n, k_total, tau, score, capacity, w, out, order);
}

// RewardOracle::token_len per child hash (the lognormal draw with glibc's
// own exp / log / cos, ctl_rng.h).
__global__ void token_len_kernel(const u64* h, int n, spex_workload wl, int* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = lognormal_tokens(h[i], kSaltTokens, wl.token_mu, wl.token_sigma, wl.token_min, wl.token_max);
}

// is_terminal / reward / answer_label per node (path hashes in CSR).
__global__ void content_kernel(const u64* path, const int* off, int n, u64 query_seed, int max_depth,
                               spex_workload wl, int* terminal, double* reward, int* label) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) content_eval(path + off[i], off[i + 1] - off[i], query_seed, max_depth, wl, terminal + i, reward + i,
                          label + i);
}

// DecodeEngine::advance (sim.cpp:305-384), one block: joins in staged order,
// the epoch cost series from the active set's unique KV tokens (distinct
// ancestor keys flagged in parallel, sim.cpp:54-78), epochs to the first
// completion / the limit / a pending join, completions in active order. The
// stream tables come in and go back out in the reference's vector order.
__global__ void __launch_bounds__(256) engine_advance_kernel(spex_engine_hw hw, double now, double limit,
                                                             spex_engine_stream* act, int* n_act,
                                                             spex_engine_stream* stg, int* n_stg,
                                                             const int* anc_key, const int* anc_tokens, int n_keys,
                                                             int* key_flag, spex_engine_finished* out, int cap,
                                                             int* n_out, double* now_out, int* status) {
  __shared__ GState cost;  // compute_, mem_a_, mem_d_ of the cached series
  __shared__ int s_flag, s_target, s_mlimit, s_min;
  __shared__ long long s_u;
  __shared__ double s_now;
  const int tid = threadIdx.x;
  if (tid == 0) {
    s_now = now;
    *n_out = 0;
    *status = 0;
  }
  __syncthreads();
  bool dirty = true;
  for (int guard = 0; guard < (1 << 24); ++guard) {
    if (tid == 0) {
      // joins: staged streams whose ready time has arrived, in staged order
      int na = *n_act, w = 0;
      bool joined = false;
      for (int j = 0; j < *n_stg; ++j) {
        if (stg[j].ready <= s_now + kTimeEps) {
          act[na++] = stg[j];
          joined = true;
        } else {
          stg[w++] = stg[j];
        }
      }
      *n_act = na;
      *n_stg = w;
      s_flag = joined ? 1 : 0;
      if (na == 0) {
        if (w == 0) {
          s_flag = 2;  // return limit
        } else {
          double r = HUGE_VAL;
          for (int j = 0; j < w; ++j) r = stg[j].ready < r ? stg[j].ready : r;
          if (r > limit + kTimeEps) {
            s_flag = 2;
          } else {
            s_now = r;
            s_flag = 3;  // retry the joins
          }
        }
      }
    }
    __syncthreads();
    if (s_flag == 2) {
      if (tid == 0) *now_out = limit;
      return;
    }
    if (s_flag == 3) continue;
    if (s_flag == 1) dirty = true;
    const int na = *n_act;
    if (dirty) {
      // refresh_costs: U = sum of partial tokens + distinct strict-ancestor tokens
      for (int k = tid; k < n_keys; k += blockDim.x) key_flag[k] = 0;
      if (tid == 0) s_u = 0;
      __syncthreads();
      long long part = 0;
      for (int i = tid; i < na; i += blockDim.x) {
        part += act[i].done;
        for (int a = act[i].anc_off; a < act[i].anc_off + act[i].anc_n; ++a) key_flag[anc_key[a]] = 1;
      }
      __syncthreads();
      for (int k = tid; k < n_keys; k += blockDim.x)
        if (key_flag[k]) part += anc_tokens[k];
      atomicAdd(reinterpret_cast<unsigned long long*>(&s_u), static_cast<unsigned long long>(part));
      __syncthreads();
      if (tid == 0) {
        cost.compute_ = static_cast<double>(na) * hw.flops_per_token / hw.peak_compute;
        const double kv_bytes = hw.kv_bytes_per_token * static_cast<double>(s_u);
        cost.mem_a_ = (hw.weight_bytes + kv_bytes) / hw.mem_bandwidth;
        cost.mem_d_ = hw.kv_bytes_per_token * static_cast<double>(na) / hw.mem_bandwidth;
      }
      dirty = false;
    }
    if (tid == 0) {
      int m_complete = act[0].remaining;
      for (int i = 1; i < na; ++i) m_complete = act[i].remaining < m_complete ? act[i].remaining : m_complete;
      const int m_limit = eng_steps_within(&cost, limit - s_now, m_complete);
      int target = m_complete;
      if (*n_stg > 0) {
        double r = HUGE_VAL;
        for (int j = 0; j < *n_stg; ++j) r = stg[j].ready < r ? stg[j].ready : r;
        const int cap2 = m_complete < m_limit ? m_complete : m_limit;
        if (cap2 >= 1 && s_now + eng_elapsed(&cost, cap2) >= r - kTimeEps) {
          int lo = 1, hi = cap2;
          while (hi > lo) {
            const int mid = lo + (hi - lo) / 2;
            if (s_now + eng_elapsed(&cost, mid) >= r - kTimeEps)
              hi = mid;
            else
              lo = mid + 1;
          }
          target = lo;
        }
      }
      s_mlimit = m_limit;
      s_target = target;
    }
    __syncthreads();
    if (s_target > s_mlimit) {
      // partial epoch: stop at the last boundary inside the window
      const int m = s_mlimit;
      if (m > 0) {
        for (int i = tid; i < na; i += blockDim.x) {
          act[i].done += m;
          act[i].remaining -= m;
        }
      }
      __syncthreads();
      if (tid == 0) *now_out = m > 0 ? s_now + eng_elapsed(&cost, m) : s_now;
      return;
    }
    const int target = s_target;
    for (int i = tid; i < na; i += blockDim.x) {
      act[i].done += target;
      act[i].remaining -= target;
    }
    __syncthreads();
    if (tid == 0) {
      s_now += eng_elapsed(&cost, target);
      int w = 0, f = 0;
      for (int i = 0; i < na; ++i) {
        if (act[i].remaining <= 0) {
          if (f < cap) {
            out[f].id = act[i].id;
            out[f].tokens_done = act[i].done;
            out[f].cancelled = act[i].cancelled;
            out[f].time = s_now;
          } else {
            *status = ERR_CAP_STAGE;
          }
          ++f;
        } else {
          act[w++] = act[i];
        }
      }
      *n_act = w;
      *n_out = f;
      s_flag = f > 0 ? 1 : 0;
    }
    dirty = true;
    __syncthreads();
    if (s_flag) {
      if (tid == 0) *now_out = s_now;
      return;
    }
  }
  if (tid == 0) *status = ERR_STALLED;
}

// Device buffers of the host-facing calls (one stream, serialised).
std::mutex g_hook_mu;
cudaStream_t g_hook_stream = nullptr;

struct Dev {
  std::vector<void*> ptrs;
  template <class T>
  T* put(const T* h, size_t n) {
    T* d = nullptr;
    if (cudaMallocAsync(reinterpret_cast<void**>(&d), sizeof(T) * (n ? n : 1), g_hook_stream) != cudaSuccess)
      return nullptr;
    ptrs.push_back(d);
    if (h && n) cudaMemcpyAsync(d, h, sizeof(T) * n, cudaMemcpyHostToDevice, g_hook_stream);
    return d;
  }
  template <class T>
  void get(T* h, const T* d, size_t n) {
    if (n) cudaMemcpyAsync(h, d, sizeof(T) * n, cudaMemcpyDeviceToHost, g_hook_stream);
  }
  ~Dev() {
    for (void* p : ptrs) cudaFreeAsync(p, g_hook_stream);
  }
};

int finish() {
  cudaError_t e = cudaStreamSynchronize(g_hook_stream);
  if (e == cudaSuccess) e = cudaGetLastError();
  return e == cudaSuccess ? 0 : 200;
}

int ensure_stream() {
  if (!g_hook_stream && cudaStreamCreateWithFlags(&g_hook_stream, cudaStreamNonBlocking) != cudaSuccess) return 200;
  return 0;
}

}  // namespace
}  // namespace spex

using namespace spex;

extern "C" int spex_policy_ucb_score(const double* value, const int* child_visits, const int* parent_visits, int n,
                                     double exploration_c, double* out, int* status) {
  std::lock_guard<std::mutex> lk(g_hook_mu);
  if (int rc = ensure_stream()) return rc;
  if (n <= 0) return 0;
  int rc;
  {
    Dev d;
    double* dv = d.put(value, n);
    int* dc = d.put(child_visits, n);
    int* dp = d.put(parent_visits, n);
    double* dout = d.put<double>(nullptr, n);
    int* dst = d.put<int>(nullptr, n);
    if (!dv || !dc || !dp || !dout || !dst) return 200;
    ucb_score_kernel<<<(n + 127) / 128, 128, 0, g_hook_stream>>>(dv, dc, dp, n, exploration_c, dout, dst);
    d.get(out, dout, n);
    d.get(status, dst, n);
    rc = finish();
  }
  return rc ? rc : finish();
}

extern "C" int spex_policy_ucb_select(const double* value, const int* visits, const int* pruned, const int* offsets,
                                      const int* parent_visits, int n_problems, double exploration_c, int* out,
                                      int* status) {
  std::lock_guard<std::mutex> lk(g_hook_mu);
  if (int rc = ensure_stream()) return rc;
  if (n_problems <= 0) return 0;
  const int n = offsets[n_problems];
  int rc;
  {
    Dev d;
    double* dv = d.put(value, n);
    int* dvi = d.put(visits, n);
    int* dpr = d.put(pruned, n);
    int* doff = d.put(offsets, n_problems + 1);
    int* dpv = d.put(parent_visits, n_problems);
    int* dout = d.put<int>(nullptr, n_problems);
    int* dst = d.put<int>(nullptr, n_problems);
    if (!dv || !dvi || !dpr || !doff || !dpv || !dout || !dst) return 200;
    ucb_select_kernel<<<(n_problems + 127) / 128, 128, 0, g_hook_stream>>>(dv, dvi, dpr, doff, dpv, n_problems,
                                                                          exploration_c, dout, dst);
    d.get(out, dout, n_problems);
    d.get(status, dst, n_problems);
    rc = finish();
  }
  return rc ? rc : finish();
}

extern "C" int spex_policy_rebase_widths(const double* rewards, const int* offsets, const int* budgets, int n_problems,
                                         double temperature, int sum_preserving, int* widths, int* status) {
  std::lock_guard<std::mutex> lk(g_hook_mu);
  if (int rc = ensure_stream()) return rc;
  if (n_problems <= 0) return 0;
  const int n = offsets[n_problems];
  int rc;
  {
    Dev d;
    double* dr = d.put(rewards, n);
    int* doff = d.put(offsets, n_problems + 1);
    int* db = d.put(budgets, n_problems);
    int* dw = d.put<int>(nullptr, n);
    double* sd = d.put<double>(nullptr, 2 * static_cast<size_t>(n));
    int* si = d.put<int>(nullptr, n);
    int* dst = d.put<int>(nullptr, n_problems);
    GState* dg = d.put<GState>(nullptr, n_problems);
    if (!dr || !doff || !db || !dw || !sd || !si || !dst || !dg) return 200;
    rebase_widths_kernel<<<(n_problems + 127) / 128, 128, 0, g_hook_stream>>>(dr, doff, db, n_problems, temperature,
                                                                             sum_preserving, dw, sd, si, dg, dst);
    d.get(widths, dw, n);
    d.get(status, dst, n_problems);
    rc = finish();
  }
  return rc ? rc : finish();
}

extern "C" int spex_budget_k_total(const double* hw4, int active_batch, double avg_kv_bytes, int cap, int* out) {
  std::lock_guard<std::mutex> lk(g_hook_mu);
  if (int rc = ensure_stream()) return rc;
  int rc;
  {
    Dev d;
    int* dout = d.put<int>(nullptr, 1);
    if (!dout) return 200;
    k_total_kernel<<<1, 1, 0, g_hook_stream>>>(hw4[0], hw4[1], hw4[2], hw4[3], active_batch, avg_kv_bytes, cap, dout);
    d.get(out, dout, 1);
    rc = finish();
  }
  return rc ? rc : finish();
}

extern "C" int spex_budget_allocate(const int* capacity, const double* hit_ema, const double* kv_bytes, int n,
                                    int k_total, double tau, double weight_bytes, int* out) {
  std::lock_guard<std::mutex> lk(g_hook_mu);
  for (int i = 0; i < n; ++i) out[i] = 0;
  if (n <= 0 || k_total <= 0) return 0;  // budget.cpp:48
  if (int rc = ensure_stream()) return rc;
  int rc;
  {
    Dev d;
    int* dc = d.put(capacity, n);
    double* dh = d.put(hit_ema, n);
    double* dk = d.put(kv_bytes, n);
    double* ds = d.put<double>(nullptr, n);
    double* dw = d.put<double>(nullptr, n);
    int* dout = d.put<int>(nullptr, n);
    int* dord = d.put<int>(nullptr, n);
    if (!dc || !dh || !dk || !ds || !dw || !dout || !dord) return 200;
    allocate_kernel<<<1, 256, 0, g_hook_stream>>>(dc, dh, dk, n, k_total, tau, weight_bytes, ds, dw, dout, dord);
    d.get(out, dout, n);
    rc = finish();
  }
  return rc ? rc : finish();
}

extern "C" int spex_content_token_len(const uint64_t* child_hash, int n, const spex_workload* wl, int* out) {
  std::lock_guard<std::mutex> lk(g_hook_mu);
  if (int rc = ensure_stream()) return rc;
  if (n <= 0) return 0;
  int rc;
  {
    Dev d;
    const u64* dh = d.put(reinterpret_cast<const u64*>(child_hash), n);
    int* dout = d.put<int>(nullptr, n);
    if (!dh || !dout) return 200;
    token_len_kernel<<<(n + 127) / 128, 128, 0, g_hook_stream>>>(dh, n, *wl, dout);
    d.get(out, dout, n);
    rc = finish();
  }
  return rc ? rc : finish();
}

extern "C" int spex_content_eval(const uint64_t* path_hash, const int* offsets, int n, uint64_t query_seed,
                                 int max_depth, const spex_workload* wl, int* terminal, double* reward, int* label) {
  std::lock_guard<std::mutex> lk(g_hook_mu);
  if (int rc = ensure_stream()) return rc;
  if (n <= 0) return 0;
  const int np = offsets[n];
  int rc;
  {
    Dev d;
    const u64* dp = d.put(reinterpret_cast<const u64*>(path_hash), np);
    const int* doff = d.put(offsets, n + 1);
    int* dt = d.put<int>(nullptr, n);
    double* dr = d.put<double>(nullptr, n);
    int* dl = d.put<int>(nullptr, n);
    if (!dp || !doff || !dt || !dr || !dl) return 200;
    content_kernel<<<(n + 127) / 128, 128, 0, g_hook_stream>>>(dp, doff, n, query_seed, max_depth, *wl, dt, dr, dl);
    d.get(terminal, dt, n);
    d.get(reward, dr, n);
    d.get(label, dl, n);
    rc = finish();
  }
  return rc ? rc : finish();
}

extern "C" int spex_engine_advance(const spex_engine_hw* hw, double now, double limit, spex_engine_stream* active,
                                   int* n_active, spex_engine_stream* staged, int* n_staged, const int* anc_key,
                                   const int* anc_tokens, int n_keys, spex_engine_finished* out, int cap, int* n_out,
                                   double* now_out) {
  std::lock_guard<std::mutex> lk(g_hook_mu);
  if (int rc = ensure_stream()) return rc;
  const int na = *n_active, ns = *n_staged, tot = na + ns;
  int n_anc = 0;
  for (int i = 0; i < na; ++i) n_anc = std::max(n_anc, active[i].anc_off + active[i].anc_n);
  for (int i = 0; i < ns; ++i) n_anc = std::max(n_anc, staged[i].anc_off + staged[i].anc_n);
  int rc, status = 0;
  {
    Dev d;
    spex_engine_stream* da = d.put<spex_engine_stream>(nullptr, tot);
    spex_engine_stream* ds = d.put<spex_engine_stream>(nullptr, tot);
    if (!da || !ds) return 200;
    if (na) cudaMemcpyAsync(da, active, sizeof(spex_engine_stream) * na, cudaMemcpyHostToDevice, g_hook_stream);
    if (ns) cudaMemcpyAsync(ds, staged, sizeof(spex_engine_stream) * ns, cudaMemcpyHostToDevice, g_hook_stream);
    int cnt[2] = {na, ns};
    int* dcnt = d.put(cnt, 2);
    const int* dk = d.put(anc_key, n_anc);
    const int* dtok = d.put(anc_tokens, n_keys);
    int* dflag = d.put<int>(nullptr, n_keys);
    spex_engine_finished* dout = d.put<spex_engine_finished>(nullptr, std::max(cap, 1));
    int* dn = d.put<int>(nullptr, 2);
    double* dnow = d.put<double>(nullptr, 1);
    if (!dcnt || !dk || !dtok || !dflag || !dout || !dn || !dnow) return 200;
    engine_advance_kernel<<<1, 256, 0, g_hook_stream>>>(*hw, now, limit, da, dcnt, ds, dcnt + 1, dk, dtok, n_keys,
                                                         dflag, dout, cap, dn, dnow, dn + 1);
    d.get(cnt, dcnt, 2);
    int nres[2];
    d.get(nres, dn, 2);
    d.get(now_out, dnow, 1);
    rc = finish();
    if (rc) return rc;
    *n_active = cnt[0];
    *n_staged = cnt[1];
    *n_out = nres[0];
    status = nres[1];
    if (cnt[0]) cudaMemcpyAsync(active, da, sizeof(spex_engine_stream) * cnt[0], cudaMemcpyDeviceToHost, g_hook_stream);
    if (cnt[1]) cudaMemcpyAsync(staged, ds, sizeof(spex_engine_stream) * cnt[1], cudaMemcpyDeviceToHost, g_hook_stream);
    if (nres[0]) d.get(out, dout, std::min(nres[0], cap));
    rc = finish();
  }
  if (rc) return rc;
  return status ? status : finish();
}

extern "C" int spex_termination_should_terminate(const int* counts, const double* weights, const int* offsets,
                                                 const int* n_total, int n_tallies, int min_answers, double alpha,
                                                 int* out) {
  std::lock_guard<std::mutex> lk(g_hook_mu);
  if (int rc = ensure_stream()) return rc;
  if (n_tallies <= 0) return 0;
  const int n = offsets[n_tallies];
  int rc;
  {
    Dev d;
    int* dc = d.put(counts, n);
    double* dw = d.put(weights, n);
    int* doff = d.put(offsets, n_tallies + 1);
    int* dn = d.put(n_total, n_tallies);
    int* dout = d.put<int>(nullptr, n_tallies);
    if ((n > 0 && (!dc || !dw)) || !doff || !dn || !dout) return 200;
    terminate_kernel<<<(n_tallies + 127) / 128, 128, 0, g_hook_stream>>>(dc, dw, doff, dn, n_tallies, min_answers,
                                                                          alpha, dout);
    d.get(out, dout, n_tallies);
    rc = finish();
  }
  return rc ? rc : finish();
}

extern "C" int spex_speculation_dfs_plan(const int32_t* parent, const uint8_t* status, const uint8_t* bits,
                                         const double* reward, const int32_t* visits, const double* value,
                                         const int32_t* depth, int n_nodes, int terminal_answers, int family,
                                         double exploration_c, int width, const int32_t* depth_widths,
                                         int n_depth_widths, int target_answers, int k, uint32_t* out_node,
                                         int32_t* out_dist, int* n_out) {
  *n_out = 0;
  if (k < 0 || k > 64) return ERR_INVALID_ARGUMENT;  // spec_k <= 64 (config.cpp)
  HookTree t;
  if (!hook_tree_build(t, parent, status, bits, reward, visits, value, depth, n_nodes, terminal_answers, family,
                       exploration_c, width, depth_widths, n_depth_widths, target_answers, k))
    return ERR_INVALID_ARGUMENT;
  if (family == kRebaseBfs || k == 0) return 0;  // frontier policies plan by allocation (speculation.cpp:125-126)
  std::lock_guard<std::mutex> lk(g_hook_mu);
  if (int rc = ensure_stream()) return rc;
  int rc, n = 0;
  {
    Dev d;
    Run R{};
    R.cfg = t.cfg;
    R.n_parent = d.put(t.parent.data(), t.cap);
    R.n_first_child = d.put(t.first_child.data(), t.cap);
    R.n_next_sib = d.put(t.next_sib.data(), t.cap);
    R.n_status = d.put(t.status.data(), t.cap);
    R.n_flags = d.put(t.flags.data(), t.cap);
    R.n_reward = d.put(t.reward.data(), t.cap);
    R.n_value = d.put(t.value.data(), t.cap);
    R.n_visits = d.put(t.visits.data(), t.cap);
    R.n_depth = d.put(t.depth.data(), t.cap);
    R.n_nchildren = d.put(t.nchildren.data(), t.cap);
    R.qs = d.put(&t.qr, 1);
    GState g{};
    R.g = d.put(&g, 1);
    R.sp_visits = d.put<int>(nullptr, t.S);
    R.sp_value = d.put<double>(nullptr, t.S);
    R.sp_nchild = d.put<int>(nullptr, t.S);
    R.sp_stack = d.put<u32>(nullptr, t.S);
    R.sp_dbl = d.put<double>(nullptr, 3 * static_cast<size_t>(t.S));
    R.sp_int = d.put<int>(nullptr, 3 * static_cast<size_t>(t.S));
    R.log_tab = nullptr;
    R.log_tab_n = 0;  // log via glibc::log itself (the table only caches it)
    Run* dR = d.put(&R, 1);
    u32* dn = d.put<u32>(nullptr, 64);
    int* dd = d.put<int>(nullptr, 64);
    int* dc = d.put<int>(nullptr, 1);
    if (!dR || !dn || !dd || !dc || !R.sp_dbl || !R.n_parent) return 200;
    dfs_plan_kernel<<<1, 1, 0, g_hook_stream>>>(dR, k, dn, dd, dc);
    d.get(&n, dc, 1);
    rc = finish();
    if (!rc && n > 0) {
      d.get(out_node, dn, n);
      d.get(out_dist, dd, n);
      rc = finish();
    }
  }
  if (rc) return rc;
  if (n < 0) return ERR_INTERNAL;
  *n_out = n;
  return finish();
}

extern "C" int spex_tree_transition_legal(const uint8_t* from, const uint8_t* to, int n, uint8_t* out) {
  std::lock_guard<std::mutex> lk(g_hook_mu);
  if (int rc = ensure_stream()) return rc;
  if (n <= 0) return 0;
  int rc;
  {
    Dev d;
    u8* df = d.put(from, n);
    u8* dt = d.put(to, n);
    u8* dout = d.put<u8>(nullptr, n);
    if (!df || !dt || !dout) return 200;
    transition_kernel<<<(n + 127) / 128, 128, 0, g_hook_stream>>>(df, dt, n, dout);
    d.get(out, dout, n);
    rc = finish();
  }
  return rc ? rc : finish();
}

extern "C" int spex_tree_prune_subtree(const int32_t* parent, uint8_t* status, int n_nodes, uint32_t id, int* pruned) {
  *pruned = 0;
  HookTree t;
  if (!hook_tree_build_min(t, parent, status, n_nodes)) return ERR_INVALID_ARGUMENT;
  if (id >= static_cast<uint32_t>(n_nodes)) return ERR_UNKNOWN_NODE;  // check_known (tree.cpp:96-99)
  std::lock_guard<std::mutex> lk(g_hook_mu);
  if (int rc = ensure_stream()) return rc;
  int rc, cnt = 0;
  {
    Dev d;
    Run R{};
    R.cfg = t.cfg;
    R.n_parent = d.put(t.parent.data(), t.cap);
    R.n_first_child = d.put(t.first_child.data(), t.cap);
    R.n_next_sib = d.put(t.next_sib.data(), t.cap);
    R.n_status = d.put(t.status.data(), t.cap);
    R.n_flags = d.put(t.flags.data(), t.cap);
    R.n_tokens = d.put(t.tokens.data(), t.cap);
    R.qs = d.put(&t.qr, 1);
    GState g{};
    R.g = d.put(&g, 1);
    R.sp_stack = d.put<u32>(nullptr, t.S);
    R.sp_visits = d.put<int>(nullptr, t.S);
    R.sp_value = d.put<double>(nullptr, t.S);
    R.sp_nchild = d.put<int>(nullptr, t.S);
    R.sp_dbl = d.put<double>(nullptr, 3 * static_cast<size_t>(t.S));
    R.sp_int = d.put<int>(nullptr, 3 * static_cast<size_t>(t.S));
    Run* dR = d.put(&R, 1);
    int* dc = d.put<int>(nullptr, 1);
    if (!dR || !dc || !R.sp_stack || !R.n_status) return 200;
    prune_kernel<<<1, 1, 0, g_hook_stream>>>(dR, id, dc);
    d.get(&cnt, dc, 1);
    d.get(t.status.data(), R.n_status, t.cap);
    rc = finish();
  }
  if (rc) return rc;
  if (cnt < 0) return ERR_INTERNAL;
  for (int i = 0; i < n_nodes; ++i) status[i] = t.status[i];
  *pruned = cnt;
  return finish();
}
