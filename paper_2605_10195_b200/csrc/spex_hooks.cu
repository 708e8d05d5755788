// spex_hooks.cu — the reference's policy and budget hooks as batched device
// calls over the C ABI (include/spex.h, SURVEY.md §8b "policy hooks"):
//
//   spex_policy_ucb_score      <- totsim::ucb_score        (policy.cpp:22-30)
//   spex_policy_ucb_select     <- totsim::ucb_select       (policy.cpp:32-51)
//   spex_policy_rebase_widths  <- totsim::rebase_widths    (policy.cpp:65-118)
//   spex_budget_k_total        <- totsim::roofline_k_total (budget.cpp:23-39)
//   spex_budget_allocate       <- totsim::allocate_budgets (budget.cpp:45-96)
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

#include "ctl_run.h"

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
