// ctl_kernel.cu — the persistent frontier-expansion control kernel (sm_100a).
//
// One CTA of 512 threads (16 warps) runs the whole consumer loop of one run
// (executor.cpp:785-807) on device: engine epochs, completion handling,
// reward events, per-query follow-ups, T1/T2 scheduling and T3 termination,
// with block barriers between phases and warp-per-query items inside them.
// No host round trip gates any expansion; the host only launches the kernel
// and reads the totals/event log back at the end.
//
// Compiled with --fmad=false: every fp64 operation of the control path must
// round like the reference's x86-64 -O2 build (no FMA contraction).
#include <cuda_runtime.h>

#include <cstdlib>

#include "ctl_run.h"

namespace spex {

struct DevExec {
  int tid, nthr, warp, nwarp, lane, lanes;
  int* sm;
  double* smd;
  i64* sml;
  __device__ __forceinline__ void sync() { __syncthreads(); }
};

// Copy n bytes (multiple of 16, 16-aligned) with the whole block.
__device__ __forceinline__ void block_copy16(void* dst, const void* src, size_t n) {
  int4* d = reinterpret_cast<int4*>(dst);
  const int4* s = reinterpret_cast<const int4*>(src);
  for (size_t i = threadIdx.x; i < n / 16; i += blockDim.x) d[i] = s[i];
}

__global__ void __launch_bounds__(512, 1) spex_control_kernel(const Run* __restrict__ d_run, int dyn_bytes) {
  __shared__ Run sR;
  __shared__ int sm[1024 + 8];
  __shared__ double smd[32];
  __shared__ long long sml[32];
  __shared__ int warp_off[512 * 3];  // per-thread item staging offsets
  // The per-query records and the run scalars are touched by every phase of
  // every consumer iteration: when they fit, they live in shared memory for
  // the whole run (generic pointers, so the control code is unchanged) and are
  // written back at the end. The control CTA owns its SM (512 x 128 registers),
  // so this shared memory costs the forward nothing.
  extern __shared__ __align__(16) unsigned char dsm[];
  if (threadIdx.x == 0) sR = d_run[blockIdx.x];  // a batch launch runs one search per CTA
  __syncthreads();
  QueryRun* const g_qs = sR.qs;
  GState* const g_g = sR.g;
  const size_t qbytes = static_cast<size_t>(sR.cfg.n_queries) * sizeof(QueryRun);
  const bool staged = static_cast<size_t>(dyn_bytes) >= qbytes + sizeof(GState);
  if (staged) {
    block_copy16(dsm, g_qs, qbytes);
    block_copy16(dsm + qbytes, g_g, sizeof(GState));
    __syncthreads();
    if (threadIdx.x == 0) {
      sR.qs = reinterpret_cast<QueryRun*>(dsm);
      sR.g = reinterpret_cast<GState*>(dsm + qbytes);
    }
    __syncthreads();
  }
  DevExec ex;
  ex.tid = threadIdx.x;
  ex.nthr = blockDim.x;
  ex.warp = threadIdx.x >> 5;
  ex.nwarp = blockDim.x >> 5;
  ex.lane = threadIdx.x & 31;
  ex.lanes = 32;
  ex.sm = sm;
  ex.smd = smd;
  ex.sml = sml;
  run_loop(&sR, ex, warp_off);
  __syncthreads();
  if (staged) {
    block_copy16(g_qs, dsm, qbytes);
    block_copy16(g_g, dsm + qbytes, sizeof(GState));
  }
}

// The control path is a call tree of non-inlined device functions (kept out of
// line so the hot loop fits the instruction cache); reserve a per-thread stack
// deep enough for its longest chain (ptxas reports the cumulative size).
static void ensure_control_stack() {
  static bool done = false;
  if (done) return;
  done = true;
  cudaFuncAttributes fa{};
  size_t need = 4096;
  if (cudaFuncGetAttributes(&fa, spex_control_kernel) == cudaSuccess && fa.localSizeBytes + 1024 > need)
    need = fa.localSizeBytes + 1024;
  size_t cur = 0;
  cudaDeviceGetLimit(&cur, cudaLimitStackSize);
  if (cur < need) cudaDeviceSetLimit(cudaLimitStackSize, need);
}

static int control_dyn_smem(int n_queries) {
  ensure_control_stack();
  const size_t need = static_cast<size_t>(n_queries) * sizeof(QueryRun) + sizeof(GState);
  constexpr size_t kMax = 200 * 1024;
  if (need > kMax) return 0;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(spex_control_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kMax));
    attr = true;
  }
  return static_cast<int>(need);
}

}  // namespace spex

extern "C" int spex_launch_control_async(spex::Run* d_run, int n_queries, int nthreads, cudaStream_t stream,
                                         cudaEvent_t a, cudaEvent_t b) {
  if (nthreads < 64 || nthreads > 512 || (nthreads & 31)) nthreads = 512;
  const int dyn = std::getenv("SPEX_CTL_NO_SMEM") ? (spex::ensure_control_stack(), 0) : spex::control_dyn_smem(n_queries);
  cudaEventRecord(a, stream);
  spex::spex_control_kernel<<<1, nthreads, dyn, stream>>>(d_run, dyn);
  cudaError_t e = cudaGetLastError();
  cudaEventRecord(b, stream);
  return static_cast<int>(e);
}

extern "C" int spex_launch_control_batch_async(spex::Run* d_runs, int n_runs, int n_queries, int nthreads,
                                               cudaStream_t stream, cudaEvent_t a, cudaEvent_t b) {
  if (nthreads < 64 || nthreads > 512 || (nthreads & 31)) nthreads = 512;
  const int dyn = std::getenv("SPEX_CTL_NO_SMEM") ? (spex::ensure_control_stack(), 0) : spex::control_dyn_smem(n_queries);
  cudaEventRecord(a, stream);
  spex::spex_control_kernel<<<n_runs, nthreads, dyn, stream>>>(d_runs, dyn);
  cudaError_t e = cudaGetLastError();
  cudaEventRecord(b, stream);
  return static_cast<int>(e);
}

extern "C" int spex_launch_control(spex::Run* d_run, int n_queries, int nthreads, cudaStream_t stream, float* ms) {
  if (nthreads < 64 || nthreads > 512 || (nthreads & 31)) nthreads = 512;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int dyn = std::getenv("SPEX_CTL_NO_SMEM") ? (spex::ensure_control_stack(), 0) : spex::control_dyn_smem(n_queries);
  cudaEventRecord(a, stream);
  spex::spex_control_kernel<<<1, nthreads, dyn, stream>>>(d_run, dyn);
  cudaError_t e = cudaGetLastError();
  cudaEventRecord(b, stream);
  cudaError_t s = cudaEventSynchronize(b);
  if (e == cudaSuccess) e = s;
  if (e == cudaSuccess) e = cudaGetLastError();
  float t = 0.f;
  cudaEventElapsedTime(&t, a, b);
  if (ms) *ms = t;
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return static_cast<int>(e);
}
