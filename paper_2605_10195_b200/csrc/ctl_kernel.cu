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

#include "ctl_run.h"

namespace spex {

struct DevExec {
  int tid, nthr, warp, nwarp, lane, lanes;
  int* sm;
  double* smd;
  i64* sml;
  __device__ __forceinline__ void sync() { __syncthreads(); }
};

__global__ void __launch_bounds__(512, 1) spex_control_kernel(const Run* __restrict__ d_run) {
  __shared__ Run sR;
  __shared__ int sm[1024 + 8];
  __shared__ double smd[32];
  __shared__ long long sml[32];
  __shared__ int warp_off[32 * 3];
  if (threadIdx.x == 0) sR = *d_run;
  __syncthreads();
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
}

}  // namespace spex

extern "C" int spex_launch_control_async(spex::Run* d_run, int nthreads, cudaStream_t stream, cudaEvent_t a,
                                         cudaEvent_t b) {
  if (nthreads < 64 || nthreads > 512 || (nthreads & 31)) nthreads = 512;
  cudaEventRecord(a, stream);
  spex::spex_control_kernel<<<1, nthreads, 0, stream>>>(d_run);
  cudaError_t e = cudaGetLastError();
  cudaEventRecord(b, stream);
  return static_cast<int>(e);
}

extern "C" int spex_launch_control(spex::Run* d_run, int nthreads, cudaStream_t stream, float* ms) {
  if (nthreads < 64 || nthreads > 512 || (nthreads & 31)) nthreads = 512;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a, stream);
  spex::spex_control_kernel<<<1, nthreads, 0, stream>>>(d_run);
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
