// gemm_tc.cu — K2: hand-written tcgen05 GEMM for the policy / PRM projections,
// with the elementwise work of the forward fused into its epilogue.
//
//   Y[M x N] = X[M x K] . W[N x K]^T      (bf16 operands, fp32 accumulate in TMEM)
//
// Persistent: one CTA per SM walks 128 x 256 output tiles (UMMA M=128, N=256,
// K=16 per instruction, cta_group::1) with two TMEM accumulators (2 x 256 fp32
// columns = all of TMEM), so the epilogue of tile i overlaps the MMAs of tile
// i+1. Warp roles:
//   warp 0      TMA producer: 128x64 bf16 boxes of X and W (128-byte swizzle)
//               into a 4-stage shared-memory ring (full/empty mbarriers)
//   warp 1      TMEM allocator (512 columns) and MMA issuer: one elected lane
//               issues 4 tcgen05.mma per stage from shared-memory descriptors,
//               tcgen05.commit frees the stage / signals the epilogue
//   warps 2..5  epilogue: tcgen05.ld of the accumulator (one TMEM lane = one
//               output row per thread, 128 columns per pass), then one of
//     EPI_STORE    y (+)= acc                       (O / down projections: residual add)
//     EPI_ROPE_KV  rotate-half RoPE; Q heads -> Qr (fp32, pre-scaled), K/V heads
//                  -> bf16 tree-KV pool at the row's slot     (fuses rope_kv_kernel)
//     EPI_SWIGLU   silu(gate) * up -> bf16 MLP activation, with the gate/up weight
//                  rows interleaved per 64-column block       (fuses swiglu_kernel)
//     EPI_LSE      per-row partial max / first argmax / sum exp / sum over the
//                  tile's vocab columns; a combine kernel finishes K3
//                  (the fp32 logits are never written to HBM)
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdlib>

#include "model.h"

namespace spex {

namespace tc {

constexpr int BM = 128, BK = 64;
constexpr int EN = 128;  // epilogue chunk (columns per tcgen05.ld pass)
constexpr int kStageLd = EN + 4;  // padded row of the epilogue staging buffer (conflict-free float4)
constexpr uint32_t kEpiBytes = 4 * 32 * kStageLd * 4;
constexpr int kThreads = 192;
// per tile width BN (128 or 256): pipeline depth, bytes per stage, TMEM columns
template <int BN> struct TileCfg {
  static constexpr int STAGES = BN == 256 ? 3 : 4;
  static constexpr uint32_t kStageBytes = (BM + BN) * BK * 2;  // 48 KB / 32 KB
  static constexpr uint32_t kTmemCols = BN;                    // one fp32 accumulator; two allocated
  // kind::f16 instruction descriptor: D f32, A/B bf16, both K-major, M=128, N=BN
  static constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                                     ((uint32_t)(BM >> 4) << 24);
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// K-major operand tile [rows][64 bf16] with 128-byte swizzle: 8-row atoms of
// 1024 B (SBO), LBO unused (1), descriptor version 1 (sm_100), layout SWIZZLE_128B.
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr) {
  return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

}  // namespace tc

template <int EPI, int DH, int BN>
__global__ void __launch_bounds__(tc::kThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M, int N,
                   int K, TcEpilogue ep, unsigned long long* tile_ctr, unsigned long long tile_base) {
  using namespace tc;
  using T = TileCfg<BN>;
  constexpr int STAGES = T::STAGES;
  constexpr uint32_t kStageBytes = T::kStageBytes;
  constexpr uint32_t kTmemCols = T::kTmemCols;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-byte alignment for the 128B-swizzled tiles
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* sA = smem;                          // [STAGES][BM][BK]
  unsigned char* sB = smem + STAGES * BM * BK * 2;   // [STAGES][BN][BK]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * kStageBytes);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;  // [2] accumulator ready
  uint64_t* tempty = tfull + 2;      // [2] accumulator drained by the epilogue
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  float* stage_out = reinterpret_cast<float*>(smem + STAGES * kStageBytes + 256);  // [4 warps][32][kStageLd]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kblocks = K / BK;
  const int n_nb = (N + BN - 1) / BN, n_tiles = n_nb * ((M + BM - 1) / BM);

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4);  // one arrive per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(2 * kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  // persistent with a dynamic tile queue: the producer lane claims tiles from a
  // global counter (so CTAs that start late — SMs busy with the control kernel
  // or the other forward stream — simply take fewer tiles) and passes each id to
  // the MMA lane and the epilogue through a shared ring; id -1 ends the CTA.
  // tile t = (mb, nb), nb fastest
  int* tq = reinterpret_cast<int*>(tmem_slot + 4);  // [8]
  if (warp == 0) {
    if (lane == 0) {
      int g = 0;  // k-block counter across tiles (stage ring position)
      for (int it = 0;; ++it) {
        long long tl = (long long)(atomicAdd(tile_ctr, 1ull) - tile_base);
        const int t = tl < n_tiles ? (int)tl : -1;
        tq[it & 7] = t;
        if (t < 0) {  // sentinel stage: no data, wakes the MMA lane
          const int s = g % STAGES;
          if (g >= STAGES) mbar_wait(&empty[s], ((g / STAGES) - 1) & 1);
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&full[s])) : "memory");
          break;
        }
        const int mb = t / n_nb, nb = t - mb * n_nb;
        for (int kb = 0; kb < kblocks; ++kb, ++g) {
          const int s = g % STAGES;
          if (g >= STAGES) mbar_wait(&empty[s], ((g / STAGES) - 1) & 1);
          mbar_arrive_tx(&full[s], kStageBytes);
          tma_load_2d(sA + s * BM * BK * 2, &tmA, kb * BK, mb * BM, &full[s]);
#pragma unroll
          for (int r = 0; r < BN / 128; ++r)  // the operand maps use 128-row boxes
            tma_load_2d(sB + s * BN * BK * 2 + r * 128 * BK * 2, &tmB, kb * BK, nb * BN + r * 128, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int g = 0;
      for (int it = 0;; ++it) {
        const int acc = it & 1;
        mbar_wait(&full[g % STAGES], (g / STAGES) & 1);  // first stage of tile `it` (or the sentinel)
        const int t = tq[it & 7];
        // accumulator `acc` must be drained before its barrier moves again
        // (also for the sentinel: two unobserved phases would alias the parity)
        if (it >= 2) mbar_wait(&tempty[acc], ((it >> 1) - 1) & 1);
        if (t < 0) {
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&tfull[acc])) : "memory");
          break;
        }
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t dt = tmem + acc * kTmemCols;
        for (int kb = 0; kb < kblocks; ++kb, ++g) {
          const int s = g % STAGES;
          if (kb > 0) mbar_wait(&full[s], (g / STAGES) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint64_t da = smem_desc(smem_u32(sA + s * BM * BK * 2));
          const uint64_t db = smem_desc(smem_u32(sB + s * BN * BK * 2));
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)  // 16 bf16 = 32 bytes = 2 descriptor units per step
            mma_bf16(dt, da + 2 * k, db + 2 * k, T::kIdesc, (kb | k) != 0);
          mma_commit(&empty[s]);
        }
        mma_commit(&tfull[acc]);
      }
    }
    __syncwarp();
  } else {
    // ---------------- epilogue: warps 2..5 own TMEM lane quarters (warp % 4)
    const int quarter = warp & 3;
    for (int it = 0;; ++it) {
      const int acc = it & 1;
      mbar_wait(&tfull[acc], (it >> 1) & 1);
      const int t = tq[it & 7];
      if (t < 0) break;
      const int mb = t / n_nb, nb = t - mb * n_nb;
      const int row = mb * BM + quarter * 32 + lane;
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t tbase = tmem + acc * kTmemCols + ((uint32_t)(quarter * 32) << 16);
#pragma unroll 1
      for (int h = 0; h < BN / EN; ++h) {
        float v[EN];
#pragma unroll
        for (int c = 0; c < EN / 32; ++c) tmem_ld32(tbase + h * EN + c * 32, v + c * 32);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (h == BN / EN - 1) {  // accumulator fully read: the MMA warp may reuse it
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0)
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&tempty[acc])) : "memory");
        }
        const int n0 = nb * BN + h * EN;
        if (n0 >= N) continue;  // partial last N tile (its B rows were zero-filled)
        const int row0 = mb * BM + quarter * 32;  // this warp's 32 rows
        if constexpr (EPI == TC_EPI_LSE) {
          if (row < M) {
            float mx = -INFINITY, sm = 0.f;
            int mi = 0;
            const int lim = min(EN, ep.V - n0);
#pragma unroll
            for (int i = 0; i < EN; ++i) {
              if (i < lim) {
                sm += v[i];
                if (v[i] > mx) {
                  mx = v[i];
                  mi = i;
                }
              }
            }
            float se = 0.f;
            const float ml2 = mx * 1.4426950408889634f;
#pragma unroll
            for (int i = 0; i < EN; ++i)
              if (i < lim) se += exp2f(fmaf(v[i], 1.4426950408889634f, -ml2));
            reinterpret_cast<float4*>(ep.part)[(long long)row * ep.n_tiles + n0 / EN] =
                make_float4(mx, se, sm, __int_as_float(n0 + mi));
          }
          continue;
        }
        // per-row transform in registers (thread = row)
        if constexpr (EPI == TC_EPI_ROPE_KV) {
          constexpr int half = DH / 2;
          const float2* cs = reinterpret_cast<const float2*>(ep.rope) + (long long)(row < M ? row : 0) * half;
#pragma unroll
          for (int h0 = 0; h0 < EN; h0 += DH) {
            const int head = (n0 + h0) / DH;
            if (head < ep.H + ep.KVH) {  // rotate-half RoPE on (x[i], x[i + half]); Q also scaled
              const float sc = head < ep.H ? ep.qscale : 1.f;
#pragma unroll
              for (int i = 0; i < half; ++i) {
                const float2 c = cs[i];
                const float a = v[h0 + i], b = v[h0 + half + i];
                v[h0 + i] = (a * c.x - b * c.y) * sc;
                v[h0 + half + i] = (a * c.y + b * c.x) * sc;
              }
            }
          }
        } else if constexpr (EPI == TC_EPI_SWIGLU) {
          // chunk n0: columns [0,64) gate j, [64,128) up j for j in [n0/2, n0/2 + 64)
#pragma unroll
          for (int i = 0; i < EN / 2; ++i) {
            const float g = v[i], u = v[EN / 2 + i];
            v[i] = g / (1.f + __expf(-g)) * u;
          }
        }
        // stage the warp's 32 x EN block in shared memory, then write it out
        // row by row with the lanes along the columns (512 B per instruction)
        float* buf = stage_out + (warp - 2) * 32 * kStageLd;
        constexpr int NW = EPI == TC_EPI_SWIGLU ? EN / 2 : EN;  // columns written
#pragma unroll
        for (int i = 0; i < NW / 4; ++i)
          *reinterpret_cast<float4*>(buf + lane * kStageLd + 4 * i) =
              make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
        __syncwarp();
        const int c = 4 * lane;  // this lane's 4 columns of each row
        for (int r = 0; r < 32; ++r) {
          const int grow = row0 + r;
          if (grow >= M) break;
          if (c >= NW) continue;
          const float4 o = *reinterpret_cast<const float4*>(buf + r * kStageLd + c);
          if constexpr (EPI == TC_EPI_STORE) {
            float4* y = reinterpret_cast<float4*>(ep.y + (long long)grow * ep.ldy + n0 + c);
            float4 w = o;
            if (ep.accumulate) {
              const float4 a = *y;
              w.x += a.x;
              w.y += a.y;
              w.z += a.z;
              w.w += a.w;
            }
            *y = w;
          } else if constexpr (EPI == TC_EPI_SWIGLU) {
            *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(ep.act) + (long long)grow * ep.F + n0 / 2 + c) =
                make_uint2(pack2(o.x, o.y), pack2(o.z, o.w));
          } else {  // TC_EPI_ROPE_KV
            const int col = n0 + c, head = col / DH, d0 = col - head * DH;
            if (head < ep.H) {
              *reinterpret_cast<float4*>(ep.Qr + ((long long)grow * ep.H + head) * DH + d0) = o;
            } else {
              const bool is_k = head < ep.H + ep.KVH;
              const int kh = is_k ? head - ep.H : head - ep.H - ep.KVH;
              __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(is_k ? ep.Kp : ep.Vp) +
                                   ((long long)kh * ep.slots + ep.rows[grow].slot) * DH + d0;
              *reinterpret_cast<uint2*>(dst) = make_uint2(pack2(o.x, o.y), pack2(o.z, o.w));
            }
          }
        }
        __syncwarp();
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * kTmemCols));
  }
}

// K3 combine: per row over the LM-head tiles' partials (first argmax on ties).
__global__ void lse_combine_kernel(const float4* __restrict__ part, int M, int n_tiles, int* amax, float* lse,
                                   float* lsum) {
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (r >= M) return;
  const float4* p = part + (long long)r * n_tiles;
  float mx = -INFINITY, sm = 0.f;
  int mi = 0x7fffffff;
  for (int t = lane; t < n_tiles; t += 32) {
    const float4 q = p[t];
    sm += q.z;
    const int qi = __float_as_int(q.w);
    if (q.x > mx || (q.x == mx && qi < mi)) {
      mx = q.x;
      mi = qi;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float om = __shfl_xor_sync(0xffffffffu, mx, o);
    const int oi = __shfl_xor_sync(0xffffffffu, mi, o);
    sm += __shfl_xor_sync(0xffffffffu, sm, o);
    if (om > mx || (om == mx && oi < mi)) mi = oi;
    mx = fmaxf(mx, om);
  }
  float se = 0.f;
  for (int t = lane; t < n_tiles; t += 32) {
    const float4 q = p[t];
    se += q.y * exp2f((q.x - mx) * 1.4426950408889634f);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
  if (lane == 0) {
    amax[r] = mi;
    lse[r] = mx + logf(se);
    lsum[r] = sm;
  }
}

// (cos, sin) of every row's absolute position, once per forward (all layers).
__global__ void rope_table_kernel(const RowDesc* __restrict__ rows, int M, const float* __restrict__ inv_freq,
                                  int half, float2* __restrict__ out) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= (long long)M * half) return;
  const int r = (int)(i / half), k = (int)(i - (long long)r * half);
  float s, c;
  sincosf((float)rows[r].abs_pos * inv_freq[k], &s, &c);
  out[i] = make_float2(c, s);
}

// Gate/up weight rows interleaved per 64-row block: out block j = [gate 64j..64j+63 ; up 64j..64j+63].
__global__ void interleave_gu_kernel(const __nv_bfloat16* __restrict__ wgu, int F, int d,
                                     __nv_bfloat16* __restrict__ out) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= 2LL * F * d) return;
  const long long orow = i / d, col = i - orow * d;
  const int blk = (int)(orow / 128), within = (int)(orow % 128);
  const long long src = within < 64 ? (long long)blk * 64 + within : (long long)F + blk * 64 + (within - 64);
  out[i] = wgu[src * d + col];
}

}  // namespace spex

using namespace spex;

template <int EPI, int DH, int BN>
static int launch_gemm_tc(const CUtensorMap* tmA, const CUtensorMap* tmB, int M, int N, int K, const TcEpilogue* ep,
                          cudaStream_t s, int grid_x, unsigned long long* tile_ctr, unsigned long long tile_base) {
  using T = tc::TileCfg<BN>;
  const size_t smem = T::STAGES * T::kStageBytes + 1024 + 256 + tc::kEpiBytes;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gemm_tc_kernel<EPI, DH, BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  gemm_tc_kernel<EPI, DH, BN><<<grid_x, tc::kThreads, smem, s>>>(*tmA, *tmB, M, N, K, *ep, tile_ctr, tile_base);
  return (int)cudaGetLastError();
}

template <int EPI, int DH>
static int launch_bn(int bn, const CUtensorMap* tmA, const CUtensorMap* tmB, int M, int N, int K,
                     const TcEpilogue* ep, cudaStream_t s, int grid_x, unsigned long long* ctr,
                     unsigned long long base) {
  return bn == 256 ? launch_gemm_tc<EPI, DH, 256>(tmA, tmB, M, N, K, ep, s, grid_x, ctr, base)
                   : launch_gemm_tc<EPI, DH, 128>(tmA, tmB, M, N, K, ep, s, grid_x, ctr, base);
}

extern "C" int spex_k_gemm_tc(const CUtensorMap* tmA, const CUtensorMap* tmB, int M, int N, int K,
                              const TcEpilogue* ep, cudaStream_t s) {
  if (M <= 0) return 0;
  if (N % tc::EN || K % tc::BK) return -1;
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  static const int cap = getenv("SPEX_TC_GRID") ? atoi(getenv("SPEX_TC_GRID")) : sms;
  const int gmax = cap > 0 && cap < sms ? cap : sms;
  // tile width: the one whose last wave is fuller (128-wide tiles cost a second
  // A-tile read per 256 columns but fill the SMs on mid-size problems)
  const int mb = (M + tc::BM - 1) / tc::BM;
  auto eff = [&](int bn) {
    const long long t = (long long)mb * ((N + bn - 1) / bn);
    const long long waves = (t + gmax - 1) / gmax;
    return (double)t / (double)(waves * gmax) * (bn == 256 ? 1.0 : 0.85);
  };
  static const int force_bn = getenv("SPEX_TC_BN") ? atoi(getenv("SPEX_TC_BN")) : 0;
  const int bn = force_bn == 128 || force_bn == 256 ? force_bn : (eff(256) >= eff(128) ? 256 : 128);
  const int tiles = mb * ((N + bn - 1) / bn);
  const int grid_x = tiles < gmax ? tiles : gmax;
  // per-stream monotone tile counter: launch j claims ids [base_j, base_j + tiles + grid).
  // Counters come from one pool; a stream seen for the first time takes the
  // least recently assigned slot (streams are per executor, so after
  // kCtrSlots newer streams the evicted one has long finished).
  constexpr int kCtrSlots = 256;
  struct Ctr {
    cudaStream_t st;
    unsigned long long base;
  };
  static Ctr ctrs[kCtrSlots];
  static unsigned long long* pool = nullptr;
  static int n_ctrs = 0;
  if (!pool) {
    if (cudaMalloc(&pool, kCtrSlots * sizeof(unsigned long long)) != cudaSuccess) return -3;
    if (cudaMemset(pool, 0, kCtrSlots * sizeof(unsigned long long)) != cudaSuccess) return -3;
  }
  Ctr* c = nullptr;
  for (int i = 0; i < n_ctrs && i < kCtrSlots; ++i)
    if (ctrs[i].st == s) c = &ctrs[i];
  if (!c) {
    c = &ctrs[n_ctrs % kCtrSlots];
    c->st = s;
    c->base = 0;
    cudaMemsetAsync(pool + (c - ctrs), 0, sizeof(unsigned long long), s);
    ++n_ctrs;
  }
  unsigned long long* const ctr = pool + (c - ctrs);
  const unsigned long long base = c->base;
  c->base += (unsigned long long)tiles + grid_x;
  switch (ep->kind) {
    case TC_EPI_STORE:
      return launch_bn<TC_EPI_STORE, 128>(bn, tmA, tmB, M, N, K, ep, s, grid_x, ctr, base);
    case TC_EPI_SWIGLU:
      return launch_bn<TC_EPI_SWIGLU, 128>(bn, tmA, tmB, M, N, K, ep, s, grid_x, ctr, base);
    case TC_EPI_LSE:
      return launch_bn<TC_EPI_LSE, 128>(bn, tmA, tmB, M, N, K, ep, s, grid_x, ctr, base);
    case TC_EPI_ROPE_KV:
      if (ep->dh == 128) return launch_bn<TC_EPI_ROPE_KV, 128>(bn, tmA, tmB, M, N, K, ep, s, grid_x, ctr, base);
      if (ep->dh == 64) return launch_bn<TC_EPI_ROPE_KV, 64>(bn, tmA, tmB, M, N, K, ep, s, grid_x, ctr, base);
      return -1;
    default:
      return -1;
  }
}

extern "C" void spex_k_lse_combine(const float* part, int M, int n_tiles, int* amax, float* lse, float* lsum,
                                   cudaStream_t s) {
  if (M <= 0) return;
  lse_combine_kernel<<<(M + 7) / 8, 256, 0, s>>>(reinterpret_cast<const float4*>(part), M, n_tiles, amax, lse, lsum);
}

extern "C" void spex_k_rope_table(const RowDesc* rows, int M, const float* inv_freq, int half, float* out,
                                  cudaStream_t s) {
  const long long n = (long long)M * half;
  if (n <= 0) return;
  rope_table_kernel<<<(int)((n + 255) / 256), 256, 0, s>>>(rows, M, inv_freq, half, reinterpret_cast<float2*>(out));
}

extern "C" void spex_k_interleave_gu(const __nv_bfloat16* wgu, int F, int d, __nv_bfloat16* out, cudaStream_t s) {
  const long long n = 2LL * F * d;
  interleave_gu_kernel<<<(int)((n + 255) / 256), 256, 0, s>>>(wgu, F, d, out);
}
