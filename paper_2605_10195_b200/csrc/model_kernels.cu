// model_kernels.cu — device kernels of the policy / PRM forward over a batch
// of tree rows (one token of one thought per row).
//
//   K1 tree_attn_kernel    decode attention over a thought's ancestor chain in
//                          the paged tree KV pool: per (row, kv head) block,
//                          64-token K/V chunks staged into shared memory by
//                          cp.async.bulk (TMA bulk copy) with an mbarrier,
//                          double-buffered, online softmax in fp32
//   K3 lm_epilogue_kernel  per-row argmax / logsumexp / checksum of the logits
//   K4 value_head_kernel   PRM score sigmoid(w . h_last)
//   plus weight init, row descriptors, embedding, RMSNorm->bf16, RoPE + KV
//   append, SwiGLU.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "ctl_state.h"
#include "model.h"

namespace spex {

__device__ __forceinline__ uint64_t d_splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

// Counter-hash uniform init (std = scale): exactly reproducible in numpy
// (oracle/model_ref.py: init_tensor).
__global__ void init_weights_kernel(__nv_bfloat16* w, long long n, uint64_t seed, uint64_t tensor_id,
                                    float scale) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    uint64_t h = d_splitmix64((tensor_id << 40) ^ (uint64_t)i ^ seed);
    float u = (float)(h >> 40) * 5.9604644775390625e-08f;  // 2^-24, exact
    float v = (u * 2.0f - 1.0f) * scale;
    w[i] = __float2bfloat16_rn(v);
  }
}

__device__ __forceinline__ int token_id(uint64_t node_hash, int pos, int V) {
  uint64_t h = d_splitmix64(node_hash ^ ((uint64_t)(pos + 1) * 0x9e3779b97f4a7c15ULL) ^ kSaltTok);
  return (int)(h % (uint64_t)V);
}

constexpr int kMaxSegFwd = 40;
__device__ int build_segments(const TreeView& t, int q, uint32_t node, int own_len, Segment* out,
                              int* abs_prefix) {
  // ancestors root-first, then the node's own prefix
  const uint32_t b = (uint32_t)q * (uint32_t)t.node_cap;
  uint32_t chain[64];
  int n = 0;
  for (uint32_t c = t.parent[b + node]; c != 0xffffffffu && n < kMaxSegFwd - 1; c = t.parent[b + c]) chain[n++] = c;
  int pre = 0;
  int k = 0;
  for (int i = n - 1; i >= 0; --i) {
    const uint32_t a = chain[i];
    const int len = t.tokens[b + a];
    if (len > 0) {
      out[k].base = t.kvbase[b + a];
      out[k].len = len;
      out[k].pad = 0;
      ++k;
    }
    pre += len;
  }
  out[k].base = t.kvbase[b + node];
  out[k].len = own_len;
  out[k].pad = 0;
  ++k;
  *abs_prefix = pre;
  return k;
}

constexpr int kMaxSeg = 40;

__global__ void build_decode_rows_kernel(TreeView t, const int* sids, const int* pos0, int n, int step,
                                         RowDesc* rows, Segment* segs) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int sid = sids[i];
  const int q = t.st_q[sid];
  const uint32_t node = t.st_node[sid];
  const int pos = pos0[i] + step;
  int pre = 0;
  int ns = build_segments(t, q, node, pos + 1, segs + (long long)i * kMaxSeg, &pre);
  const uint32_t b = (uint32_t)q * (uint32_t)t.node_cap;
  RowDesc r;
  r.q = q;
  r.node = node;
  r.pos = pos;
  r.abs_pos = pre + pos;
  r.slot = t.kvbase[b + node] + pos;
  r.seg_off = i * kMaxSeg;
  r.nseg = ns;
  r.token = token_id(t.hash[b + node], pos, t.V);
  r.pad = 0;
  rows[i] = r;
}

// PRM rows: thought k of the entry occupies rows [row_start[k], row_start[k] + len).
__global__ void build_prm_rows_kernel(TreeView t, const int* sids, const int* row_start, int n,
                                      RowDesc* rows, Segment* segs, int* last_row) {
  const int k = blockIdx.x;
  if (k >= n) return;
  const int sid = sids[k];
  const int q = t.st_q[sid];
  const uint32_t node = t.st_node[sid];
  const uint32_t b = (uint32_t)q * (uint32_t)t.node_cap;
  const int len = t.tokens[b + node];
  const int r0 = row_start[k];
  for (int j = threadIdx.x; j < len; j += blockDim.x) {
    const int i = r0 + j;
    int pre = 0;
    int ns = build_segments(t, q, node, j + 1, segs + (long long)i * kMaxSeg, &pre);
    RowDesc r;
    r.q = q;
    r.node = node;
    r.pos = j;
    r.abs_pos = pre + j;
    r.slot = t.kvbase[b + node] + j;
    r.seg_off = i * kMaxSeg;
    r.nseg = ns;
    r.token = token_id(t.hash[b + node], j, t.V);
    r.pad = 0;
    rows[i] = r;
  }
  if (threadIdx.x == 0) last_row[k] = r0 + len - 1;
}

// Root prompt rows: query q, positions 0..P-1.
__global__ void build_prompt_rows_kernel(TreeView t, int q0, int nq, RowDesc* rows, Segment* segs) {
  const int P = t.prompt_tokens;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nq * P) return;
  const int q = q0 + i / P;
  const int j = i % P;
  const uint32_t b = (uint32_t)q * (uint32_t)t.node_cap;
  Segment* s = segs + (long long)i * kMaxSeg;
  s[0].base = t.kvbase[b];
  s[0].len = j + 1;
  s[0].pad = 0;
  RowDesc r;
  r.q = q;
  r.node = 0;
  r.pos = j;
  r.abs_pos = j;
  r.slot = t.kvbase[b] + j;
  r.seg_off = i * kMaxSeg;
  r.nseg = 1;
  r.token = token_id(t.hash[b], j, t.V);
  r.pad = 0;
  rows[i] = r;
}

// PRM row counts per reward batch (sum of token_len of the scored thoughts)
// and the per-thought exclusive scan; one thread per schedule entry.
__global__ void prm_scan_all_kernel(TreeView t, const int* kind, const int* off, const int* cnt, int n_entries,
                                    const int* srow_sid, int* row_start, int* totals) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n_entries) return;
  if (kind[e] != SCHED_PRM) {
    totals[e] = 0;
    return;
  }
  int acc = 0;
  for (int k = 0; k < cnt[e]; ++k) {
    const int sid = srow_sid[off[e] + k];
    row_start[off[e] + k] = acc;
    acc += t.tokens[(uint32_t)t.st_q[sid] * (uint32_t)t.node_cap + t.st_node[sid]];
  }
  totals[e] = acc;
}

__global__ void gather_prm_kernel(const RowDesc* rows, const int* last_row, int n, const float* score,
                                  PrmOut* out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  PrmOut o;
  o.q = rows[last_row[k]].q;
  o.node = rows[last_row[k]].node;
  o.score = score[k];
  o.pad = 0;
  out[k] = o;
}

__global__ void gather_outputs_kernel(const RowDesc* rows, int M, const int* amax, const float* lse,
                                      const float* lsum, DecodeOut* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= M) return;
  DecodeOut o;
  o.q = rows[i].q;
  o.node = rows[i].node;
  o.pos = rows[i].pos;
  o.amax = amax[i];
  o.lse = lse[i];
  o.lsum = lsum[i];
  out[i] = o;
}

__global__ void embed_kernel(const RowDesc* rows, int M, const __nv_bfloat16* E, int d, float* X) {
  const int r = blockIdx.x;
  if (r >= M) return;
  const __nv_bfloat16* e = E + (long long)rows[r].token * d;
  for (int i = threadIdx.x; i < d; i += blockDim.x) X[(long long)r * d + i] = __bfloat162float(e[i]);
}

// y = bf16(x * rsqrt(mean(x^2) + eps))  (unit gains)
__global__ void rmsnorm_bf16_kernel(const float* X, int M, int d, float eps, __nv_bfloat16* Y) {
  const int r = blockIdx.x;
  if (r >= M) return;
  const float* x = X + (long long)r * d;
  float ss = 0.f;
  for (int i = threadIdx.x; i < d; i += blockDim.x) ss += x[i] * x[i];
  __shared__ float red[32];
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  const float inv = rsqrtf(red[0] / (float)d + eps);
  for (int i = threadIdx.x; i < d; i += blockDim.x) Y[(long long)r * d + i] = __float2bfloat16_rn(x[i] * inv);
}

// RoPE on q and k at the row's absolute position; append k, v (bf16) to the
// layer's KV pool at the row's slot; q (fp32, pre-scaled by 1/sqrt(dh)) to Qr.
// Pools are [KVH][slots][dh].
__global__ void rope_kv_kernel(const RowDesc* rows, int M, const float* QKV, int H, int KVH, int dh,
                               const float* inv_freq, long long slots, __nv_bfloat16* Kp, __nv_bfloat16* Vp,
                               float* Qr) {
  const int r = blockIdx.x;
  if (r >= M) return;
  const RowDesc rd = rows[r];
  const int width = (H + 2 * KVH) * dh;
  const float* src = QKV + (long long)r * width;
  const int half = dh / 2;
  const float qscale = rsqrtf((float)dh);
  for (int idx = threadIdx.x; idx < (H + KVH) * half; idx += blockDim.x) {
    const int head = idx / half;
    const int i = idx % half;
    float s, c;
    sincosf((float)rd.abs_pos * inv_freq[i], &s, &c);
    const float* x = src + head * dh;
    const float a = x[i], b = x[i + half];
    const float ya = a * c - b * s;
    const float yb = a * s + b * c;
    if (head < H) {
      float* qd = Qr + ((long long)r * H + head) * dh;
      qd[i] = ya * qscale;
      qd[i + half] = yb * qscale;
    } else {
      const int kh = head - H;
      __nv_bfloat16* kd = Kp + ((long long)kh * slots + rd.slot) * dh;
      kd[i] = __float2bfloat16_rn(ya);
      kd[i + half] = __float2bfloat16_rn(yb);
    }
  }
  for (int idx = threadIdx.x; idx < KVH * dh; idx += blockDim.x) {
    const int kh = idx / dh;
    const int i = idx % dh;
    Vp[((long long)kh * slots + rd.slot) * dh + i] = __float2bfloat16_rn(src[(H + KVH) * dh + kh * dh + i]);
  }
}

// ------------------------------------------------------------------ K1
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)),
               "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          (uint32_t)__cvta_generic_to_shared(dst)),
      "l"(src), "r"(bytes), "r"((uint32_t)__cvta_generic_to_shared(bar))
      : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = (uint32_t)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}

constexpr int kChunk = 64;
constexpr int kAttnThreads = 128;

template <int DH, int G>
__global__ void __launch_bounds__(kAttnThreads) tree_attn_kernel(const RowDesc* __restrict__ rows,
                                                                const Segment* __restrict__ segs,
                                                                const float* __restrict__ Qr, int H,
                                                                const __nv_bfloat16* __restrict__ Kp,
                                                                const __nv_bfloat16* __restrict__ Vp,
                                                                long long slots,
                                                                __nv_bfloat16* __restrict__ O) {
  constexpr int VPL = DH / 32;  // elements per lane in a K row
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __nv_bfloat16* sK = reinterpret_cast<__nv_bfloat16*>(smem_raw);            // [2][kChunk][DH]
  __nv_bfloat16* sV = sK + 2 * kChunk * DH;                                     // [2][kChunk][DH]
  float* sS = reinterpret_cast<float*>(sV + 2 * kChunk * DH);                  // [G][kChunk]
  float* sAlpha = sS + G * kChunk;                                              // [G]
  float* sL = sAlpha + G;                                                       // [G] running sum
  float* sM = sL + G;                                                           // [G] running max
  __shared__ uint64_t bar[2];

  const int r = blockIdx.x;
  const int kh = blockIdx.y;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const RowDesc rd = rows[r];
  const Segment* sg = segs + rd.seg_off;
  const __nv_bfloat16* Kh = Kp + (long long)kh * slots * DH;
  const __nv_bfloat16* Vh = Vp + (long long)kh * slots * DH;

  // q of the G heads of this group, VPL values per lane (log2e folded in)
  float qreg[G][VPL];
#pragma unroll
  for (int g = 0; g < G; ++g)
#pragma unroll
    for (int v = 0; v < VPL; ++v)
      qreg[g][v] = Qr[((long long)r * H + kh * G + g) * DH + lane * VPL + v] * 1.4426950408889634f;

  // count chunks
  int nchunks = 0;
  for (int s = 0; s < rd.nseg; ++s) nchunks += (sg[s].len + kChunk - 1) / kChunk;

  if (tid < G) {
    sM[tid] = -INFINITY;
    sL[tid] = 0.f;
  }
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // chunk cursor (identical in every thread)
  int seg_i = 0, seg_o = 0;
  auto next_chunk = [&](long long* base, int* len) {
    while (seg_i < rd.nseg && seg_o >= sg[seg_i].len) {
      ++seg_i;
      seg_o = 0;
    }
    *base = sg[seg_i].base + seg_o;
    int l = sg[seg_i].len - seg_o;
    *len = l < kChunk ? l : kChunk;
    seg_o += *len;
  };
  long long cb[2];
  int cl[2];
  // prologue: issue chunk 0 (and 1)
  for (int c = 0; c < 2 && c < nchunks; ++c) {
    next_chunk(&cb[c], &cl[c]);
    if (tid == 0) {
      const uint32_t bytes = (uint32_t)cl[c] * DH * 2;
      mbar_expect_tx(&bar[c], 2 * bytes);
      bulk_g2s(sK + c * kChunk * DH, Kh + cb[c] * DH, bytes, &bar[c]);
      bulk_g2s(sV + c * kChunk * DH, Vh + cb[c] * DH, bytes, &bar[c]);
    }
  }

  // accumulators: thread handles output dims (g, d) for d = tid % DH
  constexpr int OUT_PER_THREAD = (G * DH + kAttnThreads - 1) / kAttnThreads;
  float acc[OUT_PER_THREAD];
#pragma unroll
  for (int k = 0; k < OUT_PER_THREAD; ++k) acc[k] = 0.f;

  for (int c = 0; c < nchunks; ++c) {
    const int buf = c & 1;
    const int len = cl[buf];
    mbar_wait(&bar[buf], (uint32_t)((c >> 1) & 1));
    const __nv_bfloat16* K = sK + buf * kChunk * DH;
    const __nv_bfloat16* Vs = sV + buf * kChunk * DH;
    // scores
    for (int t = warp; t < len; t += kAttnThreads / 32) {
      float kv[VPL];
#pragma unroll
      for (int v2 = 0; v2 < VPL / 2; ++v2) {
        const __nv_bfloat162 a = *reinterpret_cast<const __nv_bfloat162*>(K + t * DH + lane * VPL + 2 * v2);
        kv[2 * v2] = __low2float(a);
        kv[2 * v2 + 1] = __high2float(a);
      }
#pragma unroll
      for (int g = 0; g < G; ++g) {
        float s = 0.f;
#pragma unroll
        for (int v = 0; v < VPL; ++v) s += qreg[g][v] * kv[v];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) sS[g * kChunk + t] = s;
      }
    }
    __syncthreads();
    // online softmax per head (warp g handles head g)
    for (int g = warp; g < G; g += kAttnThreads / 32) {
      float mx = -INFINITY;
      for (int t = lane; t < len; t += 32) mx = fmaxf(mx, sS[g * kChunk + t]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      const float m_old = sM[g];
      const float l_old = sL[g];
      const float m_new = fmaxf(m_old, mx);
      float sum = 0.f;
      for (int t = lane; t < len; t += 32) {
        const float p = exp2f(sS[g * kChunk + t] - m_new);
        sS[g * kChunk + t] = p;
        sum += p;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
      const float alpha = exp2f(m_old - m_new);
      __syncwarp();
      if (lane == 0) {
        sM[g] = m_new;
        sL[g] = l_old * alpha + sum;
        sAlpha[g] = alpha;
      }
    }
    __syncthreads();
    // PV
#pragma unroll
    for (int k = 0; k < OUT_PER_THREAD; ++k) {
      const int o = tid + k * kAttnThreads;
      if (o < G * DH) {
        const int g = o / DH, dcol = o % DH;
        float a = acc[k] * sAlpha[g];
        const float* p = sS + g * kChunk;
        for (int t = 0; t < len; ++t) a += p[t] * __bfloat162float(Vs[t * DH + dcol]);
        acc[k] = a;
      }
    }
    __syncthreads();
    // refill this buffer with chunk c + 2
    if (c + 2 < nchunks) {
      next_chunk(&cb[buf], &cl[buf]);
      if (tid == 0) {
        const uint32_t bytes = (uint32_t)cl[buf] * DH * 2;
        mbar_expect_tx(&bar[buf], 2 * bytes);
        bulk_g2s(sK + buf * kChunk * DH, Kh + cb[buf] * DH, bytes, &bar[buf]);
        bulk_g2s(sV + buf * kChunk * DH, Vh + cb[buf] * DH, bytes, &bar[buf]);
      }
    }
  }
#pragma unroll
  for (int k = 0; k < OUT_PER_THREAD; ++k) {
    const int o = tid + k * kAttnThreads;
    if (o < G * DH) {
      const int g = o / DH, dcol = o % DH;
      O[((long long)r * H + kh * G + g) * DH + dcol] = __float2bfloat16_rn(acc[k] / sL[g]);
    }
  }
}

__global__ void swiglu_kernel(const float* GU, int M, int F, __nv_bfloat16* A) {
  const long long n = (long long)M * F;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / F, j = i % F;
    const float g = GU[r * 2 * F + j];
    const float u = GU[r * 2 * F + F + j];
    A[i] = __float2bfloat16_rn(g / (1.f + __expf(-g)) * u);
  }
}

// K3: per-row argmax (first max), logsumexp and sum of the logits.
__global__ void lm_epilogue_kernel(const float* logits, int M, int V, int* amax, float* lse, float* lsum) {
  const int r = blockIdx.x;
  if (r >= M) return;
  const float* x = logits + (long long)r * V;
  float mx = -INFINITY;
  int mi = 0;
  float sm = 0.f;
  for (int i = threadIdx.x; i < V; i += blockDim.x) {
    const float v = x[i];
    if (v > mx) {
      mx = v;
      mi = i;
    }
    sm += v;
  }
  __shared__ float smx[32], ssm[32];
  __shared__ int smi[32];
  for (int o = 16; o > 0; o >>= 1) {
    const float om = __shfl_xor_sync(0xffffffffu, mx, o);
    const int oi = __shfl_xor_sync(0xffffffffu, mi, o);
    if (om > mx || (om == mx && oi < mi)) {
      mx = om;
      mi = oi;
    }
    sm += __shfl_xor_sync(0xffffffffu, sm, o);
  }
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    smx[w] = mx;
    smi[w] = mi;
    ssm[w] = sm;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < nw; ++k) {
      if (smx[k] > smx[0] || (smx[k] == smx[0] && smi[k] < smi[0])) {
        smx[0] = smx[k];
        smi[0] = smi[k];
      }
      ssm[0] += ssm[k];
    }
  }
  __syncthreads();
  const float gmax = smx[0];
  float se = 0.f;
  for (int i = threadIdx.x; i < V; i += blockDim.x) se += __expf(x[i] - gmax);
  for (int o = 16; o > 0; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) smx[w] = se;
  __syncthreads();
  if (threadIdx.x == 0) {
    float tot = 0.f;
    for (int k = 0; k < nw; ++k) tot += smx[k];
    amax[r] = smi[0];
    lse[r] = gmax + logf(tot);
    lsum[r] = ssm[0];
  }
}

// K4: PRM value head on the last token of each scored thought.
__global__ void value_head_kernel(const __nv_bfloat16* Hn, int d, const int* last_row, int n,
                                  const __nv_bfloat16* w, float* score) {
  const int k = blockIdx.x;
  if (k >= n) return;
  const __nv_bfloat16* h = Hn + (long long)last_row[k] * d;
  float s = 0.f;
  for (int i = threadIdx.x; i < d; i += blockDim.x) s += __bfloat162float(h[i]) * __bfloat162float(w[i]);
  __shared__ float red[32];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];
    score[k] = 1.f / (1.f + expf(-t));
  }
}

}  // namespace spex

// ------------------------------------------------------------------ launchers
using namespace spex;

extern "C" void spex_k_init_weights(__nv_bfloat16* w, long long n, uint64_t seed, uint64_t tid, float scale,
                                    cudaStream_t s) {
  init_weights_kernel<<<1184, 256, 0, s>>>(w, n, seed, tid, scale);
}

extern "C" void spex_k_build_decode_rows(TreeView t, const int* sids, const int* pos0, int n, int step,
                                         RowDesc* rows, Segment* segs, cudaStream_t s) {
  build_decode_rows_kernel<<<(n + 127) / 128, 128, 0, s>>>(t, sids, pos0, n, step, rows, segs);
}

extern "C" void spex_k_build_prm_rows(TreeView t, const int* sids, const int* row_start, int n, RowDesc* rows,
                                      Segment* segs, int* last_row, cudaStream_t s) {
  build_prm_rows_kernel<<<n, 128, 0, s>>>(t, sids, row_start, n, rows, segs, last_row);
}

extern "C" void spex_k_build_prompt_rows(TreeView t, int q0, int nq, RowDesc* rows, Segment* segs,
                                         cudaStream_t s) {
  const int n = nq * t.prompt_tokens;
  build_prompt_rows_kernel<<<(n + 127) / 128, 128, 0, s>>>(t, q0, nq, rows, segs);
}

extern "C" void spex_k_prm_scan_all(TreeView t, const int* kind, const int* off, const int* n, int n_entries,
                                    const int* srow_sid, int* row_start, int* totals, cudaStream_t s) {
  prm_scan_all_kernel<<<(n_entries + 127) / 128, 128, 0, s>>>(t, kind, off, n, n_entries, srow_sid, row_start,
                                                              totals);
}

extern "C" void spex_k_gather_prm(const RowDesc* rows, const int* last_row, int n, const float* score,
                                  PrmOut* out, cudaStream_t s) {
  gather_prm_kernel<<<(n + 127) / 128, 128, 0, s>>>(rows, last_row, n, score, out);
}

extern "C" void spex_k_gather_outputs(const RowDesc* rows, int M, const int* amax, const float* lse,
                                      const float* lsum, DecodeOut* out, cudaStream_t s) {
  gather_outputs_kernel<<<(M + 127) / 128, 128, 0, s>>>(rows, M, amax, lse, lsum, out);
}

extern "C" void spex_k_embed(const RowDesc* rows, int M, const __nv_bfloat16* E, int d, float* X, cudaStream_t s) {
  embed_kernel<<<M, 128, 0, s>>>(rows, M, E, d, X);
}

extern "C" void spex_k_rmsnorm(const float* X, int M, int d, float eps, __nv_bfloat16* Y, cudaStream_t s) {
  rmsnorm_bf16_kernel<<<M, 256, 0, s>>>(X, M, d, eps, Y);
}

extern "C" void spex_k_rope_kv(const RowDesc* rows, int M, const float* QKV, int H, int KVH, int dh,
                               const float* inv_freq, long long slots, __nv_bfloat16* Kp, __nv_bfloat16* Vp,
                               float* Qr, cudaStream_t s) {
  rope_kv_kernel<<<M, 128, 0, s>>>(rows, M, QKV, H, KVH, dh, inv_freq, slots, Kp, Vp, Qr);
}

template <int DH, int G>
static void launch_attn(const RowDesc* rows, const Segment* segs, const float* Qr, int H, int KVH,
                        const __nv_bfloat16* Kp, const __nv_bfloat16* Vp, long long slots, __nv_bfloat16* O, int M,
                        cudaStream_t s) {
  const size_t smem = 4 * kChunk * DH * sizeof(__nv_bfloat16) + (G * kChunk + 3 * G) * sizeof(float) + 64;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(tree_attn_kernel<DH, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  dim3 grid(M, KVH);
  tree_attn_kernel<DH, G><<<grid, kAttnThreads, smem, s>>>(rows, segs, Qr, H, Kp, Vp, slots, O);
}

extern "C" int spex_k_tree_attn(const RowDesc* rows, const Segment* segs, const float* Qr, int H, int KVH, int dh,
                                const __nv_bfloat16* Kp, const __nv_bfloat16* Vp, long long slots, __nv_bfloat16* O,
                                int M, cudaStream_t s) {
  const int G = H / KVH;
#define SPEX_ATTN_CASE(D, GG) \
  if (dh == D && G == GG) {   \
    launch_attn<D, GG>(rows, segs, Qr, H, KVH, Kp, Vp, slots, O, M, s); \
    return 0;                 \
  }
  SPEX_ATTN_CASE(128, 1)
  SPEX_ATTN_CASE(128, 2)
  SPEX_ATTN_CASE(128, 4)
  SPEX_ATTN_CASE(128, 6)
  SPEX_ATTN_CASE(128, 8)
  SPEX_ATTN_CASE(64, 1)
  SPEX_ATTN_CASE(64, 2)
  SPEX_ATTN_CASE(64, 4)
#undef SPEX_ATTN_CASE
  return -1;
}

extern "C" void spex_k_swiglu(const float* GU, int M, int F, __nv_bfloat16* A, cudaStream_t s) {
  swiglu_kernel<<<1184, 256, 0, s>>>(GU, M, F, A);
}

extern "C" void spex_k_lm_epilogue(const float* logits, int M, int V, int* amax, float* lse, float* lsum,
                                   cudaStream_t s) {
  lm_epilogue_kernel<<<M, 256, 0, s>>>(logits, M, V, amax, lse, lsum);
}

extern "C" void spex_k_value_head(const __nv_bfloat16* Hn, int d, const int* last_row, int n,
                                  const __nv_bfloat16* w, float* score, cudaStream_t s) {
  value_head_kernel<<<n, 128, 0, s>>>(Hn, d, last_row, n, w, score);
}
