// model_kernels.cu — device kernels of the policy / PRM forward over a batch
// of tree rows (one token of one thought per row).
//
//   K1 tree attention over a thought's ancestor chain in the paged tree KV
//                          pool: tree_attn_decode_kernel (decode rows, FHFMA.BF16),
//                          tree_attn_chunk_kernel (bounded chunks, opt-in),
//                          tree_attn_decode_mma_kernel (GQA decode on tensor cores),
//                          tree_attn_tile_mma_kernel (PRM/prompt rows, TMA + mma.sync),
//                          tree_attn_tile_kernel (PRM/prompt rows, dh = 64)
//   K3 lm_epilogue_kernel  per-row argmax / logsumexp / checksum of the logits
//   K4 value_head_kernel   PRM score sigmoid(w . h_last)
//   plus weight init, row descriptors, embedding, RMSNorm->bf16, RoPE + KV
//   append, SwiGLU.
#include <algorithm>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

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

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

constexpr int kMaxChain = 128;  // ancestors of one thought (deeper trees fail loudly: err bit 1)
constexpr int kPg = 16;         // tokens per tree-KV page (ctl_state.h kKvPage)

// Runs of consecutive physical pages among a thought's first `len` tokens.
__device__ __forceinline__ int count_runs(const int* __restrict__ pt, long long off, int len) {
  const int np = (len + kPg - 1) / kPg;
  int runs = 0, prev = -2;
  for (int j = 0; j < np; ++j) {
    const int p = pt[off + j];
    runs += p != prev + 1;
    prev = p;
  }
  return runs;
}

__device__ __forceinline__ int emit_runs(const int* __restrict__ pt, long long off, int len, int own, Segment* out) {
  const int np = (len + kPg - 1) / kPg;
  int k = 0;
  for (int j = 0; j < np;) {
    const int p0 = pt[off + j];
    int r = 1;
    while (j + r < np && pt[off + j + r] == p0 + r) ++r;
    const int tok = min(len - j * kPg, r * kPg);
    out[k].base = (long long)p0 * kPg;
    out[k].len = tok;
    out[k].own0 = own ? j * kPg : -1;
    ++k;
    j += r;
  }
  return k;
}

// Ancestors of `node`, root first; returns their count and the tokens they hold.
__device__ int ancestor_chain(const TreeView& t, uint32_t b, uint32_t node, uint32_t* chain, int* pre) {
  int n = 0;
  for (uint32_t c = t.parent[b + node]; c != 0xffffffffu && n < kMaxChain; c = t.parent[b + c]) ++n;
  if (n == kMaxChain) atomicOr(t.err, 1);  // deeper than the chain buffer: fail loudly
  int p = 0, i = n;
  for (uint32_t c = t.parent[b + node]; i > 0; c = t.parent[b + c]) {
    chain[--i] = c;
    p += t.tokens[b + c];
  }
  *pre = p;
  return n;
}

// Segment list of a row or thought: the ancestors' runs root-first, then the
// thought's own first `own_len` tokens (runs tagged with their positions).
// Space comes from the stream's segment pool; returns the offset (-1: full).
__device__ int build_segments(const TreeView& t, int q, uint32_t node, int own_len, Segment* segs, int* nseg,
                              int* abs_prefix) {
  const uint32_t b = (uint32_t)q * (uint32_t)t.node_cap;
  uint32_t chain[kMaxChain];
  int pre = 0;
  const int n = ancestor_chain(t, b, node, chain, &pre);
  int total = 0;
  for (int i = 0; i < n; ++i) {
    const int len = t.tokens[b + chain[i]];
    if (len > 0) total += count_runs(t.kv_pt, t.kvbase[b + chain[i]], len);
  }
  total += count_runs(t.kv_pt, t.kvbase[b + node], own_len);
  const int off = atomicAdd(t.seg_ctr, total);
  *abs_prefix = pre;
  if ((long long)off + total > t.seg_cap) {
    atomicOr(t.err, 2);
    *nseg = 0;
    return 0;
  }
  int k = 0;
  for (int i = 0; i < n; ++i) {
    const int len = t.tokens[b + chain[i]];
    if (len > 0) k += emit_runs(t.kv_pt, t.kvbase[b + chain[i]], len, 0, segs + off + k);
  }
  k += emit_runs(t.kv_pt, t.kvbase[b + node], own_len, 1, segs + off + k);
  *nseg = k;
  return off;
}

// KV slot of token `pos` of a node's thought.
__device__ __forceinline__ long long kv_slot(const TreeView& t, uint32_t b, uint32_t node, int pos) {
  return (long long)t.kv_pt[t.kvbase[b + node] + pos / kPg] * kPg + pos % kPg;
}

__global__ void build_decode_rows_kernel(TreeView t, const int* sids, const int* pos0, int n, int step,
                                         RowDesc* rows, Segment* segs) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int sid = sids[i];
  const int q = t.st_q[sid];
  const uint32_t node = t.st_node[sid];
  const int pos = pos0[i] + step;
  int pre = 0, ns = 0;
  const int off = build_segments(t, q, node, pos + 1, segs, &ns, &pre);
  const uint32_t b = (uint32_t)q * (uint32_t)t.node_cap;
  RowDesc r;
  r.q = q;
  r.node = node;
  r.pos = pos;
  r.abs_pos = pre + pos;
  r.slot = kv_slot(t, b, node, pos);
  r.seg_off = off;
  r.nseg = ns;
  r.token = token_id(t.hash[b + node], pos, t.V);
  r.pad = 0;
  rows[i] = r;
}

// PRM rows: thought k of the entry occupies rows [row_start[k], row_start[k] + len).
// The thought's rows share one segment list (ancestors + the whole thought);
// the tile kernels clip the own runs at each tile's last row (causal).
__global__ void build_prm_rows_kernel(TreeView t, const int* sids, const int* row_start, const int* tile_start,
                                      int n, RowDesc* rows, Segment* segs, int* last_row, TileDesc* tiles) {
  const int k = blockIdx.x;
  if (k >= n) return;
  const int sid = sids[k];
  const int q = t.st_q[sid];
  const uint32_t node = t.st_node[sid];
  const uint32_t b = (uint32_t)q * (uint32_t)t.node_cap;
  const int len = t.tokens[b + node];
  const int r0 = row_start[k];
  __shared__ int s_off, s_ns, s_pre;
  if (threadIdx.x == 0) {
    int ns = 0, pre = 0;
    s_off = build_segments(t, q, node, len, segs, &ns, &pre);
    s_ns = ns;
    s_pre = pre;
  }
  __syncthreads();
  for (int j = threadIdx.x; j < len; j += blockDim.x) {
    const int i = r0 + j;
    RowDesc r;
    r.q = q;
    r.node = node;
    r.pos = j;
    r.abs_pos = s_pre + j;
    r.slot = kv_slot(t, b, node, j);
    r.seg_off = s_off;
    r.nseg = s_ns;
    r.token = token_id(t.hash[b + node], j, t.V);
    r.pad = 0;
    rows[i] = r;
  }
  if (threadIdx.x == 0) last_row[k] = r0 + len - 1;
  for (int j = threadIdx.x; j * kTileRows < len; j += blockDim.x) {
    TileDesc td;
    td.row0 = r0 + j * kTileRows;
    td.nrows = len - j * kTileRows < kTileRows ? len - j * kTileRows : kTileRows;
    tiles[tile_start[k] + j] = td;
  }
}

// Root prompt rows: query q, positions 0..P-1. Nothing here reads state the
// control kernel writes (it may not have admitted the query yet): the root's
// path hash is a pure function of the run seed (generate_workload's query
// seed, sim.cpp:177-180, and the root hash, tree.cpp:57) and its pages are the
// static [q*pp, (q+1)*pp), consecutive, so each row has one segment (segs[i]).
__global__ void build_prompt_rows_kernel(TreeView t, int q0, int nq, RowDesc* rows, Segment* segs) {
  const int P = t.prompt_tokens;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nq * P) return;
  const int q = q0 + i / P;
  const int j = i % P;
  const long long base = (long long)q * t.kv_pp_root * kPg;
  const uint64_t base_seed = d_splitmix64(t.run_seed ^ 0x7175657200000008ULL);  // ctl_math.h kSaltQuery
  const uint64_t qv = (uint64_t)(q + t.q_offset) + 1 + 0x9e3779b97f4a7c15ULL;                      // ctl_math.h hash_mix
  const uint64_t root_hash = d_splitmix64(d_splitmix64(base_seed ^ (qv + (base_seed << 6) + (base_seed >> 2))));
  Segment* s = segs + i;
  s->base = base;
  s->len = j + 1;
  s->own0 = 0;
  RowDesc r;
  r.q = q;
  r.node = 0;
  r.pos = j;
  r.abs_pos = j;
  r.slot = base + j;
  r.seg_off = i;
  r.nseg = 1;
  r.token = token_id(root_hash, j, t.V);
  r.pad = 0;
  rows[i] = r;
}

// Tiles over root prompt rows: query-major, kTileRows consecutive positions.
__global__ void build_prompt_tiles_kernel(int nq, int P, TileDesc* tiles) {
  const int per = (P + kTileRows - 1) / kTileRows;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nq * per) return;
  const int q = i / per, j = i % per;
  TileDesc td;
  td.row0 = q * P + j * kTileRows;
  td.nrows = P - j * kTileRows < kTileRows ? P - j * kTileRows : kTileRows;
  tiles[i] = td;
}

// PRM row counts per reward batch (sum of token_len of the scored thoughts)
// and the per-thought exclusive scan; one thread per schedule entry.
__global__ void prm_scan_all_kernel(TreeView t, const int* kind, const int* off, const int* cnt, int n_entries,
                                    const int* srow_sid, int* row_start, int* tile_start, int* totals,
                                    int* tile_totals) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n_entries) return;
  if (kind[e] != SCHED_PRM) {
    totals[e] = 0;
    tile_totals[e] = 0;
    return;
  }
  int acc = 0, tacc = 0;
  for (int k = 0; k < cnt[e]; ++k) {
    const int sid = srow_sid[off[e] + k];
    row_start[off[e] + k] = acc;
    tile_start[off[e] + k] = tacc;
    const int len = t.tokens[(uint32_t)t.st_q[sid] * (uint32_t)t.node_cap + t.st_node[sid]];
    acc += len;
    tacc += (len + kTileRows - 1) / kTileRows;
  }
  totals[e] = acc;
  tile_totals[e] = tacc;
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
  // one warp per row, 8 bf16 per lane per step (d % 8 == 0)
  const int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (r >= M) return;
  const uint4* e = reinterpret_cast<const uint4*>(E + (long long)rows[r].token * d);
  float4* x = reinterpret_cast<float4*>(X + (long long)r * d);
  for (int i = lane; i < d / 8; i += 32) {
    const uint4 v = e[i];
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
    x[2 * i] = make_float4(__low2float(h[0]), __high2float(h[0]), __low2float(h[1]), __high2float(h[1]));
    x[2 * i + 1] = make_float4(__low2float(h[2]), __high2float(h[2]), __low2float(h[3]), __high2float(h[3]));
  }
}

// y = bf16(x * rsqrt(mean(x^2) + eps))  (unit gains)
// Programmatic dependent launch: kernels launched with the PDL attribute may
// start while the previous kernel on the stream drains; they wait here until
// its writes are visible (a no-op for a normal launch).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__global__ void rmsnorm_bf16_kernel(const float* X, int M, int d, float eps, __nv_bfloat16* Y) {
  pdl_wait();
  // one warp per row, float4 loads (d % 4 == 0); the second pass re-reads the
  // row from L1
  const int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (r >= M) return;
  const float4* x = reinterpret_cast<const float4*>(X + (long long)r * d);
  float ss = 0.f;
  for (int i = lane; i < d / 4; i += 32) {
    const float4 v = x[i];
    ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  const float inv = rsqrtf(ss / (float)d + eps);
  uint2* y = reinterpret_cast<uint2*>(Y + (long long)r * d);
  for (int i = lane; i < d / 4; i += 32) {
    const float4 v = x[i];
    uint2 o;
    o.x = pack_bf16(v.x * inv, v.y * inv);
    o.y = pack_bf16(v.z * inv, v.w * inv);
    y[i] = o;
  }
}

// The same with the row held in registers (d == 128 * NV): one pass over HBM,
// all NV loads of a lane in flight at once; identical arithmetic and order.
template <int NV>
__global__ void rmsnorm_bf16_reg_kernel(const float* X, int M, float eps, __nv_bfloat16* Y) {
  pdl_wait();
  constexpr int d = 128 * NV;
  const int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (r >= M) return;
  const float4* x = reinterpret_cast<const float4*>(X + (long long)r * d);
  float4 v[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = x[lane + 32 * k];
  float ss = 0.f;
#pragma unroll
  for (int k = 0; k < NV; ++k) ss += v[k].x * v[k].x + v[k].y * v[k].y + v[k].z * v[k].z + v[k].w * v[k].w;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  const float inv = rsqrtf(ss / (float)d + eps);
  uint2* y = reinterpret_cast<uint2*>(Y + (long long)r * d);
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    uint2 o;
    o.x = pack_bf16(v[k].x * inv, v[k].y * inv);
    o.y = pack_bf16(v[k].z * inv, v[k].w * inv);
    y[lane + 32 * k] = o;
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

// The same with an L2 eviction-priority policy (tree KV streamed once per
// step: evict_first keeps it from displacing reused lines — weights, the
// control kernel's state and code).
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                              uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          (uint32_t)__cvta_generic_to_shared(dst)),
      "l"(src), "r"(bytes), "r"((uint32_t)__cvta_generic_to_shared(bar)), "l"(policy)
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

// Tokens of a segment inside a tile's causal horizon: an own-thought run is
// cut at position `clip` (ancestor runs are whole).
__device__ __forceinline__ int seg_len_eff(const Segment& sg, int clip) {
  return sg.own0 < 0 ? sg.len : max(0, min(sg.len, clip - sg.own0));
}
constexpr int kAttnThreads = 128;


// K1 decode variant: one warp per (row, kv head) streams the row's context with
// 128-bit coalesced loads — a half-warp covers one 256-byte K (or V) row, so a
// warp consumes two tokens per load instruction and keeps UNROLL token pairs in
// flight. Scores and P.V use the sm_100 mixed-precision FMA (FHFMA.BF16:
// fp32 += bf16 x bf16, the bf16 product exact) straight on the packed K/V
// registers — no bf16->fp32 unpacking; q and p enter as bf16 exactly like the
// operands of the tensor-core tile kernel. One online-softmax update per UNROLL
// group (warp-uniform running max; the rescale is skipped when it does not
// move). No shared memory and no block barriers: decode rows have no intra-row
// reuse, occupancy is bounded only by registers.

__device__ __forceinline__ uint4 ld_stream(const __nv_bfloat16* p, uint64_t pol) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p), "l"(pol));
  return v;
}

__device__ __forceinline__ void fma2_bf16(float& acc, uint32_t a2, uint32_t b2) {
  asm("{.reg .b16 al, ah, bl, bh;\n\t"
      "mov.b32 {al, ah}, %1;\n\t"
      "mov.b32 {bl, bh}, %2;\n\t"
      "fma.rn.f32.bf16 %0, al, bl, %0;\n\t"
      "fma.rn.f32.bf16 %0, ah, bh, %0;}"
      : "+f"(acc)
      : "r"(a2), "r"(b2));
}

// acc[2e], acc[2e+1] += p * v2.{lo,hi}  (p already bf16 in both halves of p2)
__device__ __forceinline__ void fma_pv_bf16(float& a0, float& a1, uint32_t p2, uint32_t v2) {
  asm("{.reg .b16 pl, ph, vl, vh;\n\t"
      "mov.b32 {pl, ph}, %2;\n\t"
      "mov.b32 {vl, vh}, %3;\n\t"
      "fma.rn.f32.bf16 %0, pl, vl, %0;\n\t"
      "fma.rn.f32.bf16 %1, pl, vh, %1;}"
      : "+f"(a0), "+f"(a1)
      : "r"(p2), "r"(v2));
}

template <int DH, int G, int UNROLL>
__global__ void __launch_bounds__(256, (UNROLL > 4 ? 2 : (G == 1 ? 4 : (G <= 4 ? 2 : 1)))) tree_attn_decode_kernel(const RowDesc* __restrict__ rows,
                                                                 const Segment* __restrict__ segs,
                                                                 const float* __restrict__ Qr, int H, int KVH, int M,
                                                                 const __nv_bfloat16* __restrict__ Kp,
                                                                 const __nv_bfloat16* __restrict__ Vp,
                                                                 long long slots, __nv_bfloat16* __restrict__ O) {
  constexpr int EPL = 8;              // bf16 elements per lane per token (16 bytes)
  constexpr int LPT = DH / EPL;       // lanes per token (16 for DH=128, 8 for DH=64)
  constexpr int TPW = 32 / LPT;       // tokens per warp load (2 or 4)
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (gw >= M * KVH) return;
  const int r = gw / KVH, kh = gw % KVH;
  const int sub = lane / LPT;         // which token of the pair/quad
  const int li = lane % LPT;          // dim block
  const RowDesc rd = rows[r];
  const Segment* sg = segs + rd.seg_off;
  const __nv_bfloat16* Kh = Kp + (long long)kh * slots * DH + li * EPL;
  const __nv_bfloat16* Vh = Vp + (long long)kh * slots * DH + li * EPL;
  uint64_t pol;  // KV is streamed once per step: evict first, keep L2 for reused state
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  uint32_t q2[G][EPL / 2];  // q * log2(e), bf16 pairs
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const float4* qp = reinterpret_cast<const float4*>(Qr + ((long long)r * H + kh * G + g) * DH + li * EPL);
    const float4 a = qp[0], b = qp[1];
    constexpr float L2E = 1.4426950408889634f;
    q2[g][0] = pack_bf16(a.x * L2E, a.y * L2E);
    q2[g][1] = pack_bf16(a.z * L2E, a.w * L2E);
    q2[g][2] = pack_bf16(b.x * L2E, b.y * L2E);
    q2[g][3] = pack_bf16(b.z * L2E, b.w * L2E);
  }
  float m[G], l[G], acc[G][EPL];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    m[g] = -INFINITY;
    l[g] = 0.f;
#pragma unroll
    for (int e = 0; e < EPL; ++e) acc[g][e] = 0.f;
  }
  for (int si = 0; si < rd.nseg; ++si) {
    const long long base = sg[si].base;
    const int len = sg[si].len;
    for (int t0 = 0; t0 < len; t0 += TPW * UNROLL) {
      uint4 kraw[UNROLL], vraw[UNROLL];
      bool ok[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        const int t = t0 + u * TPW + sub;
        ok[u] = t < len;
        const long long off = (base + (ok[u] ? t : 0)) * DH;
        kraw[u] = ld_stream(Kh + off, pol);
        vraw[u] = ld_stream(Vh + off, pol);
      }
#pragma unroll
      for (int g = 0; g < G; ++g) {
        float sc[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
          float a = 0.f;
          fma2_bf16(a, q2[g][0], kraw[u].x);
          fma2_bf16(a, q2[g][1], kraw[u].y);
          fma2_bf16(a, q2[g][2], kraw[u].z);
          fma2_bf16(a, q2[g][3], kraw[u].w);
          sc[u] = a;
        }
#pragma unroll
        for (int o = LPT / 2; o > 0; o >>= 1)
#pragma unroll
          for (int u = 0; u < UNROLL; ++u) sc[u] += __shfl_xor_sync(0xffffffffu, sc[u], o);
        float mx = -INFINITY;
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
          if (!ok[u]) sc[u] = -INFINITY;
          mx = fmaxf(mx, sc[u]);
        }
#pragma unroll
        for (int o = LPT; o < 32; o <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if (mx > m[g]) {  // warp-uniform
          const float scale = exp2f(m[g] - mx);  // m == -inf -> 0
          l[g] *= scale;
#pragma unroll
          for (int e = 0; e < EPL; ++e) acc[g][e] *= scale;
          m[g] = mx;
        }
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
          const float p = exp2f(sc[u] - m[g]);  // masked tokens: exp2(-inf) = 0
          const __nv_bfloat16 pb = __float2bfloat16_rn(p);
          l[g] += __bfloat162float(pb);
          const uint32_t p2 = (uint32_t)__bfloat16_as_ushort(pb) * 0x10001u;
          fma_pv_bf16(acc[g][0], acc[g][1], p2, vraw[u].x);
          fma_pv_bf16(acc[g][2], acc[g][3], p2, vraw[u].y);
          fma_pv_bf16(acc[g][4], acc[g][5], p2, vraw[u].z);
          fma_pv_bf16(acc[g][6], acc[g][7], p2, vraw[u].w);
        }
      }
    }
  }
  // combine the TPW token lanes holding the same dims
#pragma unroll
  for (int g = 0; g < G; ++g) {
#pragma unroll
    for (int o = LPT; o < 32; o <<= 1) {
      l[g] += __shfl_xor_sync(0xffffffffu, l[g], o);
#pragma unroll
      for (int e = 0; e < EPL; ++e) acc[g][e] += __shfl_xor_sync(0xffffffffu, acc[g][e], o);
    }
    if (sub == 0) {
      const float inv = 1.f / l[g];
      __nv_bfloat16* op = O + ((long long)r * H + kh * G + g) * DH + li * EPL;
      uint4 packed;
      __nv_bfloat162* pk = reinterpret_cast<__nv_bfloat162*>(&packed);
#pragma unroll
      for (int e = 0; e < EPL / 2; ++e) pk[e] = __floats2bfloat162_rn(acc[g][2 * e] * inv, acc[g][2 * e + 1] * inv);
      *reinterpret_cast<uint4*>(op) = packed;
    }
  }
}

// K1 decode, bulk-copy pipeline (G = 1): a persistent grid of warps; each warp
// claims (row, kv head) items from a device counter and streams their tree
// context through its own ring of NST shared-memory stages of CH tokens (K and
// V rows of one head are contiguous in the pool, so a stage is two
// cp.async.bulk copies completing on one mbarrier). The copy engine keeps
// NST-1 chunks in flight per warp across item and segment boundaries without
// holding registers; lanes read the staged rows with 128-bit shared loads
// (half a warp per 256-byte row) into the same FHFMA.BF16 math as
// tree_attn_decode_kernel, one online-softmax update per chunk.
// One Segment (16 bytes) in a single load.
__device__ __forceinline__ void load_seg(const Segment* sp, long long& base, int& len) {
  const int4 v = __ldg(reinterpret_cast<const int4*>(sp));
  base = (long long)(((unsigned long long)(unsigned)v.y << 32) | (unsigned)v.x);
  len = v.z;
}

template <int kBulkCH, int kBulkNST, int kBulkWarps>  // tokens per stage, stages per warp, warps per block
__global__ void __launch_bounds__(kBulkWarps * 32, 1)
    tree_attn_bulk_kernel(const RowDesc* __restrict__ rows, const Segment* __restrict__ segs,
                          const float* __restrict__ Qr, int H, int KVH, int n_items,
                          const __nv_bfloat16* __restrict__ Kp, const __nv_bfloat16* __restrict__ Vp, long long slots,
                          __nv_bfloat16* __restrict__ O, int* __restrict__ item_ctr, int kv_evict_first,
                          const int* __restrict__ row_order) {
  constexpr int DH = 128, EPL = 8, LPT = 16, STAGE = kBulkCH * DH * 2;  // 4 KB of K (and of V) per stage
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ uint64_t bar[kBulkWarps][kBulkNST];
  pdl_wait();
  __shared__ int queue[kBulkWarps][8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* ring = smem_raw + (size_t)warp * kBulkNST * 2 * STAGE;  // [stage][K|V][STAGE]
  const int sub = lane / LPT, li = lane % LPT;
  if (lane == 0) {
    for (int i = 0; i < kBulkNST; ++i) mbar_init(&bar[warp][i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  uint64_t kv_pol;  // KV is streamed once per step: evict first
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(kv_pol));
  // ---- producer cursor (lane 0 only). The producer lane is on the critical
  // path of every stage: per stage it only issues the two copies from running
  // K / V pointers; a segment costs one 16-byte load (the GQA kernel's lesson,
  // profiles/r02zt_k1_gqa_tma_ab.txt).
  int p_q = 0;                   // items claimed so far (queue position)
  int p_item = -1, p_seg = 0, p_nseg = 0;
  long long p_segoff = 0;
  const Segment* p_sg = nullptr;
  const __nv_bfloat16* p_k = nullptr;  // next chunk's K / V rows
  const __nv_bfloat16* p_v = nullptr;
  int p_left = 0;                      // tokens left in the current segment
  bool p_done = false;
  int issued = 0;
  auto produce = [&]() {  // lane 0: issue the next chunk into stage issued % NST
    while (!p_done) {
      if (p_left > 0) {
        const int n = p_left < kBulkCH ? p_left : kBulkCH;
        const int st = issued % kBulkNST;
        unsigned char* kb = ring + st * 2 * STAGE;
        mbar_expect_tx(&bar[warp][st], 2u * n * DH * 2);
        if (kv_evict_first) {
          bulk_g2s_hint(kb, p_k, n * DH * 2, &bar[warp][st], kv_pol);
          bulk_g2s_hint(kb + STAGE, p_v, n * DH * 2, &bar[warp][st], kv_pol);
        } else {
          bulk_g2s(kb, p_k, n * DH * 2, &bar[warp][st]);
          bulk_g2s(kb + STAGE, p_v, n * DH * 2, &bar[warp][st]);
        }
        p_k += kBulkCH * DH;
        p_v += kBulkCH * DH;
        p_left -= n;
        ++issued;
        return;
      }
      if (p_item >= 0 && p_seg < p_nseg) {  // next segment of the item
        long long base;
        load_seg(p_sg + p_seg, base, p_left);
        ++p_seg;
        p_k = Kp + (p_segoff + base) * DH;
        p_v = Vp + (p_segoff + base) * DH;
        continue;
      }
      const int it = atomicAdd(item_ctr, 1);  // next item
      if (it >= n_items) {
        queue[warp][p_q & 7] = -1;
        p_done = true;
        // item_ctr[1] counts warps past their last claim; the last one
        // re-zeroes both, so the next launch needs no memset
        if (atomicAdd(item_ctr + 1, 1) == (int)gridDim.x * kBulkWarps - 1) {
          item_ctr[1] = 0;
          atomicExch(item_ctr, 0);
        }
        return;
      }
      queue[warp][p_q & 7] = it;
      ++p_q;
      p_item = it;
      const RowDesc rd = rows[row_order ? row_order[it / KVH] : it / KVH];
      p_sg = segs + rd.seg_off;
      p_nseg = rd.nseg;
      p_seg = 0;
      p_segoff = (long long)(it % KVH) * slots;
    }
  };
  if (lane == 0)
    for (int i = 0; i < kBulkNST - 1; ++i) produce();
  __syncwarp();
  // ---- consumer cursor (all lanes)
  int c_q = 0, consumed = 0;
  for (;;) {
    const int it = queue[warp][c_q & 7];
    if (it < 0) break;
    ++c_q;
    const int r = row_order ? row_order[it / KVH] : it / KVH, kh = it % KVH;
    const RowDesc rd = rows[r];
    const Segment* sg = segs + rd.seg_off;
    uint32_t q2[EPL / 2];
    {
      const float4* qp = reinterpret_cast<const float4*>(Qr + ((long long)r * H + kh) * DH + li * EPL);
      const float4 a = qp[0], b = qp[1];
      constexpr float L2E = 1.4426950408889634f;
      q2[0] = pack_bf16(a.x * L2E, a.y * L2E);
      q2[1] = pack_bf16(a.z * L2E, a.w * L2E);
      q2[2] = pack_bf16(b.x * L2E, b.y * L2E);
      q2[3] = pack_bf16(b.z * L2E, b.w * L2E);
    }
    float m = -INFINITY, l = 0.f, acc[EPL];
#pragma unroll
    for (int e = 0; e < EPL; ++e) acc[e] = 0.f;
    // segment lengths: 32 at a time, one per lane (one load latency instead of one per segment)
    int seg_len = 0;
    for (int si = 0; si < rd.nseg; ++si) {
      if ((si & 31) == 0) seg_len = si + lane < rd.nseg ? sg[si + lane].len : 0;
      const int len = __shfl_sync(0xffffffffu, seg_len, si & 31);
      for (int off = 0; off < len; off += kBulkCH) {
        const int n = min(kBulkCH, len - off);
        if (lane == 0) produce();  // keep NST-1 chunks in flight (stage consumed last round is free)
        const int st = consumed % kBulkNST;
        mbar_wait(&bar[warp][st], (uint32_t)((consumed / kBulkNST) & 1));
        const unsigned char* kb = ring + st * 2 * STAGE;
        float sc[kBulkCH / 2];
        uint4 vr[kBulkCH / 2];
#pragma unroll
        for (int u = 0; u < kBulkCH / 2; ++u) {
          const int t = 2 * u + sub;
          const uint4 kr = *reinterpret_cast<const uint4*>(kb + t * DH * 2 + li * 16);
          vr[u] = *reinterpret_cast<const uint4*>(kb + STAGE + t * DH * 2 + li * 16);
          float a = 0.f;
          fma2_bf16(a, q2[0], kr.x);
          fma2_bf16(a, q2[1], kr.y);
          fma2_bf16(a, q2[2], kr.z);
          fma2_bf16(a, q2[3], kr.w);
          sc[u] = a;
        }
#pragma unroll
        for (int o = LPT / 2; o > 0; o >>= 1)
#pragma unroll
          for (int u = 0; u < kBulkCH / 2; ++u) sc[u] += __shfl_xor_sync(0xffffffffu, sc[u], o);
        float mx = -INFINITY;
#pragma unroll
        for (int u = 0; u < kBulkCH / 2; ++u) {
          if (2 * u + sub >= n) sc[u] = -INFINITY;
          mx = fmaxf(mx, sc[u]);
        }
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, LPT));
        if (mx > m) {  // warp-uniform
          const float scale = exp2f(m - mx);
          l *= scale;
#pragma unroll
          for (int e = 0; e < EPL; ++e) acc[e] *= scale;
          m = mx;
        }
#pragma unroll
        for (int u = 0; u < kBulkCH / 2; ++u) {
          if (2 * u + sub < n) {  // staged rows beyond n are stale: never touch them
            const __nv_bfloat16 pb = __float2bfloat16_rn(exp2f(sc[u] - m));
            l += __bfloat162float(pb);
            const uint32_t p2 = (uint32_t)__bfloat16_as_ushort(pb) * 0x10001u;
            fma_pv_bf16(acc[0], acc[1], p2, vr[u].x);
            fma_pv_bf16(acc[2], acc[3], p2, vr[u].y);
            fma_pv_bf16(acc[4], acc[5], p2, vr[u].z);
            fma_pv_bf16(acc[6], acc[7], p2, vr[u].w);
          }
        }
        ++consumed;
        __syncwarp();  // stage st fully read before lane 0 refills it
      }
    }
    // combine the two token halves, write O
    l += __shfl_xor_sync(0xffffffffu, l, LPT);
#pragma unroll
    for (int e = 0; e < EPL; ++e) acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], LPT);
    if (sub == 0) {
      const float inv = 1.f / l;
      uint4 packed;
      packed.x = pack_bf16(acc[0] * inv, acc[1] * inv);
      packed.y = pack_bf16(acc[2] * inv, acc[3] * inv);
      packed.z = pack_bf16(acc[4] * inv, acc[5] * inv);
      packed.w = pack_bf16(acc[6] * inv, acc[7] * inv);
      *reinterpret_cast<uint4*>(O + ((long long)r * H + kh) * DH + li * EPL) = packed;
    }
  }
}

// ----------------------------------------------------------------------------
// K1 tile variant on tensor cores (PRM / prompt prefill rows, DH = 128).
// K/V chunks of 64 tokens arrive by TMA (2D tensor maps over the pool viewed as
// [KVH*slots][128], two 64-element boxes per chunk, 128-byte swizzle) into a
// double buffer guarded by mbarriers. Each warp takes (head g, token slice of
// 64/SPLIT tokens): S = Q K^T and O += P V with mma.sync m16n8k16 (bf16 in,
// fp32 accumulate), fragments via ldmatrix (.trans for V), online softmax in
// registers; warps of the same head merge (m, l, O) through shared memory.
// ----------------------------------------------------------------------------
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(map), "r"(c0), "r"(c1),
      "r"((uint32_t)__cvta_generic_to_shared(bar))
      : "memory");
}

// 4D box (64 columns, rows, 2 column halves, K|V): ONE copy lands a whole
// decode stage — K then V, each as [half][row][64] (tree_attn_wmma_kernel,
// spex_tmap_kv16)
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
      "l"(map), "r"(0), "r"(c1), "r"(0), "r"(0), "r"((uint32_t)__cvta_generic_to_shared(bar))
      : "memory");
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}

__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}

__device__ __forceinline__ void mma_bf16(float* c, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}


// byte offset of (row, 16-byte chunk c in [0,16)) in a swizzled [2 halves][64 rows][128 B] chunk buffer
__device__ __forceinline__ uint32_t swz(int row, int c) {
  const int half = c >> 3, cc = c & 7;
  return (uint32_t)(half * 8192 + row * 128 + ((cc ^ (row & 7)) << 4));
}

template <int G>
__global__ void __launch_bounds__(128) tree_attn_tile_mma_kernel(const __grid_constant__ CUtensorMap kvmap,
                                                                const TileDesc* __restrict__ tiles,
                                                                const RowDesc* __restrict__ rows,
                                                                const Segment* __restrict__ segs,
                                                                const float* __restrict__ Qr, int H, long long slots,
                                                                __nv_bfloat16* __restrict__ O, int Gt) {
  // G query heads per block; a KV head's Gt heads are split over Gt / G blocks
  // (blockIdx.y = kh * (Gt / G) + part), e.g. Gt = 6 -> 3 blocks of 2 heads
  constexpr int DH = 128;
  constexpr int SPLIT = 4 / G;          // warps per head
  constexpr int TW = kChunk / SPLIT;    // tokens per warp per chunk (16, 32 or 64)
  constexpr int NT = TW / 8;            // n8 score tiles per warp
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* sbase = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // [buf][K|V][16 KB]
  __shared__ uint64_t bar[2];
  __shared__ int sPos[kTileRows];
  __shared__ float sMl[4][2][kTileRows];  // per warp: m, l per row
  const TileDesc td = tiles[blockIdx.x];
  const int parts = Gt / G;
  const int kh = blockIdx.y / parts, hbase = kh * Gt + (blockIdx.y - kh * parts) * G;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = warp / SPLIT, slice = warp % SPLIT;
  const RowDesc last = rows[td.row0 + td.nrows - 1];
  const Segment* sg = segs + last.seg_off;
  const int nseg = last.nseg;
  if (tid < kTileRows) sPos[tid] = tid < td.nrows ? rows[td.row0 + tid].pos : -1;
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  int nchunks = 0;
  const int clip = last.pos + 1;  // the tile's causal horizon inside its own thought
  for (int s = 0; s < nseg; ++s) nchunks += (seg_len_eff(sg[s], clip) + kChunk - 1) / kChunk;
  // Q fragments (A operand, 16 rows x 128), rows beyond nrows are zero
  const int gq = lane >> 2, tq = lane & 3;
  uint32_t qa[8][4];
  {
    const int r0 = gq, r1 = gq + 8;
    const bool v0 = r0 < td.nrows, v1 = r1 < td.nrows;
    const float* q0 = Qr + ((long long)(td.row0 + (v0 ? r0 : 0)) * H + hbase + g) * DH;
    const float* q1 = Qr + ((long long)(td.row0 + (v1 ? r1 : 0)) * H + hbase + g) * DH;
    const float sc = 1.4426950408889634f;
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      const int k0 = ks * 16 + tq * 2;
      const float2 x00 = v0 ? *reinterpret_cast<const float2*>(q0 + k0) : make_float2(0.f, 0.f);
      const float2 x10 = v1 ? *reinterpret_cast<const float2*>(q1 + k0) : make_float2(0.f, 0.f);
      const float2 x01 = v0 ? *reinterpret_cast<const float2*>(q0 + k0 + 8) : make_float2(0.f, 0.f);
      const float2 x11 = v1 ? *reinterpret_cast<const float2*>(q1 + k0 + 8) : make_float2(0.f, 0.f);
      qa[ks][0] = pack_bf16(x00.x * sc, x00.y * sc);
      qa[ks][1] = pack_bf16(x10.x * sc, x10.y * sc);
      qa[ks][2] = pack_bf16(x01.x * sc, x01.y * sc);
      qa[ks][3] = pack_bf16(x11.x * sc, x11.y * sc);
    }
  }
  __syncthreads();
  int seg_i = 0, seg_o = 0;
  long long cb[2];
  int cl[2], cown[2];
  auto next_chunk = [&](int b) {
    while (seg_i < nseg && seg_o >= seg_len_eff(sg[seg_i], clip)) {
      ++seg_i;
      seg_o = 0;
    }
    cb[b] = sg[seg_i].base + seg_o;
    const int l = seg_len_eff(sg[seg_i], clip) - seg_o;
    cl[b] = l < kChunk ? l : kChunk;
    cown[b] = sg[seg_i].own0 >= 0 ? sg[seg_i].own0 + seg_o : -1;
    seg_o += cl[b];
  };
  auto issue = [&](int b) {
    unsigned char* kb = sbase + b * 32768;
    unsigned char* vb = kb + 16384;
    const int rowc = (int)((long long)kh * slots + cb[b]);
    mbar_expect_tx(&bar[b], 32768);
    tma_load_4d(kb, &kvmap, rowc, &bar[b]);  // one copy: K at kb, V at kb + 16384 (= vb)
    (void)vb;
  };
  for (int c = 0; c < 2 && c < nchunks; ++c) {
    next_chunk(c);
    if (tid == 0) issue(c);
  }
  float oacc[16][4];
#pragma unroll
  for (int n = 0; n < 16; ++n) oacc[n][0] = oacc[n][1] = oacc[n][2] = oacc[n][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;  // rows gq and gq+8
  const int pos0 = sPos[gq], pos1 = sPos[gq + 8];
  for (int c = 0; c < nchunks; ++c) {
    const int b = c & 1;
    const int len = cl[b], own0 = cown[b];
    mbar_wait(&bar[b], (uint32_t)((c >> 1) & 1));
    const uint32_t kb = (uint32_t)__cvta_generic_to_shared(sbase + b * 32768);
    const uint32_t vb = kb + 16384;
    const int t_base = slice * TW;
    // S = Q K^T for this warp's token slice
    float sacc[NT][4];
#pragma unroll
    for (int n = 0; n < NT; ++n) sacc[n][0] = sacc[n][1] = sacc[n][2] = sacc[n][3] = 0.f;
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
#pragma unroll
      for (int n2 = 0; n2 < NT / 2; ++n2) {
        // two n8 tiles (16 tokens) x k16: matrices {tok 0-7,k0-7},{tok 0-7,k8-15},{tok 8-15,k0-7},{tok 8-15,k8-15}
        const int mi = lane >> 3, ri = lane & 7;
        const int tok = t_base + n2 * 16 + (mi >> 1) * 8 + ri;
        const int chunk16 = ks * 2 + (mi & 1);
        uint32_t b0, b1, b2, b3;
        ldsm_x4(kb + swz(tok, chunk16), b0, b1, b2, b3);
        mma_bf16(sacc[2 * n2], qa[ks][0], qa[ks][1], qa[ks][2], qa[ks][3], b0, b1);
        mma_bf16(sacc[2 * n2 + 1], qa[ks][0], qa[ks][1], qa[ks][2], qa[ks][3], b2, b3);
      }
    }
    // mask and online softmax (rows gq: c0,c1; gq+8: c2,c3)
    float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
    for (int n = 0; n < NT; ++n) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int t = t_base + n * 8 + tq * 2 + e;
        const bool in = t < len;
        const bool ok0 = in && (own0 < 0 || own0 + t <= pos0);
        const bool ok1 = in && (own0 < 0 || own0 + t <= pos1);
        sacc[n][e] = ok0 ? sacc[n][e] : -INFINITY;
        sacc[n][2 + e] = ok1 ? sacc[n][2 + e] : -INFINITY;
        mx0 = fmaxf(mx0, sacc[n][e]);
        mx1 = fmaxf(mx1, sacc[n][2 + e]);
      }
    }
#pragma unroll
    for (int o = 1; o < 4; o <<= 1) {
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, o));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, o));
    }
    const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
    const float a0 = mn0 == -INFINITY ? 1.f : exp2f(m0 - mn0);
    const float a1 = mn1 == -INFINITY ? 1.f : exp2f(m1 - mn1);
    float ps0 = 0.f, ps1 = 0.f;
    uint32_t pa[NT / 2][4];
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      const float p00 = mn0 == -INFINITY ? 0.f : exp2f(sacc[n][0] - mn0);
      const float p01 = mn0 == -INFINITY ? 0.f : exp2f(sacc[n][1] - mn0);
      const float p10 = mn1 == -INFINITY ? 0.f : exp2f(sacc[n][2] - mn1);
      const float p11 = mn1 == -INFINITY ? 0.f : exp2f(sacc[n][3] - mn1);
      ps0 += p00 + p01;
      ps1 += p10 + p11;
      // C layout of n8 tile n -> A layout of k16 step n/2 (regs 0,1 for even n, 2,3 for odd n)
      if ((n & 1) == 0) {
        pa[n / 2][0] = pack_bf16(p00, p01);
        pa[n / 2][1] = pack_bf16(p10, p11);
      } else {
        pa[n / 2][2] = pack_bf16(p00, p01);
        pa[n / 2][3] = pack_bf16(p10, p11);
      }
    }
    l0 = l0 * a0 + ps0;
    l1 = l1 * a1 + ps1;
    m0 = mn0;
    m1 = mn1;
#pragma unroll
    for (int n = 0; n < 16; ++n) {
      oacc[n][0] *= a0;
      oacc[n][1] *= a0;
      oacc[n][2] *= a1;
      oacc[n][3] *= a1;
    }
    // O += P V : k = this warp's tokens (NT/2 k16 steps), n = 128 dh (16 n8 tiles)
#pragma unroll
    for (int kk = 0; kk < NT / 2; ++kk) {
#pragma unroll
      for (int n2 = 0; n2 < 8; ++n2) {
        // V^T fragments via ldmatrix.trans: matrices {tok 0-7, dh 8j..}, {tok 8-15, dh 8j..}, {tok 0-7, dh 8j+8..}, {tok 8-15, dh 8j+8..}
        const int mi = lane >> 3, ri = lane & 7;
        const int tok = t_base + kk * 16 + (mi & 1) * 8 + ri;
        const int chunk16 = n2 * 2 + (mi >> 1);
        uint32_t b0, b1, b2, b3;
        ldsm_x4_t(vb + swz(tok, chunk16), b0, b1, b2, b3);
        mma_bf16(oacc[2 * n2], pa[kk][0], pa[kk][1], pa[kk][2], pa[kk][3], b0, b1);
        mma_bf16(oacc[2 * n2 + 1], pa[kk][0], pa[kk][1], pa[kk][2], pa[kk][3], b2, b3);
      }
    }
    __syncthreads();
    if (c + 2 < nchunks) {
      next_chunk(b);
      if (tid == 0) issue(b);
    }
  }
  // row sums within the quad
#pragma unroll
  for (int o = 1; o < 4; o <<= 1) {
    l0 += __shfl_xor_sync(0xffffffffu, l0, o);
    l1 += __shfl_xor_sync(0xffffffffu, l1, o);
  }
  // merge the SPLIT warps of head g through shared memory (reuse the K/V buffers)
  float* sO = reinterpret_cast<float*>(sbase);  // [4 warps][16 rows][128] fp32 = 32 KB
  if (tq == 0) {
    sMl[warp][0][gq] = m0;
    sMl[warp][0][gq + 8] = m1;
    sMl[warp][1][gq] = l0;
    sMl[warp][1][gq + 8] = l1;
  }
  __syncthreads();
  float M0 = -INFINITY, M1 = -INFINITY;
  for (int w = g * SPLIT; w < (g + 1) * SPLIT; ++w) {
    M0 = fmaxf(M0, sMl[w][0][gq]);
    M1 = fmaxf(M1, sMl[w][0][gq + 8]);
  }
  float L0 = 0.f, L1 = 0.f;
  for (int w = g * SPLIT; w < (g + 1) * SPLIT; ++w) {
    const float mw0 = sMl[w][0][gq], mw1 = sMl[w][0][gq + 8];
    L0 += (mw0 == -INFINITY) ? 0.f : sMl[w][1][gq] * exp2f(mw0 - M0);
    L1 += (mw1 == -INFINITY) ? 0.f : sMl[w][1][gq + 8] * exp2f(mw1 - M1);
  }
  const float f0 = (m0 == -INFINITY) ? 0.f : exp2f(m0 - M0);
  const float f1 = (m1 == -INFINITY) ? 0.f : exp2f(m1 - M1);
#pragma unroll
  for (int n = 0; n < 16; ++n) {
    const int col = n * 8 + tq * 2;
    float* r0p = sO + (warp * 16 + gq) * DH + col;
    float* r1p = sO + (warp * 16 + gq + 8) * DH + col;
    r0p[0] = oacc[n][0] * f0;
    r0p[1] = oacc[n][1] * f0;
    r1p[0] = oacc[n][2] * f1;
    r1p[1] = oacc[n][3] * f1;
  }
  __syncthreads();
  // warp `slice 0` of each head writes the merged rows
  if (slice == 0) {
    for (int i = lane; i < kTileRows * DH; i += 32) {
      const int row = i / DH, col = i % DH;
      if (row >= td.nrows) continue;
      float acc = 0.f;
      for (int w = g * SPLIT; w < (g + 1) * SPLIT; ++w) acc += sO[(w * 16 + row) * DH + col];
      float Lr = 0.f, Mr = -INFINITY;
      for (int w = g * SPLIT; w < (g + 1) * SPLIT; ++w) Mr = fmaxf(Mr, sMl[w][0][row]);
      for (int w = g * SPLIT; w < (g + 1) * SPLIT; ++w) {
        const float mw = sMl[w][0][row];
        Lr += (mw == -INFINITY) ? 0.f : sMl[w][1][row] * exp2f(mw - Mr);
      }
      O[((long long)(td.row0 + row) * H + hbase + g) * DH + col] = __float2bfloat16_rn(acc / Lr);
    }
  }
  (void)L0;
  (void)L1;
}

// K1 decode, per-warp TMA pipeline on tensor cores (any GQA group G <= 16,
// dh = 128): the bulk kernel's structure — a persistent grid of warps claiming
// (row, KV head) items from a device counter, each warp streaming its items'
// tree context through its own ring of NST shared-memory stages of 16 tokens,
// loads in flight across item and segment boundaries — with the stages filled
// by 2D TMA (16-row boxes, 128-byte swizzle, so ldmatrix reads are conflict
// free) and the math on mma.sync m16n8k16: the MMA rows are the KV head's G
// query heads (zero-padded to 16), so each staged K/V row serves the whole
// group at the cost of one row-vector of MMA work. The pools are zero-filled at
// allocation, so rows of a box past a segment's end are finite (masked to p = 0).
constexpr int kMmaNST = 2;     // stages per warp
constexpr int kMmaWarps = 12;  // warps per block (12 x 2 x 8 KB = 192 KB; 170 registers)

// byte offset of (row, 16-byte chunk c in [0,16)) in a swizzled [2 halves][16 rows][128 B] box pair
__device__ __forceinline__ uint32_t swz16(int row, int c) {
  const int half = c >> 3, cc = c & 7;
  return (uint32_t)(half * 2048 + row * 128 + ((cc ^ (row & 7)) << 4));
}

template <int kNST, int kWarps, bool kSkipRescale>  // stages per warp, warps per block
__global__ void __launch_bounds__(kWarps * 32, 1)
    tree_attn_wmma_kernel(const __grid_constant__ CUtensorMap kvmap16,
                          const RowDesc* __restrict__ rows, const Segment* __restrict__ segs,
                          const float* __restrict__ Qr, int H, int KVH, int G, int n_items, long long slots,
                          __nv_bfloat16* __restrict__ O, int* __restrict__ item_ctr,
                          const int* __restrict__ row_order) {
  constexpr int DH = 128, CH = 16, STAGE = CH * DH * 2;  // 4 KB of K (and of V) per stage
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar[kWarps][kNST];
  __shared__ int queue[kWarps][8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* ring = sm + (size_t)warp * kNST * 2 * STAGE;  // [stage][K|V][STAGE]
  if (lane == 0) {
    for (int i = 0; i < kNST; ++i) mbar_init(&bar[warp][i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  // ---- producer cursor (lane 0 only)
  // The producer lane is on the critical path of every stage: per stage it only
  // issues one copy at a running row coordinate; a segment costs one 16-byte load.
  int p_q = 0, p_item = -1, p_seg = 0, p_nseg = 0, issued = 0;
  int p_row = 0, p_left = 0;  // next stage's pool row, tokens left in the current segment
  long long p_row0 = 0;
  const Segment* p_sg = nullptr;
  bool p_done = false;
  auto produce = [&]() {
    while (!p_done) {
      if (p_left > 0) {
        const int st = issued % kNST;
        unsigned char* kb = ring + st * 2 * STAGE;
        mbar_expect_tx(&bar[warp][st], 2 * STAGE);
        tma_load_4d(kb, &kvmap16, p_row, &bar[warp][st]);  // K at kb, V at kb + STAGE
        p_row += CH;
        p_left -= CH;
        ++issued;
        return;
      }
      if (p_item >= 0 && p_seg < p_nseg) {
        const int4 v = __ldg(reinterpret_cast<const int4*>(p_sg + p_seg));  // Segment {base, len, own0}
        ++p_seg;
        p_row = (int)(p_row0 + (long long)(((unsigned long long)(unsigned)v.y << 32) | (unsigned)v.x));
        p_left = v.z;
        continue;
      }
      const int it = atomicAdd(item_ctr, 1);
      if (it >= n_items) {
        queue[warp][p_q & 7] = -1;
        p_done = true;
        return;
      }
      queue[warp][p_q & 7] = it;
      ++p_q;
      p_item = it;
      const RowDesc rd = rows[row_order ? row_order[it / KVH] : it / KVH];
      p_sg = segs + rd.seg_off;
      p_nseg = rd.nseg;
      p_seg = 0;
      p_row0 = (long long)(it % KVH) * slots;
    }
  };
  if (lane == 0)
    for (int i = 0; i < kNST - 1; ++i) produce();
  __syncwarp();
  const int gq = lane >> 2, tq = lane & 3, mi = lane >> 3, ri = lane & 7;
  int c_q = 0, consumed = 0;
  for (;;) {
    const int it = queue[warp][c_q & 7];
    if (it < 0) break;
    ++c_q;
    const int r = row_order ? row_order[it / KVH] : it / KVH, kh = it % KVH;
    const RowDesc rd = rows[r];
    const Segment* sg = segs + rd.seg_off;
    // Q fragments: rows = the group's heads (gq, gq + 8 < G), dims as k
    uint32_t qa[8][4];
    {
      const bool v0 = gq < G, v1 = gq + 8 < G;
      const float* q0 = Qr + ((long long)r * H + kh * G + (v0 ? gq : 0)) * DH;
      const float* q1 = Qr + ((long long)r * H + kh * G + (v1 ? gq + 8 : 0)) * DH;
      constexpr float sc = 1.4426950408889634f;
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        const int k0 = ks * 16 + tq * 2;
        const float2 x00 = v0 ? *reinterpret_cast<const float2*>(q0 + k0) : make_float2(0.f, 0.f);
        const float2 x10 = v1 ? *reinterpret_cast<const float2*>(q1 + k0) : make_float2(0.f, 0.f);
        const float2 x01 = v0 ? *reinterpret_cast<const float2*>(q0 + k0 + 8) : make_float2(0.f, 0.f);
        const float2 x11 = v1 ? *reinterpret_cast<const float2*>(q1 + k0 + 8) : make_float2(0.f, 0.f);
        qa[ks][0] = pack_bf16(x00.x * sc, x00.y * sc);
        qa[ks][1] = pack_bf16(x10.x * sc, x10.y * sc);
        qa[ks][2] = pack_bf16(x01.x * sc, x01.y * sc);
        qa[ks][3] = pack_bf16(x11.x * sc, x11.y * sc);
      }
    }
    float oacc[16][4];
#pragma unroll
    for (int n = 0; n < 16; ++n) oacc[n][0] = oacc[n][1] = oacc[n][2] = oacc[n][3] = 0.f;
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
    for (int si = 0; si < rd.nseg; ++si) {
      const int len = sg[si].len;
      for (int off = 0; off < len; off += CH) {
        const int n = min(CH, len - off);
        if (lane == 0) produce();
        const int st = consumed % kNST;
        mbar_wait(&bar[warp][st], (uint32_t)((consumed / kNST) & 1));
        const uint32_t kb = (uint32_t)__cvta_generic_to_shared(ring + st * 2 * STAGE);
        const uint32_t vb = kb + STAGE;
        float sacc[2][4];
#pragma unroll
        for (int t = 0; t < 2; ++t) sacc[t][0] = sacc[t][1] = sacc[t][2] = sacc[t][3] = 0.f;
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          uint32_t b0, b1, b2, b3;
          ldsm_x4(kb + swz16((mi >> 1) * 8 + ri, ks * 2 + (mi & 1)), b0, b1, b2, b3);
          mma_bf16(sacc[0], qa[ks][0], qa[ks][1], qa[ks][2], qa[ks][3], b0, b1);
          mma_bf16(sacc[1], qa[ks][0], qa[ks][1], qa[ks][2], qa[ks][3], b2, b3);
        }
        float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
        for (int t = 0; t < 2; ++t)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const bool ok = t * 8 + tq * 2 + e < n;
            sacc[t][e] = ok ? sacc[t][e] : -INFINITY;
            sacc[t][2 + e] = ok ? sacc[t][2 + e] : -INFINITY;
            mx0 = fmaxf(mx0, sacc[t][e]);
            mx1 = fmaxf(mx1, sacc[t][2 + e]);
          }
#pragma unroll
        for (int o = 1; o < 4; o <<= 1) {
          mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, o));
          mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, o));
        }
        const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
        const float a0 = mn0 == -INFINITY ? 1.f : exp2f(m0 - mn0);
        const float a1 = mn1 == -INFINITY ? 1.f : exp2f(m1 - mn1);
        uint32_t pa[4];
        float ps0 = 0.f, ps1 = 0.f;
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          const float p00 = mn0 == -INFINITY ? 0.f : exp2f(sacc[t][0] - mn0);
          const float p01 = mn0 == -INFINITY ? 0.f : exp2f(sacc[t][1] - mn0);
          const float p10 = mn1 == -INFINITY ? 0.f : exp2f(sacc[t][2] - mn1);
          const float p11 = mn1 == -INFINITY ? 0.f : exp2f(sacc[t][3] - mn1);
          ps0 += p00 + p01;
          ps1 += p10 + p11;
          pa[2 * t] = pack_bf16(p00, p01);
          pa[2 * t + 1] = pack_bf16(p10, p11);
        }
        l0 = l0 * a0 + ps0;
        l1 = l1 * a1 + ps1;
        // a == 1 exactly when a row's running max did not move: the rescale can be skipped
        if (!kSkipRescale || !__all_sync(0xffffffffu, mn0 == m0 && mn1 == m1)) {
#pragma unroll
          for (int nn = 0; nn < 16; ++nn) {
            oacc[nn][0] *= a0;
            oacc[nn][1] *= a0;
            oacc[nn][2] *= a1;
            oacc[nn][3] *= a1;
          }
        }
        m0 = mn0;
        m1 = mn1;
#pragma unroll
        for (int n2 = 0; n2 < 8; ++n2) {
          uint32_t b0, b1, b2, b3;
          ldsm_x4_t(vb + swz16((mi & 1) * 8 + ri, n2 * 2 + (mi >> 1)), b0, b1, b2, b3);
          mma_bf16(oacc[2 * n2], pa[0], pa[1], pa[2], pa[3], b0, b1);
          mma_bf16(oacc[2 * n2 + 1], pa[0], pa[1], pa[2], pa[3], b2, b3);
        }
        ++consumed;
        __syncwarp();  // stage fully read before lane 0 refills it
      }
    }
#pragma unroll
    for (int o = 1; o < 4; o <<= 1) {
      l0 += __shfl_xor_sync(0xffffffffu, l0, o);
      l1 += __shfl_xor_sync(0xffffffffu, l1, o);
    }
    if (gq < G) {
      __nv_bfloat16* o0 = O + ((long long)r * H + kh * G + gq) * DH + tq * 2;
      const float inv = 1.f / l0;
#pragma unroll
      for (int nn = 0; nn < 16; ++nn)
        *reinterpret_cast<uint32_t*>(o0 + nn * 8) = pack_bf16(oacc[nn][0] * inv, oacc[nn][1] * inv);
    }
    if (gq + 8 < G) {
      __nv_bfloat16* o1 = O + ((long long)r * H + kh * G + gq + 8) * DH + tq * 2;
      const float inv = 1.f / l1;
#pragma unroll
      for (int nn = 0; nn < 16; ++nn)
        *reinterpret_cast<uint32_t*>(o1 + nn * 8) = pack_bf16(oacc[nn][2] * inv, oacc[nn][3] * inv);
    }
  }
}

// K1 tile variant for prefill-shaped rows (PRM scoring): kTileRows consecutive
// rows of one thought share their ancestors and a causal own prefix, so each
// 64-token K/V chunk is staged once per tile instead of once per row.
template <int DH, int G>
__global__ void __launch_bounds__(kAttnThreads) tree_attn_tile_kernel(const TileDesc* __restrict__ tiles,
                                                                     const RowDesc* __restrict__ rows,
                                                                     const Segment* __restrict__ segs,
                                                                     const float* __restrict__ Qr, int H,
                                                                     const __nv_bfloat16* __restrict__ Kp,
                                                                     const __nv_bfloat16* __restrict__ Vp,
                                                                     long long slots,
                                                                     __nv_bfloat16* __restrict__ O) {
  constexpr int R = kTileRows;
  constexpr int NV = R * G;             // query vectors in the tile
  constexpr int VPL = DH / 32;
  constexpr int DGRP = kAttnThreads / DH;  // threads sharing one output dim (1 or 2)
  constexpr int NACC = (NV + DGRP - 1) / DGRP;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __nv_bfloat16* sK = reinterpret_cast<__nv_bfloat16*>(smem_raw);
  __nv_bfloat16* sV = sK + 2 * kChunk * DH;
  float* sQ = reinterpret_cast<float*>(sV + 2 * kChunk * DH);  // [NV][DH]
  float* sS = sQ + NV * DH;                                    // [NV][kChunk]
  float* sM = sS + NV * kChunk;
  float* sL = sM + NV;
  float* sAlpha = sL + NV;
  __shared__ int sPos[R];
  __shared__ uint64_t bar[2];

  const TileDesc td = tiles[blockIdx.x];
  const int kh = blockIdx.y;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const RowDesc last = rows[td.row0 + td.nrows - 1];
  const Segment* sg = segs + last.seg_off;
  const int nseg = last.nseg;
  const __nv_bfloat16* Kh = Kp + (long long)kh * slots * DH;
  const __nv_bfloat16* Vh = Vp + (long long)kh * slots * DH;

  for (int i = tid; i < NV * DH; i += kAttnThreads) {
    const int v = i / DH, dcol = i % DH;
    const int ri = v / G, g = v % G;
    sQ[i] = ri < td.nrows ? Qr[((long long)(td.row0 + ri) * H + kh * G + g) * DH + dcol] * 1.4426950408889634f : 0.f;
  }
  if (tid < R) sPos[tid] = tid < td.nrows ? rows[td.row0 + tid].pos : -1;
  if (tid < NV) {
    sM[tid] = -INFINITY;
    sL[tid] = 0.f;
  }
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  int nchunks = 0;
  const int clip = last.pos + 1;  // the tile's causal horizon inside its own thought
  for (int s = 0; s < nseg; ++s) nchunks += (seg_len_eff(sg[s], clip) + kChunk - 1) / kChunk;
  __syncthreads();

  int seg_i = 0, seg_o = 0;
  long long cb[2];
  int cl[2], cown[2];  // chunk base/len; own-segment offset of the chunk (-1: ancestor)
  auto next_chunk = [&](int b) {
    while (seg_i < nseg && seg_o >= seg_len_eff(sg[seg_i], clip)) {
      ++seg_i;
      seg_o = 0;
    }
    cb[b] = sg[seg_i].base + seg_o;
    const int l = seg_len_eff(sg[seg_i], clip) - seg_o;
    cl[b] = l < kChunk ? l : kChunk;
    cown[b] = sg[seg_i].own0 >= 0 ? sg[seg_i].own0 + seg_o : -1;
    seg_o += cl[b];
  };
  for (int c = 0; c < 2 && c < nchunks; ++c) {
    next_chunk(c);
    if (tid == 0) {
      const uint32_t bytes = (uint32_t)cl[c] * DH * 2;
      mbar_expect_tx(&bar[c], 2 * bytes);
      bulk_g2s(sK + c * kChunk * DH, Kh + cb[c] * DH, bytes, &bar[c]);
      bulk_g2s(sV + c * kChunk * DH, Vh + cb[c] * DH, bytes, &bar[c]);
    }
  }
  const int dcol = tid % DH;
  const int vgrp = tid / DH;
  float acc[NACC];
#pragma unroll
  for (int k = 0; k < NACC; ++k) acc[k] = 0.f;

  for (int c = 0; c < nchunks; ++c) {
    const int buf = c & 1;
    const int len = cl[buf];
    const int own0 = cown[buf];
    mbar_wait(&bar[buf], (uint32_t)((c >> 1) & 1));
    const __nv_bfloat16* K = sK + buf * kChunk * DH;
    const __nv_bfloat16* Vs = sV + buf * kChunk * DH;
    for (int t = warp; t < len; t += kAttnThreads / 32) {
      float kv[VPL];
#pragma unroll
      for (int v2 = 0; v2 < VPL / 2; ++v2) {
        const __nv_bfloat162 a = *reinterpret_cast<const __nv_bfloat162*>(K + t * DH + lane * VPL + 2 * v2);
        kv[2 * v2] = __low2float(a);
        kv[2 * v2 + 1] = __high2float(a);
      }
#pragma unroll 4
      for (int v = 0; v < NV; ++v) {
        const float* q = sQ + v * DH + lane * VPL;
        float s = 0.f;
#pragma unroll
        for (int e = 0; e < VPL; ++e) s += q[e] * kv[e];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) {
          const bool masked = own0 >= 0 && own0 + t > sPos[v / G];
          sS[v * kChunk + t] = masked ? -INFINITY : s;
        }
      }
    }
    __syncthreads();
    for (int v = warp; v < NV; v += kAttnThreads / 32) {
      float mx = -INFINITY;
      for (int t = lane; t < len; t += 32) mx = fmaxf(mx, sS[v * kChunk + t]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      const float m_old = sM[v], l_old = sL[v];
      const float m_new = fmaxf(m_old, mx);
      float sum = 0.f;
      for (int t = lane; t < len; t += 32) {
        const float sv = sS[v * kChunk + t];
        const float p = (m_new == -INFINITY || sv == -INFINITY) ? 0.f : exp2f(sv - m_new);
        sS[v * kChunk + t] = p;
        sum += p;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
      const float alpha = (m_old == -INFINITY) ? 0.f : exp2f(m_old - m_new);
      __syncwarp();
      if (lane == 0) {
        sM[v] = m_new;
        sL[v] = l_old * alpha + sum;
        sAlpha[v] = alpha;
      }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < NACC; ++k) {
      const int v = vgrp + k * DGRP;
      if (v < NV) acc[k] *= sAlpha[v];
    }
    for (int t = 0; t < len; ++t) {
      const float vv = __bfloat162float(Vs[t * DH + dcol]);
#pragma unroll
      for (int k = 0; k < NACC; ++k) {
        const int v = vgrp + k * DGRP;
        if (v < NV) acc[k] += sS[v * kChunk + t] * vv;
      }
    }
    __syncthreads();
    if (c + 2 < nchunks) {
      next_chunk(buf);
      if (tid == 0) {
        const uint32_t bytes = (uint32_t)cl[buf] * DH * 2;
        mbar_expect_tx(&bar[buf], 2 * bytes);
        bulk_g2s(sK + buf * kChunk * DH, Kh + cb[buf] * DH, bytes, &bar[buf]);
        bulk_g2s(sV + buf * kChunk * DH, Vh + cb[buf] * DH, bytes, &bar[buf]);
      }
    }
  }
#pragma unroll
  for (int k = 0; k < NACC; ++k) {
    const int v = vgrp + k * DGRP;
    if (v < NV) {
      const int ri = v / G, g = v % G;
      if (ri < td.nrows)
        O[((long long)(td.row0 + ri) * H + kh * G + g) * DH + dcol] = __float2bfloat16_rn(acc[k] / sL[v]);
    }
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

extern "C" void spex_k_build_prm_rows(TreeView t, const int* sids, const int* row_start, const int* tile_start,
                                      int n, RowDesc* rows, Segment* segs, int* last_row, TileDesc* tiles,
                                      cudaStream_t s) {
  build_prm_rows_kernel<<<n, 128, 0, s>>>(t, sids, row_start, tile_start, n, rows, segs, last_row, tiles);
}

extern "C" void spex_k_build_prompt_rows(TreeView t, int q0, int nq, RowDesc* rows, Segment* segs,
                                         cudaStream_t s) {
  const int n = nq * t.prompt_tokens;
  build_prompt_rows_kernel<<<(n + 127) / 128, 128, 0, s>>>(t, q0, nq, rows, segs);
}

extern "C" void spex_k_build_prompt_tiles(int nq, int P, TileDesc* tiles, cudaStream_t s) {
  const int n = nq * ((P + kTileRows - 1) / kTileRows);
  build_prompt_tiles_kernel<<<(n + 127) / 128, 128, 0, s>>>(nq, P, tiles);
}

extern "C" void spex_k_prm_scan_all(TreeView t, const int* kind, const int* off, const int* n, int n_entries,
                                    const int* srow_sid, int* row_start, int* tile_start, int* totals,
                                    int* tile_totals, cudaStream_t s) {
  prm_scan_all_kernel<<<(n_entries + 127) / 128, 128, 0, s>>>(t, kind, off, n, n_entries, srow_sid, row_start,
                                                              tile_start, totals, tile_totals);
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
  embed_kernel<<<(M + 7) / 8, 256, 0, s>>>(rows, M, E, d, X);
}

// Programmatic dependent launch for the per-layer kernels of the decode step
// (RMSNorm, RoPE + KV append, K1 bulk, SwiGLU): their launch overlaps the tail
// of the kernel before them (measured -1.5% step time, profiles/r01z_pdl_ab.txt).
// SPEX_PDL=0 launches them normally.
static bool pdl_on() {
  static const bool on = !getenv("SPEX_PDL") || atoi(getenv("SPEX_PDL")) != 0;  // default on
  return on;
}
template <typename... KArgs, typename... Args>
static void launch_maybe_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                             Args... args) {
  if (!pdl_on()) {
    k<<<grid, block, smem, s>>>(static_cast<KArgs>(args)...);
    return;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

extern "C" void spex_k_rmsnorm(const float* X, int M, int d, float eps, __nv_bfloat16* Y, cudaStream_t s) {
  static const bool reg = !getenv("SPEX_RMSNORM_REG") || atoi(getenv("SPEX_RMSNORM_REG")) != 0;
  const dim3 grid((M + 7) / 8), block(256);
  if (reg) switch (d) {
      case 512: return launch_maybe_pdl(rmsnorm_bf16_reg_kernel<4>, grid, block, 0, s, X, M, eps, Y);
      case 1024: return launch_maybe_pdl(rmsnorm_bf16_reg_kernel<8>, grid, block, 0, s, X, M, eps, Y);
      case 1536: return launch_maybe_pdl(rmsnorm_bf16_reg_kernel<12>, grid, block, 0, s, X, M, eps, Y);
      case 4096: return launch_maybe_pdl(rmsnorm_bf16_reg_kernel<32>, grid, block, 0, s, X, M, eps, Y);  // Llama-3-8B
      default: break;
    }
  launch_maybe_pdl(rmsnorm_bf16_kernel, grid, block, 0, s, X, M, d, eps, Y);
}

template <int DH, int G>
static void launch_attn_decode(const RowDesc* rows, const Segment* segs, const float* Qr, int H, int KVH,
                               const __nv_bfloat16* Kp, const __nv_bfloat16* Vp, long long slots, __nv_bfloat16* O,
                               int M, cudaStream_t s) {
  const long long warps = (long long)M * KVH;
  const int blocks = (int)((warps * 32 + 255) / 256);
  // 8 token pairs in flight per lane when registers allow (G == 1: 64 regs, no spill), else 4
  static const int unroll = getenv("SPEX_K1_UNROLL") ? atoi(getenv("SPEX_K1_UNROLL")) : (G == 1 ? 8 : 4);
  if (unroll == 8)
    tree_attn_decode_kernel<DH, G, 8><<<blocks, 256, 0, s>>>(rows, segs, Qr, H, KVH, M, Kp, Vp, slots, O);
  else
    tree_attn_decode_kernel<DH, G, 4><<<blocks, 256, 0, s>>>(rows, segs, Qr, H, KVH, M, Kp, Vp, slots, O);
}



extern "C" int spex_k_tree_attn(const RowDesc* rows, const Segment* segs, const float* Qr, int H, int KVH, int dh,
                                const __nv_bfloat16* Kp, const __nv_bfloat16* Vp, long long slots, __nv_bfloat16* O,
                                int M, cudaStream_t s) {
  const int G = H / KVH;
#define SPEX_ATTN_CASE(D, GG)                                                   \
  if (dh == D && G == GG) {                                                     \
    launch_attn_decode<D, GG>(rows, segs, Qr, H, KVH, Kp, Vp, slots, O, M, s);   \
    return 0;                                                                   \
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

static int g_k1_kv_evict_first = 0;  // L2 policy of K1's bulk KV copies (set per forward)
static const int* g_k1_row_order = nullptr;  // claim order of the decode rows (set per step), or null
extern "C" void spex_k1_set_row_order(const int* order) { g_k1_row_order = order; }

// Rows of a decode step grouped by query (counting sort, one block; order
// within a query arbitrary): the bulk K1's warps then work on one tree's rows
// at the same time, so their shared prefixes are read from L2 while resident.
__global__ void __launch_bounds__(1024) order_rows_kernel(const RowDesc* __restrict__ rows, int M, int Q,
                                                           int* __restrict__ order, int lpt) {
  // Rows grouped by query (a tree's rows run together, so shared prefixes are
  // served from L2), queries taken longest context first (the longest items
  // start early instead of trailing the launch).
  constexpr int NB = 1024;
  __shared__ int hist[NB], part[NB], key[NB], rnk[NB];
  const int tid = threadIdx.x;
  // one bucket per query up to 1024 queries (buckets past nb stay empty)
  const int nb = Q > 0 && Q < NB ? Q : NB;
  hist[tid] = 0;
  key[tid] = 0;
  __syncthreads();
  auto bucket = [&](int q) { return min((int)(((long long)q * nb) / (Q > 0 ? Q : 1)), nb - 1); };
  for (int r = tid; r < M; r += 1024) {
    const int bq = bucket(rows[r].q);
    atomicAdd(&hist[bq], 1);
    if (lpt) atomicMax(&key[bq], rows[r].abs_pos + 1);
  }
  __syncthreads();
  // rank of each bucket: longer first, then by index (deterministic); the
  // empty buckets past nb rank last, in index order
  {
    int r = tid;
    if (tid < nb) {
      const int kb = key[tid];
      r = 0;
      for (int j = 0; j < nb; ++j) {
        const int kj = key[j];
        r += kj > kb || (kj == kb && j < tid);
      }
    }
    rnk[tid] = r;
  }
  __syncthreads();
  part[rnk[tid]] = hist[tid];
  __syncthreads();
  const int v = part[tid];
  for (int o = 1; o < NB; o <<= 1) {
    const int a = tid >= o ? part[tid - o] : 0;
    __syncthreads();
    part[tid] += a;
    __syncthreads();
  }
  const int excl = part[tid] - v;  // start of the bucket ranked tid
  __syncthreads();
  part[tid] = excl;
  __syncthreads();
  hist[tid] = part[rnk[tid]];  // start of bucket tid
  __syncthreads();
  for (int r = tid; r < M; r += 1024) order[atomicAdd(&hist[bucket(rows[r].q)], 1)] = r;
}

extern "C" void spex_k_order_rows(const RowDesc* rows, int M, int Q, int* order, cudaStream_t s) {
  if (M <= 0) return;
  // SPEX_K1_QLPT=0: queries in index order (round 1's claim order)
  static const int lpt = !getenv("SPEX_K1_QLPT") || atoi(getenv("SPEX_K1_QLPT")) != 0;
  order_rows_kernel<<<1, 1024, 0, s>>>(rows, M, Q, order, lpt);
}
extern "C" void spex_k1_set_kv_evict_first(int on) { g_k1_kv_evict_first = on ? 1 : 0; }

// K1 decode rows through the bulk-copy pipeline (G = 1, dh = 128); item_ctr
// points at two device ints, zero on entry and re-zeroed by the kernel.
template <int CH, int NST, int W>
static int launch_bulk(const RowDesc* rows, const Segment* segs, const float* Qr, int H, int KVH,
                       const __nv_bfloat16* Kp, const __nv_bfloat16* Vp, long long slots, __nv_bfloat16* O, int M,
                       int* item_ctr, cudaStream_t s) {
  const size_t smem = (size_t)W * NST * 2 * CH * 128 * 2;
  static int blocks = 0;
  if (!blocks) {
    cudaFuncSetAttribute(tree_attn_bulk_kernel<CH, NST, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    blocks = sms;
  }
  const int n_items = M * KVH;
  const int grid = std::min(blocks, (n_items + W - 1) / W);
  // L2 policy of the KV chunks: evict-first frees L2 for the control kernel
  // (-15% control time under load) but costs K1 its cross-row prefix hits
  // (+2.5% K1 time), so it is on only when the forward is not the bottleneck
  // (coupled shards); SPEX_K1_EVICT_FIRST=0/1 overrides.
  static const int env_ef = getenv("SPEX_K1_EVICT_FIRST") ? atoi(getenv("SPEX_K1_EVICT_FIRST")) : -1;
  const int kv_ef = env_ef >= 0 ? env_ef : g_k1_kv_evict_first;
  // item_ctr[0..1] are zero on entry and re-zeroed by the kernel's last warp
  launch_maybe_pdl(tree_attn_bulk_kernel<CH, NST, W>, dim3(grid), dim3(W * 32), smem, s, rows, segs, Qr, H, KVH,
                   n_items, Kp, Vp, slots, O, item_ctr, kv_ef, g_k1_row_order);
  return (int)cudaGetLastError();
}

// K1 decode rows through the bulk-copy pipeline (G = 1, dh = 128); item_ctr
// points at two device ints, zero before the first launch (the kernel's last
// warp re-zeroes them, so no memset per launch). Items are claimed in the
// order spex_k1_set_row_order installed for the step, else row order.
extern "C" int spex_k_tree_attn_bulk(const RowDesc* rows, const Segment* segs, const float* Qr, int H, int KVH, int dh,
                                     const __nv_bfloat16* Kp, const __nv_bfloat16* Vp, long long slots,
                                     __nv_bfloat16* O, int M, int* item_ctr, cudaStream_t s) {
  if (M <= 0) return 0;
  if (dh != 128 || H != KVH) return -1;
  // 16-token stages, 2 per warp, 14 warps: the best of an 8-point sweep on c2
  return launch_bulk<16, 2, 14>(rows, segs, Qr, H, KVH, Kp, Vp, slots, O, M, item_ctr, s);
}

// K1 decode rows on the per-warp TMA + mma.sync pipeline (G <= 16, dh = 128);
// kvmap16 is the layer's K|V pool pair as one 4D map (spex_tmap_kv16).

template <int NST, int W, bool SKIP = false>
static int launch_wmma(const CUtensorMap* kvmap16, const RowDesc* rows, const Segment* segs,
                       const float* Qr, int H, int KVH, int G, long long slots, __nv_bfloat16* O, int M,
                       int* item_ctr, cudaStream_t s) {
  const size_t smem = (size_t)W * NST * 2 * 16 * 128 * 2 + 1024;
  static int blocks = 0;
  if (!blocks) {
    cudaFuncSetAttribute(tree_attn_wmma_kernel<NST, W, SKIP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    blocks = sms;
  }
  const int n_items = M * KVH;
  const int grid = std::min(blocks, (n_items + W - 1) / W);
  cudaMemsetAsync(item_ctr, 0, sizeof(int), s);
  tree_attn_wmma_kernel<NST, W, SKIP><<<grid, W * 32, smem, s>>>(*kvmap16, rows, segs, Qr, H, KVH, G, n_items,
                                                                 slots, O, item_ctr, g_k1_row_order);
  return (int)cudaGetLastError();
}

extern "C" int spex_k_tree_attn_wmma(const CUtensorMap* kvmap16, const RowDesc* rows,
                                     const Segment* segs, const float* Qr, int H, int KVH, int dh, long long slots,
                                     __nv_bfloat16* O, int M, int* item_ctr, cudaStream_t s) {
  const int G = H / KVH;
  if (M <= 0) return 0;
  if (dh != 128 || G < 1 || G > 16) return -1;
  // 2 stages x 12 warps (8 KB per stage): the best of a stages x warps sweep on c5
  return launch_wmma<kMmaNST, kMmaWarps>(kvmap16, rows, segs, Qr, H, KVH, G, slots, O, M, item_ctr, s);
}

template <int DH, int G>
static void launch_tile(const TileDesc* tiles, int ntiles, const RowDesc* rows, const Segment* segs, const float* Qr,
                        int H, int KVH, const __nv_bfloat16* Kp, const __nv_bfloat16* Vp, long long slots,
                        __nv_bfloat16* O, cudaStream_t s) {
  constexpr int NV = kTileRows * G;
  const size_t smem = 4 * kChunk * DH * sizeof(__nv_bfloat16) + (NV * DH + NV * kChunk + 3 * NV) * sizeof(float) + 64;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(tree_attn_tile_kernel<DH, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  dim3 grid(ntiles, KVH);
  tree_attn_tile_kernel<DH, G><<<grid, kAttnThreads, smem, s>>>(tiles, rows, segs, Qr, H, Kp, Vp, slots, O);
}

extern "C" int spex_k_tree_attn_tiles_mma(const CUtensorMap* kvmap, const TileDesc* tiles,
                                          int ntiles, const RowDesc* rows, const Segment* segs, const float* Qr, int H,
                                          int KVH, int dh, long long slots, __nv_bfloat16* O, cudaStream_t s) {
  const int G = H / KVH;
  if (ntiles <= 0) return 0;
  if (dh != 128 || G < 1) return -1;
  const int Gs = G % 4 == 0 ? 4 : (G % 2 == 0 ? 2 : 1);  // heads per block
  const size_t smem = 2 * 32768 + 1024;
  dim3 grid(ntiles, KVH * (G / Gs));
#define SPEX_MMA_CASE(GG)                                                                             \
  if (Gs == GG) {                                                                                    \
    static bool attr = false;                                                                        \
    if (!attr) {                                                                                     \
      cudaFuncSetAttribute(tree_attn_tile_mma_kernel<GG>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                           (int)smem);                                                               \
      attr = true;                                                                                   \
    }                                                                                                \
    tree_attn_tile_mma_kernel<GG><<<grid, 128, smem, s>>>(*kvmap, tiles, rows, segs, Qr, H, slots, O, G);        \
    return 0;                                                                                        \
  }
  SPEX_MMA_CASE(1)
  SPEX_MMA_CASE(2)
  SPEX_MMA_CASE(4)
#undef SPEX_MMA_CASE
  return -1;
}

extern "C" int spex_k_tree_attn_tiles(const TileDesc* tiles, int ntiles, const RowDesc* rows, const Segment* segs,
                                      const float* Qr, int H, int KVH, int dh, const __nv_bfloat16* Kp,
                                      const __nv_bfloat16* Vp, long long slots, __nv_bfloat16* O, cudaStream_t s) {
  const int G = H / KVH;
  if (ntiles <= 0) return 0;
#define SPEX_TILE_CASE(D, GG)                                                        \
  if (dh == D && G == GG) {                                                          \
    launch_tile<D, GG>(tiles, ntiles, rows, segs, Qr, H, KVH, Kp, Vp, slots, O, s);  \
    return 0;                                                                        \
  }
  SPEX_TILE_CASE(128, 1)
  SPEX_TILE_CASE(128, 2)
  SPEX_TILE_CASE(128, 4)
  SPEX_TILE_CASE(128, 6)
  SPEX_TILE_CASE(64, 1)
  SPEX_TILE_CASE(64, 2)
#undef SPEX_TILE_CASE
  return -1;
}

// PRM rewards: scatter the entry's scores to their nodes, then raise the
// entry's flag for the control kernel (which spins on it in prm_reward).
__global__ void prm_publish_kernel(const RowDesc* __restrict__ rows, const int* __restrict__ last_row, int n,
                                   const float* __restrict__ score, int node_cap, float* node_score, int* done) {
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    const RowDesc r = rows[last_row[k]];
    node_score[(long long)r.q * node_cap + r.node] = score[k];
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) atomicExch(done, 1);
}

extern "C" void spex_k_prm_publish(const RowDesc* rows, const int* last_row, int n, const float* score, int node_cap,
                                   float* node_score, int* done, cudaStream_t s) {
  prm_publish_kernel<<<1, 256, 0, s>>>(rows, last_row, n, score, node_cap, node_score, done);
}

extern "C" void spex_k_value_head(const __nv_bfloat16* Hn, int d, const int* last_row, int n,
                                  const __nv_bfloat16* w, float* score, cudaStream_t s) {
  value_head_kernel<<<n, 128, 0, s>>>(Hn, d, last_row, n, w, score);
}

// Loads every kernel the forward can launch (cudaFuncGetAttributes forces the
// lazy loader), so no module load — which may synchronise the context — can
// happen while the control kernel spins on a PRM score (model mode).
namespace spex {
template <class K>
static void preload_one(K k) {
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, k);
}
}  // namespace spex

extern "C" void spex_k_preload() {
  using namespace spex;
  preload_one(init_weights_kernel);
  preload_one(build_decode_rows_kernel);
  preload_one(build_prm_rows_kernel);
  preload_one(build_prompt_rows_kernel);
  preload_one(build_prompt_tiles_kernel);
  preload_one(prm_scan_all_kernel);
  preload_one(gather_prm_kernel);
  preload_one(gather_outputs_kernel);
  preload_one(embed_kernel);
  preload_one(rmsnorm_bf16_kernel);
  preload_one(rmsnorm_bf16_reg_kernel<4>);
  preload_one(rmsnorm_bf16_reg_kernel<8>);
  preload_one(rmsnorm_bf16_reg_kernel<32>);
  preload_one(rmsnorm_bf16_reg_kernel<12>);
#define SPEX_PRELOAD_DEC(D, GG)                      \
  preload_one(tree_attn_decode_kernel<D, GG, 8>);    \
  preload_one(tree_attn_decode_kernel<D, GG, 4>);    \
  preload_one(tree_attn_tile_kernel<D, GG>);
  SPEX_PRELOAD_DEC(128, 1)
  SPEX_PRELOAD_DEC(128, 2)
  SPEX_PRELOAD_DEC(128, 4)
  SPEX_PRELOAD_DEC(128, 6)
  SPEX_PRELOAD_DEC(64, 1)
  SPEX_PRELOAD_DEC(64, 2)
#undef SPEX_PRELOAD_DEC
  preload_one(tree_attn_decode_kernel<128, 8, 8>);
  preload_one(tree_attn_decode_kernel<128, 8, 4>);
  preload_one(tree_attn_decode_kernel<64, 4, 8>);
  preload_one(tree_attn_decode_kernel<64, 4, 4>);
  preload_one(tree_attn_bulk_kernel<16, 2, 14>);
  preload_one(tree_attn_wmma_kernel<kMmaNST, kMmaWarps, false>);
  preload_one(tree_attn_tile_mma_kernel<1>);
  preload_one(tree_attn_tile_mma_kernel<2>);
  preload_one(tree_attn_tile_mma_kernel<4>);
  preload_one(order_rows_kernel);
  preload_one(value_head_kernel);
  preload_one(prm_publish_kernel);
}
