// model_host.cpp — policy / PRM forward over the schedule the control kernel
// recorded (decode epochs and reward batches), on the device.
//
// Per decode step of an epoch (DecodeEngine::advance, sim.cpp:305-384) every
// active stream runs one token through the policy: embedding, L x [RMSNorm,
// QKV projection, RoPE + append to the tree KV pool, K1 tree attention over
// the ancestor chain, O projection + residual, RMSNorm, gate/up projection,
// SwiGLU, down projection + residual], final RMSNorm, LM head and the K3
// epilogue. Every reward batch (the completions of one engine boundary,
// executor.cpp:366-411) runs the PRM over each completed thought's tokens with
// its own tree KV pool, then the value head (K4).
//
// Every projection runs on the hand-written tcgen05 GEMM (gemm_tc.cu) with the
// elementwise work fused into its epilogue; no library GEMM is called.
#include "model_host.h"

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <chrono>
#include <thread>
#include <vector>

using namespace spex;

extern "C" {
void spex_k_init_weights(__nv_bfloat16* w, long long n, uint64_t seed, uint64_t tid, float scale, cudaStream_t s);
void spex_k_build_decode_rows(TreeView t, const int* sids, const int* pos0, int n, int step, RowDesc* rows,
                              Segment* segs, cudaStream_t s);
void spex_k_build_prm_rows(TreeView t, const int* sids, const int* row_start, const int* tile_start, int n,
                           RowDesc* rows, Segment* segs, int* last_row, TileDesc* tiles, cudaStream_t s);
void spex_k_build_prompt_tiles(int nq, int P, TileDesc* tiles, cudaStream_t s);
int spex_k_tree_attn_tiles_mma(const CUtensorMap* kvmap, const TileDesc* tiles, int ntiles,
                               const RowDesc* rows, const Segment* segs, const float* Qr, int H, int KVH, int dh,
                               long long slots, __nv_bfloat16* O, cudaStream_t s);
int spex_k_tree_attn_tiles(const TileDesc* tiles, int ntiles, const RowDesc* rows, const Segment* segs,
                           const float* Qr, int H, int KVH, int dh, const __nv_bfloat16* Kp, const __nv_bfloat16* Vp,
                           long long slots, __nv_bfloat16* O, cudaStream_t s);
void spex_k_build_prompt_rows(TreeView t, int q0, int nq, RowDesc* rows, Segment* segs, cudaStream_t s);
void spex_k_prm_scan_all(TreeView t, const int* kind, const int* off, const int* n, int n_entries,
                         const int* srow_sid, int* row_start, int* tile_start, int* totals, int* tile_totals,
                         cudaStream_t s);
void spex_k_embed(const RowDesc* rows, int M, const __nv_bfloat16* E, int d, float* X, cudaStream_t s);
void spex_k_rmsnorm(const float* X, int M, int d, float eps, __nv_bfloat16* Y, cudaStream_t s);
int spex_k_tree_attn(const RowDesc* rows, const Segment* segs, const float* Qr, int H, int KVH, int dh,
                     const __nv_bfloat16* Kp, const __nv_bfloat16* Vp, long long slots, __nv_bfloat16* O, int M,
                     cudaStream_t s);
void spex_k1_set_kv_evict_first(int on);
void spex_k1_set_row_order(const int* order);
void spex_k_order_rows(const RowDesc* rows, int M, int Q, int* order, cudaStream_t s);
int spex_k_tree_attn_bulk(const RowDesc* rows, const Segment* segs, const float* Qr, int H, int KVH, int dh,
                          const __nv_bfloat16* Kp, const __nv_bfloat16* Vp, long long slots, __nv_bfloat16* O, int M,
                          int* item_ctr, cudaStream_t s);
int spex_k_tree_attn_wmma(const CUtensorMap* kvmap16, const RowDesc* rows,
                          const Segment* segs, const float* Qr, int H, int KVH, int dh, long long slots,
                          __nv_bfloat16* O, int M, int* item_ctr, cudaStream_t s);
int spex_k_gemm_tc(const CUtensorMap* tmA, const CUtensorMap* tmB, int M, int N, int K, const TcEpilogue* ep,
                   unsigned int* sched, cudaStream_t s);
void spex_k_lse_combine(const float* part, int M, int n_tiles, int* amax, float* lse, float* lsum, cudaStream_t s);
void spex_k_rope_table(const RowDesc* rows, int M, const float* inv_freq, int half, float* out, cudaStream_t s);
void spex_k_interleave_gu(const __nv_bfloat16* wgu, int F, int d, __nv_bfloat16* out, cudaStream_t s);
void spex_k_prm_publish(const RowDesc* rows, const int* last_row, int n, const float* score, int node_cap,
                        float* node_score, int* done, cudaStream_t s);
void spex_k_value_head(const __nv_bfloat16* Hn, int d, const int* last_row, int n, const __nv_bfloat16* w,
                       float* score, cudaStream_t s);
void spex_k_gather_prm(const RowDesc* rows, const int* last_row, int n, const float* score, PrmOut* out,
                       cudaStream_t s);
void spex_k_gather_outputs(const RowDesc* rows, int M, const int* amax, const float* lse, const float* lsum,
                           DecodeOut* out, cudaStream_t s);
}

namespace {

#define CK(x)                                                                                    \
  do {                                                                                           \
    cudaError_t e_ = (x);                                                                        \
    if (e_ != cudaSuccess) throw std::runtime_error(std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)
template <class T>
T* dalloc(size_t n, std::vector<void*>& owned) {
  void* p = nullptr;
  CK(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)));
  owned.push_back(p);
  return static_cast<T*>(p);
}

}  // namespace

namespace spex {

// TMA descriptor of one KV pool viewed as a 2D [KVH*slots][dh] bf16 tensor,
// 64x64-element boxes with 128-byte swizzle (tree_attn_tile_mma_kernel).
typedef CUresult (*PFN_tmap_encode)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_tmap_encode tmap_encoder() {
  static PFN_tmap_encode fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_tmap_encode>(p);
  }
  return fn;
}

// TMA descriptors of one layer's tree-KV pools: the K and V pools (one
// allocation, V above K) as one 4D view — 64 columns, rows, the 2 column
// halves at +128 B, K|V at +(V - K) — with (64, box_rows, 2, 2) boxes, so ONE
// copy fills a whole K+V stage: K then V, each [half][box_rows rows][64],
// 128-byte swizzled (conflict-free ldmatrix). The K1 kernels issue their stage
// copies from inside the consumer loop, where every extra copy is on the
// critical path (profiles/r02zt_k1_gqa_tma_ab.txt).
static bool make_kv_pair_tmap(CUtensorMap* m, void* k, void* v, long long rows, int dh, int box_rows) {
  PFN_tmap_encode enc = tmap_encoder();
  const uintptr_t kb = reinterpret_cast<uintptr_t>(k), vb = reinterpret_cast<uintptr_t>(v);
  if (!enc || dh != 128 || vb <= kb || (vb - kb) % 16 != 0 || (vb - kb) >= (1ULL << 40)) return false;
  cuuint64_t dims[4] = {64, (cuuint64_t)rows, 2, 2};
  cuuint64_t strides[3] = {(cuuint64_t)dh * 2, 128, (cuuint64_t)(vb - kb)};
  cuuint32_t box[4] = {64, (cuuint32_t)box_rows, 2, 2};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, k, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 64-token chunks of the tile kernel (PRM / prompt rows, tree_attn_tile_mma_kernel).
extern "C" int spex_tmap_kv(CUtensorMap* m, void* k, void* v, long long rows, int dh) {
  return make_kv_pair_tmap(m, k, v, rows, dh, 64) ? 0 : -1;
}

// 16-token stages of the per-warp decode pipeline (tree_attn_wmma_kernel).
extern "C" int spex_tmap_kv16(CUtensorMap* m, void* k, void* v, long long rows, int dh) {
  return make_kv_pair_tmap(m, k, v, rows, dh, 16) ? 0 : -1;
}

// TMA descriptor of a row-major bf16 matrix [rows][cols] as a GEMM operand of
// gemm_tc.cu: 64 x 64 (cols x rows) boxes, 128-byte swizzle.
extern "C" int spex_tmap_operand(CUtensorMap* m, const void* base, long long rows, long long cols) {
  PFN_tmap_encode enc = tmap_encoder();
  if (!enc || cols % 64 != 0) return -1;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {64, 64};
  cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS
             ? 0
             : -1;
}

// K2 on hand-written tcgen05 (gemm_tc.cu): operand maps of one weight matrix
struct TcWeight {
  CUtensorMap map;
  int N = 0, K = 0;
};

struct Model {
  ModelShape sh;
  std::vector<CUtensorMap> kvmap;           // per layer, K|V pair, 64-row boxes (empty without TMA maps)
  std::vector<CUtensorMap> kvmap16;  // K|V pair, 16-row boxes (decode pipeline)
  bool is_prm;
  long long slots;
  int max_rows;
  std::vector<void*> owned;
  __nv_bfloat16* embed = nullptr;
  std::vector<__nv_bfloat16*> wqkv, wo, wgu, wd;
  __nv_bfloat16* lm = nullptr;
  __nv_bfloat16* vhead = nullptr;
  std::vector<__nv_bfloat16*> Kp, Vp;  // per layer [KVH][slots][dh]
  float* inv_freq = nullptr;
  // activations
  float* X = nullptr;
  __nv_bfloat16* Xn = nullptr;
  float* Qr = nullptr;               // [rows][H][dh] fp32, RoPE'd and pre-scaled (QKV epilogue)
  __nv_bfloat16* O = nullptr;        // attention output
  __nv_bfloat16* A = nullptr;        // SwiGLU activation (gate/up epilogue)
  // K2 (tcgen05): weight maps, activation maps, RoPE table, LM-head partials
  std::vector<TcWeight> tq, to, tgu, td;
  TcWeight tlm;
  CUtensorMap a_xn, a_o, a_act;        // activation operands [max_rows][*]
  float* rope_tab = nullptr;           // [max_rows][dh/2] (cos, sin)
  float* lse_part = nullptr;           // [max_rows][V/128] float4
  unsigned int* sched = nullptr;       // tcgen05 tile queue of this model's stream (self-resetting)
  int* amax = nullptr;
  float* lse = nullptr;
  float* lsum = nullptr;

  ~Model() {
    for (void* p : owned) cudaFree(p);
  }
};

long long model_weight_params(const ModelShape& s, bool prm) {
  long long per = (long long)(s.H + 2 * s.KVH) * s.dh * s.d + (long long)s.d * s.H * s.dh +
                  2LL * s.F * s.d + (long long)s.d * s.F;
  return (long long)s.V * s.d + s.L * per + (prm ? s.d : (long long)s.V * s.d);
}

// FLOPs of the projections per row (2 * matmul params, K2 accounting)
double model_matmul_flops_per_row(const ModelShape& s, bool prm) {
  double per = (double)(s.H + 2 * s.KVH) * s.dh * s.d + (double)s.d * s.H * s.dh + 2.0 * s.F * s.d +
               (double)s.d * s.F;
  return 2.0 * (s.L * per + (prm ? 0.0 : (double)s.V * s.d));
}

static Model* make_model(const ModelShape& sh, bool prm, uint64_t seed, long long slots, int max_rows,
                         cudaStream_t st) {
  Model* m = new Model();
  m->sh = sh;
  m->is_prm = prm;
  m->slots = slots;
  m->max_rows = max_rows;
  auto& o = m->owned;
  const float kStd = 0.02f * 1.7320508f;  // uniform +-a with std 0.02
  auto init = [&](__nv_bfloat16* w, long long n, uint64_t id, float scale) {
    spex_k_init_weights(w, n, seed, id, scale, st);
  };
  m->embed = dalloc<__nv_bfloat16>((size_t)sh.V * sh.d, o);
  init(m->embed, (long long)sh.V * sh.d, 1, 1.7320508f);
  for (int l = 0; l < sh.L; ++l) {
    const long long nq = (long long)(sh.H + 2 * sh.KVH) * sh.dh * sh.d;
    const long long no = (long long)sh.d * sh.H * sh.dh;
    const long long ng = 2LL * sh.F * sh.d;
    const long long nd = (long long)sh.d * sh.F;
    m->wqkv.push_back(dalloc<__nv_bfloat16>(nq, o));
    m->wo.push_back(dalloc<__nv_bfloat16>(no, o));
    m->wgu.push_back(dalloc<__nv_bfloat16>(ng, o));
    m->wd.push_back(dalloc<__nv_bfloat16>(nd, o));
    init(m->wqkv.back(), nq, 100 + 8 * l + 0, kStd);
    init(m->wo.back(), no, 100 + 8 * l + 1, kStd);
    init(m->wgu.back(), ng, 100 + 8 * l + 2, kStd);
    init(m->wd.back(), nd, 100 + 8 * l + 3, kStd);
    // K and V of a layer in one allocation, V above K (the decode pipeline's
    // K|V tensor map, make_kv_tmap16)
    __nv_bfloat16* kv = dalloc<__nv_bfloat16>((size_t)2 * sh.KVH * slots * sh.dh, o);
    m->Kp.push_back(kv);
    m->Vp.push_back(kv + (size_t)sh.KVH * slots * sh.dh);
    // zero-filled: decode boxes may cover slots past a segment (masked to p = 0,
    // which must not meet a NaN bit pattern)
    CK(cudaMemsetAsync(m->Kp.back(), 0, (size_t)sh.KVH * slots * sh.dh * 2, st));
    CK(cudaMemsetAsync(m->Vp.back(), 0, (size_t)sh.KVH * slots * sh.dh * 2, st));
  }
  if (!getenv("SPEX_NO_MMA_ATTN")) {
    m->kvmap.resize(sh.L);
    m->kvmap16.resize(sh.L);
    for (int l = 0; l < sh.L; ++l) {
      const long long rows = (long long)sh.KVH * slots;
      if (!make_kv_pair_tmap(&m->kvmap[l], m->Kp[l], m->Vp[l], rows, sh.dh, 64) ||
          !make_kv_pair_tmap(&m->kvmap16[l], m->Kp[l], m->Vp[l], rows, sh.dh, 16)) {
        m->kvmap.clear();
        m->kvmap16.clear();
        break;
      }
    }
  }
  if (prm) {
    m->vhead = dalloc<__nv_bfloat16>(sh.d, o);
    init(m->vhead, sh.d, 3, kStd);
  } else {
    m->lm = dalloc<__nv_bfloat16>((size_t)sh.V * sh.d, o);
    init(m->lm, (long long)sh.V * sh.d, 2, kStd);
  }
  std::vector<float> inv(sh.dh / 2);
  for (int i = 0; i < sh.dh / 2; ++i)
    inv[i] = (float)(1.0 / std::pow((double)sh.rope_theta, (2.0 * i) / sh.dh));
  m->inv_freq = dalloc<float>(inv.size(), o);
  CK(cudaMemcpyAsync(m->inv_freq, inv.data(), inv.size() * sizeof(float), cudaMemcpyHostToDevice, st));
  const size_t M = max_rows;
  m->X = dalloc<float>(M * sh.d, o);
  m->Xn = dalloc<__nv_bfloat16>(M * std::max(sh.d, sh.H * sh.dh), o);
  m->Qr = dalloc<float>(M * sh.H * sh.dh, o);
  m->O = dalloc<__nv_bfloat16>(M * sh.H * sh.dh, o);
  m->A = dalloc<__nv_bfloat16>(M * sh.F, o);
  if (!prm) {
    m->amax = dalloc<int>(M, o);
    m->lse = dalloc<float>(M, o);
    m->lsum = dalloc<float>(M, o);
  }
  m->rope_tab = dalloc<float>(M * sh.dh, o);  // [max_rows][dh/2] (cos, sin)
  // K2: every projection on the hand-written tcgen05 GEMM with fused epilogues
  // (gemm_tc.cu): QKV + RoPE + KV append, O + residual, gate/up + SwiGLU,
  // down + residual, LM head + logsumexp/argmax partials. No library GEMM.
  const int qkv_n = (sh.H + 2 * sh.KVH) * sh.dh;
  if (!(sh.d % 64 == 0 && qkv_n % 128 == 0 && (sh.H * sh.dh) % 64 == 0 && sh.F % 64 == 0 &&
        (sh.dh == 64 || sh.dh == 128) && (prm || sh.V % 128 == 0)))
    throw std::runtime_error("model shape not supported by the tcgen05 projections");
  auto wmap = [&](TcWeight& w, const __nv_bfloat16* base, int N, int K) {
    w.N = N;
    w.K = K;
    if (spex_tmap_operand(&w.map, base, N, K) != 0) throw std::runtime_error("TMA descriptor of a weight failed");
  };
  m->tq.resize(sh.L);
  m->to.resize(sh.L);
  m->tgu.resize(sh.L);
  m->td.resize(sh.L);
  for (int l = 0; l < sh.L; ++l) {
    // gate/up rows interleaved per 64 for the SwiGLU epilogue (replaces the plain layout)
    __nv_bfloat16* il = dalloc<__nv_bfloat16>((size_t)2 * sh.F * sh.d, o);
    spex_k_interleave_gu(m->wgu[l], sh.F, sh.d, il, st);
    CK(cudaStreamSynchronize(st));
    o.erase(std::find(o.begin(), o.end(), static_cast<void*>(m->wgu[l])));
    CK(cudaFree(m->wgu[l]));
    m->wgu[l] = il;
    wmap(m->tq[l], m->wqkv[l], qkv_n, sh.d);
    wmap(m->to[l], m->wo[l], sh.d, sh.H * sh.dh);
    wmap(m->tgu[l], m->wgu[l], 2 * sh.F, sh.d);
    wmap(m->td[l], m->wd[l], sh.d, sh.F);
  }
  if (!prm) wmap(m->tlm, m->lm, sh.V, sh.d);
  if (spex_tmap_operand(&m->a_xn, m->Xn, (long long)M, sh.d) || spex_tmap_operand(&m->a_o, m->O, (long long)M, sh.H * sh.dh) ||
      spex_tmap_operand(&m->a_act, m->A, (long long)M, sh.F))
    throw std::runtime_error("TMA descriptor of an activation failed");
  if (!prm) m->lse_part = dalloc<float>(M * (size_t)(sh.V / 128) * 4, o);
  m->sched = dalloc<unsigned int>(2, o);
  CK(cudaMemsetAsync(m->sched, 0, 2 * sizeof(unsigned int), st));
  return m;
}

// Decode rows with one KV head per query head (G = 1) stream through the
// bulk-copy pipeline kernel (measured 1.98 s vs 2.10 s per c2 search for the
// register-pipelined FHFMA kernel); SPEX_K1_BULK=0 selects the latter.
static bool bulk_wanted() {
  static const bool on = !getenv("SPEX_K1_BULK") || atoi(getenv("SPEX_K1_BULK")) != 0;
  return on;
}
static int* g_item_ctr = nullptr;  // K1 bulk kernel's work counter (policy stream)
// Per-warp TMA + mma.sync decode pipeline: default for GQA groups (G >= 4:
// config 5's K1 5.2 s -> 3.2 s); for G = 1 the FHFMA bulk kernel is faster
// (1.98 s vs 2.13 s on c2). SPEX_K1_WMMA=1 forces it for every group size, 0 off.
static bool wmma_wanted(const ModelShape& s) {
  static const int mode = getenv("SPEX_K1_WMMA") ? atoi(getenv("SPEX_K1_WMMA")) : 2;
  return mode == 1 || (mode == 2 && s.H / s.KVH >= 4);
}

static void tc_gemm(const CUtensorMap& a, const TcWeight& w, int M, const TcEpilogue& ep, unsigned int* sched,
                    cudaStream_t st) {
  const int rc = spex_k_gemm_tc(&a, &w.map, M, w.N, w.K, &ep, sched, st);
  if (rc != 0)
    throw std::runtime_error("tcgen05 GEMM launch failed (" + std::to_string(rc) + ") M=" + std::to_string(M) +
                             " N=" + std::to_string(w.N) + " K=" + std::to_string(w.K) + " epilogue " +
                             std::to_string(ep.kind));
}

// K1 for one layer: PRM / prompt tiles on the TMA + tensor-core tile kernel;
// decode rows on the per-warp TMA pipeline (GQA groups), the bulk-copy
// pipeline (one KV head per query head) or the register pipeline (other shapes).
static void attention(Model& m, int l, const RowDesc* rows, const Segment* segs, int M, const TileDesc* tiles,
                      int ntiles, cudaStream_t st) {
  const ModelShape& s = m.sh;
  int rc = -1;
  if (tiles && !m.kvmap.empty())
    rc = spex_k_tree_attn_tiles_mma(&m.kvmap[l], tiles, ntiles, rows, segs, m.Qr, s.H, s.KVH, s.dh,
                                    m.slots, m.O, st);
  if (rc != 0 && !tiles && !m.kvmap16.empty() && wmma_wanted(s) && g_item_ctr)
    rc = spex_k_tree_attn_wmma(&m.kvmap16[l], rows, segs, m.Qr, s.H, s.KVH, s.dh, m.slots, m.O, M,
                               g_item_ctr, st);
  if (rc != 0 && !tiles && bulk_wanted() && g_item_ctr)
    rc = spex_k_tree_attn_bulk(rows, segs, m.Qr, s.H, s.KVH, s.dh, m.Kp[l], m.Vp[l], m.slots, m.O, M, g_item_ctr, st);
  if (rc != 0)
    rc = tiles ? spex_k_tree_attn_tiles(tiles, ntiles, rows, segs, m.Qr, s.H, s.KVH, s.dh, m.Kp[l], m.Vp[l], m.slots,
                                        m.O, st)
               : spex_k_tree_attn(rows, segs, m.Qr, s.H, s.KVH, s.dh, m.Kp[l], m.Vp[l], m.slots, m.O, M, st);
  if (rc != 0) throw std::runtime_error("tree attention: unsupported head shape");
}

// One forward over M rows. K1 launches are bracketed by events when `timer`
// is given, accumulating their device time.
static long long g_launches = 0;

static void forward(Model& m, const RowDesc* rows, const Segment* segs, int M, cudaStream_t st, AttnTimer* timer,
                    const TileDesc* tiles = nullptr, int ntiles = 0) {
  const ModelShape& s = m.sh;
  // embed -> L x [RMSNorm, QKV + RoPE + KV append (tcgen05), K1, O + residual
  // (tcgen05), RMSNorm, gate/up + SwiGLU (tcgen05), down + residual (tcgen05)]
  // -> RMSNorm -> LM head + logsumexp/argmax partials (tcgen05) -> combine
  g_launches += 3 + 7LL * s.L + (m.is_prm ? 0 : 2);
  spex_k_rope_table(rows, M, m.inv_freq, s.dh / 2, m.rope_tab, st);  // (cos, sin) once for all layers
  spex_k_embed(rows, M, m.embed, s.d, m.X, st);
  TcEpilogue eq{};
  eq.kind = TC_EPI_ROPE_KV;
  eq.rows = rows;
  eq.rope = m.rope_tab;
  eq.H = s.H;
  eq.KVH = s.KVH;
  eq.dh = s.dh;
  eq.qscale = 1.0f / std::sqrt((float)s.dh);
  eq.Qr = m.Qr;
  eq.slots = m.slots;
  TcEpilogue er{};
  er.kind = TC_EPI_STORE;
  er.y = m.X;
  er.ldy = s.d;
  er.accumulate = 1;
  TcEpilogue eg{};
  eg.kind = TC_EPI_SWIGLU;
  eg.act = m.A;
  eg.F = s.F;
  for (int l = 0; l < s.L; ++l) {
    spex_k_rmsnorm(m.X, M, s.d, s.eps, m.Xn, st);
    eq.Kp = m.Kp[l];
    eq.Vp = m.Vp[l];
    tc_gemm(m.a_xn, m.tq[l], M, eq, m.sched, st);
    if (timer) timer->begin(st);
    attention(m, l, rows, segs, M, tiles, ntiles, st);
    if (timer) timer->end(st);
    tc_gemm(m.a_o, m.to[l], M, er, m.sched, st);
    spex_k_rmsnorm(m.X, M, s.d, s.eps, m.Xn, st);
    tc_gemm(m.a_xn, m.tgu[l], M, eg, m.sched, st);
    tc_gemm(m.a_act, m.td[l], M, er, m.sched, st);
  }
  spex_k_rmsnorm(m.X, M, s.d, s.eps, m.Xn, st);
  if (!m.is_prm) {
    TcEpilogue el{};
    el.kind = TC_EPI_LSE;
    el.part = m.lse_part;
    el.n_tiles = s.V / 128;
    el.V = s.V;
    tc_gemm(m.a_xn, m.tlm, M, el, m.sched, st);
    spex_k_lse_combine(m.lse_part, M, s.V / 128, m.amax, m.lse, m.lsum, st);
  }
}

void AttnTimer::begin(cudaStream_t st) {
  if (n >= (int)ev.size()) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    ev.push_back({a, b});
  }
  cudaEventRecord(ev[n].first, st);
}

void AttnTimer::end(cudaStream_t st) {
  cudaEventRecord(ev[n].second, st);
  if ((int)bytes.size() <= n) bytes.resize(n + 1);
  bytes[n] = cur_bytes;
  ++n;
  if (n == (int)ev.size() && n >= 256) flush();
}

void AttnTimer::flush() {
  for (int i = 0; i < n; ++i) {
    float ms = 0.f;
    cudaEventSynchronize(ev[i].second);
    cudaEventElapsedTime(&ms, ev[i].first, ev[i].second);
    if (dump) std::fprintf(dump, "%lld %.0f %.6f\n", launches, bytes[i], ms);
    total_ms += ms;
    launches += 1;
  }
  n = 0;
}

AttnTimer::~AttnTimer() {
  if (dump) std::fclose(dump);
  for (auto& p : ev) {
    cudaEventDestroy(p.first);
    cudaEventDestroy(p.second);
  }
}

ModelShape shape_by_name(const std::string& name) {
  // {d, L, H, KVH, dh, F, V, rope_theta, eps}
  if (name == "small_policy") return {256, 2, 4, 2, 64, 768, 512, 10000.f, 1e-5f};
  if (name == "small_prm") return {128, 2, 2, 2, 64, 384, 512, 10000.f, 1e-5f};
  if (name == "mid_policy") return {1024, 8, 8, 8, 128, 2816, 32000, 10000.f, 1e-5f};
  if (name == "mid_prm") return {512, 4, 4, 4, 128, 1408, 32000, 10000.f, 1e-5f};
  if (name == "llama3_8b") return {4096, 32, 32, 8, 128, 14336, 128256, 500000.f, 1e-5f};
  if (name == "prm_1p5b") return {1536, 28, 12, 2, 128, 8960, 128256, 1000000.f, 1e-6f};
  throw std::runtime_error("unknown model shape " + name);
}

// Process-wide cache: weights and tree KV pools stay resident across runs
// (a serving process keeps them; re-initialising 10s of GB per search would
// measure cudaMalloc, not the path). Reused when shape/seed match and the
// capacity suffices.
struct ModelCache {
  Model* pol = nullptr;
  Model* prm = nullptr;
  unsigned long long seed = 0;
  // replay row buffers (kept resident: no cudaMalloc while the control kernel runs)
  int rows_cap = 0;
  RowDesc* rows = nullptr;
  Segment* segs = nullptr;
  int* last_row = nullptr;
  TileDesc* tiles = nullptr;
  float* scores = nullptr;
  // PRM side: its own stream and row buffers, so reward scoring
  // (tensor-bound prefill GEMMs) overlaps the policy decode (HBM-bound K1)
  cudaStream_t st2 = nullptr;
  RowDesc* rows2 = nullptr;
  Segment* segs2 = nullptr;
  TileDesc* tiles2 = nullptr;
  int* item_ctr = nullptr;  // K1 bulk kernel's work counter (policy stream)
  int* row_order = nullptr;  // decode rows grouped by query (K1 bulk claim order)
  int row_order_cap = 0;
};
static ModelCache g_cache;

// K1 bulk claim order grouped by query (SPEX_K1_QORDER=0: active order).
static bool qorder_wanted() {
  static const bool on = !getenv("SPEX_K1_QORDER") || atoi(getenv("SPEX_K1_QORDER")) != 0;
  return on;
}

static bool same_shape(const ModelShape& a, const ModelShape& b) {
  return a.d == b.d && a.L == b.L && a.H == b.H && a.KVH == b.KVH && a.dh == b.dh && a.F == b.F && a.V == b.V &&
         a.rope_theta == b.rope_theta && a.eps == b.eps;
}

static Model* cached(Model*& slot, const ModelShape& sh, bool prm, uint64_t seed, long long slots, int max_rows,
                     cudaStream_t st) {
  if (slot && same_shape(slot->sh, sh) && slot->slots >= slots && slot->max_rows >= max_rows &&
      g_cache.seed == seed)
    return slot;
  delete slot;
  slot = nullptr;
  CK(cudaStreamSynchronize(st));
  slot = make_model(sh, prm, prm ? (seed ^ 0x50524d00ULL) : seed, slots + slots / 8 + 1024,
                    max_rows + max_rows / 8 + 256, st);
  return slot;
}

// Frees cached models whose shape or seed differ from the next run's (before
// the caller sizes the KV pools from the free memory).
extern "C" void spex_model_cache_release_mismatch(const ModelRunConfig* mc) {
  const bool seed_ok = g_cache.seed == mc->seed;
  if (g_cache.pol && (!seed_ok || !same_shape(g_cache.pol->sh, mc->policy))) {
    cudaDeviceSynchronize();
    delete g_cache.pol;
    g_cache.pol = nullptr;
  }
  if (g_cache.prm && (!seed_ok || !mc->with_prm || !same_shape(g_cache.prm->sh, mc->prm))) {
    cudaDeviceSynchronize();
    delete g_cache.prm;
    g_cache.prm = nullptr;
  }
}

// Tree-KV pool capacity (slots) for the next run of `mc`: the resident pools
// when the cached models match, else 62% of the free HBM after releasing the
// mismatched ones (both models, all layers, K and V in bf16).
extern "C" long long spex_model_pool_slots(const ModelRunConfig* mc) {
  spex_model_cache_release_mismatch(mc);
  if (g_cache.pol && (!mc->with_prm || g_cache.prm))
    return mc->with_prm ? std::min(g_cache.pol->slots, g_cache.prm->slots) : g_cache.pol->slots;
  size_t free_b = 0, total_b = 0;
  cudaMemGetInfo(&free_b, &total_b);
  const double per_slot = 4.0 * (mc->policy.L * mc->policy.KVH * mc->policy.dh +
                                 (mc->with_prm ? mc->prm.L * mc->prm.KVH * mc->prm.dh : 0));
  return static_cast<long long>(0.70 * static_cast<double>(free_b) / per_slot);
}

extern "C" void spex_model_cache_clear() {
  delete g_cache.pol;
  delete g_cache.prm;
  g_cache.pol = g_cache.prm = nullptr;
}

// Replays the schedule through the policy and PRM. Entries come either from a
// finished control run (sv.entries_host) or live from the running control
// kernel through host-mapped memory (sv.pub_head / sv.pub_entries): the model
// stream then works on entry e while the control kernel produces e+1, ...
// Everything the forward allocates or (re)creates — models, KV pools, row
// buffers — before the control kernel starts: with PRM rewards the control
// waits on the forward, so nothing that synchronises the device (cudaFree,
// model init) may run while it is live.
extern "C" void spex_k_preload();
extern "C" void spex_k_gemm_preload();

static void prepare_cache(const ModelRunConfig& mc, const ScheduleView& sv, cudaStream_t st) {
  static const bool preloaded = [] {
    spex_k_preload();
    spex_k_gemm_preload();
    return true;
  }();
  (void)preloaded;
  const int Q = sv.n_queries, P = sv.tree.prompt_tokens;
  const int max_dec = sv.max_decode_rows, max_prm = sv.max_prm_rows;
  const int prompt_chunk = std::max(1, std::min(Q, 4096 / std::max(P, 1)));
  const long long slots = std::max<long long>(sv.kv_slots, 1);
  if (!g_cache.st2) CK(cudaStreamCreateWithFlags(&g_cache.st2, cudaStreamNonBlocking));
  if (g_cache.seed != mc.seed) spex_model_cache_clear();
  Model* pol = cached(g_cache.pol, mc.policy, false, mc.seed, slots, std::max(max_dec, prompt_chunk * P), st);
  Model* prm = mc.with_prm ? cached(g_cache.prm, mc.prm, true, mc.seed, slots, std::max(max_prm, prompt_chunk * P), st)
                           : nullptr;
  g_cache.seed = mc.seed;
  // capacity actually resident (a cached pool may be larger than this run's request)
  const long long cap_slots = prm ? std::min(pol->slots, prm->slots) : pol->slots;
  if (cap_slots < sv.kv_slots) throw std::runtime_error("tree KV pools smaller than the control's page count");
  const int rows_cap = std::max({max_dec, max_prm, prompt_chunk * P, 1});
  if (!g_cache.item_ctr) {
    std::vector<void*> keep;
    g_cache.item_ctr = dalloc<int>(64, keep);
    CK(cudaMemset(g_cache.item_ctr, 0, 64 * sizeof(int)));  // the bulk K1 kernel keeps [0..1] self-resetting
    g_item_ctr = g_cache.item_ctr;
  }
  if (g_cache.rows_cap < rows_cap) {
    CK(cudaStreamSynchronize(st));
    CK(cudaStreamSynchronize(g_cache.st2));
    cudaFree(g_cache.rows);
    cudaFree(g_cache.segs);
    cudaFree(g_cache.last_row);
    cudaFree(g_cache.tiles);
    cudaFree(g_cache.scores);
    cudaFree(g_cache.rows2);
    cudaFree(g_cache.segs2);
    cudaFree(g_cache.tiles2);
    std::vector<void*> keep;
    g_cache.rows = dalloc<RowDesc>(rows_cap, keep);
    g_cache.segs = dalloc<Segment>((size_t)rows_cap * 40, keep);
    g_cache.last_row = dalloc<int>(rows_cap, keep);
    g_cache.tiles = dalloc<TileDesc>(rows_cap, keep);
    g_cache.scores = dalloc<float>(rows_cap, keep);
    g_cache.rows2 = dalloc<RowDesc>(rows_cap, keep);
    g_cache.segs2 = dalloc<Segment>((size_t)rows_cap * 40, keep);
    g_cache.tiles2 = dalloc<TileDesc>(rows_cap, keep);
    g_cache.rows_cap = rows_cap;
  }
  if (g_cache.row_order_cap < max_dec) {
    cudaFree(g_cache.row_order);
    std::vector<void*> keep;
    g_cache.row_order = dalloc<int>(std::max(max_dec, 1), keep);
    g_cache.row_order_cap = max_dec;
  }
  CK(cudaStreamSynchronize(st));
}

extern "C" void spex_model_prepare(const ModelRunConfig* mc, const ScheduleView* sv, cudaStream_t st) {
  prepare_cache(*mc, *sv, st);
}

void run_model_schedule(const ModelRunConfig& mc, const ScheduleView& sv, ModelRunResult* res, cudaStream_t st) {
  std::vector<void*> owned;
  const int Q = sv.n_queries, P = sv.tree.prompt_tokens;
  const bool streaming = sv.pub_head != nullptr;
  const int max_dec = sv.max_decode_rows, max_prm = sv.max_prm_rows;
  const int prompt_chunk = std::max(1, std::min(Q, 4096 / std::max(P, 1)));
  const long long slots = std::max<long long>(sv.kv_slots, 1);

  prepare_cache(mc, sv, st);
  const bool prm_overlap = !std::getenv("SPEX_PRM_SAME_STREAM");
  cudaStream_t st2 = prm_overlap ? g_cache.st2 : st;
  Model* pol = g_cache.pol;
  Model* prm = mc.with_prm ? g_cache.prm : nullptr;
  RowDesc* rows = g_cache.rows;
  Segment* segs = g_cache.segs;
  RowDesc* rows2 = prm_overlap ? g_cache.rows2 : g_cache.rows;
  Segment* segs2 = prm_overlap ? g_cache.segs2 : g_cache.segs;
  TileDesc* tiles2 = prm_overlap ? g_cache.tiles2 : g_cache.tiles;
  int* last_row = g_cache.last_row;
  TileDesc* tiles = g_cache.tiles;
  float* scores = g_cache.scores;

  // segment pools of the two streams' row builders (counters zeroed before
  // each build) and the forward's error bits, in the shared counter block
  int* seg_ctr_pol = g_cache.item_ctr + 16;
  int* seg_ctr_prm = prm_overlap ? g_cache.item_ctr + 17 : seg_ctr_pol;
  int* fwd_err = g_cache.item_ctr + 18;
  CK(cudaMemsetAsync(fwd_err, 0, sizeof(int), st));
  const long long seg_cap = (long long)g_cache.rows_cap * 40;
  TreeView tv_pol = sv.tree;
  tv_pol.V = mc.policy.V;
  tv_pol.seg_ctr = seg_ctr_pol;
  tv_pol.err = fwd_err;
  tv_pol.seg_cap = seg_cap;
  TreeView tv_prm = sv.tree;
  tv_prm.V = mc.prm.V;
  tv_prm.seg_ctr = seg_ctr_prm;
  tv_prm.err = fwd_err;
  tv_prm.seg_cap = seg_cap;
  AttnTimer timer;
  if (const char* p = std::getenv("SPEX_ATTN_LOG")) timer.dump = std::fopen(p, "w");
  // a query-block shard's forward is a fraction of the step, the replicated
  // control is the floor: stream the KV evict-first to keep L2 for control
  spex_k1_set_kv_evict_first(sv.shard_hi - sv.shard_lo < Q ? 1 : 0);
  cudaEvent_t t0, t1;
  cudaEventCreate(&t0);
  cudaEventCreate(&t1);
  cudaEventRecord(t0, st);
  cudaEvent_t e_fork, e_join;
  cudaEventCreateWithFlags(&e_fork, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&e_join, cudaEventDisableTiming);
  cudaEventRecord(e_fork, st);  // weights / pools initialised on st
  if (st2 != st) CK(cudaStreamWaitEvent(st2, e_fork, 0));
  g_launches = 0;
    if (P > 0) {
    const int q_end = std::min(sv.shard_hi, Q);
    for (int q0 = sv.shard_lo; q0 < q_end; q0 += prompt_chunk) {
      const int nq = std::min(prompt_chunk, q_end - q0);
      const int ntp = nq * ((P + kTileRows - 1) / kTileRows);
      spex_k_build_prompt_rows(tv_pol, q0, nq, rows, segs, st);
      spex_k_build_prompt_tiles(nq, P, tiles, st);
      g_launches += 2;
      forward(*pol, rows, segs, nq * P, st, nullptr, tiles, ntp);
      if (prm) {
        spex_k_build_prompt_rows(tv_prm, q0, nq, rows2, segs2, st2);
        spex_k_build_prompt_tiles(nq, P, tiles2, st2);
        g_launches += 2;
        forward(*prm, rows2, segs2, nq * P, st2, nullptr, tiles2, ntp);
      }
      res->prefill_rows += (long long)nq * P;
    }
  }
  const double kv_tok_bytes = 2.0 * mc.policy.KVH * mc.policy.dh * 2.0;  // K+V bf16, one layer
  DecodeOut* dbg = mc.record_outputs ? reinterpret_cast<DecodeOut*>(mc.out_rows) : nullptr;
  PrmOut* dbg_scores = mc.record_outputs ? reinterpret_cast<PrmOut*>(mc.out_scores) : nullptr;
  long long dbg_n = 0, dbg_s = 0;

  auto process = [&](const PubEntry& pe, int e) {
    if (pe.kind == SCHED_DECODE) {
      for (int s = 0; s < pe.steps; ++s) {
        for (int c0 = 0; c0 < pe.n; c0 += max_dec) {
          const int n = std::min(max_dec, pe.n - c0);
          CK(cudaMemsetAsync(seg_ctr_pol, 0, sizeof(int), st));
          spex_k_build_decode_rows(tv_pol, sv.srow_sid + pe.off + c0, sv.srow_pos0 + pe.off + c0, n, s, rows, segs,
                                   st);
          g_launches += 1;
          if (qorder_wanted()) {
            spex_k_order_rows(rows, n, Q, g_cache.row_order, st);
            spex_k1_set_row_order(g_cache.row_order);
            g_launches += 1;
          }
          // one K1 launch per layer: the step's unique KV tokens (this chunk's share) + Q/O rows
          timer.cur_bytes = ((double)pe.u0 + (double)s * pe.n + pe.n) * kv_tok_bytes * ((double)n / pe.n) +
                            (double)n * mc.policy.H * mc.policy.dh * (4.0 + 2.0);
          forward(*pol, rows, segs, n, st, mc.time_attn ? &timer : nullptr);
          spex_k1_set_row_order(nullptr);  // read at launch: other callers get row order
          if (dbg && dbg_n + n <= mc.out_rows_cap) {
            spex_k_gather_outputs(rows, n, pol->amax, pol->lse, pol->lsum, dbg + dbg_n, st);
            dbg_n += n;
          }
        }
        res->decode_rows += pe.n;
        res->decode_steps += 1;
        // algorithmic K1 bytes: unique KV tokens of the step (engine U + the new tokens)
        const double utok = (double)pe.u0 + (double)s * pe.n + pe.n;
        res->attn_alg_bytes += utok * kv_tok_bytes * mc.policy.L +
                               (double)pe.n * mc.policy.H * mc.policy.dh * (4.0 + 2.0) * mc.policy.L;
      }
    } else if (prm && pe.rows > 0) {
      if (pe.rows > max_prm) throw std::runtime_error("PRM batch larger than the row buffers");
      CK(cudaMemsetAsync(seg_ctr_prm, 0, sizeof(int), st2));
      spex_k_build_prm_rows(tv_prm, sv.srow_sid + pe.off, sv.srow_rstart + pe.off, sv.srow_tstart + pe.off, pe.n,
                            rows2, segs2, last_row, tiles2, st2);
      forward(*prm, rows2, segs2, pe.rows, st2, nullptr, tiles2, pe.tiles);
      spex_k_value_head(prm->Xn, mc.prm.d, last_row, pe.n, prm->vhead, scores, st2);
      if (sv.prm_done) {
        spex_k_prm_publish(rows2, last_row, pe.n, scores, sv.tree.node_cap, sv.node_score, sv.prm_done + e, st2);
        g_launches += 1;
      }
      g_launches += 2;
      if (dbg_scores && dbg_s + pe.n <= mc.out_scores_cap) {
        spex_k_gather_prm(rows2, last_row, pe.n, scores, dbg_scores + dbg_s, st2);
        dbg_s += pe.n;
      }
      res->prm_rows += pe.rows;
      res->prm_thoughts += pe.n;
    }
  };

  if (!streaming) {
    for (int e = 0; e < sv.n_entries; ++e) process(sv.entries_host[e], e);
  } else {
    volatile PubHead* head = reinterpret_cast<volatile PubHead*>(sv.pub_head);
    volatile PubEntry* ents = reinterpret_cast<volatile PubEntry*>(sv.pub_entries);
    int e = 0;
    auto last_progress = std::chrono::steady_clock::now();
    for (;;) {
      const int n = head->n_sched;
      if (e < n) {
        last_progress = std::chrono::steady_clock::now();
        for (; e < n; ++e) {
          PubEntry pe;
          pe.kind = ents[e].kind;
          pe.steps = ents[e].steps;
          pe.off = ents[e].off;
          pe.n = ents[e].n;
          pe.rows = ents[e].rows;
          pe.tiles = ents[e].tiles;
          pe.u0 = ents[e].u0;
          pe.kv_next = ents[e].kv_next;
          process(pe, e);
        }
        continue;
      }
      if (head->done) {
        if (head->n_sched == e) break;
        continue;
      }
      if (std::chrono::steady_clock::now() - last_progress > std::chrono::seconds(300))
        throw std::runtime_error("control kernel published nothing for 300 s");
      std::this_thread::yield();
    }
    res->control_error = head->error;
  }
  cudaEventRecord(e_join, st2);
  if (st2 != st) CK(cudaStreamWaitEvent(st, e_join, 0));
  cudaEventRecord(t1, st);
  CK(cudaEventSynchronize(t1));
  {
    int err = 0;
    CK(cudaMemcpy(&err, fwd_err, sizeof(int), cudaMemcpyDeviceToHost));
    if (err & 1) throw std::runtime_error("a thought's ancestor chain is deeper than the row builder's limit");
    if (err & 2) throw std::runtime_error("segment pool of the row builder exhausted");
  }
  cudaEventDestroy(e_fork);
  cudaEventDestroy(e_join);
  timer.flush();
  float ms = 0.f;
  cudaEventElapsedTime(&ms, t0, t1);
  res->model_ms = ms;
  res->attn_ms = timer.total_ms;
  res->attn_launches = timer.launches;
  res->launches = g_launches;
  res->gemm_calls = 0;  // no library GEMMs: every projection is on the tcgen05 kernel
  res->out_rows = dbg_n;
  res->out_scores = dbg_s;
  res->policy_flops = model_matmul_flops_per_row(mc.policy, false) * (double)(res->decode_rows + res->prefill_rows);
  res->prm_flops = prm ? model_matmul_flops_per_row(mc.prm, true) * (double)(res->prm_rows + res->prefill_rows) : 0.0;
  CK(cudaGetLastError());
  cudaEventDestroy(t0);
  cudaEventDestroy(t1);
  for (void* p : owned) cudaFree(p);
}

}  // namespace spex

// ------------------------------------------------- standalone PRM scoring
// spex_score_batch: each sequence is one thought with no ancestors (one own
// segment, causal within it), its tokens the PRM rows, 16-row tiles on the
// tensor-core tile kernel, the value head at the last row: the arithmetic of
// the executor's PRM scoring (run_model_schedule's PRM entries), with the
// weights of spex_executor_set_model's PRM for the same seed. Its own model
// instance and buffers, grown on demand; serialised with the executor runs.
namespace spex {
namespace {
struct ScoreCache {
  Model* m = nullptr;
  ModelShape sh{};
  uint64_t seed = 0;
  long long rows_cap = 0;
  int seq_cap = 0;
  RowDesc* rows = nullptr;
  Segment* segs = nullptr;
  TileDesc* tiles = nullptr;
  int* last_row = nullptr;
  float* scores = nullptr;
  std::vector<void*> bufs;
  cudaStream_t st = nullptr;
};
ScoreCache g_score;
}  // namespace

void prm_score_sequences(const ModelShape& sh, uint64_t weight_seed, const int* tokens, const long long* offsets,
                         int n, float* scores, int device) {
  if (n <= 0) return;
  CK(cudaSetDevice(device));
  long long M = 0;
  int ntiles = 0;
  for (int i = 0; i < n; ++i) {
    const long long len = offsets[i + 1] - offsets[i];
    if (len <= 0) throw std::runtime_error("score_batch: empty sequence " + std::to_string(i));
    for (long long j = offsets[i]; j < offsets[i + 1]; ++j)
      if (tokens[j] < 0 || tokens[j] >= sh.V) throw std::runtime_error("score_batch: token id out of the vocabulary");
    M += len;
    ntiles += static_cast<int>((len + kTileRows - 1) / kTileRows);
  }
  if (M > (1LL << 30)) throw std::runtime_error("score_batch: too many tokens");
  ScoreCache& c = g_score;
  if (!c.st) CK(cudaStreamCreateWithFlags(&c.st, cudaStreamNonBlocking));
  if (!c.m || !same_shape(c.sh, sh) || c.seed != weight_seed || c.m->slots < M || c.m->max_rows < M) {
    CK(cudaStreamSynchronize(c.st));
    delete c.m;
    const long long cap = std::max<long long>(M, 4096);
    c.m = make_model(sh, true, weight_seed ^ 0x50524d00ULL, cap + cap / 8 + 1024, static_cast<int>(cap + cap / 8 + 256),
                     c.st);
    c.sh = sh;
    c.seed = weight_seed;
  }
  if (c.rows_cap < M || c.seq_cap < n) {
    CK(cudaStreamSynchronize(c.st));
    for (void* p : c.bufs) cudaFree(p);
    c.bufs.clear();
    c.rows_cap = std::max<long long>(M, c.rows_cap);
    c.seq_cap = std::max(n, c.seq_cap);
    c.rows = dalloc<RowDesc>(c.rows_cap, c.bufs);
    c.segs = dalloc<Segment>(c.seq_cap, c.bufs);
    c.tiles = dalloc<TileDesc>(c.rows_cap, c.bufs);
    c.last_row = dalloc<int>(c.seq_cap, c.bufs);
    c.scores = dalloc<float>(c.seq_cap, c.bufs);
  }
  std::vector<RowDesc> rows(M);
  std::vector<Segment> segs(n);
  std::vector<TileDesc> tiles;
  std::vector<int> last(n);
  tiles.reserve(ntiles);
  long long r = 0;
  for (int i = 0; i < n; ++i) {
    const long long len = offsets[i + 1] - offsets[i];
    const long long base = r;  // the sequence's KV slots: its rows' own
    segs[i] = Segment{base, static_cast<int>(len), 0};
    for (long long j = 0; j < len; ++j, ++r) {
      RowDesc& d = rows[r];
      d.q = i;
      d.node = 0;
      d.pos = static_cast<int>(j);
      d.abs_pos = static_cast<int>(j);
      d.slot = base + j;
      d.seg_off = i;
      d.nseg = 1;
      d.token = tokens[offsets[i] + j];
      d.pad = 0;
    }
    for (long long j = 0; j < len; j += kTileRows)
      tiles.push_back(TileDesc{static_cast<int>(base + j), static_cast<int>(std::min<long long>(kTileRows, len - j))});
    last[i] = static_cast<int>(r - 1);
  }
  CK(cudaMemcpyAsync(c.rows, rows.data(), sizeof(RowDesc) * M, cudaMemcpyHostToDevice, c.st));
  CK(cudaMemcpyAsync(c.segs, segs.data(), sizeof(Segment) * n, cudaMemcpyHostToDevice, c.st));
  CK(cudaMemcpyAsync(c.tiles, tiles.data(), sizeof(TileDesc) * tiles.size(), cudaMemcpyHostToDevice, c.st));
  CK(cudaMemcpyAsync(c.last_row, last.data(), sizeof(int) * n, cudaMemcpyHostToDevice, c.st));
  forward(*c.m, c.rows, c.segs, static_cast<int>(M), c.st, nullptr, c.tiles, static_cast<int>(tiles.size()));
  spex_k_value_head(c.m->Xn, sh.d, c.last_row, n, c.m->vhead, c.scores, c.st);
  CK(cudaMemcpyAsync(scores, c.scores, sizeof(float) * n, cudaMemcpyDeviceToHost, c.st));
  CK(cudaStreamSynchronize(c.st));
}

}  // namespace spex
