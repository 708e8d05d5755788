// model.h — shapes and device structures of the policy / PRM forward that runs
// every decode step of the frontier (K1 tree attention, K2 projections/MLP,
// K3 LM-head epilogue) and every reward (K4 PRM scoring).
//
// The reference has no model (decode is a virtual clock, the
// reward is a hash oracle). In parity mode the control plane stays driven by
// the reference's content oracle and virtual clock, and this forward runs as
// real shadow work whose outputs are checked against oracle/model_ref.py.
#pragma once

#include <cstdint>

namespace spex {

struct ModelShape {
  int d;      // hidden size
  int L;      // layers
  int H;      // query heads
  int KVH;    // key/value heads (GQA)
  int dh;     // head dim
  int F;      // MLP hidden
  int V;      // vocab
  float rope_theta;
  float eps;
};

// Teacher-forced token ids: a pure function of the node path hash and the
// token position inside the thought (the same purity the reference's content
// oracle has, rng.hpp:7-10).
constexpr uint64_t kSaltTok = 0x746f6b5f69647300ULL;

// Row of a batched forward: one token of one thought.
struct RowDesc {
  int q;          // query
  uint32_t node;  // thought node
  int pos;        // token index inside the node's thought (0-based)
  int abs_pos;    // absolute position in the root..node sequence (RoPE)
  long long slot; // KV pool slot this token writes (kv_base(node) + pos)
  int seg_off;    // offset into the segment list
  int nseg;       // number of segments (ancestors root-first, then own prefix)
  int token;      // teacher-forced input token id
  int pad;
};

struct Segment {
  long long base;  // first KV slot
  int len;         // tokens
  int pad;
};

struct TreeView {
  const uint32_t* parent;
  const int* tokens;
  const uint64_t* hash;
  const long long* kvbase;
  const int* st_q;
  const uint32_t* st_node;
  int node_cap;
  int prompt_tokens;
  int V;
};

// Per decode row-step shadow outputs kept for verification (K3 epilogue).
struct DecodeOut {
  int q;
  uint32_t node;
  int pos;
  int amax;
  float lse;
  float lsum;
};

// A tile of consecutive rows of one thought (PRM scoring) sharing one pass
// over their common context; the last row carries the longest segment list.
struct TileDesc {
  int row0;
  int nrows;
};
constexpr int kTileRows = 16;

struct PrmOut {
  int q;
  uint32_t node;
  float score;
  int pad;
};

// Decode work list of one forward step (shared by its L K1 launches): every
// row's concatenated context is cut into at most kMaxRowChunks chunks of at
// least kMinChunk tokens; one warp per (chunk, kv head) pulled from a device
// work queue, partial softmax states merged by the last warp of the row.
constexpr int kMaxRowChunks = 8;
constexpr int kMinChunk = 128;
constexpr int kQueueSlots = 256;  // per-launch work-queue counters (one per layer)
struct ChunkItem {
  int row;
  int chunk;
};
struct DecodeChunks {
  ChunkItem* items;  // (row, chunk) in row order
  int* row_nch;     // chunks of row r
  int* row_ch;      // chunk length (tokens) of row r
  int* row_item0;   // first item of row r
  int* n_items;     // device scalar
  int* qctr;        // [kQueueSlots] work-queue heads, zeroed by the builder
  float* part;      // partial (acc, m, l) per (item, kv head): G * DH + round4(2G) floats
  int* cnt;         // [rows_cap * KVH] arrival counters (self-resetting)
};

// Query groups of one decode step (K1 tree-group kernel): the step's rows of
// one query, at most kGroupRows per group (in row order), and the union of
// their context segments with a bit mask of the rows that read each one, so a
// shared ancestor's K/V is staged once for the whole group.
constexpr int kGroupRows = 16;
struct GroupDesc {
  int nrows;
  int seg_off;  // into GroupSeg[]
  int nseg;
  int pad;
  int row[kGroupRows];
};
struct GroupSeg {
  long long base;  // first KV slot
  int len;         // tokens
  uint32_t mask;   // bit i: group row i attends to this segment
};
struct TreeGroups {
  int* q_cnt;          // [q_cap] rows per query
  int* q_off;          // [q_cap] first sorted position of query q
  int* q_goff;         // [q_cap] first group of query q
  int* q_fill;         // [q_cap]
  int* sorted;         // [rows_cap] row indices grouped by query, ascending within a query
  GroupDesc* groups;   // [rows_cap]
  GroupSeg* gsegs;     // [seg_cap]
  int* n_groups;       // device scalar
  int* seg_ctr;        // device scalar (zeroed by the builder)
  int q_cap;
  long long seg_cap;
};

// K2 tcgen05 GEMM epilogues (gemm_tc.cu)
enum TcEpi : int { TC_EPI_STORE = 0, TC_EPI_ROPE_KV = 1, TC_EPI_SWIGLU = 2, TC_EPI_LSE = 3 };
struct TcEpilogue {
  int kind;  // TcEpi
  // TC_EPI_STORE: y[row * ldy + col] (+)= acc
  float* y;
  int ldy;
  int accumulate;
  // TC_EPI_ROPE_KV
  const RowDesc* rows;
  const float* rope;  // [M][dh/2] (cos, sin) pairs at each row's absolute position
  int H, KVH, dh;
  float qscale;
  float* Qr;           // [M][H][dh] fp32, q * qscale
  void* Kp;            // bf16 [KVH][slots][dh]
  void* Vp;
  long long slots;
  // TC_EPI_SWIGLU: act[row][F] bf16 (gate/up weight rows interleaved per 64)
  void* act;
  int F;
  // TC_EPI_LSE: part[row][n_tiles] = (max, sum exp(x - max), sum x, first argmax bits)
  float* part;
  int n_tiles;
  int V;
};

// Schedule produced by the control kernel: decode epochs and reward batches.
enum : int { SCHED_DECODE = 1, SCHED_PRM = 2 };

}  // namespace spex
