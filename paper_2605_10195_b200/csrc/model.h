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

// A run of physically consecutive tree-KV slots: one thought's pages are cut
// into runs of consecutive pages (a thought on fresh pages is one run).
struct Segment {
  long long base;  // first KV slot
  int len;         // tokens
  int own0;        // -1: an ancestor's run; else the thought position of the run's first token (causal masking)
};

struct TreeView {
  const uint32_t* parent;
  const int* tokens;
  const uint64_t* hash;
  const long long* kvbase;  // first page-table entry of each node's thought (ctl_state.h n_kvbase)
  const int* kv_pt;         // page table: physical page of each entry
  const int* st_q;
  const uint32_t* st_node;
  int* seg_ctr;             // segment-pool counter of the builder's stream (zeroed before each build)
  int* err;                 // forward error bits: 1 ancestor chain deeper than kMaxChain, 2 segment pool full
  long long seg_cap;        // segment-pool capacity
  uint64_t run_seed;        // root prompts: query seeds (sim.cpp:177-180)
  int kv_pp_root;           // root prompts: static pages per query
  int q_offset;             // root prompts: local query q is the job's q + q_offset (split mode)
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
