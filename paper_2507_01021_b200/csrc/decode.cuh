// K6: batched greedy decode step kernels (Listing 1 `model.model.generate`,
// PAPER.md:57-59) over continuous-batching slots.
#pragma once

#include "common.cuh"

namespace dm {

// Shared per-engine decode state (device pointers).
struct DecodeState {
  int max_slots, d, heads, layers, ffn, vocab;
  int page_tokens;       // self-KV tokens per page (64)
  int pages_per_slot;    // page-table width (7 -> 448 positions)
  int eot;
  int prompt_len;
  const int32_t* prompt;       // [prompt_len]
  // slot bookkeeping
  const int32_t* active;       // [max_slots] slot ids, first *n_active valid
  const int32_t* n_active;     // device scalar
  int32_t* pos;                // [S] position of the token being fed
  int32_t* cur_tok;            // [S]
  int32_t* n_gen;              // [S]
  int32_t* cap;                // [S]
  int32_t* done;               // [S]
  int32_t* out_tokens;         // [S, 448]
  const int32_t* page_table;   // [S, pages_per_slot]
  uint16_t* kv_pool;           // [pages][L][2][H][page_tokens][64] bf16
  const uint16_t* xkv;         // [L][S][2][H][1500][64] bf16
  // activations (fp32)
  float* x;                    // [S, d] residual stream
  float* xn;                   // [S, d] LN output
  float* q;                    // [S, d]
  float* attn;                 // [S, d]
  float* h1;                   // [S, ffn]
  // split-K / split-KV scratch
  float* part;                 // scratch partials
  int32_t* counters;           // zero-initialised tile counters
  float* amax_val;             // [tiles, S]
  int32_t* amax_idx;           // [tiles, S]
  float* logits_dbg;           // optional [S, vocab]
  int xsplits;                 // cross-attention key splits
};

enum GemvEpi : int {
  GV_STORE = 0,     // y[slot, n] = acc + b
  GV_GELU = 1,      // y = gelu(acc + b)
  GV_RESID = 2,     // x[slot, n] += acc + b
  GV_SCALE = 3,     // y = (acc + b) * scale
  GV_QKV = 4,       // q (scaled) / append k, v to the slot's self-KV page
};

struct GemvArgs {
  const float* X;          // [S, K] fp32 (slot-indexed)
  const uint16_t* W;       // [N, K] bf16
  const uint16_t* bias;    // [N] nullable
  float* Y;                // [S, N] or residual
  int N, K;
  int epi;
  float scale;
  int layer;               // GV_QKV: layer index
  int splits;              // K splits (fixed per shape; never depends on R)
  int counter_base;        // offset into DecodeState::counters
};

int launch_gemv(const DecodeState& st, const GemvArgs& a, cudaStream_t stream);
int gemv_splits(int N, int K);
int launch_decode_ln(const DecodeState& st, const float* x, const uint16_t* g,
                     const uint16_t* b, float* y, cudaStream_t stream);
int launch_embed(const DecodeState& st, const uint16_t* embed, const uint16_t* pos_emb,
                 cudaStream_t stream);
int launch_self_attn(const DecodeState& st, int layer, cudaStream_t stream);
int launch_cross_attn(const DecodeState& st, int layer, int counter_base, cudaStream_t stream);
int launch_lm_head(const DecodeState& st, const uint16_t* embed, cudaStream_t stream);
int launch_finalize(const DecodeState& st, cudaStream_t stream);

}  // namespace dm
