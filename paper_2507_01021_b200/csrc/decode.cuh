// K6: batched greedy decode step kernels (Listing 1 `model.model.generate`,
// PAPER.md:57-59) over continuous-batching slots.
//
// Activations live in "row space": row i < n_active is the i-th active slot
// (slot = active[i]); persistent per-segment state (self-KV pages, cross-KV,
// position, cap, tokens) is slot-indexed. Activations that feed a projection
// are stored as a bf16 hi/lo pair (x = hi + lo exactly to ~2^-17 relative) so
// the projections run on tcgen05 with fp32 accumulation while keeping fp32
// activation precision (SURVEY.md §7 "Design rule").
#pragma once

#include "common.cuh"

#include <vector>

namespace dm {

constexpr int kRows = 64;          // max active slots = MMA N

struct DecodeState {
  int max_slots, d, heads, layers, ffn, vocab;
  int page_tokens;       // self-KV tokens per page (64)
  int pages_per_slot;    // page-table width (7 -> 448 positions)
  int eot;
  int prompt_len;
  const int32_t* prompt;       // [prompt_len]
  // slot bookkeeping
  const int32_t* active;       // [kRows] slot of row i
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
  // row-space activations
  float* x;                    // [kRows, d] residual stream (fp32)
  uint16_t *xh, *xl;           // [kRows, d]   LN output, bf16 hi/lo
  float* q;                    // [kRows, d]   attention query (pre-scaled)
  uint16_t *ah, *al;           // [kRows, d]   attention output hi/lo
  uint16_t *hh, *hl;           // [kRows, ffn] fc1 output hi/lo
  // scratch
  float* part;                 // split-K / split-KV partials
  int32_t* counters;           // zero-initialised tile counters
  float* amax_val;             // [vocab tiles, kRows]
  int32_t* amax_idx;           // [vocab tiles, kRows]
  float* logits_dbg;           // optional [kRows, vocab]
  float* ln_part;              // [d / 128][kRows][2]: per 128-feature tile, per row, (sum, sum sq)
                               // of the residual stream, written by its producer (embed or a
                               // residual-add projection) for the next fused LayerNorm
  int xsplits;                 // cross-attention key splits
};

enum TcGemvEpi : int {
  TV_STORE = 0,     // y[r, n] = (acc + b) * scale                 (fp32)
  TV_GELU_HILO = 1, // yh/yl[r, n] = split(gelu(acc + b))         (bf16 pair)
  TV_RESID = 2,     // x[r, n] += acc + b
  TV_QKV = 3,       // q (scaled) / append k, v to the row's self-KV page
  TV_ARGMAX = 4,    // per-row (max, lowest index) over this 128-row vocab tile
};

struct TcGemvArgs {
  const uint16_t* bias;    // [N] nullable
  int N, K;
  int epi;
  float scale;
  int layer;               // TV_QKV
  int splits;              // K splits (fixed per shape; never depends on rows)
  int counter_base;
  float* y;                // TV_STORE / TV_RESID target [kRows, N]
  uint16_t *yh, *yl;       // TV_GELU_HILO targets
  // fused LayerNorm prologue: if ln_g != nullptr the activation operand is
  // LN(ln_x) (fp32 [kRows, K]) built in shared memory instead of TMA-loaded
  const float* ln_x;
  const uint16_t *ln_g, *ln_b;
};

// Pre-encoded TMA maps of one projection: weights [N, K] and the hi/lo input.
struct TcGemvMaps {
  CUtensorMap w, xh, xl;
};

int make_tmap_2d(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer,
                 uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer);
int tc_gemv_splits(int N, int K);
size_t tc_gemv_part_floats(int N, int K);
int launch_tc_gemv(const DecodeState& st, const TcGemvMaps& maps, const TcGemvArgs& a,
                   cudaStream_t stream);
int launch_decode_ln(const DecodeState& st, const float* x, const uint16_t* g,
                     const uint16_t* b, cudaStream_t stream);
int launch_embed(const DecodeState& st, const uint16_t* embed, const uint16_t* pos_emb,
                 cudaStream_t stream);
int launch_self_attn(const DecodeState& st, const CUtensorMap& kv_map, int layer,
                     cudaStream_t stream);
int launch_cross_attn(const DecodeState& st, const CUtensorMap& xkv_map, int layer,
                      int counter_base, cudaStream_t stream);
int launch_finalize(const DecodeState& st, cudaStream_t stream);

// Persistent decode (one cooperative CTA per SM runs n_steps whole steps).
// layer_ptrs: per layer 12 pointers (ln1 g/b, qkv b, o b, ln2 g/b, xq b, xo b,
// ln3 g/b, fc1 b, fc2 b).
int mk_setup(const DecodeState& st, const std::vector<TcGemvMaps>& maps, const CUtensorMap& kv_map,
             const CUtensorMap& xkv_map, const std::vector<const uint16_t*>& layer_ptrs,
             void** handle);
void mk_free(void* handle);
int mk_launch(void* handle, const DecodeState& st, const uint16_t* lnfg, const uint16_t* lnfb,
              const uint16_t* embed, const uint16_t* pos_emb, int n_steps, cudaStream_t stream,
              unsigned long long* timing = nullptr);

}  // namespace dm
