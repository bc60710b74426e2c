// K6: batched greedy decode step kernels (Listing 1 `model.model.generate`,
// PAPER.md:57-59) over continuous-batching slots.
//
// Activations live in "row space": row i < n_active is the i-th active slot
// (slot = active[i]); persistent per-segment state (self-KV pages, cross-KV,
// position, cap, tokens) is slot-indexed. Activations that feed a projection
// are stored as a bf16 hi/lo pair (x = hi + lo exactly to ~2^-17 relative) so
// the projections run on tcgen05 with fp32 accumulation while keeping fp32
// activation precision (SURVEY.md §7 "Design rule").
//
// Step graph per decoder layer (every kernel launched with programmatic
// dependent launch; everything that does not depend on the predecessor --
// weight tiles, cross-KV blocks, LayerNorm parameters, biases -- is fetched
// before griddepcontrol.wait):
//
//   ln(+embed | +residual partials) -> qkv GEMV (K-split partials)
//   -> self-attention (reduces q/k/v partials, appends k/v to the page)
//   -> o GEMV (partials) -> ln(+residual) -> cross-q GEMV (partials)
//   -> cross-attention (reduces q; tensor-core scores / P.V per key split,
//      the 8 split results merged in split order by the last split to arrive)
//   -> cross-o GEMV (partials)
//   -> ln(+residual) -> fc1 GEMV (+GELU, hi/lo)
//   -> fc2 GEMV (partials)
//
// then ln_f(+residual) -> LM-head GEMV (per-vocab-tile argmax) -> finalize.
// K-split partial sums are reduced by the consumer in split order, so every
// reduction order depends only on K / positions, never on which or how many
// rows are active: a segment decodes bit-identically alone or in any batch.
#pragma once

#include "common.cuh"

#include <vector>

namespace dm {

constexpr int kRows = 64;          // max active slots = max MMA N
// cross-attention key splits (fixed: the merge order is part of the result):
// 4 splits of 384 keys, 2 CTAs of ~105 KB per SM (measured against 8 x 192 at
// 4 per SM: see DESIGN.md section 4)
#ifndef DM_XA_KEYS
#define DM_XA_KEYS 192
#endif
constexpr int kXaKeysPerSplit = DM_XA_KEYS;
constexpr int kXSplits = (1500 + kXaKeysPerSplit - 1) / kXaKeysPerSplit;
constexpr int kXaCtasPerSm = kXaKeysPerSplit >= 384 ? 2 : (kXaKeysPerSplit >= 192 ? 4 : 6);

struct DecodeState {
  int max_slots, d, heads, layers, ffn, vocab;
  int page_tokens;       // self-KV tokens per page (64)
  int pages_per_slot;    // page-table width (7 -> 448 positions)
  int eot;
  int prompt_len;
  int grid_rows;               // rows the step graph's per-row grids cover (>= n_active)
  const int32_t* prompt;       // [prompt_len]
  // slot bookkeeping
  const int32_t* active;       // [kRows] slot of row i (host-set before a step graph runs)
  const int32_t* n_active;     // device scalar (host-set)
  int32_t* pos;                // [S] position of the token being fed
  int32_t* cur_tok;            // [S]
  int32_t* n_gen;              // [S]
  int32_t* cap;                // [S]
  int32_t* done;               // [S]
  int32_t* out_tokens;         // [S, 448]
  const int32_t* page_table;   // [S, pages_per_slot] (host-set at admission)
  uint16_t* kv_pool;           // [pages][L][2][H][page_tokens][64] bf16
  const uint16_t* xkv;         // [L][S][2][H][1500][64] bf16
  const int32_t* enc_len;      // [S] encoder positions of the slot's segment (1500, or fewer
                               // after a length-aware encode); cross-attention keys < enc_len
  // row-space activations
  float* x;                    // [kRows, d] residual stream (fp32)
  uint16_t *xh, *xl;           // [kRows, d]   LN output, bf16 hi/lo
  uint16_t *ah, *al;           // [kRows, d]   attention output hi/lo
  uint16_t *hh, *hl;           // [kRows, ffn] fc1 output hi/lo
  // scratch
  float* part;                 // split-K partials of non-linear epilogues (last-CTA reduction)
  int32_t* counters;           // zero-initialised tile counters
  float* amax_val;             // [vocab tiles, kRows]
  int32_t* amax_idx;           // [vocab tiles, kRows]
  float* logits_dbg;           // optional [kRows, vocab]
  // optional timeline tap (debug): per kernel of the step [kTraceSlots][8] globaltimer ns:
  // min CTA entry, min / max dependency release (after griddepcontrol.wait), max exit,
  // then kernel-specific max stamps 4..7 (GEMV: operand landed, MMA done, stores issued)
  unsigned long long* trace;
  int trace_id;
};

constexpr int kTraceSlots = 512;   // timeline tap: kernels per step (32 layers x 10 + 3 fits)

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// which: 0 entry, 1 released (records min and max), 3 exit, 4..7 max stamps
__device__ __forceinline__ void trace_mark(const DecodeState& st, int which) {
  if (st.trace == nullptr) return;
  const unsigned long long t = global_ns();
  unsigned long long* p = st.trace + st.trace_id * 8;
  if (which == 0) atomicMin(p, t);
  else if (which == 1) { atomicMin(p + 1, t); atomicMax(p + 2, t); }
  else atomicMax(p + which, t);
}

// K-split partial sums of a linear projection: part[s][row][n] (fp32, no bias),
// reduced by the consumer as bias + sum_s part[s] in split order.
struct Partials {
  const float* p;
  int splits;
  int n;                       // row length N
  const uint16_t* bias;        // [N] bf16
};

enum GemvEpi : int {
  GV_PARTIAL = 0,   // part[split][r][n] = acc            (consumer reduces + adds bias)
  GV_GELU_HILO = 1, // yh/yl[r, n] = split(gelu(acc + b)) (bf16 pair)
  GV_ARGMAX = 2,    // per-row (max, lowest index) over this 128-feature vocab tile
};

struct GemvArgs {
  const uint16_t* bias;    // [N] nullable (not used by GV_PARTIAL)
  int N, K;
  int epi;
  int splits;              // K splits (fixed per shape; never depends on rows)
  int kb_per;              // 64-wide k-blocks per split
  int stages;              // weight ring depth (whole slice prefetched when it fits)
  int rgroups;             // row groups (grid z): CTA z owns rows [z * xrows / rgroups, +xrows / rgroups)
  int xrows;               // rows the activation buffer holds (multiple of 16, >= active rows)
  int gx;                  // CTAs per K split (grid x); tiles c, c + gx, ... per CTA
  int counter_base;
  float* part;             // GV_PARTIAL output [splits][kRows][N]
  uint16_t *yh, *yl;       // GV_GELU_HILO targets [kRows, N]
  // Activation source. GV_X_TMA: the hi/lo operand in global memory (TMA).
  // Steps of <= 16 rows may instead build it in shared memory from the
  // producer's raw output, saving the producer's finishing kernel:
  //   GV_X_GELU:  gelu(sum of xs_splits K-split partials xp[s][kRows][K] + xbias)
  //               (fc2 after a split fc1: what gelu_hilo_kernel computes)
  //   GV_X_XMERGE: the split-order merge of the cross-attention results xp
  //               (cross-o: what xattn_merge_kernel computes)
  // -- the same arithmetic, so every row bucket gives the same bits.
  int xsrc;
  const float* xp;
  int xs_splits;
  const uint16_t* xbias;
};
enum GemvXSrc : int { GV_X_TMA = 0, GV_X_GELU = 1, GV_X_XMERGE = 2 };

// Pre-encoded TMA maps of one projection: weights [N, K] (box 128 x 64) and the
// hi/lo activation input [kRows, K] (box 16 rows x 64, loads scale with rows).
struct TcGemvMaps {
  CUtensorMap w, xh, xl;
};

constexpr int kGvXBox = 16;

int make_tmap_2d(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer,
                 uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer);
// Plan (splits, kb_per, stages) of a projection; depends only on (N, K,
// epilogue, max_splits = the partials its consumer reduces).
GemvArgs gemv_plan(int N, int K, int epi, int max_splits = 8);
// The same plan for a step graph whose active rows are <= rows: the
// activation buffer, row groups, ring depth and grid shrink with the rows
// (two CTAs per SM when they fit); the K split -- hence every value -- stays.
GemvArgs gemv_plan_for_rows(const GemvArgs& base, int rows);
size_t gemv_part_floats(int N, int K, int epi, int max_splits = 8);   // scratch for its partial sums
int launch_gemv(const DecodeState& st, const TcGemvMaps& maps, const GemvArgs& a,
                cudaStream_t stream);

// LayerNorm of the row-space residual into the hi/lo projection operand.
// mode 0: x as is; 1: x = embed[cur_tok] + pos_emb[pos] (first layer);
// 2: x += bias + sum_s part[s] (the preceding projection's residual add).
struct LnArgs {
  int mode;
  const uint16_t *g, *b;             // LayerNorm weight / bias [d]
  const uint16_t *embed, *pos_emb;   // mode 1
  Partials res;                      // mode 2
};
int launch_ln(const DecodeState& st, const LnArgs& a, cudaStream_t stream);

// Self-attention of the fed token: q/k/v from the qkv partials (q scaled),
// k/v appended to the slot's page, keys 0..pos; output -> ah/al.
int launch_self_attn(const DecodeState& st, int layer, const Partials& qkv, float q_scale,
                     cudaStream_t stream);
// Cross-attention over the slot's 1500 cross-KV rows (q from the cross-q
// partials, scaled): per (row, head, split) tensor-core scores and P.V, the 8
// split results merged in split order by the last to arrive. xkv_map: the
// cross-KV cache as [rows, 64] bf16, box 64 x 64, 128B swizzle. xpart:
// [kRows][H][8][68] fp32 scratch, xcnt: [kRows * kMaxHeads] zero-initialised
// counters. Output: o (all heads) as the bf16 hi/lo operand st.ah / st.al of
// the cross-o GEMV. probe = 1: stream K/V and stop (roofline probe); probe = 2:
// no merge (timing probe). tail_merge = false: the splits only store their
// results and launch_xattn_merge (same arithmetic) must follow.
constexpr int kMaxHeads = 20;   // per-head scratch / partial splits a LayerNorm may reduce
constexpr int kAttnSplits = 10; // partial splits an attention kernel reduces (its q / k / v)
// Steps with at most this many active rows merge the cross-attention splits in
// the last-arriving CTA (0: never; the cross-o GEMV's operand builder does it
// for few-row steps, xattn_merge_kernel above kGvFuseRows).
constexpr int kXaTailMergeRows = 0;
// Steps with at most this many rows build the cross-o / fc2 GEMV operands in
// the GEMV (GemvArgs::xsrc) instead of running the merge / GELU kernels.
constexpr int kGvFuseRows = 8;
int launch_cross_attn(const DecodeState& st, const CUtensorMap& xkv_map, int layer,
                      const Partials& xq, float q_scale, float* xpart, int* xcnt,
                      cudaStream_t stream, int probe = 0, bool tail_merge = true);
int launch_xattn_merge(const DecodeState& st, const float* xpart, cudaStream_t stream);
// fc2's operand from fc1's K-split partials: split-order sum + bias, exact
// GELU, bf16 hi/lo (the large models' fc1 needs a K split; see record_step).
int launch_gelu_hilo(const DecodeState& st, const Partials& p, uint16_t* yh, uint16_t* yl,
                     cudaStream_t stream);
// LM head from K-split partials: split-order sum + per-tile argmax (ties ->
// lowest id) into st.amax_val / amax_idx (what the GV_ARGMAX epilogue writes).
int launch_lm_argmax(const DecodeState& st, const Partials& p, cudaStream_t stream);
int launch_finalize(const DecodeState& st, cudaStream_t stream);

}  // namespace dm
