// tcgen05 / TMEM / TMA GEMM for the encoder (K2 conv stem, K3 layer GEMMs,
// K5 cross-KV precompute). D[M, N] = A[M, K] . B[N, K]^T, bf16 inputs, fp32
// accumulation in TMEM, fused epilogues.
#pragma once

#include "common.cuh"

namespace dm {

enum EpiMode : int {
  EPI_STORE_BF16 = 0,     // out bf16 [row, n] = acc + bias
  EPI_GELU_BF16 = 1,      // out bf16 = gelu(acc + bias)
  EPI_CONV1 = 2,          // out bf16 padded [b, T+2, N] row t+1 = gelu(acc + bias)
  EPI_CONV2_POS = 3,      // out f32 [b*T+t, n] = gelu(acc + bias) + pos[t, n]
  EPI_RESID_F32 = 4,      // out f32 [row, n] += acc + bias
  EPI_QKV = 5,            // scatter q (scaled) / k to [b, h, Tp, 64], v to [b, h, 64, Tp]
  EPI_XKV = 6,            // scatter k/v of every decoder layer into slot caches
  EPI_STORE_F32 = 7,      // out f32 [row, n] = acc + bias (tests)
  EPI_W2V_PROJ = 8,       // wav2vec2 feature projection: out f32 [row, n] = acc + bias and a
                          // bf16 copy into the zero-padded grouped pos-conv operand
  EPI_W2V_POS = 9,        // wav2vec2 grouped pos-conv: x[row, ch] += gelu(acc + bias[ch])
  EPI_CTC_ARGMAX = 10,    // per-row argmax over N <= 32 logits -> int32 ids (ties: lowest)
  EPI_GELU_F32 = 11,      // out f32 [row, n] = gelu(acc + bias)
};

enum AMode : int {
  A_FLAT = 0,             // A [Bt, T, K] (row stride lda), k-block = 64 columns
  A_CONV_S1 = 1,          // conv k3 s1 over a zero-padded [Bt, T+2, C] buffer
  A_CONV_S2 = 2,          // conv k3 s2 over a zero-padded [Bt, 2T+2, C] buffer
  // Conv modes read tap `tap` of output row t from input row (stride * t + tap) of a
  // [Bt, a_rows, C] buffer (callers pre-pad it). K = taps * C. With `grouped`,
  // output tile nt (BN = 64) uses input channels [64 nt, 64 nt + 64) only.
};

struct Epilogue {
  int mode = EPI_STORE_BF16;
  const uint16_t* bias = nullptr;     // [N] bf16, nullable
  void* out = nullptr;
  int ldo = 0;                        // output row stride (elements)
  const uint16_t* pos = nullptr;      // EPI_CONV2_POS: [T, N] bf16
  // EPI_QKV
  uint16_t* q = nullptr;
  uint16_t* k = nullptr;
  uint16_t* vt = nullptr;
  int heads = 0;
  int t_pad = 0;
  float q_scale = 1.0f;
  // EPI_XKV
  const int32_t* slot_ids = nullptr;
  int n_slots = 0;
  int layers = 0;
  int seg_rows = 1500;                // EPI_QKV / EPI_XKV / W2V: rows per segment
  // wav2vec2
  const int32_t* seg_len = nullptr;   // valid rows per segment (W2V_PROJ masks the rest)
  uint16_t* grp = nullptr;            // W2V_PROJ: grouped operand [Bt][rows+128][16][64]
  int grp_pad = 64;                   // zero rows before each segment in `grp`
  int grp_cpg = 48;                   // channels per group
};

struct GemmArgs {
  const uint16_t* A = nullptr;
  int a_mode = A_FLAT;
  int K = 0;              // reduction length (A_CONV_*: 3 * C)
  int C = 0;              // A_CONV_*: channels (multiple of 64)
  int T = 0;              // output rows per batch item
  int Bt = 1;             // batch items
  int lda = 0;            // A_FLAT: row stride (elements)
  long long a_bstride = 0;// A_FLAT: batch stride (elements)
  int a_rows = 0;         // conv modes: input rows per batch item (0 -> whisper default)
  int grouped = 0;        // conv modes: grouped conv, one 64-channel group per N tile
  const uint16_t* W = nullptr;   // [N, K] bf16 (K contiguous)
  int N = 0;
  int max_ctas = 0;       // persistent grid size cap (0: one CTA per SM); SMs left to other streams
  // Live M blocks (device lists of mb = b * MT + mt): only these row blocks
  // are computed (variable-length batches skip blocks wholly past every
  // segment's end). [0]: 128-row blocks (1-SM kernel), [1]: 256-row blocks
  // (CTA pairs); null: every block.
  const int32_t* mblocks[2] = {nullptr, nullptr};
  int mblock_count[2] = {0, 0};
  Epilogue epi;
};

int launch_gemm(const GemmArgs& args, cudaStream_t stream);
bool tma_available();

}  // namespace dm
