// K8: CTC encoder-only path (BASELINE.json cfg5):
// wav2vec2-base-shaped feature encoder + 12 post-LN layers + 32-way head,
// greedy CTC (argmax per frame, collapse repeats, drop blank 0).
// Semantics restated in oracle/wav2vec2.py (transformers 5.5.0
// modeling_wav2vec2.py). Variable-length segments are batched without
// changing any segment's result: every per-segment reduction (input
// normalisation, GroupNorm over time) is masked to that segment's valid
// samples/frames, the positional conv sees zeros beyond the segment (its own
// 64-row zero pads), and attention keys are masked to the segment length.
//
//   conv0 (1->512, k10 s5) + GroupNorm + GELU : CUDA cores (K=10), recomputed
//       in a stats pass and an apply pass instead of storing fp32 activations
//   conv1..6 (k3/k2, s2)                      : tcgen05 implicit GEMM (A_CONV_S2)
//   LN + projection 512->768                  : LN kernel + GEMM (EPI_W2V_PROJ)
//   positional conv (k128, 16 groups)         : grouped tcgen05 implicit GEMM
//   12 x [QKV, FMHA, O+res, LN, fc1+GELU, fc2+res, LN] : encoder kernels
//   head 768->32 + argmax                      : GEMM epilogue (EPI_CTC_ARGMAX)
//   collapse                                   : one warp per segment (ballot)

#include <cstring>
#include <string>
#include <vector>

#include "../../include/dictamux_b200.h"
#include "common.cuh"
#include "gemm.cuh"

namespace dm {

int launch_layernorm_bf16(const float*, const uint16_t*, const uint16_t*, uint16_t*, int, int,
                          cudaStream_t, float* y32, const int32_t* seg_len = nullptr,
                          int seg_rows = 0);
int launch_attention(const uint16_t*, const uint16_t*, const uint16_t*, int, int, int, int,
                     uint16_t*, int, cudaStream_t, const int32_t* seg_len);
int make_tmap_2d(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer,
                 uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer);

constexpr int kC = 512;            // feature-encoder channels
constexpr int kNormBlocks = 64;    // input-normalisation partials per segment
constexpr int kF0 = 64;            // conv0 frames per CTA

// ------------------------------------------------------------ input stats
__global__ void ctc_norm_partials(const int16_t* __restrict__ pcm,
                                  const int64_t* __restrict__ offs,
                                  const int32_t* __restrict__ lens, double* __restrict__ part) {
  const int b = blockIdx.y, blk = blockIdx.x;
  const int n = lens[b];
  const int16_t* x = pcm + offs[b];
  double s = 0.0, q = 0.0;
  for (int i = blk * blockDim.x + threadIdx.x; i < n; i += kNormBlocks * blockDim.x) {
    const double v = double(float(x[i]) * (1.0f / 32768.0f));
    s += v;
    q += v * v;
  }
  __shared__ double rs[256], rq[256];
  rs[threadIdx.x] = s;
  rq[threadIdx.x] = q;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      rs[threadIdx.x] += rs[threadIdx.x + o];
      rq[threadIdx.x] += rq[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[(b * kNormBlocks + blk) * 2] = rs[0];
    part[(b * kNormBlocks + blk) * 2 + 1] = rq[0];
  }
}

__device__ __forceinline__ void norm_stats(const double* part, int b, int n, float& mean,
                                           float& rstd) {
  double s = 0.0, q = 0.0;
  for (int i = 0; i < kNormBlocks; ++i) {
    s += part[(b * kNormBlocks + i) * 2];
    q += part[(b * kNormBlocks + i) * 2 + 1];
  }
  const double m = n > 0 ? s / n : 0.0;
  const double var = n > 0 ? q / n - m * m : 0.0;
  mean = float(m);
  rstd = float(1.0 / sqrt((var > 0 ? var : 0.0) + 1e-7));
}

// ------------------------------------------------------------ conv0 (+ GroupNorm + GELU)
constexpr int kGramBlocks = 16;   // Gram partials per segment
constexpr int kGram = 65;         // 10 tap sums + 55 upper-triangle tap products

// GroupNorm (512 groups = channels) statistics of conv0 without running the
// convolution: for channel c, sum_t y_c(t) = w_c . A and sum_t y_c(t)^2 =
// w_c^T G w_c with A_k = sum_t x(5t + k), G_kj = sum_t x(5t + k) x(5t + j) over
// the segment's frames (x = the normalised input exactly as conv0 forms it):
// 65 double sums per segment instead of a second pass of 512-channel
// convolutions. Fixed-order reductions throughout.
__global__ void __launch_bounds__(256)
ctc_gram_partials(const int16_t* __restrict__ pcm, const int64_t* __restrict__ offs,
                  const int32_t* __restrict__ lens, const double* __restrict__ npart,
                  double* __restrict__ gram_part) {
  const int b = blockIdx.y, blk = blockIdx.x;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int n = lens[b];
  const int T0 = n >= 10 ? (n - 10) / 5 + 1 : 0;
  float mean, rstd;
  norm_stats(npart, b, n, mean, rstd);
  const int16_t* x = pcm + offs[b];
  double acc[kGram];
#pragma unroll
  for (int i = 0; i < kGram; ++i) acc[i] = 0.0;
  for (int t = blk * blockDim.x + threadIdx.x; t < T0; t += kGramBlocks * blockDim.x) {
    float xv[10];
#pragma unroll
    for (int k = 0; k < 10; ++k) {
      const int j = 5 * t + k;
      xv[k] = j < n ? (float(x[j]) * (1.0f / 32768.0f) - mean) * rstd : 0.f;
    }
    int idx = 10;
#pragma unroll
    for (int k = 0; k < 10; ++k) {
      acc[k] += double(xv[k]);
#pragma unroll
      for (int j = k; j < 10; ++j) acc[idx++] += double(xv[k]) * double(xv[j]);
    }
  }
  __shared__ double red[8][kGram];
#pragma unroll
  for (int i = 0; i < kGram; ++i) {
    double v = acc[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[warp][i] = v;
  }
  __syncthreads();
  if (threadIdx.x < kGram) {
    double v = 0.0;
    for (int w = 0; w < int(blockDim.x) / 32; ++w) v += red[w][threadIdx.x];
    gram_part[(size_t(b) * kGramBlocks + blk) * kGram + threadIdx.x] = v;
  }
}

// Per (segment, channel) mean / rstd of conv0's output from the Gram sums.
__global__ void __launch_bounds__(kC)
ctc_gn_finalize(const double* __restrict__ gram_part, const uint16_t* __restrict__ w0,
                const int32_t* __restrict__ lens, float* __restrict__ gstat) {
  const int b = blockIdx.x, c = threadIdx.x;
  __shared__ double g[kGram];
  if (c < kGram) {
    double v = 0.0;
    for (int i = 0; i < kGramBlocks; ++i) v += gram_part[(size_t(b) * kGramBlocks + i) * kGram + c];
    g[c] = v;
  }
  __syncthreads();
  const int n = lens[b];
  const int T0 = n >= 10 ? (n - 10) / 5 + 1 : 0;
  double w[10];
#pragma unroll
  for (int k = 0; k < 10; ++k) w[k] = double(bf16_to_f32(w0[c * 10 + k]));
  double s = 0.0, q = 0.0;
  int idx = 10;
#pragma unroll
  for (int k = 0; k < 10; ++k) {
    s += w[k] * g[k];
#pragma unroll
    for (int j = k; j < 10; ++j, ++idx) q += (j == k ? 1.0 : 2.0) * w[k] * w[j] * g[idx];
  }
  const double m = T0 > 0 ? s / T0 : 0.0;
  double var = T0 > 0 ? q / T0 - m * m : 0.0;
  var = var > 0 ? var : 0.0;
  gstat[(b * kC + c) * 2] = float(m);
  gstat[(b * kC + c) * 2 + 1] = float(1.0 / sqrt(var + 1e-5));
}

// conv0 -> GroupNorm -> GELU -> the bf16 conv1 operand. Frames past the
// segment (the batch is padded to its longest) get zero rows and no work.
__global__ void __launch_bounds__(256)
ctc_conv0_kernel(const int16_t* __restrict__ pcm, const int64_t* __restrict__ offs,
                 const int32_t* __restrict__ lens, const double* __restrict__ npart,
                 const uint16_t* __restrict__ w0 /*[512][10]*/,
                 const float* __restrict__ gstat /*[B][512][2] mean, rstd*/,
                 const uint16_t* __restrict__ gn_g, const uint16_t* __restrict__ gn_b,
                 uint16_t* __restrict__ out, int R0) {
  __shared__ float xs[kF0 * 5 + 8];
  __shared__ float ws[kC * 10];
  const int b = blockIdx.y, f0 = blockIdx.x * kF0;
  const int n = lens[b];
  const int T0 = n >= 10 ? (n - 10) / 5 + 1 : 0;
  if (f0 >= T0) {
    const int nf = min(kF0, R0 - f0);
    uint32_t* o32 = reinterpret_cast<uint32_t*>(out + (size_t(b) * R0 + f0) * kC);
    for (int i = threadIdx.x; i < nf * kC / 2; i += blockDim.x) o32[i] = 0u;
    return;
  }
  const int nvalid = min(kF0, T0 - f0);        // frames of this CTA inside the segment
  float mean, rstd;
  norm_stats(npart, b, n, mean, rstd);
  const int16_t* x = pcm + offs[b];
  for (int i = threadIdx.x; i < kF0 * 5 + 5; i += blockDim.x) {
    const int j = f0 * 5 + i;
    xs[i] = j < n ? (float(x[j]) * (1.0f / 32768.0f) - mean) * rstd : 0.f;
  }
  for (int i = threadIdx.x; i < kC * 10; i += blockDim.x) ws[i] = bf16_to_f32(w0[i]);
  __syncthreads();
  // both of this thread's channels (c, c + 256) per frame, two frames per
  // step from one 15-sample window: each shared-memory sample read feeds 4
  // convolution taps
  const int c0 = threadIdx.x, c1 = threadIdx.x + 256;
  float wa[10], wb[10];
#pragma unroll
  for (int k = 0; k < 10; ++k) {
    wa[k] = ws[c0 * 10 + k];
    wb[k] = ws[c1 * 10 + k];
  }
  const float ma = gstat[(b * kC + c0) * 2], ra = gstat[(b * kC + c0) * 2 + 1];
  const float ga = bf16_to_f32(gn_g[c0]), ba = bf16_to_f32(gn_b[c0]);
  const float mb = gstat[(b * kC + c1) * 2], rb = gstat[(b * kC + c1) * 2 + 1];
  const float gb2 = bf16_to_f32(gn_g[c1]), bb = bf16_to_f32(gn_b[c1]);
  static_assert(kF0 % 2 == 0 && (kF0 - 2) * 5 + 14 < kF0 * 5 + 5, "conv0 window");
#pragma unroll 1
  for (int f = 0; f < kF0; f += 2) {
    float xw[15];
#pragma unroll
    for (int k = 0; k < 15; ++k) xw[k] = xs[f * 5 + k];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int ff = f + h, t = f0 + ff;
      if (t >= R0) continue;
      if (ff >= nvalid) {                      // past the segment: zero rows
        out[(size_t(b) * R0 + t) * kC + c0] = 0;
        out[(size_t(b) * R0 + t) * kC + c1] = 0;
        continue;
      }
      float ya = 0.f, yb = 0.f;
#pragma unroll
      for (int k = 0; k < 10; ++k) {
        ya = fmaf(wa[k], xw[5 * h + k], ya);
        yb = fmaf(wb[k], xw[5 * h + k], yb);
      }
      out[(size_t(b) * R0 + t) * kC + c0] = f32_to_bf16(gelu_erf((ya - ma) * ra * ga + ba));
      out[(size_t(b) * R0 + t) * kC + c1] = f32_to_bf16(gelu_erf((yb - mb) * rb * gb2 + bb));
    }
  }
}

// ------------------------------------------------------------ CTC collapse
// One warp per segment: keep frame t if id != blank and id != id[t-1].
__global__ void ctc_collapse_kernel(const int32_t* __restrict__ ids, const int32_t* __restrict__ tlen,
                                    int R, int blank, int32_t* __restrict__ tokens,
                                    int32_t* __restrict__ counts) {
  const int b = blockIdx.x, lane = threadIdx.x;
  const int T = tlen[b];
  const int32_t* row = ids + size_t(b) * R;
  int base = 0;
  for (int t0 = 0; t0 < T; t0 += 32) {
    const int t = t0 + lane;
    int keep = 0, id = 0;
    if (t < T) {
      id = row[t];
      keep = id != blank && (t == 0 || id != row[t - 1]);
    }
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    if (keep) tokens[size_t(b) * R + base + __popc(m & ((1u << lane) - 1))] = id;
    base += __popc(m);
  }
  if (lane == 0) counts[b] = base;
}

// ------------------------------------------------------------ weight repack
// pos.w [g][out cg][tap][in cg] -> [g*64 + o][tap*64 + i] with zero padding.
__global__ void repack_posconv_kernel(const uint16_t* __restrict__ w, uint16_t* __restrict__ out,
                                      int groups, int cg, int taps) {
  const size_t total = size_t(groups) * 64 * taps * 64;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < total;
       i += size_t(gridDim.x) * blockDim.x) {
    const int ci = int(i % 64);
    const int tap = int((i / 64) % taps);
    const int row = int(i / (size_t(64) * taps));
    const int g = row / 64, o = row % 64;
    out[i] = (o < cg && ci < cg) ? w[((size_t(g) * cg + o) * taps + tap) * cg + ci] : uint16_t(0);
  }
}

// ============================================================ engine
struct CtcEngine {
  int device = 0;
  dm_ctc_config cfg;
  const uint16_t* w = nullptr;
  std::vector<int64_t> off;
  const uint16_t* W(int i) const { return w + off[i]; }
  // offsets: 0..6 conv w, 7 gn.g, 8 gn.b, 9 fp.ln.g, 10 fp.ln.b, 11 proj.w, 12 proj.b,
  //          13 pos.w, 14 pos.b, 15 enc.ln.g, 16 enc.ln.b, 17 + 12 l + {qkv.w, qkv.b, o.w, o.b,
  //          ln1.g, ln1.b, fc1.w, fc1.b, fc2.w, fc2.b, ln2.g, ln2.b}, then head.w, head.b
  int layer(int l, int j) const { return 17 + 12 * l + j; }
  int head() const { return 17 + 12 * cfg.layers; }
  uint16_t* posw = nullptr;       // repacked [1024, 128*64]
  // workspace
  int64_t* offs_dev = nullptr;
  int32_t* lens_dev = nullptr;    // [B] samples
  int32_t* tlen_dev = nullptr;    // [B] output frames
  double* npart = nullptr;
  double* gram_part = nullptr;   // [B][kGramBlocks][65] conv0 GroupNorm Gram partials
  float* gstat = nullptr;
  uint16_t *act_a = nullptr, *act_b = nullptr;   // conv ping-pong [B, R, 512]
  float* f32buf = nullptr;        // conv6 out / hidden x [B*R6, 768] fp32
  uint16_t* lnb = nullptr;        // [B*R6, 768] bf16 (also 512-wide LN out)
  uint16_t* grp = nullptr;        // [B][R6+128][1024] bf16
  uint16_t *q = nullptr, *k = nullptr, *vt = nullptr;
  uint16_t* attn = nullptr;
  uint16_t* h1 = nullptr;
  int32_t* ids = nullptr;
  int32_t* tokens = nullptr;
  int32_t* counts = nullptr;
  int64_t* host_stage = nullptr;  // pinned
  // live GEMM row-block lists of the current batch (GemmArgs::mblocks)
  static constexpr size_t kMbCap = 1 << 18;
  int32_t* mb_host = nullptr;     // pinned
  int32_t* mb_dev = nullptr;
  std::vector<void*> allocs;
  int last_n = 0, last_R6 = 0;
  std::vector<int> last_tlen;
  size_t max_frames0 = 0, max_R1 = 0, max_R6 = 0, max_tpad = 0;

  int alloc(void** p, size_t bytes) {
    DM_CHECK_CUDA(cudaMalloc(p, bytes));
    allocs.push_back(*p);
    DM_CHECK_CUDA(cudaMemset(*p, 0, bytes));
    return 0;
  }
  template <class T>
  int alloc_t(T** p, size_t n) { return alloc(reinterpret_cast<void**>(p), n * sizeof(T)); }
  ~CtcEngine() {
    for (void* p : allocs) cudaFree(p);
    if (host_stage) cudaFreeHost(host_stage);
    if (mb_host) cudaFreeHost(mb_host);
  }
};

static int conv_out(int L, int k, int s) { return L >= k ? (L - k) / s + 1 : 0; }
static int even_up(int x) { return (x + 1) & ~1; }

static int ctc_init(CtcEngine* e) {
  const dm_ctc_config& c = e->cfg;
  DM_REQUIRE(c.hidden == 768 && c.heads == 12 && c.ffn == 3072 && c.vocab <= 32,
             "CTC engine supports the wav2vec2-base shape (768/12/3072, vocab <= 32)");
  DM_REQUIRE(c.max_batch >= 1 && c.max_samples >= 400, "bad max_batch / max_samples");
  const int B = c.max_batch;
  const int T0 = conv_out(c.max_samples, 10, 5);
  int T = T0;
  e->max_frames0 = T0;
  const size_t R0 = even_up(T0) + 2;
  e->max_R1 = even_up(conv_out(T0, 3, 2)) + 2;
  const int ks[6] = {3, 3, 3, 3, 2, 2};
  for (int i = 0; i < 6; ++i) T = conv_out(T, ks[i], 2);
  e->max_R6 = even_up(T) + 2;
  e->max_tpad = ((e->max_R6 + 127) / 128) * 128;
  if (e->alloc_t(&e->posw, size_t(1024) * 128 * 64)) return 2;
  repack_posconv_kernel<<<1184, 256>>>(e->W(13), e->posw, 16, 48, 128);
  DM_CHECK_LAUNCH();
  if (e->alloc_t(&e->offs_dev, B)) return 2;
  if (e->alloc_t(&e->lens_dev, B)) return 2;
  if (e->alloc_t(&e->tlen_dev, B)) return 2;
  if (e->alloc_t(&e->npart, size_t(B) * kNormBlocks * 2)) return 2;
  if (e->alloc_t(&e->gram_part, size_t(B) * kGramBlocks * kGram)) return 2;
  if (e->alloc_t(&e->gstat, size_t(B) * kC * 2)) return 2;
  if (e->alloc_t(&e->act_a, size_t(B) * R0 * kC)) return 2;
  if (e->alloc_t(&e->act_b, size_t(B) * e->max_R1 * kC)) return 2;
  const size_t rows = size_t(B) * e->max_R6;
  if (e->alloc_t(&e->f32buf, rows * 768)) return 2;
  if (e->alloc_t(&e->lnb, rows * 768)) return 2;
  if (e->alloc_t(&e->grp, size_t(B) * (e->max_R6 + 128) * 1024)) return 2;
  if (e->alloc_t(&e->q, size_t(B) * 12 * e->max_tpad * 64)) return 2;
  if (e->alloc_t(&e->k, size_t(B) * 12 * e->max_tpad * 64)) return 2;
  if (e->alloc_t(&e->vt, size_t(B) * 12 * 64 * e->max_tpad)) return 2;
  if (e->alloc_t(&e->attn, rows * 768)) return 2;
  if (e->alloc_t(&e->h1, rows * 3072)) return 2;
  if (e->alloc_t(&e->ids, rows)) return 2;
  if (e->alloc_t(&e->tokens, rows)) return 2;
  if (e->alloc_t(&e->counts, B)) return 2;
  DM_CHECK_CUDA(cudaMallocHost(&e->host_stage, sizeof(int64_t) * 4 * B));
  DM_CHECK_CUDA(cudaMallocHost(&e->mb_host, sizeof(int32_t) * CtcEngine::kMbCap));
  if (e->alloc_t(&e->mb_dev, CtcEngine::kMbCap)) return 2;
  DM_CHECK_CUDA(cudaDeviceSynchronize());
  return 0;
}

static int ctc_forward(CtcEngine* e, const int16_t* pcm, int n, const std::vector<int>& lens,
                       cudaStream_t s) {
  const int ks[7] = {10, 3, 3, 3, 3, 2, 2};
  // frame counts per layer (max over the batch), row strides even
  std::vector<int> Tl(7, 0);
  std::vector<int> tlen(n);
  for (int b = 0; b < n; ++b) {
    int T = lens[b];
    for (int i = 0; i < 7; ++i) T = conv_out(T, ks[i], i == 0 ? 5 : 2);
    tlen[b] = T;
  }
  int T0max = 0;
  for (int b = 0; b < n; ++b) T0max = std::max(T0max, conv_out(lens[b], 10, 5));
  std::vector<int> R(7);
  R[0] = even_up(T0max) + 2;
  int Tm = T0max;
  for (int i = 1; i < 7; ++i) {
    Tm = conv_out(Tm, ks[i], 2);
    R[i] = even_up(std::max(Tm, 1)) + 2;
  }
  const int R6 = R[6];
  const int tpad = ((R6 + 127) / 128) * 128;
  DM_REQUIRE(size_t(R6) <= e->max_R6 && size_t(tpad) <= e->max_tpad, "segment longer than max_samples");
  // upload tlen
  int32_t* hs = reinterpret_cast<int32_t*>(e->host_stage);
  for (int b = 0; b < n; ++b) hs[b] = tlen[b];
  DM_CHECK_CUDA(cudaMemcpyAsync(e->tlen_dev, hs, sizeof(int32_t) * n, cudaMemcpyHostToDevice, s));
  // Live row blocks: the batch is padded to its longest segment, and a row
  // block wholly past every segment's end in it is never computed (its rows
  // feed only other padding rows: the stride-2 convs read rows < 2T + k - 1,
  // the projection zeroes rows >= T, attention masks keys >= T, the collapse
  // reads frames < T). Per conv layer i: rows t < T_i[b] of item b; the flat
  // transformer rows b * R6 + t are live for t < T_6[b].
  std::vector<std::vector<int>> Ti(7, std::vector<int>(n));
  for (int b = 0; b < n; ++b) {
    int T = lens[b];
    for (int i = 0; i < 7; ++i) Ti[i][b] = T = conv_out(T, ks[i], i == 0 ? 5 : 2);
  }
  size_t mb_used = 0;
  auto add_list = [&](GemmArgs& g, int k, const std::vector<int>& live_mb) -> int {
    DM_REQUIRE(mb_used + live_mb.size() <= CtcEngine::kMbCap, "CTC live-block list overflow");
    std::copy(live_mb.begin(), live_mb.end(), e->mb_host + mb_used);
    g.mblocks[k] = e->mb_dev + mb_used;
    g.mblock_count[k] = int(live_mb.size());
    mb_used += live_mb.size();
    return 0;
  };
  // per-item blocks (conv modes): mb = b * MT + mt, mt * BM < valid[b]
  auto per_item = [&](int T, int BM, const std::vector<int>& valid) {
    std::vector<int> v;
    const int MT = ceil_div(T, BM);
    for (int b = 0; b < n; ++b)
      for (int mt = 0; mt < MT && mt * BM < valid[b]; ++mt) v.push_back(b * MT + mt);
    return v;
  };
  // flat rows b * R6 + t: block mt live if any of its rows has t < T6[b]
  auto flat_rows = [&](int BM) {
    std::vector<int> v;
    const int M = n * R6, MT = ceil_div(M, BM);
    for (int mt = 0; mt < MT; ++mt) {
      const int r0 = mt * BM, r1 = std::min(M, r0 + BM) - 1;
      bool live = r0 % R6 < Ti[6][r0 / R6];
      for (int b = r0 / R6 + 1; !live && b <= r1 / R6; ++b) live = Ti[6][b] > 0;
      if (live) v.push_back(mt);
    }
    return v;
  };
  GemmArgs conv_g[7], flat_g, pos_g;
  for (int i = 1; i < 7; ++i) {
    if (add_list(conv_g[i], 0, per_item(R[i], 128, Ti[i]))) return 2;
    if (add_list(conv_g[i], 1, per_item(R[i], 256, Ti[i]))) return 2;
  }
  if (add_list(flat_g, 0, flat_rows(128))) return 2;
  if (add_list(flat_g, 1, flat_rows(256))) return 2;
  if (add_list(pos_g, 0, per_item(R6, 128, Ti[6]))) return 2;
  if (add_list(pos_g, 1, per_item(R6, 256, Ti[6]))) return 2;
  DM_CHECK_CUDA(cudaMemcpyAsync(e->mb_dev, e->mb_host, sizeof(int32_t) * mb_used,
                                cudaMemcpyHostToDevice, s));
  auto live = [](GemmArgs& g, const GemmArgs& lists) {
    for (int k = 0; k < 2; ++k) {
      g.mblocks[k] = lists.mblocks[k];
      g.mblock_count[k] = lists.mblock_count[k];
    }
  };
  // input normalisation stats, conv0 stats, GroupNorm stats, conv0 apply
  ctc_norm_partials<<<dim3(kNormBlocks, n), 256, 0, s>>>(pcm, e->offs_dev, e->lens_dev, e->npart);
  DM_CHECK_LAUNCH();
  const int nblk = ceil_div(std::max(R[0], 1), kF0);
  ctc_gram_partials<<<dim3(kGramBlocks, n), 256, 0, s>>>(pcm, e->offs_dev, e->lens_dev, e->npart,
                                                         e->gram_part);
  DM_CHECK_LAUNCH();
  ctc_gn_finalize<<<n, kC, 0, s>>>(e->gram_part, e->W(0), e->lens_dev, e->gstat);
  DM_CHECK_LAUNCH();
  ctc_conv0_kernel<<<dim3(nblk, n), 256, 0, s>>>(pcm, e->offs_dev, e->lens_dev, e->npart, e->W(0),
                                                 e->gstat, e->W(7), e->W(8), e->act_a, R[0]);
  DM_CHECK_LAUNCH();
  // conv1..6: stride-2 implicit GEMMs, GELU (conv6 -> fp32 for the projection LN)
  uint16_t* src = e->act_a;
  uint16_t* dst = e->act_b;
  for (int i = 1; i < 7; ++i) {
    GemmArgs g;
    live(g, conv_g[i]);
    g.A = src; g.a_mode = A_CONV_S2; g.C = kC; g.K = ks[i] * kC; g.T = R[i]; g.Bt = n;
    g.a_rows = R[i - 1]; g.W = e->W(i); g.N = kC;
    if (i < 6) {
      g.epi.mode = EPI_GELU_BF16; g.epi.out = dst; g.epi.ldo = kC;
    } else {
      g.epi.mode = EPI_GELU_F32; g.epi.out = e->f32buf; g.epi.ldo = kC;
    }
    if (int rc = launch_gemm(g, s)) return rc;
    std::swap(src, dst);
  }
  const int M = n * R6;
  // feature projection: LN(512) -> Linear(512 -> 768); fp32 h + zero-padded grouped copy
  if (int rc = launch_layernorm_bf16(e->f32buf, e->W(9), e->W(10), e->lnb, M, kC, s, nullptr,
                                     e->tlen_dev, R6))
    return rc;
  DM_CHECK_CUDA(cudaMemsetAsync(e->grp, 0, size_t(n) * (R6 + 128) * 1024 * 2, s));
  float* x = e->f32buf;                            // hidden states [M, 768] fp32
  {
    GemmArgs g;
    live(g, flat_g);
    g.A = e->lnb; g.a_mode = A_FLAT; g.K = kC; g.T = M; g.Bt = 1; g.lda = kC;
    g.W = e->W(11); g.N = 768;
    g.epi.mode = EPI_W2V_PROJ; g.epi.bias = e->W(12); g.epi.out = x; g.epi.ldo = 768;
    g.epi.seg_rows = R6; g.epi.seg_len = e->tlen_dev; g.epi.grp = e->grp;
    g.epi.grp_pad = 64; g.epi.grp_cpg = 48;
    if (int rc = launch_gemm(g, s)) return rc;
  }
  // positional conv (grouped, k128) + GELU added into x
  {
    GemmArgs g;
    live(g, pos_g);
    g.A = e->grp; g.a_mode = A_CONV_S1; g.grouped = 1; g.C = 1024; g.K = 128 * 64; g.T = R6;
    g.Bt = n; g.a_rows = R6 + 128; g.W = e->posw; g.N = 1024;
    g.epi.mode = EPI_W2V_POS; g.epi.bias = nullptr; g.epi.pos = e->W(14); g.epi.out = x;
    g.epi.ldo = 768; g.epi.grp_cpg = 48;
    if (int rc = launch_gemm(g, s)) return rc;
  }
  if (int rc = launch_layernorm_bf16(x, e->W(15), e->W(16), e->lnb, M, 768, s, x, e->tlen_dev, R6))
    return rc;
  auto flat = [&](const uint16_t* A, int K, const uint16_t* Wt, int N) {
    GemmArgs g;
    live(g, flat_g);
    g.A = A; g.a_mode = A_FLAT; g.K = K; g.T = M; g.Bt = 1; g.lda = K; g.W = Wt; g.N = N;
    return g;
  };
  for (int l = 0; l < e->cfg.layers; ++l) {
    {
      GemmArgs g = flat(e->lnb, 768, e->W(e->layer(l, 0)), 3 * 768);
      g.epi.mode = EPI_QKV; g.epi.bias = e->W(e->layer(l, 1));
      g.epi.q = e->q; g.epi.k = e->k; g.epi.vt = e->vt; g.epi.heads = 12; g.epi.t_pad = tpad;
      g.epi.q_scale = 0.125f; g.epi.seg_rows = R6;
      if (int rc = launch_gemm(g, s)) return rc;
    }
    if (int rc = launch_attention(e->q, e->k, e->vt, n, 12, R6, tpad, e->attn, 768, s, e->tlen_dev))
      return rc;
    {
      GemmArgs g = flat(e->attn, 768, e->W(e->layer(l, 2)), 768);
      g.epi.mode = EPI_RESID_F32; g.epi.bias = e->W(e->layer(l, 3)); g.epi.out = x; g.epi.ldo = 768;
      if (int rc = launch_gemm(g, s)) return rc;
    }
    if (int rc = launch_layernorm_bf16(x, e->W(e->layer(l, 4)), e->W(e->layer(l, 5)), e->lnb, M,
                                       768, s, x, e->tlen_dev, R6))
      return rc;
    {
      GemmArgs g = flat(e->lnb, 768, e->W(e->layer(l, 6)), 3072);
      g.epi.mode = EPI_GELU_BF16; g.epi.bias = e->W(e->layer(l, 7)); g.epi.out = e->h1;
      g.epi.ldo = 3072;
      if (int rc = launch_gemm(g, s)) return rc;
    }
    {
      GemmArgs g = flat(e->h1, 3072, e->W(e->layer(l, 8)), 768);
      g.epi.mode = EPI_RESID_F32; g.epi.bias = e->W(e->layer(l, 9)); g.epi.out = x; g.epi.ldo = 768;
      if (int rc = launch_gemm(g, s)) return rc;
    }
    if (int rc = launch_layernorm_bf16(x, e->W(e->layer(l, 10)), e->W(e->layer(l, 11)), e->lnb,
                                       M, 768, s, x, e->tlen_dev, R6))
      return rc;
  }
  {
    GemmArgs g = flat(e->lnb, 768, e->W(e->head()), 32);
    g.epi.mode = EPI_CTC_ARGMAX; g.epi.bias = e->W(e->head() + 1); g.epi.out = e->ids;
    if (int rc = launch_gemm(g, s)) return rc;
  }
  ctc_collapse_kernel<<<n, 32, 0, s>>>(e->ids, e->tlen_dev, R6, 0, e->tokens, e->counts);
  DM_CHECK_LAUNCH();
  e->last_n = n;
  e->last_R6 = R6;
  e->last_tlen = tlen;
  return 0;
}

}  // namespace dm

using namespace dm;

extern "C" {

int dm_ctc_create(const dm_ctc_config* cfg, const uint16_t* weights, const int64_t* offsets,
                  int n_offsets, void** handle) {
  DM_REQUIRE(cfg && weights && offsets && handle, "null argument");
  DM_REQUIRE(n_offsets == 17 + 12 * cfg->layers + 2, "CTC offset table has the wrong length");
  auto* e = new CtcEngine();
  if (cudaGetDevice(&e->device) != cudaSuccess) {
    delete e;
    DM_CHECK_CUDA(cudaGetLastError());
  }
  e->cfg = *cfg;
  e->w = weights;
  e->off.assign(offsets, offsets + n_offsets);
  if (int rc = ctc_init(e)) {
    delete e;
    return rc;
  }
  *handle = e;
  return 0;
}

int dm_ctc_destroy(void* handle) {
  if (!handle) return 0;
  DM_ON_DEVICE(static_cast<CtcEngine*>(handle)->device);
  delete static_cast<CtcEngine*>(handle);
  return 0;
}

int dm_ctc_transcribe(void* handle, const int16_t* pcm, const int64_t* offsets,
                      const int32_t* lengths, int n, void* stream) {
  auto* e = static_cast<CtcEngine*>(handle);
  DM_REQUIRE(e != nullptr, "null handle");
  DM_ON_DEVICE(e->device);
  DM_REQUIRE(n >= 1 && n <= e->cfg.max_batch, "n must be in [1, max_batch]");
  std::vector<int> lens(n);
  for (int i = 0; i < n; ++i) {
    DM_REQUIRE(lengths[i] >= 0 && lengths[i] <= e->cfg.max_samples, "segment length out of range");
    lens[i] = lengths[i];
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  DM_CHECK_CUDA(cudaStreamSynchronize(s));            // host staging reuse
  std::memcpy(e->host_stage, offsets, sizeof(int64_t) * n);
  int32_t* hl = reinterpret_cast<int32_t*>(e->host_stage + n);
  std::memcpy(hl, lengths, sizeof(int32_t) * n);
  DM_CHECK_CUDA(cudaMemcpyAsync(e->offs_dev, e->host_stage, sizeof(int64_t) * n,
                                cudaMemcpyHostToDevice, s));
  DM_CHECK_CUDA(cudaMemcpyAsync(e->lens_dev, hl, sizeof(int32_t) * n, cudaMemcpyHostToDevice, s));
  DM_CHECK_CUDA(cudaStreamSynchronize(s));
  return ctc_forward(e, pcm, n, lens, s);
}

int dm_ctc_read(void* handle, int32_t* tokens, int32_t* counts, int32_t* rows_per_segment,
                void* stream) {
  auto* e = static_cast<CtcEngine*>(handle);
  DM_REQUIRE(e != nullptr, "null handle");
  DM_ON_DEVICE(e->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (rows_per_segment) *rows_per_segment = e->last_R6;
  if (counts)
    DM_CHECK_CUDA(cudaMemcpyAsync(counts, e->counts, sizeof(int32_t) * e->last_n,
                                  cudaMemcpyDeviceToHost, s));
  if (tokens)
    DM_CHECK_CUDA(cudaMemcpyAsync(tokens, e->tokens, sizeof(int32_t) * e->last_n * e->last_R6,
                                  cudaMemcpyDeviceToHost, s));
  DM_CHECK_CUDA(cudaStreamSynchronize(s));
  return 0;
}

int dm_ctc_debug(void* handle, int which, void* host_dst, size_t bytes, void* stream) {
  auto* e = static_cast<CtcEngine*>(handle);
  DM_REQUIRE(e != nullptr, "null handle");
  DM_ON_DEVICE(e->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const void* src = nullptr;
  size_t avail = 0;
  const size_t rows = size_t(e->last_n) * e->last_R6;
  switch (which) {
    case 0: src = e->ids; avail = rows * 4; break;           // per-frame argmax ids
    case 1: src = e->f32buf; avail = rows * 768 * 4; break;  // final hidden (post-LN) fp32
    default: DM_REQUIRE(false, "unknown debug tap");
  }
  DM_REQUIRE(bytes <= avail, "debug copy larger than the tapped buffer");
  DM_CHECK_CUDA(cudaMemcpyAsync(host_dst, src, bytes, cudaMemcpyDeviceToHost, s));
  DM_CHECK_CUDA(cudaStreamSynchronize(s));
  return 0;
}

}  // extern "C"
