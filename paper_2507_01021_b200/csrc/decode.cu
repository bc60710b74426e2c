// K6 decode-step kernels. Activations stay fp32 (bf16 weights widened in
// registers) — the precision rule that keeps greedy tokens identical to the
// fp32 oracle (SURVEY.md §7 "Design rule"). Every per-slot reduction has a
// fixed order that depends only on K / positions, never on how many slots are
// active, so a segment decodes bit-identically alone or in any batch.
//
// The per-step work is HBM-bound: weights are read once per step for the
// whole batch, cross-KV (the dominant stream) once per
// active slot.

#include "decode.cuh"

namespace dm {

constexpr int kGvThreads = 256;
constexpr int kGvTileN = 64;
constexpr int kGvKC = 64;
constexpr int kGvMaxRows = 64;

// ------------------------------------------------------------ GEMV
// CTA: 64 output features x all active rows, one K split. Thread (rg, fg):
// rows 4rg..4rg+3 of the active list, features 4fg..4fg+3. X chunk staged
// transposed in smem ([k][row]); W streamed from global through L1 as
// 16-byte vectors of 8 bf16.
__device__ __forceinline__ void gemv_epilogue(const DecodeState& st, const GemvArgs& a,
                                              int slot, int n, float v) {
  if (a.bias) v += bf16_to_f32(a.bias[n]);
  switch (a.epi) {
    case GV_STORE: a.Y[size_t(slot) * a.N + n] = v; break;
    case GV_GELU: a.Y[size_t(slot) * a.N + n] = gelu_erf(v); break;
    case GV_RESID: a.Y[size_t(slot) * a.N + n] += v; break;
    case GV_SCALE: a.Y[size_t(slot) * a.N + n] = v * a.scale; break;
    case GV_QKV: {
      const int d = st.d;
      if (n < d) {
        st.q[size_t(slot) * d + n] = v * a.scale;
      } else {
        const int kv = n < 2 * d ? 0 : 1;
        const int c = n - (kv + 1) * d;
        const int h = c / 64, j = c % 64;
        const int p = st.pos[slot];
        const int page = st.page_table[slot * st.pages_per_slot + p / st.page_tokens];
        size_t idx = ((((size_t(page) * st.layers + a.layer) * 2 + kv) * st.heads + h) *
                          st.page_tokens + (p % st.page_tokens)) * 64 + j;
        st.kv_pool[idx] = f32_to_bf16(v);
      }
      break;
    }
  }
}

__global__ void __launch_bounds__(kGvThreads)
gemv_kernel(const DecodeState st, const GemvArgs a) {
  __shared__ __align__(16) float xs[kGvKC][kGvMaxRows];
  __shared__ int slots[kGvMaxRows];
  __shared__ int is_last;
  const int R = min(*st.n_active, kGvMaxRows);
  const int tid = threadIdx.x;
  const int rg = tid / 16, fg = tid % 16;
  const int n0 = blockIdx.x * kGvTileN;
  const int ks = a.K / a.splits;                  // K per split (multiple of 64)
  const int k_begin = blockIdx.y * ks;
  if (tid < kGvMaxRows) slots[tid] = tid < R ? st.active[tid] : 0;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  const bool rows_live = 4 * rg < R;
  const uint16_t* wrow[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    int n = min(n0 + 4 * fg + j, a.N - 1);
    wrow[j] = a.W + size_t(n) * a.K;
  }
  __syncthreads();
  for (int kc = k_begin; kc < k_begin + ks; kc += kGvKC) {
    // stage X chunk transposed: element e -> row = e % 64, kq = e / 64 (16 float4 per row)
    for (int e = tid; e < kGvMaxRows * 16; e += kGvThreads) {
      const int row = e % kGvMaxRows, kq = e / kGvMaxRows;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (row < R)
        v = *reinterpret_cast<const float4*>(a.X + size_t(slots[row]) * a.K + kc + 4 * kq);
      xs[4 * kq + 0][row] = v.x;
      xs[4 * kq + 1][row] = v.y;
      xs[4 * kq + 2][row] = v.z;
      xs[4 * kq + 3][row] = v.w;
    }
    __syncthreads();
    if (rows_live) {
#pragma unroll 2
      for (int k8 = 0; k8 < kGvKC; k8 += 8) {
        uint4 w[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) w[j] = __ldg(reinterpret_cast<const uint4*>(wrow[j] + kc + k8));
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const float4 xv = *reinterpret_cast<const float4*>(&xs[k8 + kk][4 * rg]);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint32_t word = (&w[j].x)[kk >> 1];
            const float wf = (kk & 1) ? __uint_as_float(word & 0xFFFF0000u)
                                      : __uint_as_float(word << 16);
            acc[0][j] = fmaf(xv.x, wf, acc[0][j]);
            acc[1][j] = fmaf(xv.y, wf, acc[1][j]);
            acc[2][j] = fmaf(xv.z, wf, acc[2][j]);
            acc[3][j] = fmaf(xv.w, wf, acc[3][j]);
          }
        }
      }
    }
    __syncthreads();
  }
  if (a.splits == 1) {
    if (!rows_live) return;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int row = 4 * rg + i;
      if (row >= R) break;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int n = n0 + 4 * fg + j;
        if (n < a.N) gemv_epilogue(st, a, slots[row], n, acc[i][j]);
      }
    }
    return;
  }
  // split-K: partials [split][row][N], last CTA of this N tile reduces in order.
  float* part = st.part;
  if (rows_live) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int row = 4 * rg + i;
      if (row >= R) break;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int n = n0 + 4 * fg + j;
        if (n < a.N) part[(size_t(blockIdx.y) * kGvMaxRows + row) * a.N + n] = acc[i][j];
      }
    }
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    int prev = atomicAdd(&st.counters[a.counter_base + blockIdx.x], 1);
    is_last = (prev == a.splits - 1);
  }
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  for (int e = tid; e < R * kGvTileN; e += kGvThreads) {
    const int row = e / kGvTileN, n = n0 + e % kGvTileN;
    if (n >= a.N) continue;
    float v = 0.f;
    for (int s = 0; s < a.splits; ++s)
      v += __ldcg(&part[(size_t(s) * kGvMaxRows + row) * a.N + n]);
    gemv_epilogue(st, a, slots[row], n, v);
  }
  if (tid == 0) st.counters[a.counter_base + blockIdx.x] = 0;
}

int gemv_splits(int N, int K) {
  const int tiles = ceil_div(N, kGvTileN);
  int s = 1;
  const int kb = K / kGvKC;
  while (s * 2 <= kb && kb % (s * 2) == 0 && tiles * s * 2 <= 2 * kNumSMs) s *= 2;
  return s;
}

int launch_gemv(const DecodeState& st, const GemvArgs& a, cudaStream_t stream) {
  DM_REQUIRE(a.K % kGvKC == 0, "gemv K must be a multiple of 64");
  DM_REQUIRE((a.K / kGvKC) % a.splits == 0, "gemv splits must divide K/64");
  DM_REQUIRE(st.max_slots <= kGvMaxRows, "at most 64 decode slots");
  dim3 grid(ceil_div(a.N, kGvTileN), a.splits);
  gemv_kernel<<<grid, kGvThreads, 0, stream>>>(st, a);
  DM_CHECK_LAUNCH();
  return 0;
}

// ------------------------------------------------------------ LayerNorm fp32
template <int V4>
__global__ void __launch_bounds__(256)
decode_ln_kernel(const DecodeState st, const float* __restrict__ x, const uint16_t* g,
                 const uint16_t* b, float* __restrict__ y) {
  const int i = blockIdx.x * 8 + threadIdx.x / 32, lane = threadIdx.x % 32;
  if (i >= *st.n_active) return;
  const int slot = st.active[i];
  const int d = st.d, n4 = d / 4;
  const float4* xr = reinterpret_cast<const float4*>(x + size_t(slot) * d);
  float4 v[V4];
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < V4; ++k) {
    int c = lane + 32 * k;
    v[k] = c < n4 ? xr[c] : make_float4(0.f, 0.f, 0.f, 0.f);
    s += (v[k].x + v[k].y) + (v[k].z + v[k].w);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const float mean = s / d;
  float q = 0.f;
#pragma unroll
  for (int k = 0; k < V4; ++k) {
    int c = lane + 32 * k;
    if (c < n4) {
      float a0 = v[k].x - mean, a1 = v[k].y - mean, a2 = v[k].z - mean, a3 = v[k].w - mean;
      q += (a0 * a0 + a1 * a1) + (a2 * a2 + a3 * a3);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
  const float rstd = rsqrtf(q / d + 1e-5f);
  float4* yr = reinterpret_cast<float4*>(y + size_t(slot) * d);
#pragma unroll
  for (int k = 0; k < V4; ++k) {
    int c = lane + 32 * k;
    if (c < n4) {
      float4 o;
      o.x = (v[k].x - mean) * rstd * bf16_to_f32(g[4 * c]) + bf16_to_f32(b[4 * c]);
      o.y = (v[k].y - mean) * rstd * bf16_to_f32(g[4 * c + 1]) + bf16_to_f32(b[4 * c + 1]);
      o.z = (v[k].z - mean) * rstd * bf16_to_f32(g[4 * c + 2]) + bf16_to_f32(b[4 * c + 2]);
      o.w = (v[k].w - mean) * rstd * bf16_to_f32(g[4 * c + 3]) + bf16_to_f32(b[4 * c + 3]);
      yr[c] = o;
    }
  }
}

int launch_decode_ln(const DecodeState& st, const float* x, const uint16_t* g,
                     const uint16_t* b, float* y, cudaStream_t stream) {
  dim3 grid(ceil_div(st.max_slots, 8));
  switch (st.d / 128) {
#define DM_DLN(n) case n: decode_ln_kernel<n><<<grid, 256, 0, stream>>>(st, x, g, b, y); break;
    DM_DLN(1) DM_DLN(2) DM_DLN(3) DM_DLN(4) DM_DLN(5) DM_DLN(6) DM_DLN(7) DM_DLN(8)
    DM_DLN(9) DM_DLN(10)
#undef DM_DLN
    default: DM_REQUIRE(false, "unsupported d");
  }
  DM_CHECK_LAUNCH();
  return 0;
}

// ------------------------------------------------------------ embedding
__global__ void embed_kernel(const DecodeState st, const uint16_t* __restrict__ embed,
                             const uint16_t* __restrict__ pos_emb) {
  const int i = blockIdx.x;
  if (i >= *st.n_active) return;
  const int slot = st.active[i];
  const int tok = st.cur_tok[slot], p = st.pos[slot];
  for (int c = threadIdx.x; c < st.d; c += blockDim.x)
    st.x[size_t(slot) * st.d + c] =
        bf16_to_f32(embed[size_t(tok) * st.d + c]) + bf16_to_f32(pos_emb[size_t(p) * st.d + c]);
}

int launch_embed(const DecodeState& st, const uint16_t* embed, const uint16_t* pos_emb,
                 cudaStream_t stream) {
  embed_kernel<<<st.max_slots, 128, 0, stream>>>(st, embed, pos_emb);
  DM_CHECK_LAUNCH();
  return 0;
}

// ------------------------------------------------------------ attention
// Lane-per-key online softmax: every lane owns whole keys (64-dim dot product
// and V accumulation in registers, no per-key shuffles); lanes, warps and
// key splits are merged at the end in a fixed order.
struct SoftmaxPart {
  float m, l;
};

__device__ __forceinline__ void dot_bf16_row(const uint16_t* __restrict__ krow,
                                             const float (&q)[64], float& s) {
  const uint4* k4 = reinterpret_cast<const uint4*>(krow);
  float acc = 0.f;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    uint4 w = __ldg(k4 + c);
    uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      acc = fmaf(q[8 * c + 2 * u], __uint_as_float(ws[u] << 16), acc);
      acc = fmaf(q[8 * c + 2 * u + 1], __uint_as_float(ws[u] & 0xFFFF0000u), acc);
    }
  }
  s = acc;
}

__device__ __forceinline__ void axpy_bf16_row(const uint16_t* __restrict__ vrow, float p,
                                              float (&o)[64]) {
  const uint4* v4 = reinterpret_cast<const uint4*>(vrow);
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    uint4 w = __ldg(v4 + c);
    uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      o[8 * c + 2 * u] = fmaf(p, __uint_as_float(ws[u] << 16), o[8 * c + 2 * u]);
      o[8 * c + 2 * u + 1] = fmaf(p, __uint_as_float(ws[u] & 0xFFFF0000u), o[8 * c + 2 * u + 1]);
    }
  }
}

// Merge (m, l, o[64]) across the 32 lanes of a warp, fixed butterfly order.
__device__ __forceinline__ void warp_merge(float& m, float& l, float (&o)[64]) {
  float mw = m;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) mw = fmaxf(mw, __shfl_xor_sync(0xffffffffu, mw, off));
  const float f = (m == -INFINITY) ? 0.f : exp2f((m - mw) * 1.4426950408889634f);
  l *= f;
#pragma unroll
  for (int i = 0; i < 64; ++i) o[i] *= f;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    l += __shfl_xor_sync(0xffffffffu, l, off);
#pragma unroll
    for (int i = 0; i < 64; ++i) o[i] += __shfl_xor_sync(0xffffffffu, o[i], off);
  }
  m = mw;
}

// Process keys [k0, k1) lane-strided; return this warp's merged state.
template <class KRowFn, class VRowFn>
__device__ __forceinline__ void attend_keys(const float (&q)[64], int k0, int k1, int stride,
                                            int first, KRowFn krow, VRowFn vrow, float& m,
                                            float& l, float (&o)[64]) {
  constexpr float kLog2e = 1.4426950408889634f;
  m = -INFINITY;
  l = 0.f;
#pragma unroll
  for (int i = 0; i < 64; ++i) o[i] = 0.f;
  for (int t = k0 + first; t < k1; t += stride) {
    float s;
    dot_bf16_row(krow(t), q, s);
    const float mn = fmaxf(m, s);
    const float corr = exp2f((m - mn) * kLog2e);
    const float p = exp2f((s - mn) * kLog2e);
    l = l * corr + p;
#pragma unroll
    for (int i = 0; i < 64; ++i) o[i] *= corr;
    axpy_bf16_row(vrow(t), p, o);
    m = mn;
  }
}

constexpr int kAttnWarps = 4;

// Cross-warp merge through smem; result written by warp 0 lanes (2 dims each).
__device__ void block_merge_store(float m, float l, const float (&o)[64], float* smem_o,
                                  float* smem_ml, float* out_o, float* out_ml, bool normalise) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (lane == 0) {
    smem_ml[2 * warp] = m;
    smem_ml[2 * warp + 1] = l;
  }
  if (lane < 1) {
#pragma unroll
    for (int i = 0; i < 64; ++i) smem_o[warp * 64 + i] = o[i];
  }
  __syncthreads();
  if (warp == 0) {
    float mm = -INFINITY;
    for (int w = 0; w < kAttnWarps; ++w) mm = fmaxf(mm, smem_ml[2 * w]);
    float ll = 0.f, o0 = 0.f, o1 = 0.f;
    for (int w = 0; w < kAttnWarps; ++w) {
      const float mw = smem_ml[2 * w];
      const float f = (mw == -INFINITY) ? 0.f : exp2f((mw - mm) * 1.4426950408889634f);
      ll += smem_ml[2 * w + 1] * f;
      o0 += smem_o[w * 64 + 2 * lane] * f;
      o1 += smem_o[w * 64 + 2 * lane + 1] * f;
    }
    if (normalise) {
      out_o[2 * lane] = o0 / ll;
      out_o[2 * lane + 1] = o1 / ll;
    } else {
      out_o[2 * lane] = o0;
      out_o[2 * lane + 1] = o1;
      if (lane == 0) {
        out_ml[0] = mm;
        out_ml[1] = ll;
      }
    }
  }
}

__global__ void __launch_bounds__(kAttnWarps * 32)
self_attn_kernel(const DecodeState st, int layer) {
  __shared__ float s_o[kAttnWarps * 64];
  __shared__ float s_ml[2 * kAttnWarps];
  const int i = blockIdx.x, h = blockIdx.y;
  if (i >= *st.n_active) return;
  const int slot = st.active[i];
  const int nk = st.pos[slot] + 1;                 // keys 0..pos (incl. current)
  float q[64];
  const float* qp = st.q + size_t(slot) * st.d + h * 64;
#pragma unroll
  for (int c = 0; c < 64; ++c) q[c] = qp[c];
  const int* pt = st.page_table + slot * st.pages_per_slot;
  const size_t kv_stride = size_t(st.heads) * st.page_tokens * 64;   // k -> v
  auto krow = [&](int t) {
    const int page = pt[t / st.page_tokens];
    return st.kv_pool + ((((size_t(page) * st.layers + layer) * 2 + 0) * st.heads + h) *
                             st.page_tokens + t % st.page_tokens) * 64;
  };
  auto vrow = [&](int t) { return krow(t) + kv_stride; };
  float m, l, o[64];
  attend_keys(q, 0, nk, kAttnWarps * 32, threadIdx.x, krow, vrow, m, l, o);
  warp_merge(m, l, o);
  block_merge_store(m, l, o, s_o, s_ml, st.attn + size_t(slot) * st.d + h * 64, nullptr, true);
}

__global__ void __launch_bounds__(kAttnWarps * 32)
cross_attn_kernel(const DecodeState st, int layer, int counter_base) {
  __shared__ float s_o[kAttnWarps * 64];
  __shared__ float s_ml[2 * kAttnWarps];
  __shared__ int is_last;
  const int i = blockIdx.x, h = blockIdx.y, sp = blockIdx.z;
  if (i >= *st.n_active) return;
  const int slot = st.active[i];
  const int xs = st.xsplits;
  const int per = ceil_div(1500, xs);
  const int k0 = sp * per, k1 = min(1500, k0 + per);
  float q[64];
  const float* qp = st.q + size_t(slot) * st.d + h * 64;
#pragma unroll
  for (int c = 0; c < 64; ++c) q[c] = qp[c];
  const uint16_t* kbase =
      st.xkv + (((size_t(layer) * st.max_slots + slot) * 2 + 0) * st.heads + h) * 1500 * 64;
  const size_t vofs = size_t(st.heads) * 1500 * 64;
  auto krow = [&](int t) { return kbase + size_t(t) * 64; };
  auto vrow = [&](int t) { return kbase + vofs + size_t(t) * 64; };
  float m, l, o[64];
  attend_keys(q, k0, k1, kAttnWarps * 32, threadIdx.x, krow, vrow, m, l, o);
  warp_merge(m, l, o);
  if (xs == 1) {
    block_merge_store(m, l, o, s_o, s_ml, st.attn + size_t(slot) * st.d + h * 64, nullptr, true);
    return;
  }
  // partial -> scratch [slot][h][split][66]
  float* part = st.part + ((size_t(slot) * st.heads + h) * xs + sp) * 66;
  block_merge_store(m, l, o, s_o, s_ml, part + 2, part, false);
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    int prev = atomicAdd(&st.counters[counter_base + slot * st.heads + h], 1);
    is_last = prev == xs - 1;
  }
  __syncthreads();
  if (!is_last || threadIdx.x >= 32) return;
  __threadfence();
  const float* pb = st.part + (size_t(slot) * st.heads + h) * xs * 66;
  float mm = -INFINITY;
  for (int s = 0; s < xs; ++s) mm = fmaxf(mm, __ldcg(pb + s * 66));
  float ll = 0.f, o0 = 0.f, o1 = 0.f;
  const int lane = threadIdx.x;
  for (int s = 0; s < xs; ++s) {
    const float ms = __ldcg(pb + s * 66);
    const float f = (ms == -INFINITY) ? 0.f : exp2f((ms - mm) * 1.4426950408889634f);
    ll += __ldcg(pb + s * 66 + 1) * f;
    o0 += __ldcg(pb + s * 66 + 2 + 2 * lane) * f;
    o1 += __ldcg(pb + s * 66 + 3 + 2 * lane) * f;
  }
  float* out = st.attn + size_t(slot) * st.d + h * 64;
  out[2 * lane] = o0 / ll;
  out[2 * lane + 1] = o1 / ll;
  if (lane == 0) st.counters[counter_base + slot * st.heads + h] = 0;
}

int launch_self_attn(const DecodeState& st, int layer, cudaStream_t stream) {
  dim3 grid(st.max_slots, st.heads);
  self_attn_kernel<<<grid, kAttnWarps * 32, 0, stream>>>(st, layer);
  DM_CHECK_LAUNCH();
  return 0;
}

int launch_cross_attn(const DecodeState& st, int layer, int counter_base, cudaStream_t stream) {
  dim3 grid(st.max_slots, st.heads, st.xsplits);
  cross_attn_kernel<<<grid, kAttnWarps * 32, 0, stream>>>(st, layer, counter_base);
  DM_CHECK_LAUNCH();
  return 0;
}

// ------------------------------------------------------------ LM head + argmax
// Tied LM head (modeling_whisper.py:966,971): logits = xn . E^T, fp32. Each
// CTA scores 64 vocabulary rows for all active slots and keeps a per-slot
// (max, lowest index) partial; finalize scans the partials in tile order.
__global__ void __launch_bounds__(kGvThreads)
lm_head_kernel(const DecodeState st, const uint16_t* __restrict__ E) {
  __shared__ __align__(16) float xs[kGvKC][kGvMaxRows];
  __shared__ int slots[kGvMaxRows];
  const int R = min(*st.n_active, kGvMaxRows);
  const int tid = threadIdx.x, rg = tid / 16, fg = tid % 16;
  const int n0 = blockIdx.x * kGvTileN;
  const int K = st.d, N = st.vocab;
  if (tid < kGvMaxRows) slots[tid] = tid < R ? st.active[tid] : 0;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  const bool rows_live = 4 * rg < R;
  const uint16_t* wrow[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) wrow[j] = E + size_t(min(n0 + 4 * fg + j, N - 1)) * K;
  __syncthreads();
  for (int kc = 0; kc < K; kc += kGvKC) {
    for (int e = tid; e < kGvMaxRows * 16; e += kGvThreads) {
      const int row = e % kGvMaxRows, kq = e / kGvMaxRows;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (row < R) v = *reinterpret_cast<const float4*>(st.xn + size_t(slots[row]) * K + kc + 4 * kq);
      xs[4 * kq + 0][row] = v.x;
      xs[4 * kq + 1][row] = v.y;
      xs[4 * kq + 2][row] = v.z;
      xs[4 * kq + 3][row] = v.w;
    }
    __syncthreads();
    if (rows_live) {
#pragma unroll 2
      for (int k8 = 0; k8 < kGvKC; k8 += 8) {
        uint4 w[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) w[j] = __ldg(reinterpret_cast<const uint4*>(wrow[j] + kc + k8));
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const float4 xv = *reinterpret_cast<const float4*>(&xs[k8 + kk][4 * rg]);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint32_t word = (&w[j].x)[kk >> 1];
            const float wf = (kk & 1) ? __uint_as_float(word & 0xFFFF0000u)
                                      : __uint_as_float(word << 16);
            acc[0][j] = fmaf(xv.x, wf, acc[0][j]);
            acc[1][j] = fmaf(xv.y, wf, acc[1][j]);
            acc[2][j] = fmaf(xv.z, wf, acc[2][j]);
            acc[3][j] = fmaf(xv.w, wf, acc[3][j]);
          }
        }
      }
    }
    __syncthreads();
  }
  // per row: max over this thread's 4 features, then over the 16 fg lanes
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = 4 * rg + i;
    float best = -INFINITY;
    int bidx = 0x7FFFFFFF;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + 4 * fg + j;
      if (n < N) {
        if (st.logits_dbg && row < R) st.logits_dbg[size_t(slots[row]) * N + n] = acc[i][j];
        if (acc[i][j] > best) { best = acc[i][j]; bidx = n; }
      }
    }
#pragma unroll
    for (int off = 8; off > 0; off >>= 1) {
      const float ob = __shfl_xor_sync(0xffffffffu, best, off);
      const int oi = __shfl_xor_sync(0xffffffffu, bidx, off);
      if (ob > best || (ob == best && oi < bidx)) { best = ob; bidx = oi; }
    }
    if (fg == 0 && row < R) {
      st.amax_val[size_t(blockIdx.x) * st.max_slots + slots[row]] = best;
      st.amax_idx[size_t(blockIdx.x) * st.max_slots + slots[row]] = bidx;
    }
  }
}

int launch_lm_head(const DecodeState& st, const uint16_t* embed, cudaStream_t stream) {
  DM_REQUIRE(st.d % kGvKC == 0, "d must be a multiple of 64");
  lm_head_kernel<<<ceil_div(st.vocab, kGvTileN), kGvThreads, 0, stream>>>(st, embed);
  DM_CHECK_LAUNCH();
  return 0;
}

// One warp per active slot: argmax over tile partials (ties -> lowest id),
// then the greedy state machine (prompt forcing, EOT, per-slot cap).
__global__ void finalize_kernel(const DecodeState st) {
  const int i = blockIdx.x * 4 + threadIdx.x / 32, lane = threadIdx.x % 32;
  if (i >= *st.n_active) return;
  const int slot = st.active[i];
  const int tiles = ceil_div(st.vocab, kGvTileN);
  float best = -INFINITY;
  int bidx = 0x7FFFFFFF;
  for (int t = lane; t < tiles; t += 32) {
    const float v = st.amax_val[size_t(t) * st.max_slots + slot];
    const int id = st.amax_idx[size_t(t) * st.max_slots + slot];
    if (v > best || (v == best && id < bidx)) { best = v; bidx = id; }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const float ob = __shfl_xor_sync(0xffffffffu, best, off);
    const int oi = __shfl_xor_sync(0xffffffffu, bidx, off);
    if (ob > best || (ob == best && oi < bidx)) { best = ob; bidx = oi; }
  }
  if (lane != 0 || st.done[slot]) return;
  const int p = st.pos[slot];
  if (p + 1 < st.prompt_len) {                 // still feeding the prompt
    st.cur_tok[slot] = st.prompt[p + 1];
    st.pos[slot] = p + 1;
    return;
  }
  if (bidx == st.eot) { st.done[slot] = 1; return; }
  const int g = st.n_gen[slot];
  st.out_tokens[slot * 448 + g] = bidx;
  st.n_gen[slot] = g + 1;
  if (g + 1 >= st.cap[slot]) { st.done[slot] = 1; return; }
  st.cur_tok[slot] = bidx;
  st.pos[slot] = p + 1;
}

int launch_finalize(const DecodeState& st, cudaStream_t stream) {
  finalize_kernel<<<ceil_div(st.max_slots, 4), 128, 0, stream>>>(st);
  DM_CHECK_LAUNCH();
  return 0;
}

}  // namespace dm
