// K6 decode-step kernels. Projections (QKV, out, cross-q, MLP, tied LM head)
// run on tcgen05: the weight tile is the M=128 operand streamed by TMA, the
// active rows (N=64) are the bf16 hi/lo split of the fp32 activations, so each
// output is W.(hi + lo) accumulated in fp32 TMEM. Attention keeps fp32 math
// with bf16 K/V. Every per-row reduction has a fixed order that depends only on
// K / positions, never on which or how many rows are active, so a segment
// decodes bit-identically alone or in any batch.
//
// Per step the HBM stream is the weights (once for the whole batch) plus every
// active slot's cross-KV; both are read exactly once.

#include "decode.cuh"

namespace dm {

// ============================================================ tcgen05 GEMV
constexpr int kTvThreads = 192;     // w0 TMA, w1 MMA, w2..5 epilogue
constexpr int kTvStages = 4;
constexpr int kTvWBytes = 128 * 64 * 2;   // W tile: 128 rows x 64 k
constexpr int kTvXBytes = kRows * 64 * 2; // X tile: 64 rows x 64 k (hi or lo)
constexpr int kTvStageBytes = kTvWBytes + 2 * kTvXBytes;
constexpr int kTvSmem = kTvStages * kTvStageBytes + 1024 + 128 + 4096;

__device__ __forceinline__ void split_hilo(float v, uint16_t& hi, uint16_t& lo) {
  hi = f32_to_bf16(v);
  lo = f32_to_bf16(v - bf16_to_f32(hi));
}

__global__ void __launch_bounds__(kTvThreads, 1)
tc_gemv_kernel(const __grid_constant__ CUtensorMap tw, const __grid_constant__ CUtensorMap txh,
               const __grid_constant__ CUtensorMap txl, const DecodeState st,
               const TcGemvArgs a) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024 - (raw_addr & 1023)) & 1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kTvStages * kTvStageBytes);
  uint64_t* empty = full + kTvStages;
  uint64_t* mma_done = empty + kTvStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(mma_done + 1);
  int* is_last = reinterpret_cast<int*>(tmem_slot + 1);
  float* red_v = reinterpret_cast<float*>(smem + kTvStages * kTvStageBytes + 128);   // [4][64]
  int* red_i = reinterpret_cast<int*>(red_v + 4 * kRows);                            // [4][64]

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int tile = blockIdx.x, split = blockIdx.y;
  const int tiles = gridDim.x;
  const int kb_per = (a.K / 64) / a.splits;
  const int kb0 = split * kb_per;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tw);
    tma_prefetch_desc(&txh);
    tma_prefetch_desc(&txl);
    for (int s = 0; s < kTvStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(mma_done, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 64);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (elect_one()) {
      for (int i = 0; i < kb_per; ++i) {
        const int s = i % kTvStages;
        mbar_wait(&empty[s], ((i / kTvStages) & 1) ^ 1);
        uint8_t* base = smem + s * kTvStageBytes;
        mbar_arrive_expect_tx(&full[s], kTvStageBytes);
        const int kc = (kb0 + i) * 64;
        tma_load_2d(base, &tw, &full[s], kc, tile * 128);
        tma_load_2d(base + kTvWBytes, &txh, &full[s], kc, 0);
        tma_load_2d(base + kTvWBytes + kTvXBytes, &txl, &full[s], kc, 0);
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = umma_idesc_bf16(128, kRows);
    for (int i = 0; i < kb_per; ++i) {
      const int s = i % kTvStages;
      mbar_wait(&full[s], (i / kTvStages) & 1);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t sw = smem_u32(smem + s * kTvStageBytes);
        const uint32_t sh = sw + kTvWBytes, sl = sh + kTvXBytes;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          umma_bf16_ss(tmem, umma_desc_sw128(sw + k * 32), umma_desc_sw128(sh + k * 32), idesc,
                       (i | k) != 0);
          umma_bf16_ss(tmem, umma_desc_sw128(sw + k * 32), umma_desc_sw128(sl + k * 32), idesc, 1);
        }
        umma_commit(&empty[s]);
        if (i == kb_per - 1) umma_commit(mma_done);
      }
      __syncwarp();
    }
  } else {
    const int quad = warp & 3;
    const int f = quad * 32 + lane;                // feature within the tile
    const int n = tile * 128 + f;
    const int R = min(*st.n_active, kRows);
    mbar_wait(mma_done, 0);
    tc_fence_after();
    float v[kRows];
    {
      uint32_t r[32];
      tmem_ld32(tmem + (uint32_t(quad * 32) << 16), r);
      tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
      tmem_ld32(tmem + (uint32_t(quad * 32) << 16) + 32, r);
      tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < 32; ++i) v[32 + i] = __uint_as_float(r[i]);
    }
    if (a.splits > 1) {
      float* part = st.part;
      const size_t base = (size_t(split) * tiles + tile) * kRows * 128;
#pragma unroll
      for (int r = 0; r < kRows; ++r) part[base + size_t(r) * 128 + f] = v[r];
      __threadfence();
      named_bar_sync(1, 128);
      if (threadIdx.x == 64) {
        const int prev = atomicAdd(&st.counters[a.counter_base + tile], 1);
        *is_last = (prev == a.splits - 1);
      }
      named_bar_sync(1, 128);
      if (!*is_last) goto done;
      __threadfence();
#pragma unroll
      for (int r = 0; r < kRows; ++r) {
        float acc = 0.f;
        for (int s = 0; s < a.splits; ++s)
          acc += __ldcg(&part[(size_t(s) * tiles + tile) * kRows * 128 + size_t(r) * 128 + f]);
        v[r] = acc;
      }
      if (threadIdx.x == 64) st.counters[a.counter_base + tile] = 0;
    }
    {
      const bool nvalid = n < a.N;
      const float b = (nvalid && a.bias) ? bf16_to_f32(a.bias[n]) : 0.f;
      switch (a.epi) {
        case TV_STORE:
          if (nvalid)
#pragma unroll
            for (int r = 0; r < kRows; ++r) a.y[size_t(r) * a.N + n] = (v[r] + b) * a.scale;
          break;
        case TV_GELU_HILO:
          if (nvalid)
#pragma unroll
            for (int r = 0; r < kRows; ++r) {
              uint16_t hi, lo;
              split_hilo(gelu_erf(v[r] + b), hi, lo);
              a.yh[size_t(r) * a.N + n] = hi;
              a.yl[size_t(r) * a.N + n] = lo;
            }
          break;
        case TV_RESID:
          if (nvalid)
#pragma unroll
            for (int r = 0; r < kRows; ++r) a.y[size_t(r) * a.N + n] += v[r] + b;
          break;
        case TV_QKV: {
          if (!nvalid) break;
          const int d = st.d;
          if (n < d) {
#pragma unroll
            for (int r = 0; r < kRows; ++r) st.q[size_t(r) * d + n] = (v[r] + b) * a.scale;
          } else {
            const int kv = n < 2 * d ? 0 : 1;
            const int c = n - (kv + 1) * d;
            const int h = c / 64, j = c % 64;
#pragma unroll
            for (int r = 0; r < kRows; ++r) {
              if (r >= R) break;
              const int slot = st.active[r];
              const int p = st.pos[slot];
              const int page = st.page_table[slot * st.pages_per_slot + p / st.page_tokens];
              const size_t idx = ((((size_t(page) * st.layers + a.layer) * 2 + kv) * st.heads + h) *
                                      st.page_tokens + (p % st.page_tokens)) * 64 + j;
              st.kv_pool[idx] = f32_to_bf16(v[r] + b);
            }
          }
          break;
        }
        case TV_ARGMAX: {
          // per row: max over this tile's 128 vocabulary ids, ties -> lowest id
#pragma unroll
          for (int r = 0; r < kRows; ++r) {
            float best = nvalid ? v[r] : -INFINITY;
            int bidx = nvalid ? n : 0x7FFFFFFF;
            if (st.logits_dbg && nvalid && r < R) st.logits_dbg[size_t(r) * st.vocab + n] = v[r];
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
              const float ob = __shfl_xor_sync(0xffffffffu, best, off);
              const int oi = __shfl_xor_sync(0xffffffffu, bidx, off);
              if (ob > best || (ob == best && oi < bidx)) { best = ob; bidx = oi; }
            }
            if (lane == 0) {
              red_v[quad * kRows + r] = best;
              red_i[quad * kRows + r] = bidx;
            }
          }
          named_bar_sync(1, 128);
          if (threadIdx.x >= 64 && threadIdx.x < 64 + kRows) {
            const int r = threadIdx.x - 64;
            float best = red_v[r];
            int bidx = red_i[r];
            for (int qd = 1; qd < 4; ++qd) {
              const float ob = red_v[qd * kRows + r];
              const int oi = red_i[qd * kRows + r];
              if (ob > best || (ob == best && oi < bidx)) { best = ob; bidx = oi; }
            }
            st.amax_val[size_t(tile) * kRows + r] = best;
            st.amax_idx[size_t(tile) * kRows + r] = bidx;
          }
          break;
        }
      }
    }
  done:;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 64);
  }
}

int tc_gemv_splits(int N, int K) {
  const int tiles = ceil_div(N, 128);
  const int kb = K / 64;
  for (int s = 1; s <= kb; ++s) {
    if (kb % s) continue;
    if (kb / s <= 8 || tiles * s * 2 > 2 * kNumSMs) return s;
  }
  return kb;
}

size_t tc_gemv_part_floats(int N, int K) {
  const int s = tc_gemv_splits(N, K);
  return s > 1 ? size_t(s) * ceil_div(N, 128) * kRows * 128 : 0;
}

int launch_tc_gemv(const DecodeState& st, const TcGemvMaps& maps, const TcGemvArgs& a,
                   cudaStream_t stream) {
  DM_REQUIRE(a.K % 64 == 0, "K must be a multiple of 64");
  DM_REQUIRE((a.K / 64) % a.splits == 0, "splits must divide K/64");
  static bool attr = false;
  if (!attr) {
    DM_CHECK_CUDA(cudaFuncSetAttribute(tc_gemv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       kTvSmem));
    attr = true;
  }
  dim3 grid(ceil_div(a.N, 128), a.splits);
  tc_gemv_kernel<<<grid, kTvThreads, kTvSmem, stream>>>(maps.w, maps.xh, maps.xl, st, a);
  DM_CHECK_LAUNCH();
  return 0;
}

// ============================================================ LayerNorm
// fp32 residual row -> bf16 hi/lo (the next projection's operand).
template <int V4>
__global__ void __launch_bounds__(256)
decode_ln_kernel(const DecodeState st, const float* __restrict__ x, const uint16_t* g,
                 const uint16_t* b) {
  const int r = blockIdx.x * 8 + threadIdx.x / 32, lane = threadIdx.x % 32;
  if (r >= *st.n_active) return;
  const int d = st.d, n4 = d / 4;
  const float4* xr = reinterpret_cast<const float4*>(x + size_t(r) * d);
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
  uint2* yh = reinterpret_cast<uint2*>(st.xh + size_t(r) * d);
  uint2* yl = reinterpret_cast<uint2*>(st.xl + size_t(r) * d);
#pragma unroll
  for (int k = 0; k < V4; ++k) {
    int c = lane + 32 * k;
    if (c < n4) {
      float o[4] = {v[k].x, v[k].y, v[k].z, v[k].w};
      uint16_t hi[4], lo[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float val = (o[u] - mean) * rstd * bf16_to_f32(g[4 * c + u]) + bf16_to_f32(b[4 * c + u]);
        split_hilo(val, hi[u], lo[u]);
      }
      yh[c] = make_uint2(uint32_t(hi[0]) | (uint32_t(hi[1]) << 16), uint32_t(hi[2]) | (uint32_t(hi[3]) << 16));
      yl[c] = make_uint2(uint32_t(lo[0]) | (uint32_t(lo[1]) << 16), uint32_t(lo[2]) | (uint32_t(lo[3]) << 16));
    }
  }
}

int launch_decode_ln(const DecodeState& st, const float* x, const uint16_t* g,
                     const uint16_t* b, cudaStream_t stream) {
  dim3 grid(kRows / 8);
  switch (st.d / 128) {
#define DM_DLN(n) case n: decode_ln_kernel<n><<<grid, 256, 0, stream>>>(st, x, g, b); break;
    DM_DLN(1) DM_DLN(2) DM_DLN(3) DM_DLN(4) DM_DLN(5) DM_DLN(6) DM_DLN(7) DM_DLN(8)
    DM_DLN(9) DM_DLN(10)
#undef DM_DLN
    default: DM_REQUIRE(false, "unsupported d");
  }
  DM_CHECK_LAUNCH();
  return 0;
}

// ============================================================ embedding
__global__ void embed_kernel(const DecodeState st, const uint16_t* __restrict__ embed,
                             const uint16_t* __restrict__ pos_emb) {
  const int r = blockIdx.x;
  if (r >= *st.n_active) return;
  const int slot = st.active[r];
  const int tok = st.cur_tok[slot], p = st.pos[slot];
  for (int c = threadIdx.x; c < st.d; c += blockDim.x)
    st.x[size_t(r) * st.d + c] =
        bf16_to_f32(embed[size_t(tok) * st.d + c]) + bf16_to_f32(pos_emb[size_t(p) * st.d + c]);
}

int launch_embed(const DecodeState& st, const uint16_t* embed, const uint16_t* pos_emb,
                 cudaStream_t stream) {
  embed_kernel<<<kRows, 128, 0, stream>>>(st, embed, pos_emb);
  DM_CHECK_LAUNCH();
  return 0;
}

// ============================================================ attention
// Lane-per-key online softmax: every lane owns whole keys (64-dim dot product
// and V accumulation in registers, no per-key shuffles); lanes, warps and
// key splits are merged at the end in a fixed order.
__device__ __forceinline__ float dot_bf16_row(const uint16_t* __restrict__ krow,
                                              const float (&q)[64]) {
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
  return acc;
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

constexpr float kLog2e = 1.4426950408889634f;

// Merge (m, l, o[64]) across the 32 lanes of a warp, fixed butterfly order.
__device__ __forceinline__ void warp_merge(float& m, float& l, float (&o)[64]) {
  float mw = m;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) mw = fmaxf(mw, __shfl_xor_sync(0xffffffffu, mw, off));
  const float f = (m == -INFINITY) ? 0.f : exp2f((m - mw) * kLog2e);
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

template <class KRowFn, class VRowFn>
__device__ __forceinline__ void attend_keys(const float (&q)[64], int k0, int k1, int stride,
                                            int first, KRowFn krow, VRowFn vrow, float& m,
                                            float& l, float (&o)[64]) {
  m = -INFINITY;
  l = 0.f;
#pragma unroll
  for (int i = 0; i < 64; ++i) o[i] = 0.f;
  for (int t = k0 + first; t < k1; t += stride) {
    const float s = dot_bf16_row(krow(t), q);
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

// Cross-warp merge through smem. Warp 0 lanes then hold dims (2 lane, 2 lane+1)
// of the merged (m, l, o); returns them via out refs.
__device__ void block_merge(float m, float l, const float (&o)[64], float* smem_o,
                            float* smem_ml, float& mm, float& ll, float& o0, float& o1) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (lane == 0) {
    smem_ml[2 * warp] = m;
    smem_ml[2 * warp + 1] = l;
#pragma unroll
    for (int i = 0; i < 64; ++i) smem_o[warp * 64 + i] = o[i];
  }
  __syncthreads();
  mm = -INFINITY;
  for (int w = 0; w < kAttnWarps; ++w) mm = fmaxf(mm, smem_ml[2 * w]);
  ll = 0.f; o0 = 0.f; o1 = 0.f;
  for (int w = 0; w < kAttnWarps; ++w) {
    const float mw = smem_ml[2 * w];
    const float f = (mw == -INFINITY) ? 0.f : exp2f((mw - mm) * kLog2e);
    ll += smem_ml[2 * w + 1] * f;
    o0 += smem_o[w * 64 + 2 * lane] * f;
    o1 += smem_o[w * 64 + 2 * lane + 1] * f;
  }
}

__device__ __forceinline__ void store_hilo2(const DecodeState& st, int r, int h, int lane,
                                            float a, float b) {
  uint16_t h0, l0, h1, l1;
  split_hilo(a, h0, l0);
  split_hilo(b, h1, l1);
  const size_t idx = size_t(r) * st.d + h * 64 + 2 * lane;
  *reinterpret_cast<uint32_t*>(st.ah + idx) = uint32_t(h0) | (uint32_t(h1) << 16);
  *reinterpret_cast<uint32_t*>(st.al + idx) = uint32_t(l0) | (uint32_t(l1) << 16);
}

__global__ void __launch_bounds__(kAttnWarps * 32)
self_attn_kernel(const DecodeState st, int layer) {
  __shared__ float s_o[kAttnWarps * 64];
  __shared__ float s_ml[2 * kAttnWarps];
  const int r = blockIdx.x, h = blockIdx.y;
  if (r >= *st.n_active) return;
  const int slot = st.active[r];
  const int nk = st.pos[slot] + 1;                 // keys 0..pos (incl. current)
  float q[64];
  const float* qp = st.q + size_t(r) * st.d + h * 64;
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
  float mm, ll, o0, o1;
  block_merge(m, l, o, s_o, s_ml, mm, ll, o0, o1);
  if (threadIdx.x < 32) store_hilo2(st, r, h, threadIdx.x, o0 / ll, o1 / ll);
}

__global__ void __launch_bounds__(kAttnWarps * 32)
cross_attn_kernel(const DecodeState st, int layer, int counter_base) {
  __shared__ float s_o[kAttnWarps * 64];
  __shared__ float s_ml[2 * kAttnWarps];
  __shared__ int is_last;
  const int r = blockIdx.x, h = blockIdx.y, sp = blockIdx.z;
  if (r >= *st.n_active) return;
  const int slot = st.active[r];
  const int xs = st.xsplits;
  const int per = ceil_div(1500, xs);
  const int k0 = sp * per, k1 = min(1500, k0 + per);
  float q[64];
  const float* qp = st.q + size_t(r) * st.d + h * 64;
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
  float mm, ll, o0, o1;
  block_merge(m, l, o, s_o, s_ml, mm, ll, o0, o1);
  if (xs == 1) {
    if (threadIdx.x < 32) store_hilo2(st, r, h, threadIdx.x, o0 / ll, o1 / ll);
    return;
  }
  // partial -> scratch [row][h][split][66]
  const int lane = threadIdx.x;
  float* part = st.part + ((size_t(r) * st.heads + h) * xs + sp) * 66;
  if (lane < 32) {
    part[2 + 2 * lane] = o0;
    part[3 + 2 * lane] = o1;
    if (lane == 0) { part[0] = mm; part[1] = ll; }
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const int prev = atomicAdd(&st.counters[counter_base + r * st.heads + h], 1);
    is_last = prev == xs - 1;
  }
  __syncthreads();
  if (!is_last || threadIdx.x >= 32) return;
  __threadfence();
  const float* pb = st.part + (size_t(r) * st.heads + h) * xs * 66;
  float gm = -INFINITY;
  for (int s = 0; s < xs; ++s) gm = fmaxf(gm, __ldcg(pb + s * 66));
  float gl = 0.f, g0 = 0.f, g1 = 0.f;
  for (int s = 0; s < xs; ++s) {
    const float ms = __ldcg(pb + s * 66);
    const float f = (ms == -INFINITY) ? 0.f : exp2f((ms - gm) * kLog2e);
    gl += __ldcg(pb + s * 66 + 1) * f;
    g0 += __ldcg(pb + s * 66 + 2 + 2 * lane) * f;
    g1 += __ldcg(pb + s * 66 + 3 + 2 * lane) * f;
  }
  store_hilo2(st, r, h, lane, g0 / gl, g1 / gl);
  if (lane == 0) st.counters[counter_base + r * st.heads + h] = 0;
}

int launch_self_attn(const DecodeState& st, int layer, cudaStream_t stream) {
  dim3 grid(kRows, st.heads);
  self_attn_kernel<<<grid, kAttnWarps * 32, 0, stream>>>(st, layer);
  DM_CHECK_LAUNCH();
  return 0;
}

int launch_cross_attn(const DecodeState& st, int layer, int counter_base, cudaStream_t stream) {
  dim3 grid(kRows, st.heads, st.xsplits);
  cross_attn_kernel<<<grid, kAttnWarps * 32, 0, stream>>>(st, layer, counter_base);
  DM_CHECK_LAUNCH();
  return 0;
}

// ============================================================ finalize
// One warp per active row: argmax over the vocab-tile partials (ties -> lowest
// id), then the greedy state machine (prompt forcing, EOT, per-slot cap).
__global__ void finalize_kernel(const DecodeState st) {
  const int r = blockIdx.x * 4 + threadIdx.x / 32, lane = threadIdx.x % 32;
  if (r >= *st.n_active) return;
  const int slot = st.active[r];
  const int tiles = ceil_div(st.vocab, 128);
  float best = -INFINITY;
  int bidx = 0x7FFFFFFF;
  for (int t = lane; t < tiles; t += 32) {
    const float v = st.amax_val[size_t(t) * kRows + r];
    const int id = st.amax_idx[size_t(t) * kRows + r];
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
  finalize_kernel<<<kRows / 4, 128, 0, stream>>>(st);
  DM_CHECK_LAUNCH();
  return 0;
}

}  // namespace dm
