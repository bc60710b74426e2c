// K4: encoder self-attention (non-causal, 1500 x 1500 x 64 per head) on
// tcgen05. One CTA per (two 128-query tiles, segment*head). Warp roles:
//   w0: TMA producer (both Q tiles once, then K / V^T tiles through a 2-stage ring)
//   w1: MMA issuer (S_t = Q_t K_j^T into TMEM, PV_t = P_t V_j into TMEM,
//       alternating between the two query tiles t)
//   w2..9: softmax, two warpgroups (one per query tile), one query row per
//       thread (TMEM lane = row): row max (3-input FMNMX) /
//       exp2 / row sum entirely in registers (no shuffles), P_j written as
//       packed bf16 into TMEM, where the P.V MMA reads it as its A operand
//       (shared memory then only carries Q, K and V: a P round trip through
//       smem cost 128 KB of smem bandwidth per key block pair, the kernel's
//       bound), O accumulated in TMEM with a lazy rescale.
// Q arrives pre-scaled by head_dim^-0.5 (modeling_whisper.py:310) from the
// QKV GEMM epilogue; V arrives transposed ([dims, positions]) so both MMAs
// are K-major. Keys >= 1500 (the 1536-padded tail) are masked to -inf.

#include "common.cuh"

namespace dm {

#ifdef DM_ATTN_TRACE
// phase timeline of one CTA (clock64): [tile][j][sfull, ld, off, emit] and
// MMA warp [tile][j][S issue, PV issue]
__device__ unsigned long long g_attn_trace[2 * 16 * 4 + 2 * 16 * 2 + 1];
#define ATRACE(idx) do { if (traced && lane == 0) g_attn_trace[idx] = clock64(); } while (0)
#define ATRACE_E(idx) do { if (traced) g_attn_trace[idx] = clock64(); } while (0)
#else
#define ATRACE(idx) do {} while (0)
#define ATRACE_E(idx) do {} while (0)
#endif

constexpr int kQBytes = 128 * 128;   // 128 rows x 64 bf16
constexpr int kKBytes = 128 * 128;
constexpr int kVBytes = 2 * 64 * 128;  // two 64-key boxes of [64 dims x 64 keys]

// NT query tiles per CTA (w0 TMA, w1 MMA, one softmax warpgroup per tile) and
// a KS-deep K/V ring. NT = 1 (default): 256 TMEM columns and a 2-deep ring, so
// two independent CTAs share an SM -- their exponential phases drift apart
// instead of running in lockstep, and short sequences hide each other's
// setup (whisper-large-v3 layer, 12 segments: 253 -> 239 µs; CTC 78 -> 72 µs).
// NT = 2: two tiles share every K/V tile, one CTA per SM (512 columns).
template <int NT>
struct AttnCfg {
  static constexpr int kThreads = (2 + 4 * NT) * 32;
  static constexpr int kKS = NT == 2 ? 4 : 2;
  static constexpr int kTmemCols = 256 * NT;        // S NT x 128, O NT x 64, P NT x 64
  static constexpr int q = 0;                       // [NT tiles]
  static constexpr int k = q + NT * kQBytes;
  static constexpr int v = k + kKS * kKBytes;
  static constexpr int bars = v + kKS * kVBytes;
  static constexpr int total = bars + 256 + 1024;
};

__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
__device__ __forceinline__ float ex2(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// One CTA per (pair of 128-query tiles, segment*head). The two tiles share
// every K/V tile; each has its own S (128 TMEM cols), O (64 cols), P (64 cols)
// and its own softmax warpgroup, so the tensor core works on one tile while
// the other tile's softmax runs.
template <int NT>
__global__ void __launch_bounds__(AttnCfg<NT>::kThreads, 3 - NT)
attn_tcgen05_kernel(const __grid_constant__ CUtensorMap tm_q,
                    const __grid_constant__ CUtensorMap tm_k,
                    const __grid_constant__ CUtensorMap tm_vt, int T_rows, int t_pad,
                    int heads, uint16_t* __restrict__ out, int ldo,
                    const int32_t* __restrict__ seg_len) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024 - (raw_addr & 1023)) & 1023);
  using L = AttnCfg<NT>;
  constexpr int kAttnKS = L::kKS;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::bars);
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;            // [KS]
  uint64_t* kv_empty = kv_full + kAttnKS;  // [KS]
  uint64_t* s_full = kv_empty + kAttnKS;   // [2 tiles]
  uint64_t* s_empty = s_full + 2;          // [2 tiles]
  uint64_t* p_full = s_empty + 2;          // [2 tiles]
  uint64_t* o_full = p_full + 2;           // [2 tiles]
  uint64_t* o_empty = o_full + 2;          // [2 tiles]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_empty + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int qp = blockIdx.x, bh = blockIdx.y;
  // per-segment valid length (variable-length CTC batches); whisper: all 1500
  const int T = seg_len ? seg_len[bh / heads] : T_rows;
  if (qp * 128 * NT >= T) return;
  const int nb = ceil_div(T, 128);
#ifdef DM_ATTN_TRACE
  const bool traced = qp == 2 && bh == 5 && nb <= 16;
  if (traced && threadIdx.x == 0) g_attn_trace[192] = clock64();
#endif

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_vt);
    mbar_init(q_full, 1);
    for (int i = 0; i < kAttnKS; ++i) { mbar_init(&kv_full[i], 1); mbar_init(&kv_empty[i], 1); }
    for (int i = 0; i < NT; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], 4);
      mbar_init(&p_full[i], 4);
      mbar_init(&o_full[i], 1);
      mbar_init(&o_empty[i], 4);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, L::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // TMEM columns: S tile t at 128 t, O tile t at kO + 64 t, P tile t at kP + 64 t
  constexpr uint32_t kO = 128 * NT, kP = 192 * NT;

  if (warp == 0) {
    if (elect_one()) {
      mbar_arrive_expect_tx(q_full, NT * kQBytes);
      for (int t = 0; t < NT; ++t)
        tma_load_2d(smem + L::q + t * kQBytes, &tm_q, q_full, 0, bh * t_pad + qp * 128 * NT + 128 * t);
      for (int j = 0; j < nb; ++j) {
        const int st = j % kAttnKS;
        mbar_wait(&kv_empty[st], ((j / kAttnKS) & 1) ^ 1);
        mbar_arrive_expect_tx(&kv_full[st], kKBytes + kVBytes);
        tma_load_2d(smem + L::k + st * kKBytes, &tm_k, &kv_full[st], 0,
                    bh * t_pad + j * 128);
        uint8_t* sv = smem + L::v + st * kVBytes;
        tma_load_2d(sv, &tm_vt, &kv_full[st], j * 128, bh * 64);
        tma_load_2d(sv + 64 * 128, &tm_vt, &kv_full[st], j * 128 + 64, bh * 64);
      }
    }
  } else if (warp == 1) {
    // Issue order per tile t: as soon as softmax_t(j) has published P_t(j)
    // (which also frees S_t): S_t(j + 1), then PV_t(j). Each tile's next
    // scores neither wait on the other tile's softmax nor queue behind PV.
    constexpr uint32_t idesc_s = umma_idesc_bf16(128, 128);
    constexpr uint32_t idesc_o = umma_idesc_bf16(128, 64);
    mbar_wait(q_full, 0);
    auto issue_s = [&](int t, int j) {           // S_t = Q_t K_j^T
      const uint32_t sk = smem_u32(smem + L::k + (j % kAttnKS) * kKBytes);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t sq = smem_u32(smem + L::q + t * kQBytes);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          umma_bf16_ss(tmem + t * 128, umma_desc_sw128(sq + kk * 32),
                       umma_desc_sw128(sk + kk * 32), idesc_s, kk != 0);
        umma_commit(&s_full[t]);
      }
      __syncwarp();
    };
    mbar_wait(&kv_full[0], 0);
    if (lane == 0) ATRACE_E(128 + 0);
    issue_s(0, 0);
    if (lane == 0) ATRACE_E(128 + 32);
    if (NT == 2) issue_s(1, 0);
    for (int j = 0; j < nb; ++j) {
      const int st = j % kAttnKS;
      const uint32_t ph = j & 1;
      const uint32_t sv = smem_u32(smem + L::v + st * kVBytes);
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        // S_t(j + 1) as soon as softmax_t(j) has read S_t(j) out of TMEM (before
        // it finishes P_t(j)): the tile's next scores overlap its own exp/pack
        if (j + 1 < nb) {
          if (t == 0) mbar_wait(&kv_full[(j + 1) % kAttnKS], ((j + 1) / kAttnKS) & 1);
          mbar_wait(&s_empty[t], ph);
          if (lane == 0) ATRACE_E(128 + (t * 16 + j + 1) * 2);
          issue_s(t, j + 1);
        }
        // softmax_t(j) done: P_t(j) written and O_t rescaled if its max moved
        mbar_wait(&p_full[t], ph);
        if (lane == 0) ATRACE_E(128 + (t * 16 + j) * 2 + 1);
        tc_fence_after();
        if (elect_one()) {                   // O_t += P_t V_j (P from TMEM, O in TMEM)
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const uint32_t bb = sv + (kk >> 2) * (64 * 128) + (kk & 3) * 32;
            umma_bf16_ts(tmem + kO + t * 64, tmem + kP + t * 64 + kk * 8, umma_desc_sw128(bb),
                         idesc_o, (j | kk) != 0);
          }
          umma_commit(&o_full[t]);
          if (t == NT - 1) umma_commit(&kv_empty[st]);
        }
        __syncwarp();
      }
    }
  } else {
    const int t = (warp - 2) >> 2;                        // query tile of this warpgroup
    const int quad = warp & 3;
    const int r = quad * 32 + lane;                       // query row in tile
    const uint32_t lane_off = uint32_t(quad * 32) << 16;
    const uint32_t s_col = t * 128, o_col = kO + t * 64, p_col = kP + t * 64;
    constexpr float kLog2e = 1.4426950408889634f;
    // O_t accumulates in TMEM across key blocks. The exponent offset m_run
    // only moves when the block max exceeds it by more than 2^8 (then O_t's
    // row is rescaled in TMEM before the next P.V accumulates): P <= 256 fits
    // bf16, and numerator and row sum share the same offset.
    float m_run = -INFINITY, l_run = 0.f;
    for (int j = 0; j < nb; ++j) {
      mbar_wait(&s_full[t], j & 1);
      if (quad == 0) ATRACE((t * 16 + j) * 4 + 0);
      tc_fence_after();
      const int kvalid = T - j * 128;                     // < 128 only on the tail block
      float alpha = 1.f, m_use = m_run, mscaled = 0.f;
      // exponent offset for this block (and O_t rescale when it moves)
      auto offset = [&](float mx) {
        bool resc = false;
        if (j == 0) {
          m_use = mx;
        } else if ((mx - m_run) * kLog2e > 8.f) {
          alpha = ex2((m_run - mx) * kLog2e);
          m_use = mx;
          resc = true;
        }
        mscaled = m_use * kLog2e;
        if (j >= 1) {
          // PV_t(j - 1) done: P_t is free and O_t holds blocks 0..j-1
          mbar_wait(&o_full[t], (j - 1) & 1);
          tc_fence_after();
          if (__any_sync(0xffffffffu, resc)) {
#pragma unroll 1
            for (int c = 0; c < 2; ++c) {
              uint32_t ov[32];
              tmem_ld32(tmem + lane_off + o_col + c * 32, ov);
              tmem_wait_ld();
#pragma unroll
              for (int i = 0; i < 32; ++i) ov[i] = __float_as_uint(__uint_as_float(ov[i]) * alpha);
              tmem_st32(tmem + lane_off + o_col + c * 32, ov);
            }
            tmem_wait_st();
          }
        }
      };
      // p = exp2(s log2e - m log2e), row sum, bf16 P into TMEM
      float rs0 = 0.f, rs1 = 0.f, rs2 = 0.f, rs3 = 0.f;
      auto emit = [&](int c, const uint32_t (&v)[32], bool full) {
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          float p0, p1;
          if (full) {
            p0 = ex2(fmaf(__uint_as_float(v[2 * i]), kLog2e, -mscaled));
            p1 = ex2(fmaf(__uint_as_float(v[2 * i + 1]), kLog2e, -mscaled));
          } else {
            p0 = (c * 32 + 2 * i < kvalid) ? ex2(fmaf(__uint_as_float(v[2 * i]), kLog2e, -mscaled)) : 0.f;
            p1 = (c * 32 + 2 * i + 1 < kvalid)
                     ? ex2(fmaf(__uint_as_float(v[2 * i + 1]), kLog2e, -mscaled)) : 0.f;
          }
          if (i & 1) { rs2 += p0; rs3 += p1; } else { rs0 += p0; rs1 += p1; }
          pk[i] = pack_bf16x2(p0, p1);
        }
        tmem_st16(tmem + lane_off + p_col + c * 16, pk);   // keys 32c..32c+31
      };
      auto release_s = [&]() {                   // the MMA warp may issue S_t(j + 1)
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_empty[t]);
      };
      if (kvalid >= 128) {
        // the whole S row in registers with one wait; S_t is released at once
        uint32_t s0[32], s1[32], s2[32], s3[32];
        tmem_ld32(tmem + lane_off + s_col, s0);
        tmem_ld32(tmem + lane_off + s_col + 32, s1);
        tmem_ld32(tmem + lane_off + s_col + 64, s2);
        tmem_ld32(tmem + lane_off + s_col + 96, s3);
        tmem_wait_ld();
        release_s();
        if (quad == 0) ATRACE((t * 16 + j) * 4 + 1);
        float m0 = m_run, m1 = m_run, m2 = m_run, m3 = m_run;
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          m0 = fmax3(m0, __uint_as_float(s0[i]), __uint_as_float(s0[i + 1]));
          m1 = fmax3(m1, __uint_as_float(s1[i]), __uint_as_float(s1[i + 1]));
          m2 = fmax3(m2, __uint_as_float(s2[i]), __uint_as_float(s2[i + 1]));
          m3 = fmax3(m3, __uint_as_float(s3[i]), __uint_as_float(s3[i + 1]));
        }
        offset(fmaxf(fmaxf(m0, m1), fmaxf(m2, m3)));
        if (quad == 0) ATRACE((t * 16 + j) * 4 + 2);
        emit(0, s0, true);
        emit(1, s1, true);
        emit(2, s2, true);
        emit(3, s3, true);
      } else {
        uint32_t sr[32];
        float mx = m_run;
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
          tmem_ld32(tmem + lane_off + s_col + c * 32, sr);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (c * 32 + i < kvalid) mx = fmaxf(mx, __uint_as_float(sr[i]));
        }
        offset(mx);
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
          tmem_ld32(tmem + lane_off + s_col + c * 32, sr);
          tmem_wait_ld();
          if (c == 3) release_s();
          emit(c, sr, false);
        }
      }
      const float rs = (rs0 + rs1) + (rs2 + rs3);
      if (quad == 0) ATRACE((t * 16 + j) * 4 + 3);
      tmem_wait_st();
      tc_fence_before();                      // P_t (and an O_t rescale) before the next P.V
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[t]);
      l_run = l_run * alpha + rs;
      m_run = m_use;
    }
    mbar_wait(&o_full[t], (nb - 1) & 1);
    tc_fence_after();
    // normalise and store this query row
    const int tq = qp * 128 * NT + t * 128 + r;
    const float inv = 1.0f / l_run;
    const int b = bh / heads, h = bh % heads;
#pragma unroll 1
    for (int c = 0; c < 2; ++c) {
      uint32_t ov[32];
      tmem_ld32(tmem + lane_off + o_col + c * 32, ov);
      tmem_wait_ld();
      if (tq < T) {
        uint4* dst = reinterpret_cast<uint4*>(out + (size_t(b) * T_rows + tq) * ldo + h * 64 + c * 32);
#pragma unroll
        for (int i = 0; i < 4; ++i)
          dst[i] = make_uint4(
              pack_bf16x2(__uint_as_float(ov[8 * i]) * inv, __uint_as_float(ov[8 * i + 1]) * inv),
              pack_bf16x2(__uint_as_float(ov[8 * i + 2]) * inv, __uint_as_float(ov[8 * i + 3]) * inv),
              pack_bf16x2(__uint_as_float(ov[8 * i + 4]) * inv, __uint_as_float(ov[8 * i + 5]) * inv),
              pack_bf16x2(__uint_as_float(ov[8 * i + 6]) * inv, __uint_as_float(ov[8 * i + 7]) * inv));
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, L::kTmemCols);
  }
}

// ------------------------------------------------------------ LayerNorm
// fp32 rows -> bf16 rows (encoder pre-LN and final LN). One warp per row,
// two-pass mean/variance in registers, eps 1e-5.
template <int V4>  // float4 per lane
__global__ void __launch_bounds__(256)
layernorm_bf16_kernel(const float* __restrict__ x, const uint16_t* __restrict__ g,
                      const uint16_t* __restrict__ bta, uint16_t* __restrict__ y, int rows,
                      int d, float* __restrict__ y32, const int32_t* __restrict__ seg_len,
                      int seg_rows) {
  const int row = blockIdx.x * 8 + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (row >= rows) return;
  if (seg_len && row % seg_rows >= seg_len[row / seg_rows]) return;   // padding row: skipped
  const float4* xr = reinterpret_cast<const float4*>(x + size_t(row) * d);
  const int n4 = d / 4;
  float4 v[V4];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < V4; ++i) {
    int c = lane + 32 * i;
    v[i] = c < n4 ? xr[c] : make_float4(0.f, 0.f, 0.f, 0.f);
    s += (v[i].x + v[i].y) + (v[i].z + v[i].w);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const float mean = s / d;
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < V4; ++i) {
    int c = lane + 32 * i;
    if (c < n4) {
      float a = v[i].x - mean, b = v[i].y - mean, cc = v[i].z - mean, e = v[i].w - mean;
      q += (a * a + b * b) + (cc * cc + e * e);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
  const float rstd = rsqrtf(q / d + 1e-5f);
  uint2* yr = reinterpret_cast<uint2*>(y + size_t(row) * d);
#pragma unroll
  for (int i = 0; i < V4; ++i) {
    int c = lane + 32 * i;
    if (c < n4) {
      const uint2 gw = __ldg(reinterpret_cast<const uint2*>(g) + c);     // 4 bf16 each
      const uint2 bw = __ldg(reinterpret_cast<const uint2*>(bta) + c);
      float o0 = (v[i].x - mean) * rstd * __uint_as_float(gw.x << 16) + __uint_as_float(bw.x << 16);
      float o1 = (v[i].y - mean) * rstd * __uint_as_float(gw.x & 0xFFFF0000u) + __uint_as_float(bw.x & 0xFFFF0000u);
      float o2 = (v[i].z - mean) * rstd * __uint_as_float(gw.y << 16) + __uint_as_float(bw.y << 16);
      float o3 = (v[i].w - mean) * rstd * __uint_as_float(gw.y & 0xFFFF0000u) + __uint_as_float(bw.y & 0xFFFF0000u);
      yr[c] = make_uint2(pack_bf16x2(o0, o1), pack_bf16x2(o2, o3));
      if (y32) reinterpret_cast<float4*>(y32 + size_t(row) * d)[c] = make_float4(o0, o1, o2, o3);
    }
  }
}

int launch_layernorm_bf16(const float* x, const uint16_t* g, const uint16_t* b, uint16_t* y,
                          int rows, int d, cudaStream_t stream, float* y32,
                          const int32_t* seg_len, int seg_rows) {
  DM_REQUIRE(d % 128 == 0 && d <= 1280, "layernorm d must be a multiple of 128, <= 1280");
  dim3 grid(ceil_div(rows, 8));
  const int v4 = d / 128;
  switch (v4) {
#define DM_LN_CASE(n) \
  case n: layernorm_bf16_kernel<n><<<grid, 256, 0, stream>>>(x, g, b, y, rows, d, y32, seg_len, seg_rows); break;
    DM_LN_CASE(1) DM_LN_CASE(2) DM_LN_CASE(3) DM_LN_CASE(4) DM_LN_CASE(5)
    DM_LN_CASE(6) DM_LN_CASE(7) DM_LN_CASE(8) DM_LN_CASE(9) DM_LN_CASE(10)
#undef DM_LN_CASE
    default: DM_REQUIRE(false, "unsupported d");
  }
  DM_CHECK_LAUNCH();
  return 0;
}

// host: tensor maps for Q/K ([BH*Tp, 64]) and V^T ([BH*64, Tp])
int make_attn_maps(const uint16_t* q, const uint16_t* k, const uint16_t* vt, int bh, int t_pad,
                   CUtensorMap* mq, CUtensorMap* mk, CUtensorMap* mv);

int launch_attention(const uint16_t* q, const uint16_t* k, const uint16_t* vt, int n_seg,
                     int heads, int T, int t_pad, uint16_t* out, int ldo, cudaStream_t stream,
                     const int32_t* seg_len) {
  DM_REQUIRE(t_pad % 128 == 0 && t_pad >= T, "t_pad must be a multiple of 128 >= T");
  CUtensorMap mq, mk, mv;
  if (make_attn_maps(q, k, vt, n_seg * heads, t_pad, &mq, &mk, &mv)) return 2;
  // one query tile per CTA, two CTAs per SM (DM_ATTN_NT1_MAX_T: longest T that
  // uses it; experiments)
  static const int nt1_max = std::getenv("DM_ATTN_NT1_MAX_T") ? std::atoi(std::getenv("DM_ATTN_NT1_MAX_T"))
                                                               : 1 << 30;
  if (T <= nt1_max) {
    using L = AttnCfg<1>;
    DM_SMEM_ATTR(attn_tcgen05_kernel<1>, L::total);
    attn_tcgen05_kernel<1><<<dim3(ceil_div(T, 128), n_seg * heads), L::kThreads, L::total, stream>>>(
        mq, mk, mv, T, t_pad, heads, out, ldo, seg_len);
  } else {
    using L = AttnCfg<2>;
    DM_SMEM_ATTR(attn_tcgen05_kernel<2>, L::total);
    attn_tcgen05_kernel<2><<<dim3(ceil_div(T, 256), n_seg * heads), L::kThreads, L::total, stream>>>(
        mq, mk, mv, T, t_pad, heads, out, ldo, seg_len);
  }
  DM_CHECK_LAUNCH();
  return 0;
}

#ifdef DM_ATTN_TRACE
extern "C" __attribute__((visibility("default"))) int dm_attn_trace_read(unsigned long long* host) {
  return (int)cudaMemcpyFromSymbol(host, g_attn_trace, sizeof(g_attn_trace));
}
#endif

}  // namespace dm
