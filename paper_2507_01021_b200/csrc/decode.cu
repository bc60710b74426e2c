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

#include <vector>

namespace dm {

// ============================================================ tcgen05 GEMV
constexpr int kTvThreads = 192;     // w0 TMA, w1 MMA, w2..5 epilogue
constexpr int kTvStages = 3;
constexpr int kTvWBytes = 128 * 64 * 2;   // W tile: 128 rows x 64 k
constexpr int kTvXBytes = kRows * 64 * 2; // X tile: 64 rows x 64 k (hi or lo)
constexpr int kTvStageBytes = kTvWBytes + 2 * kTvXBytes;
constexpr int kTvSmem = kTvStages * kTvStageBytes + 1024 + 128 + 4096;

__device__ __forceinline__ void split_hilo(float v, uint16_t& hi, uint16_t& lo) {
  hi = f32_to_bf16(v);
  lo = f32_to_bf16(v - bf16_to_f32(hi));
}

// Epilogue on 32 rows [r0, r0+32) of one feature column n (values v[0..32)).
template <int EPI>
__device__ __forceinline__ void tv_epilogue32(const DecodeState& st, const TcGemvArgs& a, int n,
                                              bool nvalid, float b, int r0, const float (&v)[32],
                                              const long long* kvbase, float* tr, int f,
                                              int R = kRows) {
  if (EPI != TV_ARGMAX && r0 >= R) return;        // inactive rows: nothing to write
  switch (EPI) {
    case TV_STORE:
      if (nvalid) {
        float* __restrict__ y = a.y + n;
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (r0 + i < R) y[size_t(r0 + i) * a.N] = (v[i] + b) * a.scale;
      }
      break;
    case TV_GELU_HILO:
      if (nvalid) {
        uint16_t* __restrict__ yh = a.yh + n;
        uint16_t* __restrict__ yl = a.yl + n;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          if (r0 + i >= R) continue;
          uint16_t hi, lo;
          split_hilo(gelu_erf(v[i] + b), hi, lo);
          yh[size_t(r0 + i) * a.N] = hi;
          yl[size_t(r0 + i) * a.N] = lo;
        }
      }
      break;
    case TV_RESID:
      if (nvalid) {
        float* __restrict__ y = a.y + n;
        float old[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) old[i] = r0 + i < R ? __ldcg(y + size_t(r0 + i) * a.N) : 0.f;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const float nv = old[i] + (v[i] + b);
          if (r0 + i < R) y[size_t(r0 + i) * a.N] = nv;
          if (tr) tr[(r0 + i) * 129 + f] = nv;     // row statistics for the next LayerNorm
        }
      } else if (tr) {
#pragma unroll
        for (int i = 0; i < 32; ++i) tr[(r0 + i) * 129 + f] = 0.f;
      }
      break;
    case TV_QKV: {
      if (!nvalid) break;
      const int d = st.d;
      if (n < d) {
        float* __restrict__ q = st.q + n;
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (r0 + i < R) q[size_t(r0 + i) * d] = (v[i] + b) * a.scale;
      } else {
        const int kv = n < 2 * d ? 0 : 1;
        const int c = n - (kv + 1) * d;
        const int h = c / 64, j = c % 64;
        const long long col = (long long)(kv * st.heads + h) * st.page_tokens * 64 + j;
        uint16_t* __restrict__ pool = st.kv_pool;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const long long base = kvbase[r0 + i];
          if (base >= 0) pool[base + col] = f32_to_bf16(v[i] + b);
        }
      }
      break;
    }
    case TV_ARGMAX: {
      const int R = *st.n_active;
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const float val = nvalid ? v[i] : -INFINITY;
        tr[(r0 + i) * 129 + f] = val;
        if (st.logits_dbg && nvalid && r0 + i < R)
          st.logits_dbg[size_t(r0 + i) * st.vocab + n] = val;
      }
      break;
    }
  }
}

// Persistent-over-N GEMV: CTA (c, split) owns N tiles c, c + gridDim.x, ...
// for one K split. Its activation operand (all k-blocks of the split, hi and
// lo, <= 128 KB) is loaded once; weight tiles stream through a 3-stage TMA
// ring (the first stages are issued before griddepcontrol.wait: weights never
// depend on the predecessor); accumulators alternate between two 64-column
// TMEM buffers so the epilogue of tile i overlaps the MMAs of tile i + 1.
constexpr int kTvWStages = 3;
constexpr int kTvMaxKb = 8;
__host__ __device__ constexpr int tv_smem_bytes(int kb, bool argmax) {
  return kb * 2 * kTvXBytes + kTvWStages * kTvWBytes + (argmax ? kRows * 129 * 4 : 0) + 1024 + 2048;
}
__host__ __device__ constexpr bool tv_uses_tr(int epi) { return epi == TV_ARGMAX || epi == TV_RESID;
  // (misc: barriers + flags at +0, kvbase[64] at +256, LN stats[64][2] at +768)
}

template <int EPI, bool SPLIT>
__global__ void __launch_bounds__(kTvThreads, 1)
tc_gemv_kernel(const __grid_constant__ CUtensorMap tw, const __grid_constant__ CUtensorMap txh,
               const __grid_constant__ CUtensorMap txl, const DecodeState st,
               const TcGemvArgs a) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024 - (raw_addr & 1023)) & 1023);
  const int kb_per = (a.K / 64) / a.splits;
  uint8_t* xs = smem;                                        // [kb][hi 8K | lo 8K]
  uint8_t* ws = smem + kb_per * 2 * kTvXBytes;               // [stage] 16K
  constexpr bool kTr = EPI == TV_ARGMAX || EPI == TV_RESID;
  float* tr = reinterpret_cast<float*>(ws + kTvWStages * kTvWBytes);   // ARGMAX / RESID stats
  uint8_t* misc = reinterpret_cast<uint8_t*>(tr) + (kTr ? kRows * 129 * 4 : 0);
  uint64_t* wfull = reinterpret_cast<uint64_t*>(misc);
  uint64_t* wempty = wfull + kTvWStages;
  uint64_t* xfull = wempty + kTvWStages;
  uint64_t* tm_full = xfull + 1;                             // [2]
  uint64_t* tm_empty = tm_full + 2;                          // [2]
  uint64_t* xready = tm_empty + 2;                           // fused-LN operand written
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(xready + 1);
  int* is_last = reinterpret_cast<int*>(tmem_slot + 1);
  long long* kvbase = reinterpret_cast<long long*>(misc + 256);
  const bool fused_ln = a.ln_g != nullptr;

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int split = blockIdx.y;
  const int tiles = ceil_div(a.N, 128);
  const int kb0 = split * kb_per;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tw);
    tma_prefetch_desc(&txh);
    tma_prefetch_desc(&txl);
    for (int s = 0; s < kTvWStages; ++s) {
      mbar_init(&wfull[s], 1);
      mbar_init(&wempty[s], 1);
    }
    mbar_init(xfull, 1);
    mbar_init(xready, 4);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tm_full[s], 1);
      mbar_init(&tm_empty[s], 4);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 128);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (elect_one()) {
      // weight stream: independent of the predecessor kernel
      int wi = 0;
      auto issue_w = [&](int tile, int i) {
        const int s = wi % kTvWStages;
        mbar_wait(&wempty[s], ((wi / kTvWStages) & 1) ^ 1);
        mbar_arrive_expect_tx(&wfull[s], kTvWBytes);
        tma_load_2d(ws + s * kTvWBytes, &tw, &wfull[s], (kb0 + i) * 64, tile * 128);
        ++wi;
      };
      const int total = ((tiles - 1 - int(blockIdx.x)) / int(gridDim.x) + 1) * kb_per;
      const int pre = total < kTvWStages ? total : kTvWStages;
      for (int q = 0; q < pre; ++q)
        issue_w(blockIdx.x + (q / kb_per) * gridDim.x, q % kb_per);
      pdl_wait();
      pdl_trigger();
      if (!fused_ln) {
        mbar_arrive_expect_tx(xfull, kb_per * 2 * kTvXBytes);
        for (int i = 0; i < kb_per; ++i) {
          tma_load_2d(xs + i * 2 * kTvXBytes, &txh, xfull, (kb0 + i) * 64, 0);
          tma_load_2d(xs + i * 2 * kTvXBytes + kTvXBytes, &txl, xfull, (kb0 + i) * 64, 0);
        }
      }
      for (int q = pre; q < total; ++q) issue_w(blockIdx.x + (q / kb_per) * gridDim.x, q % kb_per);
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = umma_idesc_bf16(128, kRows);
    mbar_wait(fused_ln ? xready : xfull, 0);
    int wi = 0, it = 0;
    for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++it) {
      const int buf = it & 1;
      mbar_wait(&tm_empty[buf], ((it >> 1) & 1) ^ 1);
      tc_fence_after();
      for (int i = 0; i < kb_per; ++i, ++wi) {
        const int s = wi % kTvWStages;
        mbar_wait(&wfull[s], (wi / kTvWStages) & 1);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t sw = smem_u32(ws + s * kTvWBytes);
          const uint32_t sh = smem_u32(xs + i * 2 * kTvXBytes), sl = sh + kTvXBytes;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            umma_bf16_ss(tmem + buf * 64, umma_desc_sw128(sw + k * 32),
                         umma_desc_sw128(sh + k * 32), idesc, (i | k) != 0);
            umma_bf16_ss(tmem + buf * 64, umma_desc_sw128(sw + k * 32),
                         umma_desc_sw128(sl + k * 32), idesc, 1);
          }
          umma_commit(&wempty[s]);
          if (i == kb_per - 1) umma_commit(&tm_full[buf]);
        }
        __syncwarp();
      }
    }
  } else {
    const int quad = warp & 3;
    const int f = quad * 32 + lane;                // feature within the tile
    const int et = threadIdx.x - 64;               // 0..127 among epilogue threads
    pdl_wait();
    const int R = min(*st.n_active, kRows);
    if (fused_ln) {
      // LayerNorm of the active rows into the 128B-swizzled K-major operand
      // tiles of this CTA's K range. (a) statistics: two threads per row, many
      // independent L2 loads per thread; (b) normalise + split hi/lo + store,
      // one 16-byte chunk per thread per step, coalesced along the row.
      float* stats = reinterpret_cast<float*>(kvbase + kRows);   // [kRows][2]
      const int K = a.K;
      if (et < kRows) {
        // statistics from the producer's per-tile partials (fixed tile order)
        const int r = et, nt = K / 128;
        float s1 = 0.f, s2 = 0.f;
        if (r < R)
          for (int t = 0; t < nt; ++t) {
            s1 += __ldcg(st.ln_part + (size_t(t) * kRows + r) * 2);
            s2 += __ldcg(st.ln_part + (size_t(t) * kRows + r) * 2 + 1);
          }
        const float mean = s1 / K;
        const float var = fmaxf(s2 / K - mean * mean, 0.f);
        stats[2 * r] = mean;
        stats[2 * r + 1] = rsqrtf(var + 1e-5f);
      }
      named_bar_sync(1, 128);
      const int nck = kb_per * 8;                 // 16-byte chunks per row in this K range
#pragma unroll 4
      for (int idx = et; idx < R * nck; idx += 128) {
        const int r = idx / nck, cl = idx % nck;
        const int ci = kb0 * 8 + cl;              // chunk index within the row
        const float4* xr = reinterpret_cast<const float4*>(a.ln_x + size_t(r) * K + ci * 8);
        const float4 x0 = __ldcg(xr), x1 = __ldcg(xr + 1);
        const float e[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
        const float mean = stats[2 * r], rstd = stats[2 * r + 1];
        const uint4 gw = __ldg(reinterpret_cast<const uint4*>(a.ln_g) + ci);
        const uint4 bw = __ldg(reinterpret_cast<const uint4*>(a.ln_b) + ci);
        const uint32_t gs[4] = {gw.x, gw.y, gw.z, gw.w}, bs[4] = {bw.x, bw.y, bw.z, bw.w};
        uint32_t hi[4], lo[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          uint16_t h0, l0, h1, l1;
          split_hilo((e[2 * u] - mean) * rstd * __uint_as_float(gs[u] << 16) +
                         __uint_as_float(bs[u] << 16), h0, l0);
          split_hilo((e[2 * u + 1] - mean) * rstd * __uint_as_float(gs[u] & 0xFFFF0000u) +
                         __uint_as_float(bs[u] & 0xFFFF0000u), h1, l1);
          hi[u] = uint32_t(h0) | (uint32_t(h1) << 16);
          lo[u] = uint32_t(l0) | (uint32_t(l1) << 16);
        }
        const int kb = cl / 8, j = cl % 8;
        uint8_t* tile = xs + kb * 2 * kTvXBytes + r * 128 + ((j ^ (r & 7)) << 4);
        *reinterpret_cast<uint4*>(tile) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
        *reinterpret_cast<uint4*>(tile + kTvXBytes) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(xready);
    }
    if (EPI == TV_QKV) {
      if (et < kRows) {
        long long off = -1;
        if (et < R) {
          const int slot = st.active[et];
          const int p = st.pos[slot];
          const int page = st.page_table[slot * st.pages_per_slot + p / st.page_tokens];
          off = ((long long)(page * st.layers + a.layer) * 2 * st.heads * st.page_tokens +
                 (p % st.page_tokens)) * 64;
        }
        kvbase[et] = off;
      }
      named_bar_sync(1, 128);
    }
    int it = 0;
    for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++it) {
      const int n = tile * 128 + f;
      const bool nvalid = n < a.N;
      const float b = (nvalid && a.bias) ? bf16_to_f32(a.bias[n]) : 0.f;
      const int buf = it & 1;
      mbar_wait(&tm_full[buf], (it >> 1) & 1);
      tc_fence_after();
      float v0[32], v1[32];
      {
        uint32_t rr[32];
        tmem_ld32(tmem + (uint32_t(quad * 32) << 16) + buf * 64, rr);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 32; ++i) v0[i] = __uint_as_float(rr[i]);
        tmem_ld32(tmem + (uint32_t(quad * 32) << 16) + buf * 64 + 32, rr);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 32; ++i) v1[i] = __uint_as_float(rr[i]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tm_empty[buf]);
      if (SPLIT) {
        float* part = st.part;
        const size_t base = (size_t(split) * tiles + tile) * kRows * 128;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          part[base + size_t(i) * 128 + f] = v0[i];
          part[base + size_t(32 + i) * 128 + f] = v1[i];
        }
        __threadfence();
        named_bar_sync(1, 128);
        if (et == 0) {
          const int prev = atomicAdd(&st.counters[a.counter_base + tile], 1);
          *is_last = (prev == a.splits - 1);
        }
        named_bar_sync(1, 128);
        const int last = *is_last;
        named_bar_sync(1, 128);
        if (!last) continue;
        __threadfence();
#pragma unroll
        for (int i = 0; i < 32; ++i) { v0[i] = 0.f; v1[i] = 0.f; }
        for (int s = 0; s < a.splits; ++s) {
          const float* ps = part + (size_t(s) * tiles + tile) * kRows * 128 + f;
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            v0[i] += __ldcg(ps + size_t(i) * 128);
            v1[i] += __ldcg(ps + size_t(32 + i) * 128);
          }
        }
        if (et == 0) st.counters[a.counter_base + tile] = 0;
      }
      float* trp = (EPI == TV_ARGMAX || (EPI == TV_RESID && st.ln_part)) ? tr : nullptr;
      tv_epilogue32<EPI>(st, a, n, nvalid, b, 0, v0, kvbase, trp, f, R);
      tv_epilogue32<EPI>(st, a, n, nvalid, b, 32, v1, kvbase, trp, f, R);
      if (EPI == TV_RESID && st.ln_part) {
        // per-row (sum, sum sq) of the updated residual over this 128-feature tile
        named_bar_sync(1, 128);
        const int r = et >> 1, half = et & 1;
        const float* row = tr + r * 129 + half * 64;
        float s1 = 0.f, s2 = 0.f;
#pragma unroll 8
        for (int i = 0; i < 64; ++i) { s1 += row[i]; s2 += row[i] * row[i]; }
        s1 += __shfl_xor_sync(0xffffffffu, s1, 1);
        s2 += __shfl_xor_sync(0xffffffffu, s2, 1);
        if (half == 0) {
          st.ln_part[(size_t(tile) * kRows + r) * 2] = s1;
          st.ln_part[(size_t(tile) * kRows + r) * 2 + 1] = s2;
        }
        named_bar_sync(1, 128);                    // tr reused by the next tile
      }
      if (EPI == TV_ARGMAX) {
        // per row: max over this tile's 128 vocabulary ids, ties -> lowest id
        named_bar_sync(1, 128);
        const int r = et >> 1, half = et & 1;
        float best = -INFINITY;
        int bidx = 0x7FFFFFFF;
        const float* row = tr + r * 129 + half * 64;
        for (int i = 0; i < 64; ++i) {
          const float x = row[i];
          if (x > best) { best = x; bidx = tile * 128 + half * 64 + i; }
        }
        const float ob = __shfl_xor_sync(0xffffffffu, best, 1);
        const int oi = __shfl_xor_sync(0xffffffffu, bidx, 1);
        if (ob > best || (ob == best && oi < bidx)) { best = ob; bidx = oi; }
        if (half == 0) {
          st.amax_val[size_t(tile) * kRows + r] = best;
          st.amax_idx[size_t(tile) * kRows + r] = bidx;
        }
        named_bar_sync(1, 128);                    // tr reused by the next tile
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 128);
  }
}

// Smallest K split (a divisor of K/64) that leaves <= 8 k-blocks per CTA, so
// the CTA's activation operand fits in shared memory. Depends only on K.
int tc_gemv_splits(int N, int K) {
  (void)N;
  const int kb = K / 64;
  for (int s = 1; s <= kb; ++s)
    if (kb % s == 0 && kb / s <= kTvMaxKb) return s;
  return kb;
}

size_t tc_gemv_part_floats(int N, int K) {
  const int s = tc_gemv_splits(N, K);
  return s > 1 ? size_t(s) * ceil_div(N, 128) * kRows * 128 : 0;
}

template <int EPI, bool SPLIT>
static int launch_tv(const DecodeState& st, const TcGemvMaps& maps, const TcGemvArgs& a,
                     cudaStream_t stream) {
  const int kb_per = (a.K / 64) / a.splits;
  DM_REQUIRE(kb_per <= kTvMaxKb, "decode GEMV: at most 8 k-blocks per split");
  const int smem = tv_smem_bytes(kTvMaxKb, tv_uses_tr(EPI));
  static bool attr = false;
  if (!attr) {
    DM_CHECK_CUDA(cudaFuncSetAttribute(tc_gemv_kernel<EPI, SPLIT>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr = true;
  }
  const int tiles = ceil_div(a.N, 128);
  const int per_split = std::max(1, std::min(tiles, kNumSMs / a.splits));
  dim3 grid(per_split, a.splits);
  DM_CHECK_CUDA(launch_pdl(tc_gemv_kernel<EPI, SPLIT>, grid, dim3(kTvThreads),
                           size_t(tv_smem_bytes(kb_per, tv_uses_tr(EPI))), stream, maps.w,
                           maps.xh, maps.xl, st, a));
  return 0;
}

int launch_tc_gemv(const DecodeState& st, const TcGemvMaps& maps, const TcGemvArgs& a,
                   cudaStream_t stream) {
  DM_REQUIRE(a.K % 64 == 0, "K must be a multiple of 64");
  DM_REQUIRE((a.K / 64) % a.splits == 0, "splits must divide K/64");
  const bool sp = a.splits > 1;
  switch (a.epi) {
    case TV_STORE: return sp ? launch_tv<TV_STORE, true>(st, maps, a, stream)
                             : launch_tv<TV_STORE, false>(st, maps, a, stream);
    case TV_GELU_HILO: return sp ? launch_tv<TV_GELU_HILO, true>(st, maps, a, stream)
                                 : launch_tv<TV_GELU_HILO, false>(st, maps, a, stream);
    case TV_RESID: return sp ? launch_tv<TV_RESID, true>(st, maps, a, stream)
                             : launch_tv<TV_RESID, false>(st, maps, a, stream);
    case TV_QKV: return sp ? launch_tv<TV_QKV, true>(st, maps, a, stream)
                           : launch_tv<TV_QKV, false>(st, maps, a, stream);
    case TV_ARGMAX: return sp ? launch_tv<TV_ARGMAX, true>(st, maps, a, stream)
                              : launch_tv<TV_ARGMAX, false>(st, maps, a, stream);
    default: DM_REQUIRE(false, "unknown epilogue");
  }
}

// ============================================================ LayerNorm
// fp32 residual row -> bf16 hi/lo (the next projection's operand).
template <int V4>
__global__ void __launch_bounds__(256)
decode_ln_kernel(const DecodeState st, const float* __restrict__ x, const uint16_t* g,
                 const uint16_t* b) {
  const int r = blockIdx.x * 8 + threadIdx.x / 32, lane = threadIdx.x % 32;
  pdl_wait();
  pdl_trigger();
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
#define DM_DLN(n) \
  case n: DM_CHECK_CUDA(launch_pdl(decode_ln_kernel<n>, grid, dim3(256), 0, stream, st, x, g, b)); break;
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
  pdl_wait();
  pdl_trigger();
  if (r >= *st.n_active) return;
  const int slot = st.active[r];
  const int tok = st.cur_tok[slot], p = st.pos[slot];
  float s1 = 0.f, s2 = 0.f;
  for (int c = threadIdx.x; c < st.d; c += blockDim.x) {
    const float v =
        bf16_to_f32(embed[size_t(tok) * st.d + c]) + bf16_to_f32(pos_emb[size_t(p) * st.d + c]);
    st.x[size_t(r) * st.d + c] = v;
    s1 += v;
    s2 += v * v;
  }
  if (st.ln_part) {
    // (sum, sum sq) of the row for the fused LayerNorm: per 128-feature tile t,
    // threads t*128 .. own features c = t*128 + threadIdx.x (blockDim == 128)
    __shared__ float red[2][4];
    const int d = st.d, nt = d / 128;
    for (int t = 0; t < nt; ++t) {
      const int c = t * 128 + threadIdx.x;
      float v = 0.f;
      if (c < d)
        v = bf16_to_f32(embed[size_t(tok) * d + c]) + bf16_to_f32(pos_emb[size_t(p) * d + c]);
      float a1 = v, a2 = v * v;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        a1 += __shfl_xor_sync(0xffffffffu, a1, o);
        a2 += __shfl_xor_sync(0xffffffffu, a2, o);
      }
      if ((threadIdx.x & 31) == 0) { red[0][threadIdx.x >> 5] = a1; red[1][threadIdx.x >> 5] = a2; }
      __syncthreads();
      if (threadIdx.x == 0) {
        st.ln_part[(size_t(t) * kRows + r) * 2] = (red[0][0] + red[0][1]) + (red[0][2] + red[0][3]);
        st.ln_part[(size_t(t) * kRows + r) * 2 + 1] = (red[1][0] + red[1][1]) + (red[1][2] + red[1][3]);
      }
      __syncthreads();
    }
  }
  (void)s1; (void)s2;
}

int launch_embed(const DecodeState& st, const uint16_t* embed, const uint16_t* pos_emb,
                 cudaStream_t stream) {
  DM_CHECK_CUDA(launch_pdl(embed_kernel, dim3(kRows), dim3(128), 0, stream, st, embed, pos_emb));
  return 0;
}

// ============================================================ attention
// Lane-per-key online softmax: every lane owns whole keys (64-dim dot product
// and V accumulation in registers, no per-key shuffles); lanes, warps and
// key splits are merged at the end in a fixed order.
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

constexpr int kDaWarps = 4;                    // compute warps (lane = key)
constexpr int kDaThreads = (kDaWarps + 1) * 32; // + 1 TMA producer warp
constexpr int kDaKeys = 128;                    // keys per stage (2 boxes of 64)
constexpr int kDaStages = 3;
constexpr int kDaBox = 64 * 128;                // 64 keys x 128 B
constexpr int kDaStageBytes = 4 * kDaBox;       // K0 K1 V0 V1
constexpr int kDaSmem = kDaStages * kDaStageBytes + 1024 + 2048;

// Cross-warp merge of (m, l, o[64]) through smem; afterwards every lane of
// the calling warps holds dims (2 lane, 2 lane + 1) of the merged state.
__device__ void block_merge(float m, float l, const float (&o)[64], float* smem_o,
                            float* smem_ml, float& mm, float& ll, float& o0, float& o1) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (lane == 0) {
    smem_ml[2 * warp] = m;
    smem_ml[2 * warp + 1] = l;
#pragma unroll
    for (int i = 0; i < 64; ++i) smem_o[warp * 64 + i] = o[i];
  }
  named_bar_sync(1, kDaWarps * 32);
  mm = -INFINITY;
  for (int w = 0; w < kDaWarps; ++w) mm = fmaxf(mm, smem_ml[2 * w]);
  ll = 0.f; o0 = 0.f; o1 = 0.f;
  for (int w = 0; w < kDaWarps; ++w) {
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

// Decode attention for one (row, head[, key split]). K/V tiles stream through
// a 2-stage smem ring by TMA (128B-swizzled, so a lane reading its own key row
// chunk-by-chunk is bank-conflict free while q stays in registers); every
// compute lane owns whole keys. kCross: keys = the slot's 1500 cross-KV rows
// (split over blockIdx.z); else: keys 0..pos of the paged self-KV cache.
template <bool kCross>
__global__ void __launch_bounds__(kDaThreads)
dec_attn_kernel(const __grid_constant__ CUtensorMap tm, const DecodeState st, int layer,
                int counter_base) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024 - (raw_addr & 1023)) & 1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kDaStages * kDaStageBytes);
  uint64_t* empty = full + kDaStages;
  float* s_ml = reinterpret_cast<float*>(empty + kDaStages);     // [2 * warps]
  float* s_o = s_ml + 2 * kDaWarps;                                // [warps * 64]
  int* is_last = reinterpret_cast<int*>(s_o + kDaWarps * 64);

  const int r = blockIdx.x, h = blockIdx.y, sp = blockIdx.z;
  // n_active / active[] are host-set before the step graph: safe before pdl_wait
  if (r >= *st.n_active) return;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int slot = st.active[r];
  if (!kCross) pdl_wait();                 // pos / self-KV come from predecessors
  int k0, k1;
  if (kCross) {
    const int per = ceil_div(ceil_div(1500, st.xsplits), kDaKeys) * kDaKeys;
    k0 = sp * per;
    k1 = min(1500, k0 + per);
  } else {
    k0 = 0;
    k1 = st.pos[slot] + 1;
  }
  const int nchunks = k1 > k0 ? ceil_div(k1 - k0, kDaKeys) : 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kDaStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kDaWarps);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == kDaWarps) {
    // ---------------- TMA producer
    if (elect_one()) {
      tma_prefetch_desc(&tm);
      const int* pt = st.page_table + slot * st.pages_per_slot;
      for (int c = 0; c < nchunks; ++c) {
        const int s = c % kDaStages;
        mbar_wait(&empty[s], ((c / kDaStages) & 1) ^ 1);
        uint8_t* base = smem + s * kDaStageBytes;
        mbar_arrive_expect_tx(&full[s], kDaStageBytes);
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          const int t = k0 + c * kDaKeys + half * 64;
          int row_k, row_v;
          if (kCross) {
            row_k = (((layer * st.max_slots + slot) * 2 + 0) * st.heads + h) * 1500 + t;
            row_v = row_k + st.heads * 1500;
          } else {
            const int page = pt[min(t / st.page_tokens, st.pages_per_slot - 1)];
            row_k = (((page * st.layers + layer) * 2 + 0) * st.heads + h) * st.page_tokens;
            row_v = row_k + st.heads * st.page_tokens;
          }
          tma_load_2d(base + half * kDaBox, &tm, &full[s], 0, row_k);
          tma_load_2d(base + (2 + half) * kDaBox, &tm, &full[s], 0, row_v);
        }
      }
    }
    return;
  }

  // ---------------- compute warps: lane owns key (chunk base + 32 warp + lane)
  if (kCross) pdl_wait();                  // q comes from the predecessor
  pdl_trigger();
  float q[64];
  {
    const float4* qp = reinterpret_cast<const float4*>(st.q + size_t(r) * st.d + h * 64);
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      const float4 v = qp[c];
      q[4 * c] = v.x; q[4 * c + 1] = v.y; q[4 * c + 2] = v.z; q[4 * c + 3] = v.w;
    }
  }
  float m = -INFINITY, l = 0.f, o[64];
#pragma unroll
  for (int i = 0; i < 64; ++i) o[i] = 0.f;
  const int half = warp >> 1;
  const int rr = (warp & 1) * 32 + lane;              // row within the 64-key box
  const int sw = rr & 7;                              // 128B swizzle phase
  for (int c = 0; c < nchunks; ++c) {
    const int s = c % kDaStages;
    mbar_wait(&full[s], (c / kDaStages) & 1);
    const int t = k0 + c * kDaKeys + warp * 32 + lane;
    if (t < k1) {
      const uint8_t* krow = smem + s * kDaStageBytes + half * kDaBox + rr * 128;
      const uint8_t* vrow = krow + 2 * kDaBox;
      float sc = 0.f;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint4 w = *reinterpret_cast<const uint4*>(krow + ((j ^ sw) << 4));
        const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          sc = fmaf(q[8 * j + 2 * u], __uint_as_float(ws[u] << 16), sc);
          sc = fmaf(q[8 * j + 2 * u + 1], __uint_as_float(ws[u] & 0xFFFF0000u), sc);
        }
      }
      const float mn = fmaxf(m, sc);
      const float corr = exp2f((m - mn) * kLog2e);
      const float p = exp2f((sc - mn) * kLog2e);
      l = l * corr + p;
      m = mn;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint4 w = *reinterpret_cast<const uint4*>(vrow + ((j ^ sw) << 4));
        const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          o[8 * j + 2 * u] = fmaf(o[8 * j + 2 * u], corr, p * __uint_as_float(ws[u] << 16));
          o[8 * j + 2 * u + 1] =
              fmaf(o[8 * j + 2 * u + 1], corr, p * __uint_as_float(ws[u] & 0xFFFF0000u));
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  warp_merge(m, l, o);
  float mm, ll, o0, o1;
  block_merge(m, l, o, s_o, s_ml, mm, ll, o0, o1);
  if (!kCross || st.xsplits == 1) {
    if (warp == 0) store_hilo2(st, r, h, lane, o0 / ll, o1 / ll);
    return;
  }
  // split partial -> scratch [row][h][split][66]; last split CTA merges in order
  const int xs = st.xsplits;
  float* part = st.part + ((size_t(r) * st.heads + h) * xs + sp) * 66;
  if (warp == 0) {
    part[2 + 2 * lane] = o0;
    part[3 + 2 * lane] = o1;
    if (lane == 0) { part[0] = mm; part[1] = ll; }
    __threadfence();
  }
  named_bar_sync(1, kDaWarps * 32);
  if (threadIdx.x == 0) {
    const int prev = atomicAdd(&st.counters[counter_base + r * st.heads + h], 1);
    *is_last = prev == xs - 1;
  }
  named_bar_sync(1, kDaWarps * 32);
  if (!*is_last || warp != 0) return;
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

int launch_self_attn(const DecodeState& st, const CUtensorMap& kv_map, int layer,
                     cudaStream_t stream) {
  static bool attr = false;
  if (!attr) {
    DM_CHECK_CUDA(cudaFuncSetAttribute(dec_attn_kernel<false>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, kDaSmem));
    attr = true;
  }
  dim3 grid(kRows, st.heads, 1);
  DM_CHECK_CUDA(launch_pdl(dec_attn_kernel<false>, grid, dim3(kDaThreads), kDaSmem, stream, kv_map,
                           st, layer, 0));
  return 0;
}

int launch_cross_attn(const DecodeState& st, const CUtensorMap& xkv_map, int layer,
                      int counter_base, cudaStream_t stream) {
  static bool attr = false;
  if (!attr) {
    DM_CHECK_CUDA(cudaFuncSetAttribute(dec_attn_kernel<true>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, kDaSmem));
    attr = true;
  }
  dim3 grid(kRows, st.heads, st.xsplits);
  DM_CHECK_CUDA(launch_pdl(dec_attn_kernel<true>, grid, dim3(kDaThreads), kDaSmem, stream, xkv_map,
                           st, layer, counter_base));
  return 0;
}

// ============================================================ finalize
// One warp per active row: argmax over the vocab-tile partials (ties -> lowest
// id), then the greedy state machine (prompt forcing, EOT, per-slot cap).
__global__ void finalize_kernel(const DecodeState st) {
  const int r = blockIdx.x * 4 + threadIdx.x / 32, lane = threadIdx.x % 32;
  pdl_wait();
  pdl_trigger();
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
  DM_CHECK_CUDA(launch_pdl(finalize_kernel, dim3(kRows / 4), dim3(128), 0, stream, st));
  return 0;
}



// ============================================================ persistent decode
// One cooperative CTA per SM runs whole greedy decode steps: every phase of
// the step (embed, per layer LN / QKV / self-attn / O / LN / cross-q /
// cross-attn / cross-o / LN / fc1 / fc2, final LN, LM head, finalize) is a
// list of work items spread over the CTAs, separated by grid barriers. This
// removes the ~70 dependent kernel launches (and their TMEM allocation,
// barrier setup and tail) per step; the TMA ring, the two TMEM accumulators
// and all mbarriers persist across phases and steps. Per-item arithmetic is
// identical to the standalone kernels above (same fixed reduction orders).
constexpr int kMkThreads = 256;          // w0 TMA, w1 MMA, w4..7 epilogue / attention roles
constexpr int kMkStages = 3;
constexpr int kMkStage = 32768;          // GEMV: W 16K + Xh 8K + Xl 8K; attention: K0 K1 V0 V1
constexpr int kMkTr = kRows * 129 * 4;   // argmax transpose
constexpr int kMkSmem = kMkStages * kMkStage + kMkTr + 4096 + 1024;

struct MkLayerW {
  const uint16_t *ln1g, *ln1b, *qkvb, *ob, *ln2g, *ln2b, *xqb, *xob, *ln3g, *ln3b, *fc1b, *fc2b;
};

struct MkParams {
  DecodeState st;
  const TcGemvMaps* maps;          // device [Ld * 6 + 1]
  const CUtensorMap* attn_maps;    // device [2]: self-KV pool, cross-KV cache
  const MkLayerW* lw;              // device [Ld]
  const uint16_t *lnfg, *lnfb, *embed, *pos_emb;
  unsigned* gbar;                  // grid barrier counter, zero at launch
  unsigned long long* timing;      // optional: globaltimer at each barrier (block 0)
  int n_steps;
  int sp_qkv, sp_dd, sp_fc1, sp_fc2;
};

struct MkBars {
  uint64_t full[kMkStages], empty[kMkStages];
  uint64_t tm_full[2], tm_empty[2];
  uint64_t afull[kMkStages], aempty[kMkStages];
  uint32_t tmem;
  int flag;
};

struct MkRing {
  int p = 0, m = 0, mn = 0, en = 0, ap = 0, ac = 0;
};

__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

__device__ __forceinline__ void mk_grid_sync(unsigned* bar, unsigned& target,
                                             unsigned long long* timing = nullptr) {
  // bar.sync orders the CTA's phase writes before thread 0's release-add
  // (cumulative at gpu scope); thread 0's acquire-load + bar.sync orders every
  // thread's next-phase reads after all CTAs' writes. Cross-CTA data is read
  // with ld.global.cg or TMA (L2), never through a possibly stale L1 line.
  __syncthreads();
  if (threadIdx.x == 0) {
    target += gridDim.x;
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
    unsigned v;
    long long spins = 0;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
      if (++spins > (1ll << 30)) asm volatile("trap;");
    } while (v < target);
    if (timing && blockIdx.x == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
      timing[target / gridDim.x - 1] = t;
    }
  }
  __syncthreads();
}

// LN of row r: fp32 x -> bf16 hi/lo (runtime d <= 1280)
__device__ __forceinline__ void mk_ln_row(const DecodeState& st, int r, const uint16_t* g,
                                          const uint16_t* b) {
  const int lane = threadIdx.x % 32, d = st.d, n4 = d / 4;
  const float4* xr = reinterpret_cast<const float4*>(st.x + size_t(r) * d);
  float4 v[10];
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 10; ++k) {
    const int c = lane + 32 * k;
    v[k] = c < n4 ? __ldcg(xr + c) : make_float4(0.f, 0.f, 0.f, 0.f);
    s += (v[k].x + v[k].y) + (v[k].z + v[k].w);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const float mean = s / d;
  float q = 0.f;
#pragma unroll
  for (int k = 0; k < 10; ++k) {
    const int c = lane + 32 * k;
    if (c < n4) {
      const float a0 = v[k].x - mean, a1 = v[k].y - mean, a2 = v[k].z - mean, a3 = v[k].w - mean;
      q += (a0 * a0 + a1 * a1) + (a2 * a2 + a3 * a3);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
  const float rstd = rsqrtf(q / d + 1e-5f);
  uint2* yh = reinterpret_cast<uint2*>(st.xh + size_t(r) * d);
  uint2* yl = reinterpret_cast<uint2*>(st.xl + size_t(r) * d);
#pragma unroll
  for (int k = 0; k < 10; ++k) {
    const int c = lane + 32 * k;
    if (c < n4) {
      const float o[4] = {v[k].x, v[k].y, v[k].z, v[k].w};
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

__device__ __noinline__ void mk_ln_phase(const DecodeState& st, int R, const uint16_t* g,
                                            const uint16_t* b) {
  const int gw = blockIdx.x * (kMkThreads / 32) + threadIdx.x / 32;
  for (int r = gw; r < R; r += gridDim.x * (kMkThreads / 32)) mk_ln_row(st, r, g, b);
}

__device__ __forceinline__ void mk_embed_phase(const MkParams& P, int R) {
  const DecodeState& st = P.st;
  const int gw = blockIdx.x * (kMkThreads / 32) + threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int r = gw; r < R; r += gridDim.x * (kMkThreads / 32)) {
    const int slot = st.active[r];
    const int tok = __ldcg(st.cur_tok + slot), p = __ldcg(st.pos + slot);
    for (int c = lane; c < st.d; c += 32)
      st.x[size_t(r) * st.d + c] =
          bf16_to_f32(P.embed[size_t(tok) * st.d + c]) + bf16_to_f32(P.pos_emb[size_t(p) * st.d + c]);
  }
}

__device__ __forceinline__ void mk_finalize_phase(const DecodeState& st, int R) {
  const int gw = blockIdx.x * (kMkThreads / 32) + threadIdx.x / 32, lane = threadIdx.x % 32;
  const int tiles = ceil_div(st.vocab, 128);
  for (int r = gw; r < R; r += gridDim.x * (kMkThreads / 32)) {
    const int slot = st.active[r];
    float best = -INFINITY;
    int bidx = 0x7FFFFFFF;
    for (int t = lane; t < tiles; t += 32) {
      const float v = __ldcg(st.amax_val + size_t(t) * kRows + r);
      const int id = __ldcg(st.amax_idx + size_t(t) * kRows + r);
      if (v > best || (v == best && id < bidx)) { best = v; bidx = id; }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const float ob = __shfl_xor_sync(0xffffffffu, best, off);
      const int oi = __shfl_xor_sync(0xffffffffu, bidx, off);
      if (ob > best || (ob == best && oi < bidx)) { best = ob; bidx = oi; }
    }
    if (lane != 0 || __ldcg(st.done + slot)) continue;
    const int p = __ldcg(st.pos + slot);
    if (p + 1 < st.prompt_len) {
      st.cur_tok[slot] = st.prompt[p + 1];
      st.pos[slot] = p + 1;
      continue;
    }
    if (bidx == st.eot) { st.done[slot] = 1; continue; }
    const int g = __ldcg(st.n_gen + slot);
    st.out_tokens[slot * 448 + g] = bidx;
    st.n_gen[slot] = g + 1;
    if (g + 1 >= __ldcg(st.cap + slot)) { st.done[slot] = 1; continue; }
    st.cur_tok[slot] = bidx;
    st.pos[slot] = p + 1;
  }
}

template <int EPI, bool SPLIT>
__device__ __noinline__ void mk_gemv(const DecodeState& st, const TcGemvMaps* maps, const TcGemvArgs& a,
                        uint8_t* smem, MkBars& B, MkRing& rg, float* tr, long long* kvbase, int R) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int tiles = ceil_div(a.N, 128), items = tiles * a.splits;
  const int kb_per = (a.K / 64) / a.splits;
  if (warp == 0) {
    if (lane == 0) {
      fence_proxy_async_global();          // activations written by generic stores
      for (int item = blockIdx.x; item < items; item += gridDim.x) {
        const int tile = item % tiles, split = item / tiles;
        for (int i = 0; i < kb_per; ++i, ++rg.p) {
          const int s = rg.p % kMkStages;
          mbar_wait(&B.empty[s], ((rg.p / kMkStages) & 1) ^ 1);
          uint8_t* base = smem + s * kMkStage;
          mbar_arrive_expect_tx(&B.full[s], kMkStage);
          const int kc = (split * kb_per + i) * 64;
          tma_load_2d(base, &maps->w, &B.full[s], kc, tile * 128);
          tma_load_2d(base + kTvWBytes, &maps->xh, &B.full[s], kc, 0);
          tma_load_2d(base + kTvWBytes + kTvXBytes, &maps->xl, &B.full[s], kc, 0);
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = umma_idesc_bf16(128, kRows);
    for (int item = blockIdx.x; item < items; item += gridDim.x, ++rg.mn) {
      const int buf = rg.mn & 1;
      mbar_wait(&B.tm_empty[buf], ((rg.mn >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = B.tmem + buf * 64;
      for (int i = 0; i < kb_per; ++i, ++rg.m) {
        const int s = rg.m % kMkStages;
        mbar_wait(&B.full[s], (rg.m / kMkStages) & 1);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t sw = smem_u32(smem + s * kMkStage);
          const uint32_t sh = sw + kTvWBytes, sl = sh + kTvXBytes;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            umma_bf16_ss(d_tmem, umma_desc_sw128(sw + k * 32), umma_desc_sw128(sh + k * 32), idesc,
                         (i | k) != 0);
            umma_bf16_ss(d_tmem, umma_desc_sw128(sw + k * 32), umma_desc_sw128(sl + k * 32), idesc, 1);
          }
          umma_commit(&B.empty[s]);
          if (i == kb_per - 1) umma_commit(&B.tm_full[buf]);
        }
        __syncwarp();
      }
    }
  } else if (warp >= 4) {
    const int quad = warp & 3;
    const int f = quad * 32 + lane;
    const int et = threadIdx.x - 128;                  // 0..127
    if (EPI == TV_QKV) {
      if (et < kRows) {
        long long off = -1;
        if (et < R) {
          const int slot = st.active[et];
          const int p = __ldcg(st.pos + slot);
          const int page = st.page_table[slot * st.pages_per_slot + p / st.page_tokens];
          off = ((long long)(page * st.layers + a.layer) * 2 * st.heads * st.page_tokens +
                 (p % st.page_tokens)) * 64;
        }
        kvbase[et] = off;
      }
      named_bar_sync(1, 128);
    }
    for (int item = blockIdx.x; item < items; item += gridDim.x, ++rg.en) {
      const int tile = item % tiles, split = item / tiles;
      const int n = tile * 128 + f;
      const bool nvalid = n < a.N;
      const float b = (nvalid && a.bias) ? bf16_to_f32(a.bias[n]) : 0.f;
      const int buf = rg.en & 1;
      mbar_wait(&B.tm_full[buf], (rg.en >> 1) & 1);
      tc_fence_after();
      float v0[32], v1[32];
      {
        uint32_t rr[32];
        tmem_ld32(B.tmem + (uint32_t(quad * 32) << 16) + buf * 64, rr);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 32; ++i) v0[i] = __uint_as_float(rr[i]);
        tmem_ld32(B.tmem + (uint32_t(quad * 32) << 16) + buf * 64 + 32, rr);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 32; ++i) v1[i] = __uint_as_float(rr[i]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&B.tm_empty[buf]);
      if (SPLIT) {
        float* part = st.part;
        const size_t base = (size_t(split) * tiles + tile) * kRows * 128;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          part[base + size_t(i) * 128 + f] = v0[i];
          part[base + size_t(32 + i) * 128 + f] = v1[i];
        }
        __threadfence();
        named_bar_sync(1, 128);
        if (et == 0) {
          const int prev = atomicAdd(&st.counters[a.counter_base + tile], 1);
          B.flag = (prev == a.splits - 1);
        }
        named_bar_sync(1, 128);
        const int last = B.flag;
        named_bar_sync(1, 128);                      // flag consumed before the next item
        if (!last) continue;
        __threadfence();
#pragma unroll
        for (int i = 0; i < 32; ++i) { v0[i] = 0.f; v1[i] = 0.f; }
        for (int s = 0; s < a.splits; ++s) {
          const float* ps = part + (size_t(s) * tiles + tile) * kRows * 128 + f;
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            v0[i] += __ldcg(ps + size_t(i) * 128);
            v1[i] += __ldcg(ps + size_t(32 + i) * 128);
          }
        }
        if (et == 0) st.counters[a.counter_base + tile] = 0;
      }
      tv_epilogue32<EPI>(st, a, n, nvalid, b, 0, v0, kvbase, tr, f);
      tv_epilogue32<EPI>(st, a, n, nvalid, b, 32, v1, kvbase, tr, f);
      if (EPI == TV_ARGMAX) {
        named_bar_sync(1, 128);
        const int r = et >> 1, half = et & 1;
        float best = -INFINITY;
        int bidx = 0x7FFFFFFF;
        const float* row = tr + r * 129 + half * 64;
        for (int i = 0; i < 64; ++i) {
          const float x = row[i];
          if (x > best) { best = x; bidx = tile * 128 + half * 64 + i; }
        }
        const float ob = __shfl_xor_sync(0xffffffffu, best, 1);
        const int oi = __shfl_xor_sync(0xffffffffu, bidx, 1);
        if (ob > best || (ob == best && oi < bidx)) { best = ob; bidx = oi; }
        if (half == 0) {
          st.amax_val[size_t(tile) * kRows + r] = best;
          st.amax_idx[size_t(tile) * kRows + r] = bidx;
        }
        named_bar_sync(1, 128);                      // tr reused by the next item
      }
    }
  }
}

template <bool kCross>
__device__ __noinline__ void mk_attn(const DecodeState& st, const CUtensorMap* tm, int layer, uint8_t* smem,
                        MkBars& B, MkRing& rg, float* s_o, float* s_ml, int counter_base, int R) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int xs = kCross ? st.xsplits : 1;
  const int items = R * st.heads * xs;
  for (int item = blockIdx.x; item < items; item += gridDim.x) {
    const int r = item / (st.heads * xs), h = (item / xs) % st.heads, sp = item % xs;
    const int slot = st.active[r];
    int k0, k1;
    if (kCross) {
      const int per = ceil_div(ceil_div(1500, xs), kDaKeys) * kDaKeys;
      k0 = sp * per;
      k1 = min(1500, k0 + per);
    } else {
      k0 = 0;
      k1 = __ldcg(st.pos + slot) + 1;
    }
    const int nchunks = k1 > k0 ? ceil_div(k1 - k0, kDaKeys) : 0;
    if (warp == kDaWarps) {
      if (lane == 0) {
        fence_proxy_async_global();
        const int* pt = st.page_table + slot * st.pages_per_slot;
        for (int c = 0; c < nchunks; ++c, ++rg.ap) {
          const int s = rg.ap % kMkStages;
          mbar_wait(&B.aempty[s], ((rg.ap / kMkStages) & 1) ^ 1);
          uint8_t* base = smem + s * kMkStage;
          mbar_arrive_expect_tx(&B.afull[s], kDaStageBytes);
#pragma unroll
          for (int half = 0; half < 2; ++half) {
            const int t = k0 + c * kDaKeys + half * 64;
            int row_k, row_v;
            if (kCross) {
              row_k = (((layer * st.max_slots + slot) * 2 + 0) * st.heads + h) * 1500 + t;
              row_v = row_k + st.heads * 1500;
            } else {
              const int page = pt[min(t / st.page_tokens, st.pages_per_slot - 1)];
              row_k = (((page * st.layers + layer) * 2 + 0) * st.heads + h) * st.page_tokens;
              row_v = row_k + st.heads * st.page_tokens;
            }
            tma_load_2d(base + half * kDaBox, tm, &B.afull[s], 0, row_k);
            tma_load_2d(base + (2 + half) * kDaBox, tm, &B.afull[s], 0, row_v);
          }
        }
      }
      continue;
    }
    if (warp > kDaWarps) continue;
    float q[64];
    {
      const float4* qp = reinterpret_cast<const float4*>(st.q + size_t(r) * st.d + h * 64);
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        const float4 v = __ldcg(qp + c);
        q[4 * c] = v.x; q[4 * c + 1] = v.y; q[4 * c + 2] = v.z; q[4 * c + 3] = v.w;
      }
    }
    float m = -INFINITY, l = 0.f, o[64];
#pragma unroll
    for (int i = 0; i < 64; ++i) o[i] = 0.f;
    const int half = warp >> 1;
    const int rr = (warp & 1) * 32 + lane;
    const int sw = rr & 7;
    for (int c = 0; c < nchunks; ++c, ++rg.ac) {
      const int s = rg.ac % kMkStages;
      mbar_wait(&B.afull[s], (rg.ac / kMkStages) & 1);
      const int t = k0 + c * kDaKeys + warp * 32 + lane;
      if (t < k1) {
        const uint8_t* krow = smem + s * kMkStage + half * kDaBox + rr * 128;
        const uint8_t* vrow = krow + 2 * kDaBox;
        float sc = 0.f;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint4 w = *reinterpret_cast<const uint4*>(krow + ((j ^ sw) << 4));
          const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            sc = fmaf(q[8 * j + 2 * u], __uint_as_float(ws[u] << 16), sc);
            sc = fmaf(q[8 * j + 2 * u + 1], __uint_as_float(ws[u] & 0xFFFF0000u), sc);
          }
        }
        const float mn = fmaxf(m, sc);
        const float corr = exp2f((m - mn) * kLog2e);
        const float p = exp2f((sc - mn) * kLog2e);
        l = l * corr + p;
        m = mn;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint4 w = *reinterpret_cast<const uint4*>(vrow + ((j ^ sw) << 4));
          const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            o[8 * j + 2 * u] = fmaf(o[8 * j + 2 * u], corr, p * __uint_as_float(ws[u] << 16));
            o[8 * j + 2 * u + 1] =
                fmaf(o[8 * j + 2 * u + 1], corr, p * __uint_as_float(ws[u] & 0xFFFF0000u));
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&B.aempty[s]);
    }
    warp_merge(m, l, o);
    float mm, ll, o0, o1;
    block_merge(m, l, o, s_o, s_ml, mm, ll, o0, o1);
    if (!kCross || xs == 1) {
      if (warp == 0) store_hilo2(st, r, h, lane, o0 / ll, o1 / ll);
    } else {
      float* part = st.part + ((size_t(r) * st.heads + h) * xs + sp) * 66;
      if (warp == 0) {
        part[2 + 2 * lane] = o0;
        part[3 + 2 * lane] = o1;
        if (lane == 0) { part[0] = mm; part[1] = ll; }
        __threadfence();
      }
      named_bar_sync(1, kDaWarps * 32);
      if (threadIdx.x == 0) {
        const int prev = atomicAdd(&st.counters[counter_base + r * st.heads + h], 1);
        B.flag = prev == xs - 1;
      }
      named_bar_sync(1, kDaWarps * 32);
      if (B.flag && warp == 0) {
        __threadfence();
        const float* pb = st.part + (size_t(r) * st.heads + h) * xs * 66;
        float gm = -INFINITY;
        for (int s = 0; s < xs; ++s) gm = fmaxf(gm, __ldcg(pb + s * 66));
        float gl = 0.f, g0 = 0.f, g1 = 0.f;
        for (int s = 0; s < xs; ++s) {
          const float ms = __ldcg(pb + s * 66);
          const float fct = (ms == -INFINITY) ? 0.f : exp2f((ms - gm) * kLog2e);
          gl += __ldcg(pb + s * 66 + 1) * fct;
          g0 += __ldcg(pb + s * 66 + 2 + 2 * lane) * fct;
          g1 += __ldcg(pb + s * 66 + 3 + 2 * lane) * fct;
        }
        store_hilo2(st, r, h, lane, g0 / gl, g1 / gl);
        if (lane == 0) st.counters[counter_base + r * st.heads + h] = 0;
      }
    }
    named_bar_sync(1, kDaWarps * 32);                // s_o / s_ml / flag reused next item
  }
}

__global__ void __launch_bounds__(kMkThreads, 1) decode_mega_kernel(const MkParams P) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024 - (raw_addr & 1023)) & 1023);
  float* tr = reinterpret_cast<float*>(smem + kMkStages * kMkStage);
  uint8_t* misc = smem + kMkStages * kMkStage + kMkTr;
  MkBars& B = *reinterpret_cast<MkBars*>(misc);
  long long* kvbase = reinterpret_cast<long long*>(misc + 512);
  float* s_o = reinterpret_cast<float*>(misc + 1024);          // [4 * 64]
  float* s_ml = s_o + 4 * 64;                                   // [8]
  const DecodeState& st = P.st;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kMkStages; ++s) {
      mbar_init(&B.full[s], 1);
      mbar_init(&B.empty[s], 1);
      mbar_init(&B.afull[s], 1);
      mbar_init(&B.aempty[s], kDaWarps);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&B.tm_full[s], 1);
      mbar_init(&B.tm_empty[s], 4);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(&B.tmem, 128);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  MkRing rg;
  unsigned target = 0;
  const int R = min(*st.n_active, kRows);
  const int d = st.d, F = st.ffn;
  for (int step = 0; step < P.n_steps; ++step) {
    mk_embed_phase(P, R);
    mk_grid_sync(P.gbar, target, P.timing);
    for (int l = 0; l < st.layers; ++l) {
      const MkLayerW& w = P.lw[l];
      const TcGemvMaps* m = P.maps + size_t(l) * 6;
      TcGemvArgs a{};
      a.layer = l;
      a.counter_base = 0;
      mk_ln_phase(st, R, w.ln1g, w.ln1b);
      mk_grid_sync(P.gbar, target, P.timing);
      a.bias = w.qkvb; a.N = 3 * d; a.K = d; a.scale = 0.125f; a.splits = P.sp_qkv;
      if (a.splits > 1) mk_gemv<TV_QKV, true>(st, m + 0, a, smem, B, rg, tr, kvbase, R);
      else mk_gemv<TV_QKV, false>(st, m + 0, a, smem, B, rg, tr, kvbase, R);
      mk_grid_sync(P.gbar, target, P.timing);
      mk_attn<false>(st, &P.attn_maps[0], l, smem, B, rg, s_o, s_ml, 4096, R);
      mk_grid_sync(P.gbar, target, P.timing);
      a.bias = w.ob; a.N = d; a.K = d; a.scale = 1.f; a.splits = P.sp_dd; a.y = st.x;
      if (a.splits > 1) mk_gemv<TV_RESID, true>(st, m + 1, a, smem, B, rg, tr, kvbase, R);
      else mk_gemv<TV_RESID, false>(st, m + 1, a, smem, B, rg, tr, kvbase, R);
      mk_grid_sync(P.gbar, target, P.timing);
      mk_ln_phase(st, R, w.ln2g, w.ln2b);
      mk_grid_sync(P.gbar, target, P.timing);
      a.bias = w.xqb; a.scale = 0.125f; a.y = st.q;
      if (a.splits > 1) mk_gemv<TV_STORE, true>(st, m + 2, a, smem, B, rg, tr, kvbase, R);
      else mk_gemv<TV_STORE, false>(st, m + 2, a, smem, B, rg, tr, kvbase, R);
      mk_grid_sync(P.gbar, target, P.timing);
      mk_attn<true>(st, &P.attn_maps[1], l, smem, B, rg, s_o, s_ml, 4096, R);
      mk_grid_sync(P.gbar, target, P.timing);
      a.bias = w.xob; a.scale = 1.f; a.y = st.x;
      if (a.splits > 1) mk_gemv<TV_RESID, true>(st, m + 3, a, smem, B, rg, tr, kvbase, R);
      else mk_gemv<TV_RESID, false>(st, m + 3, a, smem, B, rg, tr, kvbase, R);
      mk_grid_sync(P.gbar, target, P.timing);
      mk_ln_phase(st, R, w.ln3g, w.ln3b);
      mk_grid_sync(P.gbar, target, P.timing);
      a.bias = w.fc1b; a.N = F; a.K = d; a.splits = P.sp_fc1; a.yh = st.hh; a.yl = st.hl;
      if (a.splits > 1) mk_gemv<TV_GELU_HILO, true>(st, m + 4, a, smem, B, rg, tr, kvbase, R);
      else mk_gemv<TV_GELU_HILO, false>(st, m + 4, a, smem, B, rg, tr, kvbase, R);
      mk_grid_sync(P.gbar, target, P.timing);
      a.bias = w.fc2b; a.N = d; a.K = F; a.splits = P.sp_fc2; a.y = st.x;
      if (a.splits > 1) mk_gemv<TV_RESID, true>(st, m + 5, a, smem, B, rg, tr, kvbase, R);
      else mk_gemv<TV_RESID, false>(st, m + 5, a, smem, B, rg, tr, kvbase, R);
      mk_grid_sync(P.gbar, target, P.timing);
    }
    mk_ln_phase(st, R, P.lnfg, P.lnfb);
    mk_grid_sync(P.gbar, target, P.timing);
    {
      TcGemvArgs a{};
      a.N = st.vocab; a.K = d; a.scale = 1.f; a.splits = 1;
      mk_gemv<TV_ARGMAX, false>(st, P.maps + size_t(st.layers) * 6, a, smem, B, rg, tr, kvbase, R);
    }
    mk_grid_sync(P.gbar, target, P.timing);
    mk_finalize_phase(st, R);
    mk_grid_sync(P.gbar, target, P.timing);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(B.tmem, 128);
  }
}

int launch_decode_mega(const MkParams& P, cudaStream_t stream);

__global__ void __launch_bounds__(kMkThreads, 1) grid_barrier_bench_kernel(unsigned* bar, int iters) {
  unsigned target = 0;
  for (int i = 0; i < iters; ++i) mk_grid_sync(bar, target);
}

int bench_grid_barrier(int iters, float* us_per_barrier) {
  unsigned* bar = nullptr;
  DM_CHECK_CUDA(cudaMalloc(&bar, 256));
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    DM_CHECK_CUDA(cudaMemset(bar, 0, 256));
    cudaEvent_t a, b;
    DM_CHECK_CUDA(cudaEventCreate(&a));
    DM_CHECK_CUDA(cudaEventCreate(&b));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(kNumSMs);
    cfg.blockDim = dim3(kMkThreads);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    DM_CHECK_CUDA(cudaEventRecord(a));
    DM_CHECK_CUDA(cudaLaunchKernelEx(&cfg, grid_barrier_bench_kernel, bar, iters));
    DM_CHECK_CUDA(cudaEventRecord(b));
    DM_CHECK_CUDA(cudaEventSynchronize(b));
    float ms = 0.f;
    DM_CHECK_CUDA(cudaEventElapsedTime(&ms, a, b));
    best = fminf(best, ms);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  }
  cudaFree(bar);
  *us_per_barrier = best * 1000.f / iters;
  return 0;
}

// Host-side builder: device copies of the per-layer pointers and tensor maps.
struct MkHost {
  MkLayerW* lw = nullptr;
  TcGemvMaps* maps = nullptr;
  CUtensorMap* attn_maps = nullptr;
  unsigned* gbar = nullptr;
};

int mk_setup(const DecodeState& st, const std::vector<TcGemvMaps>& maps, const CUtensorMap& kv_map,
             const CUtensorMap& xkv_map, const std::vector<const uint16_t*>& layer_ptrs,
             void** handle) {
  auto* h = new MkHost();
  const int L = st.layers;
  std::vector<MkLayerW> lw(L);
  for (int l = 0; l < L; ++l) {
    const uint16_t* const* p = &layer_ptrs[size_t(l) * 12];
    lw[l] = MkLayerW{p[0], p[1], p[2], p[3], p[4], p[5], p[6], p[7], p[8], p[9], p[10], p[11]};
  }
  DM_CHECK_CUDA(cudaMalloc(&h->lw, sizeof(MkLayerW) * L));
  DM_CHECK_CUDA(cudaMemcpy(h->lw, lw.data(), sizeof(MkLayerW) * L, cudaMemcpyHostToDevice));
  DM_CHECK_CUDA(cudaMalloc(&h->maps, sizeof(TcGemvMaps) * maps.size()));
  DM_CHECK_CUDA(cudaMemcpy(h->maps, maps.data(), sizeof(TcGemvMaps) * maps.size(),
                           cudaMemcpyHostToDevice));
  CUtensorMap am[2] = {kv_map, xkv_map};
  DM_CHECK_CUDA(cudaMalloc(&h->attn_maps, sizeof(am)));
  DM_CHECK_CUDA(cudaMemcpy(h->attn_maps, am, sizeof(am), cudaMemcpyHostToDevice));
  DM_CHECK_CUDA(cudaMalloc(&h->gbar, 256));
  *handle = h;
  return 0;
}

void mk_free(void* handle) {
  auto* h = static_cast<MkHost*>(handle);
  if (!h) return;
  cudaFree(h->lw);
  cudaFree(h->maps);
  cudaFree(h->attn_maps);
  cudaFree(h->gbar);
  delete h;
}

int mk_launch(void* handle, const DecodeState& st, const uint16_t* lnfg, const uint16_t* lnfb,
              const uint16_t* embed, const uint16_t* pos_emb, int n_steps, cudaStream_t stream,
              unsigned long long* timing) {
  auto* h = static_cast<MkHost*>(handle);
  MkParams P{};
  P.st = st;
  P.maps = h->maps;
  P.attn_maps = h->attn_maps;
  P.lw = h->lw;
  P.lnfg = lnfg; P.lnfb = lnfb; P.embed = embed; P.pos_emb = pos_emb;
  P.gbar = h->gbar;
  P.timing = timing;
  P.n_steps = n_steps;
  P.sp_qkv = tc_gemv_splits(3 * st.d, st.d);
  P.sp_dd = tc_gemv_splits(st.d, st.d);
  P.sp_fc1 = tc_gemv_splits(st.ffn, st.d);
  P.sp_fc2 = tc_gemv_splits(st.d, st.ffn);
  return launch_decode_mega(P, stream);
}

int launch_decode_mega(const MkParams& P, cudaStream_t stream) {
  static bool attr = false;
  if (!attr) {
    DM_CHECK_CUDA(cudaFuncSetAttribute(decode_mega_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, kMkSmem));
    attr = true;
  }
  DM_CHECK_CUDA(cudaMemsetAsync(P.gbar, 0, sizeof(unsigned), stream));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(kNumSMs);
  cfg.blockDim = dim3(kMkThreads);
  cfg.dynamicSmemBytes = kMkSmem;
  cfg.stream = stream;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeCooperative;
  attrs[0].val.cooperative = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  DM_CHECK_CUDA(cudaLaunchKernelEx(&cfg, decode_mega_kernel, P));
  return 0;
}

}  // namespace dm
