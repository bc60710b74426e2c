// K6 decode-step kernels (see decode.cuh for the step graph). Projections run
// on tcgen05: the weight tile is the M=128 operand streamed by TMA, the active
// rows are the N operand (bf16 hi/lo split of the fp32 activations, N = active
// rows rounded up to 16), each output is W.(hi + lo) accumulated in fp32 TMEM.
// Attention keeps fp32 math with bf16 K/V.
//
// Latency structure (measured with the globaltimer tap, scripts/step_trace.py):
// the step is a chain of ~70 dependent kernels, each paying the release of its
// predecessor plus its own post-release critical path. Everything a kernel can
// fetch without its predecessor's output -- the whole weight slice of a GEMV
// CTA, a cross-attention CTA's K/V block, LayerNorm parameters and biases -- is
// issued before griddepcontrol.wait, so after the release only the (small)
// activation operand is read.
//
// Per step the HBM stream is the weights (once for the whole batch) plus every
// active slot's cross-KV and self-KV; each is read once.

#include "decode.cuh"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

namespace dm {

constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ void split_hilo(float v, uint16_t& hi, uint16_t& lo) {
  hi = f32_to_bf16(v);
  lo = f32_to_bf16(v - bf16_to_f32(hi));
}

// Sum of up to kMaxSplits K-split partials p[s * stride] in split order. All
// loads are issued before the first add (a runtime-trip loop would serialise
// one L2 round trip per split on the consumer's critical path).
constexpr int kMaxSplits = 10;
__device__ __forceinline__ float sum_splits(const float* p, size_t stride, int splits) {
  float v[kMaxSplits];
#pragma unroll
  for (int s = 0; s < kMaxSplits; ++s) v[s] = s < splits ? __ldcg(p + s * stride) : 0.f;
  float a = v[0];
#pragma unroll
  for (int s = 1; s < kMaxSplits; ++s)
    if (s < splits) a += v[s];
  return a;
}
template <int MAXS = kMaxSplits>
__device__ __forceinline__ float4 sum_splits4(const float* p, size_t stride, int splits) {
  float4 v[MAXS];
#pragma unroll
  for (int s = 0; s < MAXS; ++s)
    v[s] = s < splits ? __ldcg(reinterpret_cast<const float4*>(p + s * stride))
                      : make_float4(0.f, 0.f, 0.f, 0.f);
  float4 a = v[0];
#pragma unroll
  for (int s = 1; s < MAXS; ++s)
    if (s < splits) { a.x += v[s].x; a.y += v[s].y; a.z += v[s].z; a.w += v[s].w; }
  return a;
}

// ------------------------------------------------------------ cluster / bulk-copy PTX
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\t"
               "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t dsmem_addr(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_dsmem_f32(uint32_t addr, float v) {
  asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}
__device__ __forceinline__ void cluster_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
}
// arrive (release, cluster scope) on an mbarrier in another CTA's shared memory
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], "
        "%2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}
// 1-D bulk copy global -> own shared memory, completion on an mbarrier
__device__ __forceinline__ void bulk_load(void* smem_dst, const void* gsrc, uint32_t bytes,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(gsrc)), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// 1-D bulk prefetch global -> L2 (no completion; the later loads hit L2)
__device__ __forceinline__ void bulk_prefetch_l2(const void* gsrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(reinterpret_cast<uint64_t>(gsrc)),
               "r"(bytes)
               : "memory");
}

template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl_cluster(void (*kernel)(KArgs...), dim3 grid, dim3 block,
                                      dim3 cluster, size_t smem, cudaStream_t stream,
                                      Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = cluster.x;
  attr[1].val.clusterDim.y = cluster.y;
  attr[1].val.clusterDim.z = cluster.z;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

constexpr int kXpStride = 68;                 // floats per split result: o[64], max, sum, pad

__device__ __forceinline__ float4 bf16x4_to_f32(uint2 w) {
  return make_float4(__uint_as_float(w.x << 16), __uint_as_float(w.x & 0xFFFF0000u),
                     __uint_as_float(w.y << 16), __uint_as_float(w.y & 0xFFFF0000u));
}

// Cross-attention output of (row r, head h, dimension c): the split-order
// merge of its splits' (o, max, sum) in `xpart` (the last-arriver tail, the
// merge kernel and the cross-o GEMV's operand builder all use this).
__device__ __forceinline__ float xattn_merged(const DecodeState& st, const float* xpart, int r,
                                              int h, int nsplit, int c) {
  const float* base = xpart + (size_t(r) * st.heads + h) * kXSplits * kXpStride;
  float mv[kXSplits], lv[kXSplits], ov[kXSplits];
#pragma unroll
  for (int s = 0; s < kXSplits; ++s) {        // splits past the window: empty
    mv[s] = s < nsplit ? __ldcg(base + s * kXpStride + 64) : -INFINITY;
    lv[s] = s < nsplit ? __ldcg(base + s * kXpStride + 65) : 0.f;
    ov[s] = s < nsplit ? __ldcg(base + s * kXpStride + c) : 0.f;
  }
  float M = -INFINITY;
#pragma unroll
  for (int s = 0; s < kXSplits; ++s) M = fmaxf(M, mv[s]);
  float Ls = 0.f, O = 0.f;
#pragma unroll
  for (int s = 0; s < kXSplits; ++s) {
    const float f = exp2f((mv[s] - M) * kLog2e);
    Ls += lv[s] * f;
    O += ov[s] * f;
  }
  return O / Ls;
}

// xattn_merged for dimensions c .. c + 3 (c % 4 == 0): each lane of the result
// is computed exactly as xattn_merged computes it (same operations, same
// order); the max / sum loads are shared and o is read as float4.
__device__ __forceinline__ float4 xattn_merged4(const DecodeState& st, const float* xpart, int r,
                                                int h, int nsplit, int c) {
  const float* base = xpart + (size_t(r) * st.heads + h) * kXSplits * kXpStride;
  float mv[kXSplits], lv[kXSplits];
  float4 ov[kXSplits];
#pragma unroll
  for (int s = 0; s < kXSplits; ++s) {
    mv[s] = s < nsplit ? __ldcg(base + s * kXpStride + 64) : -INFINITY;
    lv[s] = s < nsplit ? __ldcg(base + s * kXpStride + 65) : 0.f;
    ov[s] = s < nsplit ? __ldcg(reinterpret_cast<const float4*>(base + s * kXpStride + c))
                       : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  float M = -INFINITY;
#pragma unroll
  for (int s = 0; s < kXSplits; ++s) M = fmaxf(M, mv[s]);
  float Ls = 0.f;
  float4 O = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int s = 0; s < kXSplits; ++s) {
    const float f = exp2f((mv[s] - M) * kLog2e);
    Ls += lv[s] * f;
    O.x += ov[s].x * f;
    O.y += ov[s].y * f;
    O.z += ov[s].z * f;
    O.w += ov[s].w * f;
  }
  return make_float4(O.x / Ls, O.y / Ls, O.z / Ls, O.w / Ls);
}

// element (row n, k) of a K-major SW128 operand tile with 128-byte rows
__device__ __forceinline__ int sw128_off(int n, int k) {
  return n * 128 + ((((k >> 3) ^ n) & 7) << 4) + (k & 7) * 2;
}

// ============================================================ tcgen05 GEMV
// CTA (c, split) owns N tiles c, c + gridDim.x, ... for one K split. Warp
// roles: w0 TMA, w1 MMA (+ TMEM alloc), w2..5 epilogue (thread = output
// feature of the 128-row tile). Before the dependency wait the producer fills
// the weight ring (the whole slice when it fits); after it, it loads only the
// active rows of the activation operand (16-row boxes). Accumulators
// alternate between two 64-column TMEM buffers so the epilogue of tile i
// overlaps the MMAs of tile i + 1.
constexpr int kGvThreads = 192;
constexpr int kGvWBytes = 128 * 64 * 2;        // W block: 128 features x 64 k
constexpr int kGvXBytes = kRows * 64 * 2;      // X block: 64 rows x 64 k (hi or lo)
constexpr int kSmPerSm = 233472;               // shared memory per SM (228 KB)
constexpr int kGvTr = kRows * 129 * 4;         // GV_ARGMAX transpose / GELU staging (64 rows)
__host__ __device__ constexpr int gemv_tr_bytes(int xrows) { return (xrows <= 16 ? 16 : kRows) * 129 * 4; }
constexpr int kGvMaxStages = 8;
constexpr int kGvMisc = 1024;
constexpr int kSmemOptin = 232448;             // 227 KB per CTA (sm_100)

__host__ __device__ constexpr int gemv_smem_bytes(int kb_per, int stages, int epi, int rgroups,
                                                  int xrows = kRows) {
  return 1024 + kb_per * 2 * (xrows * 128 / rgroups) + stages * kGvWBytes +
         (epi != GV_PARTIAL ? gemv_tr_bytes(xrows) : 0) + kGvMisc;
}

// XR: rows of the register / staging layout (16: step graphs of <= 16 active
// rows, smaller shared memory; 64 otherwise)
template <int EPI, bool SPLIT, int XR>
__global__ void __launch_bounds__(kGvThreads, 1)
gemv_kernel(const __grid_constant__ CUtensorMap tw, const __grid_constant__ CUtensorMap txh,
            const __grid_constant__ CUtensorMap txl, const DecodeState st, const GemvArgs a) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024 - (raw_addr & 1023)) & 1023);
  const int kb_per = a.kb_per, NS = a.stages;
  uint8_t* xs = smem;                                        // [kb][hi | lo], RG rows each
  const int RG = a.xrows / int(gridDim.z);                  // rows per row group
  uint8_t* ws = xs + kb_per * 2 * RG * 128;                  // [stage] 16K
  float* tr = reinterpret_cast<float*>(ws + NS * kGvWBytes); // GV_ARGMAX / GELU staging
  uint8_t* misc = reinterpret_cast<uint8_t*>(tr) + (EPI != GV_PARTIAL ? gemv_tr_bytes(XR) : 0);
  constexpr int V0N = XR < 32 ? XR : 32;           // rows held in v0 (v1: rows 32..63)
  constexpr bool V1 = XR > 32;
  uint64_t* wfull = reinterpret_cast<uint64_t*>(misc);
  uint64_t* wempty = wfull + kGvMaxStages;
  uint64_t* xfull = wempty + kGvMaxStages;
  uint64_t* tm_full = xfull + 1;                             // [2]
  uint64_t* tm_empty = tm_full + 2;                          // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tm_empty + 2);
  int* is_last = reinterpret_cast<int*>(tmem_slot + 1);
  if (threadIdx.x == 0) trace_mark(st, 0);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int split = blockIdx.y;
  const int tiles = ceil_div(a.N, 128);
  const int kb0 = split * kb_per;
  // rows of this CTA's row group: [r0, r0 + R); n_active is host-set before
  // the step graph runs, so it is safe to read before the wait
  const int r0 = int(blockIdx.z) * RG;
  const int R = min(*st.n_active - r0, RG);
  if (R <= 0 && blockIdx.z > 0) return;                      // empty row group
  const int G = R > 0 ? ceil_div(R, kGvXBox) : 1;            // 16-row activation boxes
  const int Np = G * kGvXBox;                                // MMA N
  const int XB = RG * 128;                                   // one hi or lo k-block

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tw);
    tma_prefetch_desc(&txh);
    tma_prefetch_desc(&txl);
    for (int s = 0; s < NS; ++s) {
      mbar_init(&wfull[s], 1);
      mbar_init(&wempty[s], 1);
    }
    mbar_init(xfull, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tm_full[s], 1);
      mbar_init(&tm_empty[s], 4);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // dependents may launch now and prefetch their own inputs. Not before the
  // TMEM allocation: a dependent's CTAs that allocate TMEM and then wait for
  // this grid must never hold the columns one of its CTAs still needs.
  pdl_trigger();

  if (warp == 0) {
    if (elect_one()) {
      const int my_tiles = (tiles - 1 - int(blockIdx.x)) / int(gridDim.x) + 1;
      const int total = my_tiles * kb_per;
      int wi = 0;
      const uint64_t keep = l2_policy_evict_last();      // weights: re-read every step
      auto issue_w = [&](int q) {
        const int s = wi % NS;
        mbar_wait(&wempty[s], ((wi / NS) & 1) ^ 1);
        mbar_arrive_expect_tx(&wfull[s], kGvWBytes);
        tma_load_2d_hint(ws + s * kGvWBytes, &tw, &wfull[s], (kb0 + q % kb_per) * 64,
                         (int(blockIdx.x) + (q / kb_per) * int(gridDim.x)) * 128, keep);
        ++wi;
      };
      const int pre = total < NS ? total : NS;
      if (total <= NS) {
        // whole weight slice resident: one barrier for all of it, so the MMA
        // warp needs a single wait instead of one handshake per k-block
        mbar_arrive_expect_tx(&wfull[0], total * kGvWBytes);
        for (int q = 0; q < total; ++q)
          tma_load_2d_hint(ws + q * kGvWBytes, &tw, &wfull[0], (kb0 + q % kb_per) * 64,
                           (int(blockIdx.x) + (q / kb_per) * int(gridDim.x)) * 128, keep);
        wi = total;
      } else {
        for (int q = 0; q < pre; ++q) issue_w(q);   // weights never depend on the predecessor
      }
      pdl_wait();
      trace_mark(st, 1);
      if (a.xsrc == GV_X_TMA) {                 // (else the epilogue warps build it)
        mbar_arrive_expect_tx(xfull, kb_per * 2 * G * kGvXBox * 128);
        for (int i = 0; i < kb_per; ++i) {
          uint8_t* xb = xs + i * 2 * XB;        // [hi: Np rows | lo: Np rows], 128 B rows
          for (int g = 0; g < G; ++g) {
            tma_load_2d(xb + g * kGvXBox * 128, &txh, xfull, (kb0 + i) * 64, r0 + g * kGvXBox);
            tma_load_2d(xb + (Np + g * kGvXBox) * 128, &txl, xfull, (kb0 + i) * 64, r0 + g * kGvXBox);
          }
        }
      }
      for (int q = pre; q < total; ++q) issue_w(q);
    }
  } else if (warp == 1) {
    // one MMA per k-step: B = [x_hi rows ; x_lo rows] (N = 2 Np), so the
    // weight tile (the A operand, the smem-read-bound side at small N) is read
    // once for both halves; D columns [0, Np) hold W.x_hi, [Np, 2 Np) W.x_lo
    const uint32_t idesc = umma_idesc_bf16(128, 2 * Np);
    const int my_tiles = (tiles - 1 - int(blockIdx.x)) / int(gridDim.x) + 1;
    const bool resident = my_tiles * kb_per <= NS;
    mbar_wait(xfull, 0);
    if (lane == 0) trace_mark(st, 4);
    int wi = 0, it = 0;
    if (resident) {
      // all operands landed after two waits: issue every MMA back to back
      mbar_wait(&wfull[0], 0);
      tc_fence_after();
      for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++it) {
        const int buf = it & 1;
        mbar_wait(&tm_empty[buf], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t d = tmem + buf * 128;
          for (int i = 0; i < kb_per; ++i) {
            const uint64_t aw = umma_desc_sw128(smem_u32(ws + (it * kb_per + i) * kGvWBytes));
            const uint64_t bx = umma_desc_sw128(smem_u32(xs + i * 2 * XB));
#pragma unroll
            for (int k = 0; k < 4; ++k)      // +32 B per k-step = +2 in the address field
              umma_bf16_ss(d, aw + 2 * k, bx + 2 * k, idesc, (i | k) != 0);
          }
          trace_mark(st, 7);
          umma_commit(&tm_full[buf]);
        }
        __syncwarp();
      }
    }
    for (int tile = resident ? tiles : int(blockIdx.x); tile < tiles; tile += gridDim.x, ++it) {
      const int buf = it & 1;
      mbar_wait(&tm_empty[buf], ((it >> 1) & 1) ^ 1);
      tc_fence_after();
      for (int i = 0; i < kb_per; ++i, ++wi) {
        const int s = wi % NS;
        mbar_wait(&wfull[s], (wi / NS) & 1);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t sw = smem_u32(ws + s * kGvWBytes);
          const uint32_t sh = smem_u32(xs + i * 2 * XB);
#pragma unroll
          for (int k = 0; k < 4; ++k)
            umma_bf16_ss(tmem + buf * 128, umma_desc_sw128(sw + k * 32),
                         umma_desc_sw128(sh + k * 32), idesc, (i | k) != 0);
          umma_commit(&wempty[s]);
          if (i == kb_per - 1) {
            trace_mark(st, 7);
            umma_commit(&tm_full[buf]);
          }
        }
        __syncwarp();
      }
    }
    // release TMEM as soon as the epilogue has read the last accumulators,
    // while its global stores are still draining
    for (int k = it - 2; k < it; ++k)
      if (k >= 0) mbar_wait(&tm_empty[k & 1], (k >> 1) & 1);
    tc_fence_after();
    tmem_dealloc(tmem, 256);
  } else {
    const int quad = warp & 3;
    const int f = quad * 32 + lane;                // feature within the tile
    const int et = threadIdx.x - 64;               // 0..127 among epilogue threads
    float bcur = 0.f;
    if (EPI != GV_PARTIAL && a.bias != nullptr && int(blockIdx.x) * 128 + f < a.N)
      bcur = bf16_to_f32(a.bias[blockIdx.x * 128 + f]);
    pdl_wait();
    if (a.xsrc != GV_X_TMA) {
      // build this CTA's activation slice (rows [r0, r0 + Np), k-blocks kb0..)
      // in the SW128 layout the TMA would have produced, 4 k per item
      const int kq = kb_per * 16;
#pragma unroll 2
      for (int e = et; e < Np * kq; e += 128) {
        const int row = e / kq, kk = (e % kq) * 4;
        float v[4] = {0.f, 0.f, 0.f, 0.f};
        if (row < R) {
          const int gr = r0 + row, gk = kb0 * 64 + kk;
          float4 y;
          if (a.xsrc == GV_X_GELU) {       // gelu_hilo_kernel's arithmetic
            const float4 sa = sum_splits4<8>(a.xp + size_t(gr) * a.K + gk, size_t(kRows) * a.K,
                                             a.xs_splits);
            const float4 bb = bf16x4_to_f32(*reinterpret_cast<const uint2*>(a.xbias + gk));
            y = make_float4(gelu_erf(sa.x + bb.x), gelu_erf(sa.y + bb.y), gelu_erf(sa.z + bb.z),
                            gelu_erf(sa.w + bb.w));
          } else {                         // xattn_merge_kernel's arithmetic
            const int nsplit = ceil_div(st.enc_len[st.active[gr]], kXaKeysPerSplit);
            y = xattn_merged4(st, a.xp, gr, gk >> 6, nsplit, gk & 63);
          }
          v[0] = y.x; v[1] = y.y; v[2] = y.z; v[3] = y.w;
        }
        uint16_t h[4], l[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) split_hilo(v[u], h[u], l[u]);
        uint8_t* xb = xs + (kk >> 6) * 2 * XB;
        *reinterpret_cast<uint2*>(xb + sw128_off(row, kk & 63)) =
            make_uint2(uint32_t(h[0]) | (uint32_t(h[1]) << 16), uint32_t(h[2]) | (uint32_t(h[3]) << 16));
        *reinterpret_cast<uint2*>(xb + sw128_off(Np + row, kk & 63)) =
            make_uint2(uint32_t(l[0]) | (uint32_t(l[1]) << 16), uint32_t(l[2]) | (uint32_t(l[3]) << 16));
      }
      fence_proxy_async_smem();
      named_bar_sync(1, 128);
      if (et == 0) mbar_arrive(xfull);
    }
    int it = 0;
    for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++it) {
      const int n = tile * 128 + f;
      const bool nvalid = n < a.N;
      const float b = bcur;
      {
        const int nn = n + int(gridDim.x) * 128;   // next tile's bias, off the critical path
        bcur = (EPI != GV_PARTIAL && a.bias != nullptr && nn < a.N) ? bf16_to_f32(a.bias[nn]) : 0.f;
      }
      const int buf = it & 1;
      mbar_wait(&tm_full[buf], (it >> 1) & 1);
      tc_fence_after();
      if (et == 0) trace_mark(st, 5);
      float v0[32], v1[32];
      {
        // row r: W.x_hi (column r) + W.x_lo (column Np + r)
        const uint32_t base = tmem + (uint32_t(quad * 32) << 16) + buf * 128;
        // hi and lo columns in flight together, one wait
        uint32_t ra[32], rb[32];
        tmem_ld32(base, ra);
        tmem_ld32(base + Np, rb);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 32; ++i) v0[i] = __uint_as_float(ra[i]) + __uint_as_float(rb[i]);
        if (Np > 32) {
          tmem_ld32(base + 32, ra);
          tmem_ld32(base + Np + 32, rb);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) v1[i] = __uint_as_float(ra[i]) + __uint_as_float(rb[i]);
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) v1[i] = 0.f;
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tm_empty[buf]);
      if (EPI == GV_PARTIAL) {
        if (nvalid) {
          float* __restrict__ p = a.part + (size_t(split) * kRows + r0) * a.N + n;
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (i < R) p[size_t(i) * a.N] = v0[i];
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (32 + i < R) p[size_t(32 + i) * a.N] = v1[i];
        }
        continue;
      }
      if (SPLIT) {
        // last-CTA reduction of the K splits (fixed split order)
        float* part = st.part;
        const size_t base = (size_t(split) * tiles + tile) * kRows * 128;
#pragma unroll
        for (int i = 0; i < V0N; ++i) part[base + size_t(i) * 128 + f] = v0[i];
        if (V1) {
#pragma unroll
          for (int i = 0; i < 32; ++i) part[base + size_t(32 + i) * 128 + f] = v1[i];
        }
        named_bar_sync(1, 128);
        if (et == 0) {                 // one release (cumulative over the barrier)
          __threadfence();
          const int prev = atomicAdd(&st.counters[a.counter_base + tile], 1);
          *is_last = (prev == a.splits - 1);
          if (*is_last) __threadfence();
        }
        named_bar_sync(1, 128);
        const int last = *is_last;
        named_bar_sync(1, 128);
        if (!last) continue;
#pragma unroll
        for (int i = 0; i < 32; ++i) { v0[i] = 0.f; v1[i] = 0.f; }
        for (int s = 0; s < a.splits; ++s) {
          const float* ps = part + (size_t(s) * tiles + tile) * kRows * 128 + f;
#pragma unroll
          for (int i = 0; i < V0N; ++i) v0[i] += __ldcg(ps + size_t(i) * 128);
          if (V1) {
#pragma unroll
            for (int i = 0; i < 32; ++i) v1[i] += __ldcg(ps + size_t(32 + i) * 128);
          }
        }
        if (et == 0) st.counters[a.counter_base + tile] = 0;
      }
      if (EPI == GV_GELU_HILO) {
        if (nvalid) {
          uint16_t* __restrict__ yh = a.yh + size_t(r0) * a.N + n;
          uint16_t* __restrict__ yl = a.yl + size_t(r0) * a.N + n;
          // stage the rows in this thread's smem column (conflict-free), then
          // one compact loop over the active rows (no unrolled erf copies)
          float* col = tr + f;
#pragma unroll
          for (int i = 0; i < V0N; ++i) col[i * 129] = v0[i];
          if (V1) {
#pragma unroll
            for (int i = 0; i < 32; ++i) col[(32 + i) * 129] = v1[i];
          }
#pragma unroll 4
          for (int i = 0; i < R; ++i) {
            uint16_t hi, lo;
            split_hilo(gelu_erf(col[i * 129] + b), hi, lo);
            yh[size_t(i) * a.N] = hi;
            yl[size_t(i) * a.N] = lo;
          }
        }
      }
      if (EPI == GV_ARGMAX) {
#pragma unroll
        for (int i = 0; i < V0N; ++i) tr[i * 129 + f] = nvalid ? v0[i] : -INFINITY;
        if (V1) {
#pragma unroll
          for (int i = 0; i < 32; ++i) tr[(32 + i) * 129 + f] = nvalid ? v1[i] : -INFINITY;
        }
        if (st.logits_dbg && nvalid) {
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            if (i < R) st.logits_dbg[size_t(i) * st.vocab + n] = v0[i];
            if (32 + i < R) st.logits_dbg[size_t(32 + i) * st.vocab + n] = v1[i];
          }
        }
        // per row: max over this tile's 128 vocabulary ids, ties -> lowest id
        named_bar_sync(1, 128);
        const int r = (et >> 1) % XR, half = et & 1;    // (rows >= XR repeat row r: unused)
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
        if (half == 0 && (et >> 1) < XR) {
          st.amax_val[size_t(tile) * kRows + r] = best;
          st.amax_idx[size_t(tile) * kRows + r] = bidx;
        }
        named_bar_sync(1, 128);                    // tr reused by the next tile
      }
    }
  }
  if (warp >= 2 && lane == 0) trace_mark(st, 6);
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) trace_mark(st, 3);
}

GemvArgs gemv_plan(int N, int K, int epi, int max_splits) {
  GemvArgs a{};
  a.N = N;
  a.K = K;
  a.epi = epi;
  const int KB = K / 64;
  if (epi == GV_PARTIAL) {
    // K split: as many CTAs as fill the GPU (several per SM at low rows, where
    // the activation buffer is small) with the shortest weight slice each,
    // each extra partial costing its consumer a little; at most max_splits
    // partials (what the consumer reduces) and 8 k-blocks per CTA
    const int tiles_n = ceil_div(N, 128);
    float best = 1e30f;
    a.kb_per = KB;
    for (int kb = 1; kb <= 8 && kb <= KB; ++kb) {
      if (KB % kb || KB / kb > max_splits) continue;
      const int ctas = tiles_n * (KB / kb);
      const int smem16 = gemv_smem_bytes(kb, kb, epi, 1, 16) + 1024;
      const int cps = std::max(1, std::min(4, kSmPerSm / smem16));
      const int waves = ceil_div(ctas, cps * kNumSMs);
      const float cost = float(waves * kb) + 0.25f * float(KB / kb);
      if (cost < best - 1e-6f) { best = cost; a.kb_per = kb; }
    }
  } else {
    // non-linear epilogue: as few K splits as fit (<= 8 k-blocks per CTA)
    a.kb_per = KB;
    for (int s = 1; s <= KB; ++s)
      if (KB % s == 0 && KB / s <= 8) { a.kb_per = KB / s; break; }
  }
  a.splits = KB / a.kb_per;
  // fc1-style projections (non-linear, unsplit): four row groups of 16 so each
  // CTA holds its whole weight slice plus a quarter of the activation rows
  a.rgroups = (epi == GV_GELU_HILO && a.splits == 1) ? 4 : 1;
  const int tiles = ceil_div(N, 128);
  const int gx = std::max(1, std::min(tiles, kNumSMs / a.splits));
  const int per_cta = ceil_div(tiles, gx) * a.kb_per;
  const int fixed = gemv_smem_bytes(a.kb_per, 0, epi, a.rgroups);
  a.stages = std::min({kGvMaxStages, (kSmemOptin - fixed) / kGvWBytes, per_cta});
  a.xrows = kRows;
  a.gx = gx;
  return a;
}

GemvArgs gemv_plan_for_rows(const GemvArgs& base, int rows) {
  GemvArgs a = base;
  static const int mode = std::getenv("DM_GV_ROWPLAN") ? std::atoi(std::getenv("DM_GV_ROWPLAN")) : 1;
  if (mode == 0) return a;
  if (mode == 2 && a.epi != GV_PARTIAL) return a;
  const int xr = std::min(kRows, std::max(kGvXBox, ceil_div(rows, kGvXBox) * kGvXBox));
  int rg = a.rgroups;
  while (rg > 1 && xr % (rg * kGvXBox) != 0) rg /= 2;
  a.xrows = xr;
  a.rgroups = rg;
  const int tiles = ceil_div(a.N, 128);
  // two CTAs per SM when the activation buffer is small enough that half an
  // SM still holds the whole weight slice (or a ring of >= 4 stages): more
  // CTAs, fewer tiles each
  for (int cps = 4; cps >= 1; --cps) {
    const int gx = std::max(1, std::min(tiles, cps * kNumSMs / a.splits));
    const int per_cta = ceil_div(tiles, gx) * a.kb_per;
    const int fixed = gemv_smem_bytes(a.kb_per, 0, a.epi, rg, xr);
    int room = (kSmemOptin - fixed) / kGvWBytes;
    if (cps > 1) room = std::min(room, (kSmPerSm / cps - 1024 - fixed) / kGvWBytes);
    const int stages = std::min({kGvMaxStages, room, per_cta});
    if (cps == 1 || stages >= std::min(per_cta, 4)) {
      a.gx = gx;
      a.stages = stages;
      break;
    }
  }
  return a;
}

size_t gemv_part_floats(int N, int K, int epi, int max_splits) {
  const GemvArgs a = gemv_plan(N, K, epi, max_splits);
  if (epi == GV_PARTIAL) return size_t(a.splits) * kRows * N;
  return a.splits > 1 ? size_t(a.splits) * ceil_div(N, 128) * kRows * 128 : 0;
}

template <int EPI, bool SPLIT, int XR>
static int launch_gv(const DecodeState& st, const TcGemvMaps& maps, const GemvArgs& a,
                     cudaStream_t stream) {
  DM_SMEM_ATTR((gemv_kernel<EPI, SPLIT, XR>), kSmemOptin);
  DM_CHECK_CUDA(launch_pdl(gemv_kernel<EPI, SPLIT, XR>, dim3(a.gx, a.splits, a.rgroups),
                           dim3(kGvThreads),
                           size_t(gemv_smem_bytes(a.kb_per, a.stages, EPI, a.rgroups, a.xrows)),
                           stream, maps.w, maps.xh, maps.xl, st, a));
  return 0;
}

template <int EPI, bool SPLIT>
static int launch_gv_rows(const DecodeState& st, const TcGemvMaps& maps, const GemvArgs& a,
                          cudaStream_t stream) {
  return a.xrows <= 16 ? launch_gv<EPI, SPLIT, 16>(st, maps, a, stream)
                       : launch_gv<EPI, SPLIT, kRows>(st, maps, a, stream);
}

int launch_gemv(const DecodeState& st, const TcGemvMaps& maps, const GemvArgs& a,
                cudaStream_t stream) {
  DM_REQUIRE(a.K % 64 == 0 && a.kb_per >= 1 && a.splits * a.kb_per * 64 == a.K, "bad K split");
  DM_REQUIRE(a.stages >= 1 && a.stages <= kGvMaxStages, "bad weight ring depth");
  DM_REQUIRE(a.rgroups == 1 || a.rgroups == 2 || a.rgroups == 4, "GEMV row groups: 1, 2 or 4");
  DM_REQUIRE(a.rgroups == 1 || (a.epi != GV_ARGMAX && a.splits == 1), "row groups: linear / fc1 only");
  DM_REQUIRE(gemv_smem_bytes(a.kb_per, a.stages, a.epi, a.rgroups, a.xrows) <= kSmemOptin,
             "GEMV slice exceeds smem");
  DM_REQUIRE(a.xrows % (16 * a.rgroups) == 0 && a.xrows <= kRows && a.gx >= 1,
             "GEMV activation rows / grid");
  DM_REQUIRE(a.xsrc == GV_X_TMA ||
                 (a.xrows <= 16 && a.rgroups == 1 && a.xp != nullptr &&
                  (a.xsrc == GV_X_XMERGE || (a.xbias != nullptr && a.xs_splits >= 1 && a.xs_splits <= 8))),
             "GEMV operand builder: <= 16 rows, one row group, source set");
  const bool sp = a.splits > 1;
  switch (a.epi) {
    case GV_PARTIAL:
      DM_REQUIRE(a.part != nullptr, "partial output missing");
      return launch_gv_rows<GV_PARTIAL, false>(st, maps, a, stream);
    case GV_GELU_HILO: return sp ? launch_gv_rows<GV_GELU_HILO, true>(st, maps, a, stream)
                                 : launch_gv_rows<GV_GELU_HILO, false>(st, maps, a, stream);
    case GV_ARGMAX: return sp ? launch_gv_rows<GV_ARGMAX, true>(st, maps, a, stream)
                              : launch_gv_rows<GV_ARGMAX, false>(st, maps, a, stream);
    default: DM_REQUIRE(false, "unknown epilogue");
  }
}

// ============================================================ LayerNorm
// One CTA per row, d/4 threads (thread t owns features 4t..4t+3). Parameters
// are fetched before the dependency wait; after it, one round of loads (x and
// the residual partials, or the embedding rows), two block reductions (mean,
// then the centred second moment), and the hi/lo operand stores.

__device__ __forceinline__ float block_sum_fixed(float v, float* red) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nw = blockDim.x / 32;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) red[warp] = v;
  __syncthreads();
  float s = 0.f;
  for (int w = 0; w < nw; ++w) s += red[w];
  __syncthreads();
  return s;
}

// MODE 2 brings the residual row and every partial row into shared memory
// with one bulk copy each, all issued by one thread onto one mbarrier: a
// single L2 round trip however many partials there are (per-thread loads
// issue in groups of ~6 -- the SASS scoreboard limit -- so 8-20 partials would
// cost 2-4 dependent round trips).
// block_sum_fixed without the trailing barrier: the caller gives each
// reduction its own per-warp slots (same order: xor tree, then warps 0..n-1)
__device__ __forceinline__ float block_sum_once(float v, float* slots) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nw = blockDim.x / 32;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) slots[warp] = v;
  __syncthreads();
  float s = 0.f;
  for (int w = 0; w < nw; ++w) s += slots[w];
  return s;
}

template <int MODE>
__global__ void __launch_bounds__(320) ln_kernel(const DecodeState st, const LnArgs a) {
  extern __shared__ __align__(16) float ln_rows[];      // MODE 2: [1 + splits][d]
  __shared__ float red[20];                              // two reductions' per-warp slots
  __shared__ __align__(8) uint64_t ln_bar;
  const int r = blockIdx.x, t = threadIdx.x, d = st.d;
  if (t == 0) trace_mark(st, 0);
  pdl_trigger();
  const int R = *st.n_active;
  const float4 gm = bf16x4_to_f32(__ldg(reinterpret_cast<const uint2*>(a.g) + t));
  const float4 bt = bf16x4_to_f32(__ldg(reinterpret_cast<const uint2*>(a.b) + t));
  float4 rb = make_float4(0.f, 0.f, 0.f, 0.f);
  if (MODE == 2 && a.res.bias) rb = bf16x4_to_f32(__ldg(reinterpret_cast<const uint2*>(a.res.bias) + t));
  const int slot = r < R ? st.active[r] : 0;
  if (MODE == 2) {
    if (t == 0) {
      mbar_init(&ln_bar, 1);
      fence_barrier_init();
    }
    // every thread polls ln_bar after the wait: it must be initialised first
    // (without this barrier a warp that runs ahead of warp 0 -- common when
    // the SM is shared with another stream's CTAs -- waits on stale shared
    // memory and the CTA faults)
    __syncthreads();
  }
  pdl_wait();
  if (t == 0) trace_mark(st, 1);
  if (r >= R) return;
  float4 x;
  float* xr = st.x + size_t(r) * d;
  if (MODE == 1) {
    const int tok = st.cur_tok[slot], p = st.pos[slot];
    const float4 e = bf16x4_to_f32(__ldg(reinterpret_cast<const uint2*>(a.embed + size_t(tok) * d) + t));
    const float4 pe = bf16x4_to_f32(__ldg(reinterpret_cast<const uint2*>(a.pos_emb + size_t(p) * d) + t));
    x = make_float4(e.x + pe.x, e.y + pe.y, e.z + pe.z, e.w + pe.w);
    reinterpret_cast<float4*>(xr)[t] = x;
  } else if (MODE == 2) {
    const int ns = a.res.splits;
    if (t == 0) {
      mbar_arrive_expect_tx(&ln_bar, uint32_t(ns + 1) * d * 4);
      bulk_load(ln_rows, xr, d * 4, &ln_bar);
      for (int s = 0; s < ns; ++s)
        bulk_load(ln_rows + (s + 1) * d, a.res.p + (size_t(s) * kRows + r) * a.res.n, d * 4, &ln_bar);
    }
    mbar_wait(&ln_bar, 0);
    x = reinterpret_cast<const float4*>(ln_rows)[t];
    float4 acc = reinterpret_cast<const float4*>(ln_rows + d)[t];
    for (int s = 1; s < ns; ++s) {
      const float4 v = reinterpret_cast<const float4*>(ln_rows + (s + 1) * d)[t];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    x.x += acc.x + rb.x; x.y += acc.y + rb.y; x.z += acc.z + rb.z; x.w += acc.w + rb.w;
    reinterpret_cast<float4*>(xr)[t] = x;
  } else {
    x = __ldcg(reinterpret_cast<const float4*>(xr) + t);
  }
  if (t == 0) trace_mark(st, 4);
  const float mean = block_sum_once((x.x + x.y) + (x.z + x.w), red) / d;
  const float c0 = x.x - mean, c1 = x.y - mean, c2 = x.z - mean, c3 = x.w - mean;
  const float var = block_sum_once((c0 * c0 + c1 * c1) + (c2 * c2 + c3 * c3), red + 10) / d;
  if (t == 0) trace_mark(st, 5);
  const float rstd = rsqrtf(var + 1e-5f);
  uint16_t h[4], l[4];
  split_hilo(c0 * rstd * gm.x + bt.x, h[0], l[0]);
  split_hilo(c1 * rstd * gm.y + bt.y, h[1], l[1]);
  split_hilo(c2 * rstd * gm.z + bt.z, h[2], l[2]);
  split_hilo(c3 * rstd * gm.w + bt.w, h[3], l[3]);
  reinterpret_cast<uint2*>(st.xh + size_t(r) * d)[t] =
      make_uint2(uint32_t(h[0]) | (uint32_t(h[1]) << 16), uint32_t(h[2]) | (uint32_t(h[3]) << 16));
  reinterpret_cast<uint2*>(st.xl + size_t(r) * d)[t] =
      make_uint2(uint32_t(l[0]) | (uint32_t(l[1]) << 16), uint32_t(l[2]) | (uint32_t(l[3]) << 16));
  if (t == 0) trace_mark(st, 3);
}

int launch_ln(const DecodeState& st, const LnArgs& a, cudaStream_t stream) {
  DM_REQUIRE(st.d % 128 == 0 && st.d / 4 <= 320, "LayerNorm: d must be a multiple of 128, <= 1280");
  DM_REQUIRE(a.mode != 2 || (a.res.p != nullptr && a.res.splits >= 1 &&
                             a.res.splits <= kMaxHeads && a.res.n == st.d),
             "LayerNorm: residual partials missing");
  const dim3 grid(st.grid_rows), block(st.d / 4);
  switch (a.mode) {
    case 0: DM_CHECK_CUDA(launch_pdl(ln_kernel<0>, grid, block, 0, stream, st, a)); break;
    case 1: DM_CHECK_CUDA(launch_pdl(ln_kernel<1>, grid, block, 0, stream, st, a)); break;
    case 2: {
      const int smem = (a.res.splits + 1) * st.d * 4;
      DM_SMEM_ATTR(ln_kernel<2>, (kMaxHeads + 1) * 1280 * 4);
      DM_CHECK_CUDA(launch_pdl(ln_kernel<2>, grid, block, smem, stream, st, a));
      break;
    }
    default: DM_REQUIRE(false, "LayerNorm: unknown mode");
  }
  return 0;
}

// ============================================================ attention
// Two-pass softmax per (row, head[, key split]): scores lane-per-key (q in
// shared memory, fp32 dot products over the bf16 key row), block max, exp2 and
// block sum in a fixed order, then P.V lane-per-dimension (warp w takes keys
// w, w + 8, ...) merged across warps in a fixed order. Every order depends
// only on key positions, never on the batch.
__device__ __forceinline__ float block_max(float v, float* red) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nw = blockDim.x / 32;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  if (lane == 0) red[warp] = v;
  __syncthreads();
  float m = -INFINITY;
  for (int w = 0; w < nw; ++w) m = fmaxf(m, red[w]);
  __syncthreads();
  return m;
}

__device__ __forceinline__ void store_hilo1(const DecodeState& st, int r, int c, float v) {
  uint16_t hi, lo;
  split_hilo(v, hi, lo);
  st.ah[size_t(r) * st.d + c] = hi;
  st.al[size_t(r) * st.d + c] = lo;
}

#ifndef DM_SA_THREADS
#define DM_SA_THREADS 256
#endif
#ifndef DM_SA_PREPAGES
#define DM_SA_PREPAGES 2
#endif
constexpr int kSaThreads = DM_SA_THREADS;
constexpr int kSaWarps = kSaThreads / 32;
constexpr int kSaMaxKeys = 448;
constexpr int kSaPageBytes = 64 * 128;                         // one page block: 64 keys x 64 dims
constexpr int kSaPrePages = DM_SA_PREPAGES;                    // pages staged in shared memory

// Self-attention for (row, head). The fed token's position and the slot's
// earlier keys/values do not depend on this step's predecessors (positions
// advance only in the previous step's finalize), so the K and V page blocks
// of positions 0..min(pos, 128)-1 are bulk-copied into shared memory before
// the dependency wait (later positions are read from global memory). After it: reduce the fed token's q/k/v from the qkv
// partials, append k/v (bf16) at `pos`, scores (cached keys read chunk-wise in
// XOR order -- conflict-free -- plus the fed key), two-pass softmax, P.V.
__global__ void __launch_bounds__(kSaThreads)
self_attn_kernel(const DecodeState st, int layer, const Partials qkv, float q_scale) {
  extern __shared__ __align__(128) uint8_t sa_smem[];          // [pages][K 8K | V 8K] + bar
  __shared__ __align__(16) float qs[64];
  __shared__ float kc[64], vc[64];
  __shared__ float sc[kSaMaxKeys];
  __shared__ float redm[kSaWarps], reds[kSaWarps];
  __shared__ float op[kSaWarps][64];
  const int r = blockIdx.x, h = blockIdx.y, tid = threadIdx.x;
  const int warp = tid / 32, lane = tid % 32;
  if (tid == 0) trace_mark(st, 0);
  pdl_trigger();
  if (r >= *st.n_active) return;                 // host-set: safe before the wait
  const int slot = st.active[r];
  // a slot that finished (EOT / cap) in an earlier step stays in the active
  // list until the host's next poll; its outputs are never read again
  if (st.done[slot]) return;
  const int d = st.d, H = st.heads, L = st.layers;
  const int p = st.pos[slot];                    // final since the previous step
  const int np = min(ceil_div(p, 64), kSaPrePages);   // staged pages of positions < p
  const int* pt = st.page_table + slot * st.pages_per_slot;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sa_smem + kSaPrePages * 2 * kSaPageBytes);
  const size_t kv_off = size_t(H) * 64 * 64;     // k -> v within a (page, layer)
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_barrier_init();
    if (np > 0) {
      mbar_arrive_expect_tx(bar, np * 2 * kSaPageBytes);
      for (int g = 0; g < np; ++g) {
        const uint16_t* kb = st.kv_pool + ((size_t(pt[g]) * L + layer) * 2 * H + h) * 64 * 64;
        bulk_load(sa_smem + g * 2 * kSaPageBytes, kb, kSaPageBytes, bar);
        bulk_load(sa_smem + g * 2 * kSaPageBytes + kSaPageBytes, kb + kv_off, kSaPageBytes, bar);
      }
    }
  } else if (tid < 32) {
    // later pages (positions >= 64 * kSaPrePages) are read from global memory
    // after the wait: pull them into L2 now (one lane per K or V page block)
    const int g = kSaPrePages + (tid >> 1);
    if (g < ceil_div(p, 64)) {
      const uint16_t* kb = st.kv_pool + ((size_t(pt[g]) * L + layer) * 2 * H + h) * 64 * 64;
      bulk_prefetch_l2((tid & 1) ? kb + kv_off : kb, kSaPageBytes);
    }
  }
  float bq = 0.f, bk = 0.f, bv = 0.f;
  if (tid < 64) {
    bq = bf16_to_f32(qkv.bias[h * 64 + tid]);
    bk = bf16_to_f32(qkv.bias[d + h * 64 + tid]);
    bv = bf16_to_f32(qkv.bias[2 * d + h * 64 + tid]);
  }
  pdl_wait();
  if (tid == 0) trace_mark(st, 1);
  if (tid < 64) {
    const int c = h * 64 + tid;
    const float* pp = qkv.p + size_t(r) * qkv.n + c;
    const size_t sstr = size_t(kRows) * qkv.n;
    const float aq = sum_splits(pp, sstr, qkv.splits);
    const float ak = sum_splits(pp + d, sstr, qkv.splits);
    const float av = sum_splits(pp + 2 * d, sstr, qkv.splits);
    const uint16_t kb = f32_to_bf16(ak + bk), vb = f32_to_bf16(av + bv);
    const size_t kbase = ((size_t(pt[p >> 6]) * L + layer) * 2 * H + h) * 64 * 64 + size_t(p & 63) * 64;
    st.kv_pool[kbase + tid] = kb;
    st.kv_pool[kbase + kv_off + tid] = vb;
    qs[tid] = (aq + bq) * q_scale;
    kc[tid] = bf16_to_f32(kb);
    vc[tid] = bf16_to_f32(vb);
  }
  __syncthreads();
  if (tid == 0) trace_mark(st, 4);
  if (np > 0) mbar_wait(bar, 0);
  if (tid == 0) trace_mark(st, 5);
  const int nk = p + 1;
  float mloc = -INFINITY;
  for (int t = tid; t < nk; t += kSaThreads) {
    float s = 0.f;
    if (t < p && t >= 64 * kSaPrePages) {
      const uint4* kr = reinterpret_cast<const uint4*>(
          st.kv_pool + ((size_t(pt[t >> 6]) * L + layer) * 2 * H + h) * 64 * 64 + size_t(t & 63) * 64);
      uint4 w[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) w[j] = __ldg(kr + j);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t ws[4] = {w[j].x, w[j].y, w[j].z, w[j].w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          s = fmaf(qs[8 * j + 2 * u], __uint_as_float(ws[u] << 16), s);
          s = fmaf(qs[8 * j + 2 * u + 1], __uint_as_float(ws[u] & 0xFFFF0000u), s);
        }
      }
    } else if (t < p) {
      // chunk j of key row t read at chunk (j ^ t) & 7: 4 lanes per 16-byte
      // bank group; chunk dot products summed in that (position-fixed) order
      const uint8_t* kr = sa_smem + (t >> 6) * 2 * kSaPageBytes + (t & 63) * 128;
      const int sw = t & 7;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int cc = j ^ sw;
        const uint4 w = *reinterpret_cast<const uint4*>(kr + cc * 16);
        const float4 qa = *reinterpret_cast<const float4*>(qs + 8 * cc);
        const float4 qb = *reinterpret_cast<const float4*>(qs + 8 * cc + 4);
        float sj = qa.x * __uint_as_float(w.x << 16);
        sj = fmaf(qa.y, __uint_as_float(w.x & 0xFFFF0000u), sj);
        sj = fmaf(qa.z, __uint_as_float(w.y << 16), sj);
        sj = fmaf(qa.w, __uint_as_float(w.y & 0xFFFF0000u), sj);
        sj = fmaf(qb.x, __uint_as_float(w.z << 16), sj);
        sj = fmaf(qb.y, __uint_as_float(w.z & 0xFFFF0000u), sj);
        sj = fmaf(qb.z, __uint_as_float(w.w << 16), sj);
        sj = fmaf(qb.w, __uint_as_float(w.w & 0xFFFF0000u), sj);
        s += sj;
      }
    } else {
#pragma unroll 8
      for (int j = 0; j < 64; ++j) s = fmaf(qs[j], kc[j], s);
    }
    sc[t] = s;
    mloc = fmaxf(mloc, s);
  }
  // block max / sum with one barrier each (separate per-warp slots; same
  // reduction order as block_max / block_sum_fixed)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mloc = fmaxf(mloc, __shfl_xor_sync(0xffffffffu, mloc, o));
  if (lane == 0) redm[warp] = mloc;
  __syncthreads();
  float m = -INFINITY;
#pragma unroll
  for (int w = 0; w < kSaThreads / 32; ++w) m = fmaxf(m, redm[w]);
  float lsum = 0.f;
  for (int t = tid; t < nk; t += kSaThreads) {
    const float e = exp2f((sc[t] - m) * kLog2e);
    sc[t] = e;
    lsum += e;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
  if (lane == 0) reds[warp] = lsum;
  __syncthreads();                               // (also publishes sc[])
  float l = 0.f;
#pragma unroll
  for (int w = 0; w < kSaThreads / 32; ++w) l += reds[w];
  if (tid == 0) trace_mark(st, 6);
  float o0 = 0.f, o1 = 0.f;
#pragma unroll 8
  for (int t = warp; t < nk; t += kSaWarps) {
    float v0, v1;
    if (t < p) {
      const uint32_t w =
          t < 64 * kSaPrePages
              ? *reinterpret_cast<const uint32_t*>(sa_smem + (t >> 6) * 2 * kSaPageBytes +
                                                   kSaPageBytes + (t & 63) * 128 + lane * 4)
              : __ldg(reinterpret_cast<const uint32_t*>(
                          st.kv_pool + ((size_t(pt[t >> 6]) * L + layer) * 2 * H + h) * 64 * 64 +
                          kv_off + size_t(t & 63) * 64) + lane);
      v0 = __uint_as_float(w << 16);
      v1 = __uint_as_float(w & 0xFFFF0000u);
    } else {
      v0 = vc[2 * lane];
      v1 = vc[2 * lane + 1];
    }
    const float e = sc[t];
    o0 = fmaf(e, v0, o0);
    o1 = fmaf(e, v1, o1);
  }
  op[warp][2 * lane] = o0;
  op[warp][2 * lane + 1] = o1;
  __syncthreads();
  if (tid == 0) trace_mark(st, 7);
  if (tid < 64) {
    float a = 0.f;
#pragma unroll
    for (int w = 0; w < kSaWarps; ++w) a += op[w][tid];
    store_hilo1(st, r, h * 64 + tid, a / l);
  }
  if (tid == 0) trace_mark(st, 3);
}

int launch_self_attn(const DecodeState& st, int layer, const Partials& qkv, float q_scale,
                     cudaStream_t stream) {
  DM_REQUIRE(qkv.p != nullptr && qkv.n == 3 * st.d && qkv.bias != nullptr &&
                 qkv.splits >= 1 && qkv.splits <= kMaxSplits, "self-attn: qkv partials");
  DM_REQUIRE(st.page_tokens == 64 && st.pages_per_slot * 64 <= kSaMaxKeys, "self-attn: page geometry");
  const int smem = kSaPrePages * 2 * kSaPageBytes + 16;
  DM_SMEM_ATTR(self_attn_kernel, smem);
  DM_CHECK_CUDA(launch_pdl(self_attn_kernel, dim3(st.grid_rows, st.heads), dim3(kSaThreads), smem,
                           stream, st, layer, qkv, q_scale));
  return 0;
}

constexpr int kXaThreads = 128;                               // 4 warps = the 4 TMEM quadrants
constexpr int kXaBoxes = kXaKeysPerSplit / 64;                // 64-key TMA boxes per split
constexpr int kXaKeys = kXaKeysPerSplit;
static_assert(kXSplits * kXaKeys >= 1500 && (kXSplits - 1) * kXaKeys < 1500, "key splits");
constexpr int kXaTmemCols = (kXaBoxes + 1) * 8 <= 32 ? 32 : ((kXaBoxes + 1) * 8 <= 64 ? 64 : 128);

// Cross-attention of the fed token (modeling_whisper.py:398-406, encoder_attn
// of the decoder layer; q.64^-1/2 at :310), one CTA per (row, head, key split
// of 192 keys). The split's K and V blocks (contiguous in the slot's cross-KV
// cache) are TMA-loaded into shared memory before the dependency wait; after
// it only q is read. Scores and P.V run on the tensor cores (tcgen05, fp32
// TMEM accumulators) with fp32-equivalent operands split into bf16 hi/lo pairs:
//   S^T[64 keys x 8] = K_box[64 x 64] . [q_hi; q_lo; 0]^T   (3 boxes, M = 64)
//   s = S[:, 0] + S[:, 1]                                    (q = q_hi + q_lo)
//   O^T[64 dims x 8] = V^T[64 x 192] . [p_hi; p_lo; 0]^T     (V as the MN-major
//   A operand straight from the TMA box, M = 64)
// so the CUDA cores only do the softmax. Each split writes (o[64], max, sum)
// to global scratch and leaves; the last of the 8 splits to arrive (a
// per-(row, head) counter) merges them in split order and stores o_head as
// the bf16 hi/lo operand of the cross-o tcgen05 GEMV that follows. Every
// reduction order depends only on d and key positions, never on the batch.
// (Measured alternatives: the same math with the 8 splits as a
// cluster merging over DSMEM and the cross-o projection in the tail; a
// persistent 2-CTA/SM grid with a K/V ring; warp-level mma.sync; all slower
// at 64 rows, the cluster form faster below ~32 rows.)
constexpr int kXaQOff = 2 * kXaKeys * 128;                // B operand [q_hi; q_lo; 0] (1 KB)
constexpr int kXaPOff = kXaQOff + 1024;                   // B operand [p_hi; p_lo; 0] (1 KB per box)
constexpr int kXaBarOff = kXaPOff + kXaBoxes * 1024;
constexpr int kXaSmem = 1024 + kXaBarOff + 64;          // (align) K, V, q / p operands, mbarriers
constexpr uint32_t kXaIdescS = umma_idesc_bf16(64, 8);                 // K-major A and B
constexpr uint32_t kXaIdescO = umma_idesc_bf16(64, 8) | (1u << 15);    // A (V^T) MN-major

__device__ __forceinline__ void tmem_ld2(uint32_t taddr, uint32_t& a, uint32_t& b) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];"
               : "=r"(a), "=r"(b) : "r"(taddr));
}


// Merge of the (o, max, sum) results of a (row, head)'s splits, in split
// order, into the cross-o operand; thread `c` < 64 does head dimension c. The
// same arithmetic in the last-arriver tail and in xattn_merge_kernel, so both
// paths give the same bits.
__device__ __forceinline__ void xattn_merge_head(const DecodeState& st, const float* xpart, int r,
                                                 int h, int nsplit, int c) {
  uint16_t hi, lo;
  split_hilo(xattn_merged(st, xpart, r, h, nsplit, c), hi, lo);
  const size_t idx = size_t(r) * st.d + h * 64 + c;
  st.ah[idx] = hi;
  st.al[idx] = lo;
}

// After a split's (o, max, sum) is in `xpart`: count it; the last of the 8
// splits of (row, head) merges them in split order into the cross-o operand.
// (Few-row steps only: the release fence and the counter round trip keep every
// CTA -- and its 52 KB of K/V staging -- alive ~2 us longer, 29 of 101 us per
// layer at 64 rows; many-row steps merge in xattn_merge_kernel instead.)
__device__ __forceinline__ void xattn_finish(const DecodeState& st, const float* xpart, int* xcnt,
                                             int r, int h, int nsplit, int tid, int* is_last) {
  const int H = st.heads;
  // the CTA's result stores, then one release by thread 0 (cumulative over
  // the barrier), and the last arriver's acquire before it reads the others
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    *is_last = atomicAdd(&xcnt[r * H + h], 1) == nsplit - 1;
    if (*is_last) __threadfence();
  }
  __syncthreads();
  if (!*is_last) return;
  if (tid < 64) xattn_merge_head(st, xpart, r, h, nsplit, tid);
  if (tid == 0) {
    xcnt[r * H + h] = 0;                         // ready for the next launch of any layer
    trace_mark(st, 3);
  }
}

// The split merge as its own kernel (steps with more than kXaTailMergeRows
// rows): one thread per (row, head, dimension); the cross-attention CTAs
// store their split results and leave.
__global__ void __launch_bounds__(256)
xattn_merge_kernel(const DecodeState st, const float* __restrict__ xpart) {
  if (threadIdx.x == 0) trace_mark(st, 0);
  pdl_trigger();
  const int r = blockIdx.y, h = blockIdx.x * 4 + threadIdx.x / 64;
  pdl_wait();
  if (threadIdx.x == 0) trace_mark(st, 1);
  if (r >= *st.n_active || h >= st.heads) return;
  const int nsplit = ceil_div(st.enc_len[st.active[r]], kXaKeys);
  xattn_merge_head(st, xpart, r, h, nsplit, threadIdx.x % 64);
  if (threadIdx.x == 0) trace_mark(st, 3);
}

int launch_xattn_merge(const DecodeState& st, const float* xpart, cudaStream_t stream) {
  DM_REQUIRE(xpart != nullptr && st.heads <= kMaxHeads, "cross-attn merge: scratch");
  DM_CHECK_CUDA(launch_pdl(xattn_merge_kernel, dim3(ceil_div(st.heads, 4), st.grid_rows),
                           dim3(256), 0, stream, st, xpart));
  return 0;
}

__global__ void __launch_bounds__(kXaThreads, kXaCtasPerSm)
cross_attn_kernel(const __grid_constant__ CUtensorMap tm, const DecodeState st, int layer,
                       const Partials xq, float q_scale, float* __restrict__ xpart,
                       int* __restrict__ xcnt, int probe, int tail_merge) {
  extern __shared__ uint8_t xa_raw[];
  uint8_t* xa_smem = xa_raw + ((1024 - (smem_u32(xa_raw) & 1023)) & 1023);
  __shared__ float redm[4], reds[4];
  __shared__ uint32_t tmem_slot;
  __shared__ int is_last;
  // grid (split, head, row): a row's splits are adjacent in launch order, so the
  // splits past a short window (which leave at once) interleave with real ones
  const int sp = blockIdx.x, h = blockIdx.y, r = blockIdx.z, tid = threadIdx.x;
  const int warp = tid / 32, lane = tid % 32;
  if (tid == 0) trace_mark(st, 0);
  if (r >= *st.n_active) return;
  const int slot = st.active[r];
  const int H = st.heads;
  // splits past a (length-aware) segment's window do not exist for it: the
  // CTA leaves at once and the merge counts only the slot's own splits
  const int len = st.enc_len[slot], nsplit = ceil_div(len, kXaKeys);
  if (sp >= nsplit) return;
  const int k0 = sp * kXaKeys, nk = min(len, k0 + kXaKeys) - k0;
  float* res = xpart + ((size_t(r) * H + h) * kXSplits + sp) * kXpStride;
  uint8_t* Ks = xa_smem;
  uint8_t* Vs = xa_smem + kXaKeys * 128;
  uint8_t* Qs = xa_smem + kXaQOff;
  uint8_t* Ps = xa_smem + kXaPOff;
  uint64_t* barK = reinterpret_cast<uint64_t*>(xa_smem + kXaBarOff);
  uint64_t* barV = barK + 1;
  uint64_t* barS = barK + 2;
  uint64_t* barO = barK + 3;
  if (tid == 0) {
    mbar_init(barK, 1);
    mbar_init(barV, 1);
    mbar_init(barS, 1);
    mbar_init(barO, 1);
    fence_barrier_init();
    tma_prefetch_desc(&tm);
    const int row_k = (((layer * st.max_slots + slot) * 2 + 0) * H + h) * 1500 + k0;
    const int row_v = row_k + H * 1500;
    const uint64_t stream = l2_policy_evict_first();
    mbar_arrive_expect_tx(barK, kXaBoxes * 64 * 128);
#pragma unroll
    for (int bx = 0; bx < kXaBoxes; ++bx)
      tma_load_2d_hint(Ks + bx * 64 * 128, &tm, barK, 0, row_k + bx * 64, stream);
    mbar_arrive_expect_tx(barV, kXaBoxes * 64 * 128);
#pragma unroll
    for (int bx = 0; bx < kXaBoxes; ++bx)
      tma_load_2d_hint(Vs + bx * 64 * 128, &tm, barV, 0, row_v + bx * 64, stream);
  }
  if (warp == 1) tmem_alloc(&tmem_slot, kXaTmemCols);
  for (int i = tid; i < (1 + kXaBoxes) * 1024 / 16; i += kXaThreads) {
    const int row = (i * 16 / 128) & 7;
    if (row >= 2) reinterpret_cast<uint4*>(Qs)[i] = make_uint4(0u, 0u, 0u, 0u);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  pdl_trigger();                                 // (after the TMEM allocation, see gemv_kernel)
  const float bq = tid < 64 ? bf16_to_f32(xq.bias[h * 64 + tid]) : 0.f;
  pdl_wait();
  if (tid == 0) trace_mark(st, 1);
  if (probe == 1) {                              // (timing probe: the K/V stream alone)
    mbar_wait(barK, 0);
    mbar_wait(barV, 0);
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc(tmem, kXaTmemCols);
    return;
  }
  if (tid < 64) {
    const float* pp = xq.p + size_t(r) * xq.n + h * 64 + tid;
    const float a = sum_splits(pp, size_t(kRows) * xq.n, xq.splits);
    const float qv = (a + bq) * q_scale;
    uint16_t hi, lo;
    split_hilo(qv, hi, lo);
    *reinterpret_cast<uint16_t*>(Qs + sw128_off(0, tid)) = hi;
    *reinterpret_cast<uint16_t*>(Qs + sw128_off(1, tid)) = lo;
  }
  fence_proxy_async_smem();
  __syncthreads();
  if (tid == 0) {
    mbar_wait(barK, 0);
    tc_fence_after();
    const uint64_t bq_desc = umma_desc_sw128(smem_u32(Qs));
#pragma unroll
    for (int bx = 0; bx < kXaBoxes; ++bx) {
      const uint64_t ak = umma_desc_sw128(smem_u32(Ks + bx * 64 * 128));
#pragma unroll
      for (int k = 0; k < 4; ++k)
        umma_bf16_ss(tmem + bx * 8, ak + 2 * k, bq_desc + 2 * k, kXaIdescS, k != 0);
    }
    umma_commit(barS);
  }
  if (warp < 4) {
    const bool own = lane < 16;
    float s3[kXaBoxes], e3[kXaBoxes];
    mbar_wait(barS, 0);
    tc_fence_after();
    uint32_t a[kXaBoxes], b[kXaBoxes];
    const uint32_t lane_base = uint32_t(warp * 32) << 16;
#pragma unroll
    for (int j = 0; j < kXaBoxes; ++j) tmem_ld2(tmem + lane_base + j * 8, a[j], b[j]);
    tmem_wait_ld();
    float mloc = -INFINITY;
#pragma unroll
    for (int j = 0; j < kXaBoxes; ++j) {
      const int key = 64 * j + 16 * warp + lane;
      s3[j] = (own && key < nk) ? __uint_as_float(a[j]) + __uint_as_float(b[j]) : -INFINITY;
      mloc = fmaxf(mloc, s3[j]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mloc = fmaxf(mloc, __shfl_xor_sync(0xffffffffu, mloc, o));
    if (lane == 0) redm[warp] = mloc;
    named_bar_sync(1, 128);
    const float m = fmaxf(fmaxf(redm[0], redm[1]), fmaxf(redm[2], redm[3]));
    float es = 0.f;
#pragma unroll
    for (int j = 0; j < kXaBoxes; ++j) {
      e3[j] = s3[j] == -INFINITY ? 0.f : exp2f((s3[j] - m) * kLog2e);
      es += e3[j];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) es += __shfl_xor_sync(0xffffffffu, es, o);
    if (lane == 0) reds[warp] = es;
    if (own) {
#pragma unroll
      for (int j = 0; j < kXaBoxes; ++j) {
        uint16_t hi, lo;
        split_hilo(e3[j], hi, lo);
        const int kk = 16 * warp + lane;
        *reinterpret_cast<uint16_t*>(Ps + j * 1024 + sw128_off(0, kk)) = hi;
        *reinterpret_cast<uint16_t*>(Ps + j * 1024 + sw128_off(1, kk)) = lo;
      }
    }
    fence_proxy_async_smem();
    named_bar_sync(1, 128);
    if (tid == 0) {
      res[64] = m;
      res[65] = (reds[0] + reds[1]) + (reds[2] + reds[3]);
      mbar_wait(barV, 0);
      tc_fence_after();
#pragma unroll
      for (int j = 0; j < kXaBoxes; ++j) {
        const uint64_t bp = umma_desc_sw128(smem_u32(Ps + j * 1024));
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint64_t av = umma_desc_sw128(smem_u32(Vs + j * 64 * 128 + k * 2048));
          umma_bf16_ss(tmem + kXaBoxes * 8, av, bp + 2 * k, kXaIdescO, (j | k) != 0);
        }
      }
      umma_commit(barO);
    }
    mbar_wait(barO, 0);
    tc_fence_after();
    uint32_t oa, ob;
    tmem_ld2(tmem + lane_base + kXaBoxes * 8, oa, ob);
    tmem_wait_ld();
    if (own) res[16 * warp + lane] = __uint_as_float(oa) + __uint_as_float(ob);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, kXaTmemCols);
  if (!tail_merge) return;                       // xattn_merge_kernel follows
  xattn_finish(st, xpart, xcnt, r, h, nsplit, tid, &is_last);
}

int launch_cross_attn(const DecodeState& st, const CUtensorMap& xkv_map, int layer,
                           const Partials& xq, float q_scale, float* xpart, int* xcnt,
                           cudaStream_t stream, int probe, bool tail_merge) {
  DM_REQUIRE(xq.p != nullptr && xq.n == st.d && xq.bias != nullptr && xq.splits >= 1 &&
                 xq.splits <= kMaxSplits, "cross-attn: q partials");
  DM_REQUIRE(xpart != nullptr && xcnt != nullptr && st.heads <= kMaxHeads, "cross-attn: scratch");
  DM_SMEM_ATTR(cross_attn_kernel, kXaSmem);
  DM_CHECK_CUDA(launch_pdl(cross_attn_kernel, dim3(kXSplits, st.heads, st.grid_rows),
                           dim3(kXaThreads), kXaSmem, stream, xkv_map, st, layer, xq, q_scale,
                           xpart, xcnt, probe, int(tail_merge && probe != 2)));
  return 0;
}

// ============================================================ split-K GELU
// fc1 of the large models: the GEMV writes K-split partials like the linear
// projections, and this kernel reduces them in split order, adds the bias,
// applies the exact GELU and writes the bf16 hi/lo operand of fc2 -- the
// epilogue spread over every SM instead of the last CTA of each tile.
__global__ void __launch_bounds__(256)
gelu_hilo_kernel(const DecodeState st, const Partials p, uint16_t* __restrict__ yh,
                 uint16_t* __restrict__ yl) {
  if (threadIdx.x == 0) trace_mark(st, 0);
  pdl_trigger();
  const int r = blockIdx.y;
  const int n4 = blockIdx.x * blockDim.x + threadIdx.x;        // 4 features each
  float4 b = make_float4(0.f, 0.f, 0.f, 0.f);
  if (4 * n4 < p.n) b = bf16x4_to_f32(__ldg(reinterpret_cast<const uint2*>(p.bias) + n4));
  pdl_wait();
  if (threadIdx.x == 0) trace_mark(st, 1);
  if (r >= *st.n_active || 4 * n4 >= p.n) return;
  // (fc1's split is 4 by default: a 4-wide load set keeps the registers and
  // the loads in flight small; same split-order sums either way)
  const float4 a = p.splits <= 4
                       ? sum_splits4<4>(p.p + size_t(r) * p.n + 4 * n4, size_t(kRows) * p.n, p.splits)
                       : sum_splits4<kMaxHeads>(p.p + size_t(r) * p.n + 4 * n4, size_t(kRows) * p.n,
                                                p.splits);
  const float v[4] = {a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w};
  uint16_t h[4], l[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) split_hilo(gelu_erf(v[i]), h[i], l[i]);
  const size_t o = size_t(r) * p.n + 4 * n4;
  *reinterpret_cast<uint2*>(yh + o) = make_uint2(uint32_t(h[0]) | (uint32_t(h[1]) << 16),
                                                 uint32_t(h[2]) | (uint32_t(h[3]) << 16));
  *reinterpret_cast<uint2*>(yl + o) = make_uint2(uint32_t(l[0]) | (uint32_t(l[1]) << 16),
                                                 uint32_t(l[2]) | (uint32_t(l[3]) << 16));
  if (threadIdx.x == 0) trace_mark(st, 3);
}

int launch_gelu_hilo(const DecodeState& st, const Partials& p, uint16_t* yh, uint16_t* yl,
                     cudaStream_t stream) {
  DM_REQUIRE(p.p != nullptr && p.bias != nullptr && p.n % 4 == 0 && p.splits >= 1 &&
                 p.splits <= kMaxHeads, "gelu: partials");
  DM_CHECK_CUDA(launch_pdl(gelu_hilo_kernel, dim3(ceil_div(p.n / 4, 256), st.grid_rows), dim3(256),
                           0, stream, st, p, yh, yl));
  return 0;
}

// ============================================================ finalize
// One warp per active row: argmax over the vocab-tile partials (ties -> lowest
// id), then the greedy state machine (prompt forcing, EOT, per-slot cap).
// LM head tail: logits = the K-split partials summed in split order, then per
// (128-id vocabulary tile, row) the argmax (ties -> lowest id) into
// amax_val / amax_idx for finalize_kernel -- the values and ties of the GEMV's
// last-CTA ARGMAX merge, without its per-tile release fence and counter.
// One warp per (tile, row), lane l covers ids 4l .. 4l + 3 of the tile (each
// lane scans its ids in increasing order, so a tie keeps the lowest id).
__global__ void __launch_bounds__(256)
lm_argmax_kernel(const DecodeState st, const Partials p) {
  if (threadIdx.x == 0) trace_mark(st, 0);
  pdl_trigger();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int tiles = ceil_div(st.vocab, 128);
  const int tile = blockIdx.x, r = blockIdx.y * 8 + warp;
  pdl_wait();
  if (threadIdx.x == 0) trace_mark(st, 1);
  if (r >= *st.n_active || tile >= tiles) return;
  const size_t stride = size_t(kRows) * p.n;
  float best = -INFINITY;
  int bidx = 0x7FFFFFFF;
  float v[4][kMaxSplits];
#pragma unroll
  for (int u = 0; u < 4; ++u) {                 // all loads first
    const int n = tile * 128 + 4 * lane + u;
    const float* q = p.p + size_t(r) * p.n + n;
#pragma unroll
    for (int s = 0; s < kMaxSplits; ++s) v[u][s] = (s < p.splits && n < st.vocab) ? __ldcg(q + s * stride) : 0.f;
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int n = tile * 128 + 4 * lane + u;
    if (n >= st.vocab) break;
    float a = v[u][0];
#pragma unroll
    for (int s = 1; s < kMaxSplits; ++s)
      if (s < p.splits) a += v[u][s];
    if (st.logits_dbg) st.logits_dbg[size_t(r) * st.vocab + n] = a;
    if (a > best) { best = a; bidx = n; }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const float ob = __shfl_xor_sync(0xffffffffu, best, off);
    const int oi = __shfl_xor_sync(0xffffffffu, bidx, off);
    if (ob > best || (ob == best && oi < bidx)) { best = ob; bidx = oi; }
  }
  if (lane == 0) {
    st.amax_val[size_t(tile) * kRows + r] = best;
    st.amax_idx[size_t(tile) * kRows + r] = bidx;
  }
  if (threadIdx.x == 0) trace_mark(st, 3);
}

int launch_lm_argmax(const DecodeState& st, const Partials& p, cudaStream_t stream) {
  DM_REQUIRE(p.p != nullptr && p.n == st.vocab && p.splits >= 1 &&
                 p.splits <= kMaxSplits, "LM head argmax: partials");
  DM_CHECK_CUDA(launch_pdl(lm_argmax_kernel, dim3(ceil_div(st.vocab, 128), ceil_div(st.grid_rows, 8)),
                           dim3(256), 0, stream, st, p));
  return 0;
}

__global__ void finalize_kernel(const DecodeState st) {
  const int r = blockIdx.x * 4 + threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) trace_mark(st, 0);
  pdl_trigger();
  pdl_wait();
  if (threadIdx.x == 0) trace_mark(st, 1);
  if (lane == 0) trace_mark(st, 3);
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

}  // namespace dm
