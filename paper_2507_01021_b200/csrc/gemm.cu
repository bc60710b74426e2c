// tcgen05 GEMM: persistent, warp-specialised, TMA -> 128B-swizzled smem ring
// -> tcgen05.mma (M=128, N=BN, K=16 per instruction, fp32 accumulators in
// TMEM, double-buffered) -> 4 epilogue warps (tcgen05.ld -> fused epilogue ->
// global). Implements the encoder's conv stem (implicit im2col: each conv tap
// is a separate K range read through its own TMA coordinates), the layer GEMMs
// and the cross-KV precompute.
//
// Batch invariance: the reduction order of every output element depends only
// on K (fixed BLOCK_K = 64, no split-K), never on M or on batch composition.

#include <cudaTypedefs.h>

#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <mutex>

#include "gemm.cuh"

namespace dm {

constexpr int kBM = 128;
constexpr int kBK = 64;
constexpr int kGemmThreads = 320;   // w0 TMA, w1 MMA + TMEM alloc, w2..9 epilogue
constexpr int kEpiWarps = 8;        // two warpgroups, each drains half of the tile's columns

__device__ __forceinline__ void tma_load_4d(void* smem_dst, const CUtensorMap* m,
                                            uint64_t* bar, int c0, int c1, int c2,
                                            int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::"
      "bytes [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1),
      "r"(c2), "r"(c3)
      : "memory");
}

struct TileGeom {
  int MT, NT, tiles, KB, cpb;   // cpb = channel blocks per conv tap
};

template <int BN, int MODE>
__device__ __forceinline__ void epilogue_chunk(const Epilogue& e, const GemmArgs& g,
                                               int b, int t, int row_valid, int n0,
                                               uint32_t (&r)[32], const float4* pre = nullptr,
                                               const uint4* bpre = nullptr) {
  float v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
  if (e.bias != nullptr) {     // (EPI_W2V_POS carries its bias in e.pos, indexed by channel)
    const uint4* bp = reinterpret_cast<const uint4*>(e.bias + n0);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      uint4 w = bpre ? bpre[i] : __ldg(bp + i);
      uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        v[i * 8 + 2 * j] += __uint_as_float(ws[j] << 16);
        v[i * 8 + 2 * j + 1] += __uint_as_float(ws[j] & 0xFFFF0000u);
      }
    }
  }
  if (!row_valid) return;
  const int N = g.N;
  switch (MODE) {
    case EPI_GELU_BF16:
    case EPI_GELU_F32:
    case EPI_CONV1:
    case EPI_CONV2_POS:
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = gelu_erf(v[i]);
      break;
    default:
      break;
  }
  switch (MODE) {
    case EPI_STORE_BF16:
    case EPI_GELU_BF16:
    case EPI_CONV1: {
      size_t row = (MODE == EPI_CONV1) ? size_t(b) * (g.T + 2) + t + 1
                                         : size_t(b) * g.T + t;
      uint4* dst = reinterpret_cast<uint4*>(static_cast<uint16_t*>(e.out) +
                                            row * e.ldo + n0);
#pragma unroll
      for (int i = 0; i < 4; ++i)
        dst[i] = make_uint4(pack_bf16x2(v[8 * i], v[8 * i + 1]),
                            pack_bf16x2(v[8 * i + 2], v[8 * i + 3]),
                            pack_bf16x2(v[8 * i + 4], v[8 * i + 5]),
                            pack_bf16x2(v[8 * i + 6], v[8 * i + 7]));
      break;
    }
    case EPI_CONV2_POS: {
      const uint4* pp = reinterpret_cast<const uint4*>(e.pos + size_t(t) * N + n0);
      float4* dst = reinterpret_cast<float4*>(static_cast<float*>(e.out) +
                                              (size_t(b) * g.T + t) * e.ldo + n0);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        uint4 w = __ldg(pp + i);
        uint32_t ws[4] = {w.x, w.y, w.z, w.w};
        float o[8];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          o[2 * j] = v[i * 8 + 2 * j] + __uint_as_float(ws[j] << 16);
          o[2 * j + 1] = v[i * 8 + 2 * j + 1] + __uint_as_float(ws[j] & 0xFFFF0000u);
        }
        dst[2 * i] = make_float4(o[0], o[1], o[2], o[3]);
        dst[2 * i + 1] = make_float4(o[4], o[5], o[6], o[7]);
      }
      break;
    }
    case EPI_RESID_F32:
    case EPI_GELU_F32:
    case EPI_STORE_F32: {
      float4* dst = reinterpret_cast<float4*>(static_cast<float*>(e.out) +
                                              (size_t(b) * g.T + t) * e.ldo + n0);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float4 o = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
        if (MODE == EPI_RESID_F32) {
          float4 rr = pre ? pre[i] : dst[i];
          o.x += rr.x; o.y += rr.y; o.z += rr.z; o.w += rr.w;
        }
        dst[i] = o;
      }
      break;
    }
    case EPI_QKV: {
      // global row -> (segment, position)
      const int d = N / 3;
      const int row = b * g.T + t;
      const int seg = row / e.seg_rows, pos = row % e.seg_rows;
      const int region = n0 / d, h = (n0 % d) / 64, j0 = n0 % 64;
      const size_t head = size_t(seg) * e.heads + h;
      if (region < 2) {
        uint16_t* base = region == 0 ? e.q : e.k;
        const float sc = region == 0 ? e.q_scale : 1.0f;
        uint4* dst = reinterpret_cast<uint4*>(base + (head * e.t_pad + pos) * 64 + j0);
#pragma unroll
        for (int i = 0; i < 4; ++i)
          dst[i] = make_uint4(pack_bf16x2(v[8 * i] * sc, v[8 * i + 1] * sc),
                              pack_bf16x2(v[8 * i + 2] * sc, v[8 * i + 3] * sc),
                              pack_bf16x2(v[8 * i + 4] * sc, v[8 * i + 5] * sc),
                              pack_bf16x2(v[8 * i + 6] * sc, v[8 * i + 7] * sc));
      } else {
        uint16_t* base = e.vt + (head * 64 + j0) * e.t_pad + pos;
#pragma unroll
        for (int i = 0; i < 32; ++i) base[size_t(i) * e.t_pad] = f32_to_bf16(v[i]);
      }
      break;
    }
    case EPI_XKV: {
      const int d = N / (2 * e.layers);
      const int row = b * g.T + t;
      const int seg = row / e.seg_rows, pos = row % e.seg_rows;
      const int slot = e.slot_ids[seg];
      const int l = n0 / (2 * d), kv = (n0 / d) % 2, h = (n0 % d) / 64, j0 = n0 % 64;
      size_t idx = ((((size_t(l) * e.n_slots + slot) * 2 + kv) * e.heads + h) * 1500 + pos) * 64 + j0;
      uint4* dst = reinterpret_cast<uint4*>(static_cast<uint16_t*>(e.out) + idx);
#pragma unroll
      for (int i = 0; i < 4; ++i)
        dst[i] = make_uint4(pack_bf16x2(v[8 * i], v[8 * i + 1]),
                            pack_bf16x2(v[8 * i + 2], v[8 * i + 3]),
                            pack_bf16x2(v[8 * i + 4], v[8 * i + 5]),
                            pack_bf16x2(v[8 * i + 6], v[8 * i + 7]));
      break;
    }
    case EPI_W2V_PROJ: {
      const int row = b * g.T + t;
      const int seg = row / e.seg_rows, pos = row % e.seg_rows;
      const bool valid = pos < e.seg_len[seg];
      float4* dst = reinterpret_cast<float4*>(static_cast<float*>(e.out) + size_t(row) * e.ldo + n0);
#pragma unroll
      for (int i = 0; i < 8; ++i)
        dst[i] = valid ? make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3])
                       : make_float4(0.f, 0.f, 0.f, 0.f);
      // grouped bf16 copy: channel ch -> group ch / cpg, slot ch % cpg (64-wide groups)
      uint16_t* gp = e.grp + (size_t(seg) * (e.seg_rows + 2 * e.grp_pad) + e.grp_pad + pos) *
                                 (size_t(N) / e.grp_cpg * 64);
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const int ch = n0 + i;
        gp[(ch / e.grp_cpg) * 64 + ch % e.grp_cpg] = valid ? f32_to_bf16(v[i]) : uint16_t(0);
      }
      break;
    }
    case EPI_W2V_POS: {
      // n0 covers 32 of a 64-wide group tile; slots >= cpg are padding
      const int grp_i = n0 / 64, j0 = n0 % 64;
      if (j0 >= e.grp_cpg) break;
      const int row = b * g.T + t;
      float* x = static_cast<float*>(e.out) + size_t(row) * e.ldo;
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const int j = j0 + i;
        if (j < e.grp_cpg) {
          const int ch = grp_i * e.grp_cpg + j;
          x[ch] += gelu_erf(v[i] + bf16_to_f32(e.pos[ch]));
        }
      }
      break;
    }
    case EPI_CTC_ARGMAX: {
      if (n0 != 0) break;
      float best = v[0];
      int bi = 0;
#pragma unroll
      for (int i = 1; i < 32; ++i)
        if (i < N && v[i] > best) { best = v[i]; bi = i; }
      static_cast<int32_t*>(e.out)[size_t(b) * g.T + t] = bi;
      break;
    }
    default:
      break;
  }
}

// fp32 residual tiles (EPI_RESID_F32, BN = 128) are TMA-loaded by the
// producer into a 64 KB shared buffer -- four 32-column boxes, 128B-swizzled
// -- as soon as the epilogue has taken the previous tile's residual into
// registers, so the epilogue never waits on a global load.
template <int BN, int STAGES, int MODE>
constexpr bool kResTma = BN == 128 && STAGES == 5 && MODE == EPI_RESID_F32;

template <int BN, int STAGES, int MODE>
struct GemmSmem {
  static constexpr int kABytes = kBM * kBK * 2;
  static constexpr int kBBytes = BN * kBK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kResBytes = kResTma<BN, STAGES, MODE> ? kBM * BN * 4 : 0;
  static constexpr int kBytes = STAGES * kStageBytes + kResBytes + 1024 /*align*/ + 256 /*bars*/;
};

template <int BN, int STAGES, int MODE>
__global__ void __launch_bounds__(kGemmThreads, 1)
gemm_tcgen05_kernel(const __grid_constant__ CUtensorMap tmap_a,
                    const __grid_constant__ CUtensorMap tmap_b,
                    const __grid_constant__ CUtensorMap tmap_r, const GemmArgs g,
                    const TileGeom geo) {
  using S = GemmSmem<BN, STAGES, MODE>;
  constexpr bool RT = kResTma<BN, STAGES, MODE>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024 - (raw_addr & 1023)) & 1023);
  uint8_t* rbuf = smem + STAGES * S::kStageBytes;                     // [4 boxes][128 rows][128 B]
  uint64_t* full = reinterpret_cast<uint64_t*>(rbuf + S::kResBytes);
  uint64_t* empty = full + STAGES;
  uint64_t* tmem_full = empty + STAGES;      // [2]
  uint64_t* tmem_empty = tmem_full + 2;      // [2]
  uint64_t* res_full = tmem_empty + 2;
  uint64_t* res_empty = res_full + 1;
  uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(res_empty + 1);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmap_a);
    tma_prefetch_desc(&tmap_b);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tmem_full[s], 1);
      mbar_init(&tmem_empty[s], kEpiWarps);   // one arrive per epilogue warp
    }
    mbar_init(res_full, 1);
    mbar_init(res_empty, kEpiWarps);
    if (RT) tma_prefetch_desc(&tmap_r);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_base_slot, 2 * BN);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_base_slot;

  if (warp == 0) {
    // ---------------- TMA producer
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int tile = blockIdx.x; tile < geo.tiles; tile += gridDim.x, ++it) {
        const int nt = tile % geo.NT;
        const int mb = g.mblocks[0] ? g.mblocks[0][tile / geo.NT] : tile / geo.NT;
        const int b = mb / geo.MT, mt = mb % geo.MT;
        if (RT) {
          // this tile's residual, once the epilogue holds the previous one in registers
          mbar_wait(res_empty, (it & 1) ^ 1);
          mbar_arrive_expect_tx(res_full, S::kResBytes);
#pragma unroll
          for (int j = 0; j < BN / 32; ++j)
            tma_load_2d(rbuf + j * (kBM * 128), &tmap_r, res_full, nt * BN + j * 32,
                        b * g.T + mt * kBM);
        }
        for (int kb = 0; kb < geo.KB; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * S::kStageBytes;
          uint8_t* sb = sa + S::kABytes;
          mbar_arrive_expect_tx(&full[stage], S::kStageBytes);
          if (g.a_mode == A_FLAT) {
            tma_load_3d(sa, &tmap_a, &full[stage], kb * kBK, mt * kBM, b);
          } else {
            const int tap = kb / geo.cpb;
            const int c0 = (kb % geo.cpb) * kBK + (g.grouped ? nt * kBK : 0);
            if (g.a_mode == A_CONV_S1)
              tma_load_3d(sa, &tmap_a, &full[stage], c0, mt * kBM + tap, b);
            else
              tma_load_4d(sa, &tmap_a, &full[stage], c0, tap & 1, mt * kBM + (tap >> 1), b);
          }
          tma_load_2d(sb, &tmap_b, &full[stage], kb * kBK, nt * BN);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer
    constexpr uint32_t idesc = umma_idesc_bf16(kBM, BN);
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (int tile = blockIdx.x; tile < geo.tiles; tile += gridDim.x, ++it) {
      const int as = it & 1;
      const uint32_t aphase = (it >> 1) & 1;
      mbar_wait(&tmem_empty[as], aphase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + as * BN;
      for (int kb = 0; kb < geo.KB; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t sa = smem_u32(smem + stage * S::kStageBytes);
          const uint32_t sb = sa + S::kABytes;
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) {
            umma_bf16_ss(d_tmem, umma_desc_sw128(sa + k * 32), umma_desc_sw128(sb + k * 32),
                         idesc, (kb | k) != 0);
          }
          umma_commit(&empty[stage]);
          if (kb == geo.KB - 1) umma_commit(&tmem_full[as]);
        }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else {
    // ---------------- epilogue warps (2..9): TMEM lane quadrant = warp % 4,
    // column half = (warp - 2) / 4
    const int quad = warp & 3;
    const int chalf = (warp - 2) >> 2;
    int it = 0;
    for (int tile = blockIdx.x; tile < geo.tiles; tile += gridDim.x, ++it) {
      const int nt = tile % geo.NT;
      const int mb = g.mblocks[0] ? g.mblocks[0][tile / geo.NT] : tile / geo.NT;
      const int b = mb / geo.MT, mt = mb % geo.MT;
      const int as = it & 1;
      const uint32_t aphase = (it >> 1) & 1;
      const int t = mt * kBM + quad * 32 + lane;
      const int row_valid = t < g.T;
      // fp32 residual of this thread's row segment: independent of the MMA, so
      // it is fetched before waiting for the accumulator (BN = 128: 64 floats)
      constexpr int kPre = BN == 128 ? BN / 8 : 1;
      float4 res[kPre];
      const bool pre = BN == 128 && MODE == EPI_RESID_F32 && row_valid &&
                       nt * BN + (chalf + 1) * (BN / 2) <= g.N;
      if (RT) {
        // rows quad*32 + lane, columns chalf*64 .. +64 = boxes 2*chalf, 2*chalf + 1;
        // 16-byte chunk q of row r sits at chunk q ^ (r & 7) (conflict-free)
        mbar_wait(res_full, it & 1);
        const int tr = quad * 32 + lane;
#pragma unroll
        for (int i = 0; i < kPre; ++i) {
          const int box = chalf * 2 + i / 8, q = i % 8;
          res[i] = *reinterpret_cast<const float4*>(rbuf + box * (kBM * 128) + tr * 128 +
                                                    ((q ^ (tr & 7)) << 4));
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(res_empty);
      } else if (pre) {
        const float4* src = reinterpret_cast<const float4*>(
            static_cast<const float*>(g.epi.out) + (size_t(b) * g.T + t) * g.epi.ldo + nt * BN +
            chalf * (BN / 2));
#pragma unroll
        for (int i = 0; i < kPre; ++i) res[i] = __ldcs(src + i);
      }
      // (and the bias of this thread's columns)
      uint4 bias_pre[BN == 128 ? 8 : 1];
      const bool bpre = BN == 128 && g.epi.bias != nullptr && nt * BN + (chalf + 1) * (BN / 2) <= g.N;
      if (bpre) {
        const uint4* bp = reinterpret_cast<const uint4*>(g.epi.bias + nt * BN + chalf * (BN / 2));
#pragma unroll
        for (int i = 0; i < (BN == 128 ? 8 : 1); ++i) bias_pre[i] = __ldg(bp + i);
      }
      // BN = 256: bias of this thread's first 32-column chunk, fetched before
      // the accumulator wait (later chunks are fetched one chunk ahead)
      uint4 bias_c[4];
      const bool wide_bias = BN != 128 && g.epi.bias != nullptr;
      auto load_bias4 = [&](int c, uint4 (&dst)[4]) {
        const int n0 = nt * BN + c;
        if (wide_bias && n0 + 32 <= g.N) {
          const uint4* bp = reinterpret_cast<const uint4*>(g.epi.bias + n0);
#pragma unroll
          for (int i = 0; i < 4; ++i) dst[i] = __ldg(bp + i);
        }
      };
      if (BN != 128) load_bias4(chalf * (BN / 2), bias_c);
      mbar_wait(&tmem_full[as], aphase);
      tc_fence_after();
      if (BN == 128) {
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
          const int c = chalf * (BN / 2) + cc * 32;
          const int n0 = nt * BN + c;
          uint32_t r[32];
          tmem_ld32(tmem_base + (uint32_t(quad * 32) << 16) + as * BN + c, r);
          tmem_wait_ld();
          if (n0 < g.N)
            epilogue_chunk<BN, MODE>(g.epi, g, b, t, row_valid, n0, r, pre ? res + cc * 8 : nullptr,
                               bpre ? bias_pre + cc * 4 : nullptr);
        }
      } else {
#pragma unroll 1
        for (int c = chalf * (BN / 2); c < (chalf + 1) * (BN / 2); c += 32) {
          const int n0 = nt * BN + c;
          uint4 bias_n[4];
          if (c + 32 < (chalf + 1) * (BN / 2)) load_bias4(c + 32, bias_n);
          uint32_t r[32];
          tmem_ld32(tmem_base + (uint32_t(quad * 32) << 16) + as * BN + c, r);
          tmem_wait_ld();
          if (n0 < g.N)
            epilogue_chunk<BN, MODE>(g.epi, g, b, t, row_valid, n0, r, nullptr,
                                     (wide_bias && n0 + 32 <= g.N) ? bias_c : nullptr);
#pragma unroll
          for (int i = 0; i < 4; ++i) bias_c[i] = bias_n[i];
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tmem_empty[as]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 2 * BN);
  }
}

// ------------------------------------------------------------ CTA-pair GEMM
// 2-SM variant (tcgen05 cta_group::2) for 256 x 256 output tiles. The two
// CTAs of a cluster each hold 128 rows of A and their half (128 rows) of the
// B tile; the leader issues tcgen05.mma.cta_group::2 (M = 256), which reads
// both CTAs' shared memory and writes each CTA's 128 accumulator rows into its
// own TMEM. Per k-block an SM ingests 16 KB of A + 16 KB of B instead of
// 16 + 32 KB: the d = 512 layer GEMMs are bound by that L2 -> SMEM stream.
// Barriers: both CTAs' TMA bytes complete on the leader's `full` barrier
// (peer bit cleared); the MMA commit multicasts to both CTAs' `empty` and
// `tmem_full`; both CTAs' epilogue warps arrive on the leader's `tmem_empty`.
// Per output element the MMA sequence is the same as the 1-SM kernel's, so
// results do not depend on which kernel ran.
constexpr int kPairBN = 256;
constexpr uint32_t kPeerBitMask = 0xFEFFFFFFu;   // clears the CTA-rank bit of a cluster smem address

template <int STAGES>
struct PairSmem {
  static constexpr int kABytes = kBM * kBK * 2;             // 16 KB
  static constexpr int kBBytes = (kPairBN / 2) * kBK * 2;   // 16 KB: this CTA's half of B
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kBytes = STAGES * kStageBytes + 1024 /*align*/ + 256 /*bars*/;
};

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void pair_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma_pair_2d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar) & kPeerBitMask), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_pair_3d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1,
                                            int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar) & kPeerBitMask), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tma_pair_4d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1,
                                            int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar) & kPeerBitMask), "r"(c0), "r"(c1), "r"(c2),
      "r"(c3)
      : "memory");
}
__device__ __forceinline__ void umma_bf16_ss_pair(uint32_t tmem_d, uint64_t a_desc, uint64_t b_desc,
                                                  uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {   // -> both CTAs' barrier
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(uint16_t(3))
      : "memory");
}

template <int STAGES, int MODE>
__global__ void __launch_bounds__(kGemmThreads, 1)
gemm_pair_kernel(const __grid_constant__ CUtensorMap tmap_a,
                 const __grid_constant__ CUtensorMap tmap_b, const GemmArgs g, const TileGeom geo) {
  using S = PairSmem<STAGES>;
  constexpr int BN = kPairBN;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024 - (raw_addr & 1023)) & 1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * S::kStageBytes);
  uint64_t* empty = full + STAGES;
  uint64_t* tmem_full = empty + STAGES;      // [2]
  uint64_t* tmem_empty = tmem_full + 2;      // [2] (the leader's counts both CTAs' epilogues)
  uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int pair = int(blockIdx.x) >> 1, npairs = int(gridDim.x) >> 1;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmap_a);
    tma_prefetch_desc(&tmap_b);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tmem_full[s], 1);
      mbar_init(&tmem_empty[s], 2 * kEpiWarps);
    }
    fence_barrier_init();
  }
  pair_cluster_sync();                       // both CTAs' barriers initialised
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_base_slot)),
                 "r"(uint32_t(2 * BN)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_base_slot;

  if (warp == 0) {
    // ---------------- TMA producer (both CTAs: own A rows, own half of B)
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = pair; tile < geo.tiles; tile += npairs) {
        const int nt = tile % geo.NT;
        const int mb = g.mblocks[1] ? g.mblocks[1][tile / geo.NT] : tile / geo.NT;
        const int b = mb / geo.MT, mt = mb % geo.MT;
        const int row0 = mt * (2 * kBM) + int(rank) * kBM;
        for (int kb = 0; kb < geo.KB; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * S::kStageBytes;
          uint8_t* sb = sa + S::kABytes;
          if (leader) mbar_arrive_expect_tx(&full[stage], 2 * S::kStageBytes);
          if (g.a_mode == A_FLAT) {
            tma_pair_3d(sa, &tmap_a, &full[stage], kb * kBK, row0, b);
          } else {
            const int tap = kb / geo.cpb;
            const int c0 = (kb % geo.cpb) * kBK;
            if (g.a_mode == A_CONV_S1)
              tma_pair_3d(sa, &tmap_a, &full[stage], c0, row0 + tap, b);
            else
              tma_pair_4d(sa, &tmap_a, &full[stage], c0, tap & 1, row0 + (tap >> 1), b);
          }
          tma_pair_2d(sb, &tmap_b, &full[stage], kb * kBK, nt * BN + int(rank) * (BN / 2));
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (leader only)
    if (leader) {
      constexpr uint32_t idesc = umma_idesc_bf16(2 * kBM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int tile = pair; tile < geo.tiles; tile += npairs, ++it) {
        const int as = it & 1;
        const uint32_t aphase = (it >> 1) & 1;
        mbar_wait(&tmem_empty[as], aphase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + as * BN;
        for (int kb = 0; kb < geo.KB; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          if (elect_one()) {
            const uint32_t sa = smem_u32(smem + stage * S::kStageBytes);
            const uint32_t sb = sa + S::kABytes;
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k)
              umma_bf16_ss_pair(d_tmem, umma_desc_sw128(sa + k * 32), umma_desc_sw128(sb + k * 32),
                                idesc, (kb | k) != 0);
            umma_commit_pair(&empty[stage]);
            if (kb == geo.KB - 1) umma_commit_pair(&tmem_full[as]);
          }
          __syncwarp();
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else {
    // ---------------- epilogue warps (2..9): this CTA's 128 rows
    const int quad = warp & 3;
    const int chalf = (warp - 2) >> 2;
    const uint32_t lead_empty0 = [&] {
      uint32_t r;
      asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(smem_u32(tmem_empty)));
      return r;
    }();
    int it = 0;
    for (int tile = pair; tile < geo.tiles; tile += npairs, ++it) {
      const int nt = tile % geo.NT;
      const int mb = g.mblocks[1] ? g.mblocks[1][tile / geo.NT] : tile / geo.NT;
      const int b = mb / geo.MT, mt = mb % geo.MT;
      const int as = it & 1;
      const uint32_t aphase = (it >> 1) & 1;
      const int t = mt * (2 * kBM) + int(rank) * kBM + quad * 32 + lane;
      const int row_valid = t < g.T;
      // bias one 32-column chunk ahead (the first before the accumulator wait)
      uint4 bias_c[4];
      const bool has_bias = g.epi.bias != nullptr;
      auto load_bias4 = [&](int c, uint4 (&dst)[4]) {
        const int n0 = nt * BN + c;
        if (has_bias && n0 + 32 <= g.N) {
          const uint4* bp = reinterpret_cast<const uint4*>(g.epi.bias + n0);
#pragma unroll
          for (int i = 0; i < 4; ++i) dst[i] = __ldg(bp + i);
        }
      };
      load_bias4(chalf * (BN / 2), bias_c);
      mbar_wait(&tmem_full[as], aphase);
      tc_fence_after();
#pragma unroll 1
      for (int c = chalf * (BN / 2); c < (chalf + 1) * (BN / 2); c += 32) {
        const int n0 = nt * BN + c;
        uint4 bias_n[4];
        if (c + 32 < (chalf + 1) * (BN / 2)) load_bias4(c + 32, bias_n);
        uint32_t r[32];
        tmem_ld32(tmem_base + (uint32_t(quad * 32) << 16) + as * BN + c, r);
        tmem_wait_ld();
        if (n0 < g.N)
          epilogue_chunk<BN, MODE>(g.epi, g, b, t, row_valid, n0, r, nullptr,
                                   (has_bias && n0 + 32 <= g.N) ? bias_c : nullptr);
#pragma unroll
        for (int i = 0; i < 4; ++i) bias_c[i] = bias_n[i];
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        const uint32_t bar = lead_empty0 + uint32_t(as) * 8;
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar) : "memory");
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  pair_cluster_sync();                       // both CTAs done with TMEM and peer smem
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(uint32_t(2 * BN)));
  }
}

// ------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
static std::once_flag g_encode_once;

bool tma_available() {
  std::call_once(g_encode_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  return g_encode != nullptr;
}

static int make_map(CUtensorMap* m, const void* ptr, int rank, const cuuint64_t* dims,
                    const cuuint64_t* strides_bytes, const cuuint32_t* box) {
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(ptr), dims,
                        strides_bytes, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed with CUresult " + std::to_string(int(r)));
    return 2;
  }
  return 0;
}

template <int BN, int STAGES, int MODE>
static int launch_bn_mode(const GemmArgs& g, cudaStream_t stream) {
  CUtensorMap ma, mb, mr;
  std::memset(&mr, 0, sizeof(mr));
  if (kResTma<BN, STAGES, MODE>) {
    // fp32 residual [rows, N] (row stride ldo), boxes of 32 columns x 128 rows, 128B swizzle
    DM_REQUIRE(g.a_mode == A_FLAT && g.Bt == 1 && g.epi.ldo % 4 == 0, "residual TMA: flat rows");
    cuuint64_t dims[2] = {cuuint64_t(g.N), cuuint64_t(g.T)};
    cuuint64_t str[1] = {cuuint64_t(g.epi.ldo) * 4};
    cuuint32_t box[2] = {32, kBM};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = g_encode(&mr, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, g.epi.out, dims, str, box, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    DM_REQUIRE(r == CUDA_SUCCESS, "residual tensor map: CUresult " + std::to_string(int(r)));
  }
  if (g.a_mode == A_FLAT) {
    cuuint64_t dims[3] = {cuuint64_t(g.K), cuuint64_t(g.T), cuuint64_t(g.Bt)};
    cuuint64_t str[2] = {cuuint64_t(g.lda) * 2, cuuint64_t(g.a_bstride) * 2};
    cuuint32_t box[3] = {kBK, kBM, 1};
    if (make_map(&ma, g.A, 3, dims, str, box)) return 2;
  } else if (g.a_mode == A_CONV_S1) {
    const int rows = g.a_rows ? g.a_rows : g.T + 2;
    cuuint64_t dims[3] = {cuuint64_t(g.C), cuuint64_t(rows), cuuint64_t(g.Bt)};
    cuuint64_t str[2] = {cuuint64_t(g.C) * 2, cuuint64_t(g.C) * 2 * rows};
    cuuint32_t box[3] = {kBK, kBM, 1};
    if (make_map(&ma, g.A, 3, dims, str, box)) return 2;
  } else {
    const int rows = g.a_rows ? g.a_rows : 2 * g.T + 2;     // must be even
    cuuint64_t dims[4] = {cuuint64_t(g.C), 2, cuuint64_t(rows / 2), cuuint64_t(g.Bt)};
    cuuint64_t str[3] = {cuuint64_t(g.C) * 2, cuuint64_t(g.C) * 4, cuuint64_t(g.C) * 2 * rows};
    cuuint32_t box[4] = {kBK, 1, kBM, 1};
    if (make_map(&ma, g.A, 4, dims, str, box)) return 2;
  }
  {
    cuuint64_t dims[2] = {cuuint64_t(g.K), cuuint64_t(g.N)};
    cuuint64_t str[1] = {cuuint64_t(g.K) * 2};
    cuuint32_t box[2] = {kBK, BN};
    if (make_map(&mb, g.W, 2, dims, str, box)) return 2;
  }
  TileGeom geo;
  geo.MT = ceil_div(g.T, kBM);
  geo.NT = ceil_div(g.N, BN);
  geo.tiles = (g.mblocks[0] ? g.mblock_count[0] : g.Bt * geo.MT) * geo.NT;
  if (geo.tiles == 0) return 0;
  geo.KB = ceil_div(g.K, kBK);
  geo.cpb = g.grouped ? 1 : (g.C > 0 ? g.C / kBK : 1);
  const int smem = GemmSmem<BN, STAGES, MODE>::kBytes;
  DM_SMEM_ATTR((gemm_tcgen05_kernel<BN, STAGES, MODE>), smem);
  const int sms = g.max_ctas > 0 ? std::min(g.max_ctas, kNumSMs) : kNumSMs;
  int grid = geo.tiles < sms ? geo.tiles : sms;
  gemm_tcgen05_kernel<BN, STAGES, MODE><<<grid, kGemmThreads, smem, stream>>>(ma, mb, mr, g, geo);
  DM_CHECK_LAUNCH();
  return 0;
}

template <int STAGES, int MODE>
static int launch_pair_mode(const GemmArgs& g, cudaStream_t stream) {
  constexpr int BN = kPairBN;
  CUtensorMap ma, mb;
  if (g.a_mode == A_FLAT) {
    cuuint64_t dims[3] = {cuuint64_t(g.K), cuuint64_t(g.T), cuuint64_t(g.Bt)};
    cuuint64_t str[2] = {cuuint64_t(g.lda) * 2, cuuint64_t(g.a_bstride) * 2};
    cuuint32_t box[3] = {kBK, kBM, 1};
    if (make_map(&ma, g.A, 3, dims, str, box)) return 2;
  } else if (g.a_mode == A_CONV_S1) {
    const int rows = g.a_rows ? g.a_rows : g.T + 2;
    cuuint64_t dims[3] = {cuuint64_t(g.C), cuuint64_t(rows), cuuint64_t(g.Bt)};
    cuuint64_t str[2] = {cuuint64_t(g.C) * 2, cuuint64_t(g.C) * 2 * rows};
    cuuint32_t box[3] = {kBK, kBM, 1};
    if (make_map(&ma, g.A, 3, dims, str, box)) return 2;
  } else {
    const int rows = g.a_rows ? g.a_rows : 2 * g.T + 2;
    cuuint64_t dims[4] = {cuuint64_t(g.C), 2, cuuint64_t(rows / 2), cuuint64_t(g.Bt)};
    cuuint64_t str[3] = {cuuint64_t(g.C) * 2, cuuint64_t(g.C) * 4, cuuint64_t(g.C) * 2 * rows};
    cuuint32_t box[4] = {kBK, 1, kBM, 1};
    if (make_map(&ma, g.A, 4, dims, str, box)) return 2;
  }
  {
    cuuint64_t dims[2] = {cuuint64_t(g.K), cuuint64_t(g.N)};
    cuuint64_t str[1] = {cuuint64_t(g.K) * 2};
    cuuint32_t box[2] = {kBK, BN / 2};          // this CTA's half of the B tile
    if (make_map(&mb, g.W, 2, dims, str, box)) return 2;
  }
  TileGeom geo;
  geo.MT = ceil_div(g.T, 2 * kBM);
  geo.NT = ceil_div(g.N, BN);
  geo.tiles = (g.mblocks[1] ? g.mblock_count[1] : g.Bt * geo.MT) * geo.NT;
  if (geo.tiles == 0) return 0;
  geo.KB = ceil_div(g.K, kBK);
  geo.cpb = g.C > 0 ? g.C / kBK : 1;
  const int smem = PairSmem<STAGES>::kBytes;
  DM_SMEM_ATTR((gemm_pair_kernel<STAGES, MODE>), smem);
  const int pairs = std::min(geo.tiles, (g.max_ctas > 0 ? std::min(g.max_ctas, kNumSMs) : kNumSMs) / 2);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * pairs);
  cfg.blockDim = dim3(kGemmThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = 2;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  DM_CHECK_CUDA(cudaLaunchKernelEx(&cfg, gemm_pair_kernel<STAGES, MODE>, ma, mb, g, geo));
  return 0;
}

template <int STAGES>
static int launch_pair(const GemmArgs& g, cudaStream_t stream) {
  switch (g.epi.mode) {
#define DM_GEMM_MODE(m) \
  case m: return launch_pair_mode<STAGES, m>(g, stream);
    DM_GEMM_MODE(EPI_STORE_BF16) DM_GEMM_MODE(EPI_GELU_BF16) DM_GEMM_MODE(EPI_CONV1)
    DM_GEMM_MODE(EPI_CONV2_POS) DM_GEMM_MODE(EPI_RESID_F32) DM_GEMM_MODE(EPI_QKV)
    DM_GEMM_MODE(EPI_XKV) DM_GEMM_MODE(EPI_STORE_F32) DM_GEMM_MODE(EPI_W2V_PROJ)
    DM_GEMM_MODE(EPI_CTC_ARGMAX) DM_GEMM_MODE(EPI_GELU_F32)
#undef DM_GEMM_MODE
    default: DM_REQUIRE(false, "unknown GEMM epilogue");
  }
}

// The epilogue mode is a template parameter: each instantiation carries only
// its own epilogue (register pressure and I-cache footprint of one mode).
template <int BN, int STAGES>
static int launch_bn(const GemmArgs& g, cudaStream_t stream) {
  switch (g.epi.mode) {
#define DM_GEMM_MODE(m) \
  case m: return launch_bn_mode<BN, STAGES, m>(g, stream);
    DM_GEMM_MODE(EPI_STORE_BF16) DM_GEMM_MODE(EPI_GELU_BF16) DM_GEMM_MODE(EPI_CONV1)
    DM_GEMM_MODE(EPI_CONV2_POS) DM_GEMM_MODE(EPI_RESID_F32) DM_GEMM_MODE(EPI_QKV)
    DM_GEMM_MODE(EPI_XKV) DM_GEMM_MODE(EPI_STORE_F32) DM_GEMM_MODE(EPI_W2V_PROJ)
    DM_GEMM_MODE(EPI_CTC_ARGMAX) DM_GEMM_MODE(EPI_GELU_F32)
#undef DM_GEMM_MODE
    default: DM_REQUIRE(false, "unknown GEMM epilogue");
  }
}

int make_tmap_2d(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer,
                 uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer) {
  DM_REQUIRE(tma_available(), "cuTensorMapEncodeTiled entry point unavailable");
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t str[1] = {row_stride_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  return make_map(m, ptr, 2, dims, str, box);
}

int make_attn_maps(const uint16_t* q, const uint16_t* k, const uint16_t* vt, int bh, int t_pad,
                   CUtensorMap* mq, CUtensorMap* mk, CUtensorMap* mv) {
  DM_REQUIRE(tma_available(), "cuTensorMapEncodeTiled entry point unavailable");
  {
    cuuint64_t dims[2] = {64, cuuint64_t(bh) * t_pad};
    cuuint64_t str[1] = {128};
    cuuint32_t box[2] = {64, 128};
    if (make_map(mq, q, 2, dims, str, box)) return 2;
    if (make_map(mk, k, 2, dims, str, box)) return 2;
  }
  {
    cuuint64_t dims[2] = {cuuint64_t(t_pad), cuuint64_t(bh) * 64};
    cuuint64_t str[1] = {cuuint64_t(t_pad) * 2};
    cuuint32_t box[2] = {64, 64};
    if (make_map(mv, vt, 2, dims, str, box)) return 2;
  }
  return 0;
}

int launch_gemm(const GemmArgs& g, cudaStream_t stream) {
  DM_REQUIRE(tma_available(), "cuTensorMapEncodeTiled entry point unavailable");
  DM_REQUIRE(g.K > 0 && g.N > 0 && g.T > 0 && g.Bt > 0, "empty GEMM");
  DM_REQUIRE(g.N % 32 == 0, "N must be a multiple of 32");
  DM_REQUIRE(g.K % 8 == 0, "K must be a multiple of 8 (16-byte rows)");
  DM_REQUIRE(g.a_mode == A_FLAT || (g.C % kBK == 0 && (g.grouped || g.K % g.C == 0)),
             "conv A needs C % 64 == 0 and K == taps * C");
  DM_REQUIRE(!g.grouped || (g.a_mode == A_CONV_S1 && g.K % kBK == 0),
             "grouped conv: stride-1 conv mode, K = taps * 64");
  DM_REQUIRE(g.a_mode != A_CONV_S2 || g.a_rows % 2 == 0, "stride-2 conv input rows must be even");
  DM_REQUIRE((reinterpret_cast<uintptr_t>(g.A) & 15) == 0 &&
                 (reinterpret_cast<uintptr_t>(g.W) & 15) == 0,
             "operands must be 16-byte aligned");
  if (g.grouped) {
    DM_REQUIRE(g.epi.mode == EPI_W2V_POS, "grouped GEMM: wav2vec2 pos-conv epilogue only");
    return launch_bn_mode<64, 8, EPI_W2V_POS>(g, stream);
  }
  // wide N, or long K (fc2, the stride-2 conv): 128 x 256 tiles cut the per-SM
  // operand stream (bytes per FLOP (128 + BN) / (128 BN)); with a long K the
  // epilogue's global traffic overlaps the next tile's mainloop
  // (experiments: DM_GEMM_PAIR_MIN_K moves the CTA-pair threshold)
  static const int pair_min_k =
      std::getenv("DM_GEMM_PAIR_MIN_K") ? std::atoi(std::getenv("DM_GEMM_PAIR_MIN_K")) : 1024;
  const bool resid_path = g.epi.mode == EPI_RESID_F32 && g.a_mode == A_FLAT && g.Bt == 1;
  if (g.N % 256 == 0 && (g.N >= 1024 || g.K >= 1536)) {
    // K >= 1024 (large-v3's projections, fc2, the stride-2 conv): the
    // mainloop's L2 -> SMEM operand stream bounds the 1-SM kernel, so 256 x 256
    // tiles run on CTA pairs (cta_group::2; measured at large-v3, 12
    // segments: cross-KV 4.64 -> 3.64 ms, qkv 144 -> 131 us, o 86 -> 81 us,
    // fc1 unchanged; whisper-base conv2 99 -> 95 us, fc2 118 -> 112 us). The
    // K = 512 GEMMs are bound by their epilogues (GELU, Q/K/V scatter) and
    // stay on the 1-SM kernel (pairs measured slower: fc1 163 -> 176 us).
    // The 128-wide TMA-prefetched residual path measured slower for the wide
    // o-projection (86 -> 166 us). DM_GEMM_NO_PAIR=1 forces the 1-SM kernel
    // (same per-element MMA sequence).
    static const bool no_pair = std::getenv("DM_GEMM_NO_PAIR") != nullptr;
    if (g.K >= pair_min_k && !no_pair) return launch_pair<6>(g, stream);
    return launch_bn<256, 4>(g, stream);
  }
  if (resid_path) return launch_bn_mode<128, 5, EPI_RESID_F32>(g, stream);  // + 64 KB residual buffer
  return launch_bn<128, 6>(g, stream);
}

}  // namespace dm
