// K1: fused pad_or_trim + log-mel front end (Whisper feature_extractor).
//
// Replaces Listing 1's `model.feature_extractor(chunk)` + `pad_or_trim`
// and the reference's sample-domain pad_or_trim
// (pkg/src/dictamux/backend.py:87-99). Semantics restated in
// oracle/logmel.py (transformers 5.5.0 feature_extraction_whisper.py:140-164).
//
// Layout: segments are concatenated int16 PCM in HBM (offsets/lengths); the
// 480,000-sample window is never materialised -- samples past the true length
// read as zero inside the loads. Per CTA: 32 consecutive frames of one
// segment. The 400-point real DFT runs as a 200-point complex FFT
// (even/odd packing), itself a 4-step 8 x 25 FFT staged through shared
// memory; the 25-point DFTs are 5 x 5 radix-5 in registers. Power -> sparse
// slaney mel -> log10(max(., 1e-10)) -> per-segment max via an
// order-preserving atomicMax.
//
// Product path (encoder operand only): pass 1 writes bf16((x + 4) / 4) --
// the normalisation WITHOUT the clamp -- straight into the time-major conv1
// operand (rows 1..3000 of a zero-padded [B, 3002, ldt] bf16 buffer); pass 2
// clamps that buffer in place to bf16((max - 8 + 4) / 4). Because
// x -> bf16((x + 4) / 4) is monotonic, max(bf16(a), bf16(b)) = bf16(max(a, b)):
// the result is bit for bit bf16((max(x, max - 8) + 4) / 4), the feature
// extractor's clamp + normalise, with 2 bytes per value written once and
// re-read once instead of an fp32 round trip. The fp32 [B, n_mels, 3000]
// feature contract (dm_logmel, and the engine's debug tap) is a separate
// output of the same passes.
//
// Frames whose 400-sample window lies entirely in the zero padding are
// skipped (their power is exactly 0, so the result is log10(1e-10)).

#include "common.cuh"

namespace dm {

constexpr int kFFT = 400;
constexpr int kHop = 160;
constexpr int kWindow = 480000;
constexpr int kFrames = 3000;
constexpr int kBins = 201;
constexpr int kFPB = 32;                               // frames per CTA
static_assert(kFrames % 4 == 0 && kFPB % 4 == 0, "float4 frame groups");
constexpr int kSpan = (kFPB - 1) * kHop + kFFT;        // 5360 samples
constexpr int kLogmelThreads = 256;
constexpr int kMelMaxBins = 16;                        // bins of the widest mel filter (host-checked)

// Twiddles / window / sparse mel bank, prepared on the host (float64 -> fp32).
struct LogmelTables {
  float2 tw200[25 * 8];    // W200^{q*k1}
  float2 tw25[25];         // W25^{j}
  float2 tw400[kBins];     // W400^{k}
  float window[kFFT];      // periodic Hann
  int mel_start[128];      // first bin of mel m
  int mel_count[128];      // bins of mel m
  int mel_woff[128];       // offset into mel_w
  float mel_w[1024];       // weights
};

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) {
  return make_float2(a.x + b.x, a.y + b.y);
}
__device__ __forceinline__ float2 csub(float2 a, float2 b) {
  return make_float2(a.x - b.x, a.y - b.y);
}

// 5-point DFT in place (forward, W5 = e^{-2 pi i / 5}).
__device__ __forceinline__ void dft5(float2& x0, float2& x1, float2& x2,
                                     float2& x3, float2& x4) {
  const float c1 = 0.30901699437494745f, c2 = -0.8090169943749475f;
  const float s1 = 0.9510565162951535f, s2 = 0.5877852522924731f;
  float2 a1 = cadd(x1, x4), b1 = csub(x1, x4);
  float2 a2 = cadd(x2, x3), b2 = csub(x2, x3);
  float2 y0 = cadd(x0, cadd(a1, a2));
  float2 t1 = make_float2(x0.x + c1 * a1.x + c2 * a2.x, x0.y + c1 * a1.y + c2 * a2.y);
  float2 t2 = make_float2(x0.x + c2 * a1.x + c1 * a2.x, x0.y + c2 * a1.y + c1 * a2.y);
  // -i * (s1*b1 + s2*b2)  and  -i * (s2*b1 - s1*b2)
  float2 u1 = make_float2(s1 * b1.x + s2 * b2.x, s1 * b1.y + s2 * b2.y);
  float2 u2 = make_float2(s2 * b1.x - s1 * b2.x, s2 * b1.y - s1 * b2.y);
  x0 = y0;
  x1 = make_float2(t1.x + u1.y, t1.y - u1.x);
  x4 = make_float2(t1.x - u1.y, t1.y + u1.x);
  x2 = make_float2(t2.x + u2.y, t2.y - u2.x);
  x3 = make_float2(t2.x - u2.y, t2.y + u2.x);
}

// 8-point DFT (forward) of z[0..7], natural order in and out.
__device__ __forceinline__ void dft8(float2 (&z)[8]) {
  const float r = 0.7071067811865476f;
  // radix-2 DIT: split even/odd
  float2 e0 = cadd(z[0], z[4]), e1 = csub(z[0], z[4]);
  float2 e2 = cadd(z[2], z[6]), e3 = csub(z[2], z[6]);
  float2 o0 = cadd(z[1], z[5]), o1 = csub(z[1], z[5]);
  float2 o2 = cadd(z[3], z[7]), o3 = csub(z[3], z[7]);
  // 4-point on evens: E[k]
  float2 E0 = cadd(e0, e2), E2 = csub(e0, e2);
  float2 E1 = make_float2(e1.x + e3.y, e1.y - e3.x);   // e1 - i e3
  float2 E3 = make_float2(e1.x - e3.y, e1.y + e3.x);   // e1 + i e3
  float2 O0 = cadd(o0, o2), O2 = csub(o0, o2);
  float2 O1 = make_float2(o1.x + o3.y, o1.y - o3.x);
  float2 O3 = make_float2(o1.x - o3.y, o1.y + o3.x);
  // twiddles W8^k: k=1: (r, -r), k=2: -i, k=3: (-r, -r)
  float2 T1 = make_float2(r * (O1.x + O1.y), r * (O1.y - O1.x));
  float2 T2 = make_float2(O2.y, -O2.x);
  float2 T3 = make_float2(r * (-O3.x + O3.y), r * (-O3.y - O3.x));
  z[0] = cadd(E0, O0); z[4] = csub(E0, O0);
  z[1] = cadd(E1, T1); z[5] = csub(E1, T1);
  z[2] = cadd(E2, T2); z[6] = csub(E2, T2);
  z[3] = cadd(E3, T3); z[7] = csub(E3, T3);
}

__device__ __forceinline__ uint32_t float_to_ordered(float f) {
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float ordered_to_float(uint32_t k) {
  uint32_t u = (k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k;
  return __uint_as_float(u);
}

struct LogmelSmem {
  float samples[kSpan];           // also reused as power[kFPB][kBins]
  float pad_[kFPB * kBins - kSpan > 0 ? kFPB * kBins - kSpan : 1];
  float2 y[kFPB * 200];           // stage A out ([frame][k1][q]) / stage B out (Z, natural order)
  float2 tw200[200];
  float2 tw25[25];
  float2 tw400[kBins];
  float window[kFFT];
  int mstart[128], mcount[128], mwoff[128];
  float mw[1024];
};

__device__ __forceinline__ float fast_log10(float x) {
  return __log2f(x) * 0.30102999566398120f;       // MUFU lg2 (abs err ~2^-22)
}

// bf16 bits of the normalised-but-unclamped value (x + 4) / 4
__device__ __forceinline__ uint32_t norm_bf16_pair(float a, float b) {
  return pack_bf16x2((a + 4.0f) / 4.0f, (b + 4.0f) / 4.0f);
}

// Pass 1. mel_t (nullable): the time-major bf16 operand, rows 1..3000 of
// [B, 3002, ldt]; out32 (nullable): fp32 unnormalised log-mel [B, n_mels, 3000].
__global__ void __launch_bounds__(kLogmelThreads)
logmel_kernel(const int16_t* __restrict__ pcm, const int64_t* __restrict__ offsets,
              const int32_t* __restrict__ lengths, const LogmelTables* __restrict__ tab,
              int n_mels, uint16_t* __restrict__ mel_t, int ldt, float* __restrict__ out32,
              uint32_t* __restrict__ segmax) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  LogmelSmem& s = *reinterpret_cast<LogmelSmem*>(smem_raw);
  const int b = blockIdx.y;
  const int f0 = blockIdx.x * kFPB;
  const int tid = threadIdx.x;
  const int nfr = min(kFPB, kFrames - f0);
  int n = lengths[b];
  n = n < 0 ? 0 : (n > kWindow ? kWindow : n);
  const int16_t* x = pcm + offsets[b];
  uint16_t* tb = mel_t ? mel_t + (size_t(b) * (kFrames + 2) + f0 + 1) * ldt : nullptr;
  float* ob = out32 ? out32 + size_t(b) * n_mels * kFrames : nullptr;
  const int np = n_mels / 2;                        // mel pairs per frame (40 or 64)

  // Frames >= first_zero have all-zero windows: start index f*160-200 >= n.
  const int first_zero = n == 0 ? 0 : min(kFrames, (n + 200 + kHop - 1) / kHop);
  if (f0 >= first_zero) {
    const float v = log10f(1e-10f);
    if (tb) {
      const uint32_t w = norm_bf16_pair(v, v);
      for (int t = tid; t < np * nfr; t += kLogmelThreads)
        reinterpret_cast<uint32_t*>(tb + size_t(t / np) * ldt)[t % np] = w;
    }
    if (ob)
      for (int i = tid; i < n_mels * nfr; i += kLogmelThreads)
        ob[size_t(i / nfr) * kFrames + f0 + i % nfr] = v;
    if (tid == 0) atomicMax(segmax + b, float_to_ordered(v));
    return;
  }

  // twiddles as [k1][q] (the table is [q][k1]): stage A's lanes run along q
  for (int i = tid; i < 200; i += kLogmelThreads) s.tw200[(i % 8) * 25 + i / 8] = tab->tw200[i];
  for (int i = tid; i < 25; i += kLogmelThreads) s.tw25[i] = tab->tw25[i];
  for (int i = tid; i < kBins; i += kLogmelThreads) s.tw400[i] = tab->tw400[i];
  for (int i = tid; i < kFFT; i += kLogmelThreads) s.window[i] = tab->window[i];
  // Samples of the padded + reflected window [f0*160-200, f0*160-200+kSpan).
  const int base = f0 * kHop - kFFT / 2;
  if (base >= 0 && base + kSpan <= n) {
    // interior span: 16-byte loads (8 samples each) from the first aligned
    // address, the unaligned head and tail sample by sample
    const int16_t* src = x + base;
    const int head = int(((16 - (reinterpret_cast<uintptr_t>(src) & 15)) & 15) >> 1);
    const int nv = (kSpan - head) >> 3;
    const uint4* v = reinterpret_cast<const uint4*>(src + head);
    for (int i = tid; i < nv; i += kLogmelThreads) {
      const uint4 w = __ldg(v + i);
      float* d = s.samples + head + 8 * i;
      const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        d[2 * u] = float(int16_t(ws[u] & 0xFFFFu)) * (1.0f / 32768.0f);
        d[2 * u + 1] = float(int16_t(ws[u] >> 16)) * (1.0f / 32768.0f);
      }
    }
    const int tail0 = head + 8 * nv;
    if (tid < head) s.samples[tid] = float(src[tid]) * (1.0f / 32768.0f);
    if (tid < kSpan - tail0) s.samples[tail0 + tid] = float(src[tail0 + tid]) * (1.0f / 32768.0f);
  } else {
    for (int i = tid; i < kSpan; i += kLogmelThreads) {
      int j = base + i;
      if (j < 0) j = -j;                                   // reflect at start
      if (j >= kWindow) j = 2 * (kWindow - 1) - j;         // reflect at end
      s.samples[i] = (j < n) ? float(x[j]) * (1.0f / 32768.0f) : 0.0f;
    }
  }
  // sparse mel bank into shared memory (read by every (mel, frame) task)
  for (int i = tid; i < n_mels; i += kLogmelThreads) {
    s.mstart[i] = tab->mel_start[i];
    s.mcount[i] = tab->mel_count[i];
    s.mwoff[i] = tab->mel_woff[i];
  }
  for (int i = tid; i < 1024; i += kLogmelThreads) s.mw[i] = tab->mel_w[i];
  __syncthreads();

  // Stage A: per (frame, q): 8-point DFT over p of z[25p+q], twiddle W200^{q k1}.
  // (250 threads as q = tid % 25, frames tid / 25 + 10 i: one division per thread)
  const int qa = tid % 25, fa = tid / 25;
  for (int fr = fa; fr < kFPB && tid < 250; fr += 10) {
    const int q = qa;
    float2 z[8];
    const float* src = s.samples + fr * kHop;
#pragma unroll
    for (int p = 0; p < 8; ++p) {
      int m = 25 * p + q;
      z[p] = make_float2(src[2 * m] * s.window[2 * m],
                         src[2 * m + 1] * s.window[2 * m + 1]);
    }
    dft8(z);
    // Y[k1][q] (k1-major: a warp's lanes store consecutive q, conflict-free)
    float2* dst = s.y + fr * 200 + q;
#pragma unroll
    for (int k1 = 0; k1 < 8; ++k1) dst[k1 * 25] = cmul(z[k1], s.tw200[k1 * 25 + q]);
  }
  __syncthreads();

  // Stage B: per (frame, k1): 25-point DFT over q (5 x 5).
  {
    const int fr = tid / 8, k1 = tid % 8;               // 256 tasks exactly
    float2 v[25];
    const float2* src = s.y + fr * 200 + k1 * 25;
#pragma unroll
    for (int q = 0; q < 25; ++q) v[q] = src[q];
    // q = 5a + c: DFT over a for each c, twiddle W25^{c e}
#pragma unroll
    for (int c = 0; c < 5; ++c) {
      dft5(v[c], v[5 + c], v[10 + c], v[15 + c], v[20 + c]);
#pragma unroll
      for (int e = 1; e < 5; ++e) v[5 * e + c] = cmul(v[5 * e + c], s.tw25[c * e]);
    }
    // DFT over c for each e: output k2 = e + 5 g
#pragma unroll
    for (int e = 0; e < 5; ++e)
      dft5(v[5 * e + 0], v[5 * e + 1], v[5 * e + 2], v[5 * e + 3], v[5 * e + 4]);
    __syncthreads();
    // v[5e + g] = Z[k1 + 8*(e + 5g)]
    float2* dst = s.y + fr * 200;
#pragma unroll
    for (int e = 0; e < 5; ++e)
#pragma unroll
      for (int g = 0; g < 5; ++g) dst[k1 + 8 * (e + 5 * g)] = v[5 * e + g];
  }
  __syncthreads();

  // Real-FFT post-processing + power: thread = bin (201 of 256), loop over frames
  float* power = s.samples;
  if (tid < kBins) {
    const int k = tid;
    const float2 tw = s.tw400[k];
    const int kz = k % 200, kc = (200 - k) % 200;
#pragma unroll 4
    for (int fr = 0; fr < kFPB; ++fr) {
      const float2* Z = s.y + fr * 200;
      float2 zk = Z[kz], zc = Z[kc];
      zc.y = -zc.y;                                      // conj(Z[200-k])
      float2 E = make_float2(0.5f * (zk.x + zc.x), 0.5f * (zk.y + zc.y));
      float2 D = make_float2(0.5f * (zk.x - zc.x), 0.5f * (zk.y - zc.y));
      float2 O = make_float2(D.y, -D.x);                 // D / i
      float2 X = cadd(E, cmul(tw, O));
      power[fr * kBins + k] = X.x * X.x + X.y * X.y;
    }
  }
  __syncthreads();

  // Sparse mel + log10: thread = (mel pair p, frame group g); the pair's bank
  // rows stay in registers, frames g, g + 4, ... (bf16 pair stores run along
  // the time-major row)
  float lmax = -INFINITY;
  const int p = tid & 63, g = tid >> 6;
  if (p < np) {
    const int m0 = 2 * p;
    const int st0 = s.mstart[m0], c0 = s.mcount[m0], w0 = s.mwoff[m0];
    const int st1 = s.mstart[m0 + 1], c1 = s.mcount[m0 + 1], w1 = s.mwoff[m0 + 1];
    // the pair's filter weights in registers for all its frames (<= kMelMaxBins
    // bins per filter: 14 at 80 mels, 9 at 128; same summation order)
    float r0[kMelMaxBins], r1[kMelMaxBins];
#pragma unroll
    for (int i = 0; i < kMelMaxBins; ++i) {
      r0[i] = i < c0 ? s.mw[w0 + i] : 0.f;
      r1[i] = i < c1 ? s.mw[w1 + i] : 0.f;
    }
    for (int fr = g; fr < nfr; fr += kLogmelThreads / 64) {
      const float* pw = power + fr * kBins;
      float a0 = 0.f, a1 = 0.f;
#pragma unroll
      for (int i = 0; i < kMelMaxBins; ++i)
        if (i < c0) a0 = fmaf(r0[i], pw[st0 + i], a0);
#pragma unroll
      for (int i = 0; i < kMelMaxBins; ++i)
        if (i < c1) a1 = fmaf(r1[i], pw[st1 + i], a1);
      const float v0 = fast_log10(fmaxf(a0, 1e-10f));
      const float v1 = fast_log10(fmaxf(a1, 1e-10f));
      if (tb) reinterpret_cast<uint32_t*>(tb + size_t(fr) * ldt)[p] = norm_bf16_pair(v0, v1);
      if (ob) {
        ob[size_t(m0) * kFrames + f0 + fr] = v0;
        ob[size_t(m0 + 1) * kFrames + f0 + fr] = v1;
      }
      lmax = fmaxf(lmax, fmaxf(v0, v1));
    }
  }
  // block max -> one atomic
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) lmax = fmaxf(lmax, __shfl_xor_sync(0xffffffffu, lmax, o));
  __shared__ float wmax[kLogmelThreads / 32];
  if ((tid & 31) == 0) wmax[tid >> 5] = lmax;
  __syncthreads();
  if (tid == 0) {
    float m = wmax[0];
    for (int i = 1; i < kLogmelThreads / 32; ++i) m = fmaxf(m, wmax[i]);
    atomicMax(segmax + b, float_to_ordered(m));
  }
}

// Pass 2 (operand): clamp the bf16 operand in place to bf16((max - 8 + 4) / 4);
// 8 channels per thread, written back only where a value rose.
__global__ void __launch_bounds__(256)
logmel_clamp_kernel(uint16_t* __restrict__ mel_t, const uint32_t* __restrict__ segmax,
                    int n_mels, int ldt, int frames) {
  const int b = blockIdx.y;
  const int vpr = n_mels / 8;                             // 16-byte vectors per frame row
  const float fl = ordered_to_float(segmax[b]) - 8.0f;
  const float floor_n = __uint_as_float(uint32_t(f32_to_bf16((fl + 4.0f) / 4.0f)) << 16);
  uint16_t* base = mel_t + (size_t(b) * (kFrames + 2) + 1) * ldt;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < frames * vpr;
       t += gridDim.x * blockDim.x) {
    uint4* pv = reinterpret_cast<uint4*>(base + size_t(t / vpr) * ldt) + (t % vpr);
    uint4 v = *pv;
    uint32_t w[4] = {v.x, v.y, v.z, v.w};
    bool changed = false;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const float lo = __uint_as_float(w[u] << 16), hi = __uint_as_float(w[u] & 0xFFFF0000u);
      const float nlo = fmaxf(lo, floor_n), nhi = fmaxf(hi, floor_n);
      changed |= (nlo != lo) | (nhi != hi);
      w[u] = (__float_as_uint(nlo) >> 16) | (__float_as_uint(nhi) & 0xFFFF0000u);
    }
    if (changed) *pv = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

// Pass 2 (fp32 feature contract): clamp to (max - 8) and normalise in place.
__global__ void __launch_bounds__(256)
logmel_normalize_kernel(float* __restrict__ out, const uint32_t* __restrict__ segmax, int n_mels) {
  const int b = blockIdx.y;
  const float floor_v = ordered_to_float(segmax[b]) - 8.0f;
  float4* o = reinterpret_cast<float4*>(out + size_t(b) * n_mels * kFrames);
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n_mels * kFrames / 4;
       t += gridDim.x * blockDim.x) {
    float4 v = o[t];
    v.x = (fmaxf(v.x, floor_v) + 4.0f) / 4.0f;
    v.y = (fmaxf(v.y, floor_v) + 4.0f) / 4.0f;
    v.z = (fmaxf(v.z, floor_v) + 4.0f) / 4.0f;
    v.w = (fmaxf(v.w, floor_v) + 4.0f) / 4.0f;
    o[t] = v;
  }
}

size_t logmel_smem_bytes() { return sizeof(LogmelSmem); }

int launch_logmel(const int16_t* pcm, const int64_t* offsets, const int32_t* lengths,
                 int n_segments, int n_mels, const LogmelTables* tables, float* out32,
                 uint16_t* mel_t, uint32_t* segmax, cudaStream_t stream, int frames) {
  DM_REQUIRE(n_mels == 80 || n_mels == 128, "n_mels must be 80 or 128");
  DM_REQUIRE(n_segments >= 0, "n_segments < 0");
  DM_REQUIRE(out32 != nullptr || mel_t != nullptr, "no log-mel output");
  if (n_segments == 0) return 0;
  const size_t smem = logmel_smem_bytes();
  DM_SMEM_ATTR(logmel_kernel, int(smem));
  DM_CHECK_CUDA(cudaMemsetAsync(segmax, 0, sizeof(uint32_t) * n_segments, stream));
  // time-major operand rows are padded to 64 (n_mels <= 64) or 128 channels
  const int ldt = n_mels <= 64 ? 64 : 128;
  // frames < 3000: only the first `frames` (the length-aware encoder's
  // window; the per-segment max is unchanged: every later frame of a shorter
  // segment is zero padding)
  DM_REQUIRE(frames >= 1 && frames <= kFrames && (out32 == nullptr || frames == kFrames),
             "log-mel frames");
  dim3 grid(ceil_div(frames, kFPB), n_segments);
  logmel_kernel<<<grid, kLogmelThreads, smem, stream>>>(pcm, offsets, lengths, tables, n_mels,
                                                         mel_t, ldt, out32, segmax);
  DM_CHECK_LAUNCH();
  if (mel_t) {
    logmel_clamp_kernel<<<dim3(24, n_segments), 256, 0, stream>>>(mel_t, segmax, n_mels, ldt,
                                                                  frames);
    DM_CHECK_LAUNCH();
  }
  if (out32) {
    logmel_normalize_kernel<<<dim3(48, n_segments), 256, 0, stream>>>(out32, segmax, n_mels);
    DM_CHECK_LAUNCH();
  }
  return 0;
}

}  // namespace dm
