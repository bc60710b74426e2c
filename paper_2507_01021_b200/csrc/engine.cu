// C-ABI entry points and the Whisper engine: owns device buffers, runs the
// encoder (log-mel -> conv stem -> L layers -> LN -> cross-KV into slots) and
// the decode step (captured once as a CUDA graph, replayed per step), and the
// K7 slot / self-KV page allocator.

#include <cstdlib>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/dictamux_b200.h"
#include "common.cuh"
#include "decode.cuh"
#include "gemm.cuh"

namespace dm {

// ------------------------------------------------------------ error state
static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }
const char* last_error() { return g_err.c_str(); }

cudaError_t set_max_smem(const void* fn, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> raised;   // (kernel, device) -> bytes
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  int& have = raised[std::make_pair(fn, dev)];
  if (have >= bytes) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) have = bytes;
  return e;
}

// forward decls (logmel.cu / attention.cu)
struct LogmelTables;
int launch_logmel(const int16_t*, const int64_t*, const int32_t*, int, int,
                  const LogmelTables*, float*, uint16_t*, uint32_t*, cudaStream_t,
                  int frames = 3000);
int launch_layernorm_bf16(const float*, const uint16_t*, const uint16_t*, uint16_t*, int, int,
                          cudaStream_t, float* y32 = nullptr, const int32_t* seg_len = nullptr,
                          int seg_rows = 0);
int launch_attention(const uint16_t*, const uint16_t*, const uint16_t*, int, int, int, int,
                     uint16_t*, int, cudaStream_t, const int32_t* seg_len = nullptr);

// ------------------------------------------------------------ log-mel tables
struct LogmelTablesHost {
  float2 tw200[25 * 8];
  float2 tw25[25];
  float2 tw400[201];
  float window[400];
  int mel_start[128];
  int mel_count[128];
  int mel_woff[128];
  float mel_w[1024];
};

static double hz_to_mel(double f) {
  if (f >= 1000.0) return 15.0 + std::log(f / 1000.0) * (27.0 / std::log(6.4));
  return 3.0 * f / 200.0;
}
static double mel_to_hz(double m) {
  if (m >= 15.0) return 1000.0 * std::exp(std::log(6.4) / 27.0 * (m - 15.0));
  return 200.0 * m / 3.0;
}

// Restates mel_filter_bank(201, n_mels, 0, 8000, 16000, "slaney", "slaney")
// (transformers audio_utils.py:453-545) in double precision.
static int build_logmel_tables(int n_mels, LogmelTablesHost* t) {
  const double PI = 3.14159265358979323846;
  for (int q = 0; q < 25; ++q)
    for (int k1 = 0; k1 < 8; ++k1) {
      double a = -2.0 * PI * q * k1 / 200.0;
      t->tw200[q * 8 + k1] = make_float2(float(std::cos(a)), float(std::sin(a)));
    }
  for (int j = 0; j < 25; ++j) {
    double a = -2.0 * PI * j / 25.0;
    t->tw25[j] = make_float2(float(std::cos(a)), float(std::sin(a)));
  }
  for (int k = 0; k < 201; ++k) {
    double a = -2.0 * PI * k / 400.0;
    t->tw400[k] = make_float2(float(std::cos(a)), float(std::sin(a)));
  }
  for (int n = 0; n < 400; ++n) t->window[n] = float(0.5 - 0.5 * std::cos(2.0 * PI * n / 400.0));
  std::vector<double> filt(n_mels + 2);
  const double m0 = hz_to_mel(0.0), m1 = hz_to_mel(8000.0);
  for (int i = 0; i < n_mels + 2; ++i) filt[i] = mel_to_hz(m0 + (m1 - m0) * i / (n_mels + 1));
  int woff = 0;
  for (int m = 0; m < n_mels; ++m) {
    const double enorm = 2.0 / (filt[m + 2] - filt[m]);
    int start = -1, count = 0;
    for (int k = 0; k < 201; ++k) {
      const double f = 8000.0 * k / 200.0;
      const double down = (f - filt[m]) / (filt[m + 1] - filt[m]);
      const double up = (filt[m + 2] - f) / (filt[m + 2] - filt[m + 1]);
      const double w = std::max(0.0, std::min(down, up)) * enorm;
      if (w > 0.0) {
        if (start < 0) start = k;
        if (woff + (k - start) >= 1024) return 1;
        t->mel_w[woff + (k - start)] = float(w);
        count = k - start + 1;
      }
    }
    if (start < 0) start = 0;
    if (count > 16) return 1;        // logmel.cu kMelMaxBins: filter weights held in registers
    t->mel_start[m] = start;
    t->mel_count[m] = count;
    t->mel_woff[m] = woff;
    woff += count;
  }
  return 0;
}

static std::mutex g_tab_mu;
static std::map<std::pair<int, int>, void*> g_tables;   // (device, n_mels) -> device ptr

static int get_logmel_tables(int n_mels, const LogmelTables** out) {
  int dev = 0;
  DM_CHECK_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_tab_mu);
  auto key = std::make_pair(dev, n_mels);
  auto it = g_tables.find(key);
  if (it == g_tables.end()) {
    LogmelTablesHost h;
    std::memset(&h, 0, sizeof(h));
    DM_REQUIRE(build_logmel_tables(n_mels, &h) == 0, "mel table overflow");
    void* d = nullptr;
    DM_CHECK_CUDA(cudaMalloc(&d, sizeof(h)));
    DM_CHECK_CUDA(cudaMemcpy(d, &h, sizeof(h), cudaMemcpyHostToDevice));
    it = g_tables.emplace(key, d).first;
  }
  *out = static_cast<const LogmelTables*>(it->second);
  return 0;
}

// ------------------------------------------------------------ weight fill
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void fill_normal_kernel(uint16_t* dst, uint64_t n, uint64_t key, float scale,
                                   float mean) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t h = splitmix64(key + i);
    const int64_t s = int64_t(h & 0xFFFF) + int64_t((h >> 16) & 0xFFFF) +
                      int64_t((h >> 32) & 0xFFFF) + int64_t(h >> 48);
    const float z = float(s - 131070);                    // exact (< 2^24)
    const float v = __fadd_rn(__fmul_rn(z, scale), mean);
    dst[i] = __bfloat16_as_ushort(__float2bfloat16_rn(v));
  }
}

// ------------------------------------------------------------ upload ring
// Pinned host chunks for the small stream-ordered uploads (slot ids, page
// table, admission args, active lists). A chunk is reused only after the copy
// that read it has executed (its event), so no call has to drain the stream.
struct UploadRing {
  static constexpr int kN = 16;
  static constexpr size_t kChunk = 16 * 1024;
  uint8_t* host = nullptr;
  cudaEvent_t ev[kN] = {};
  bool used[kN] = {};
  int next = 0;
  int init() {
    DM_CHECK_CUDA(cudaMallocHost(&host, kN * kChunk));
    for (int i = 0; i < kN; ++i) DM_CHECK_CUDA(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
    return 0;
  }
  ~UploadRing() {
    for (int i = 0; i < kN; ++i)
      if (ev[i]) cudaEventDestroy(ev[i]);
    if (host) cudaFreeHost(host);
  }
  // copy `bytes` from host memory to `dev` in stream order
  int upload(void* dev, const void* src, size_t bytes, cudaStream_t s) {
    DM_REQUIRE(bytes <= kChunk, "upload larger than a staging chunk");
    const int i = next;
    next = (next + 1) % kN;
    if (used[i]) DM_CHECK_CUDA(cudaEventSynchronize(ev[i]));
    std::memcpy(host + i * kChunk, src, bytes);
    DM_CHECK_CUDA(cudaMemcpyAsync(dev, host + i * kChunk, bytes, cudaMemcpyHostToDevice, s));
    DM_CHECK_CUDA(cudaEventRecord(ev[i], s));
    used[i] = true;
    return 0;
  }
};

// ------------------------------------------------------------ Whisper engine
constexpr int kMaxPrompt = 224;     // Whisper: n_text_ctx / 2 (previous-text context + task tokens)
constexpr int kRowBuckets = 9;
constexpr int kRowBucket[kRowBuckets] = {1, 2, 4, 8, 16, 24, 32, 48, kRows};

struct WhisperEngine {
  int device = 0;                      // the CUDA device of every buffer/stream below
  UploadRing ring;
  int32_t* admit_args_dev = nullptr;   // [2 * max_slots]
  dm_whisper_config cfg;
  int d, H, L, Ld, F, nm, Cp;
  // weights
  const uint16_t* w = nullptr;
  std::vector<int64_t> off;
  const uint16_t* W(int i) const { return w + off[i]; }
  int enc_layer_base(int l) const { return 5 + 12 * l; }
  int after_enc() const { return 5 + 12 * L; }          // enc.ln.g
  int dec_layer_base(int l) const { return after_enc() + 4 + 18 * l; }
  int after_dec() const { return after_enc() + 4 + 18 * Ld; }
  uint16_t* conv1_w_pad = nullptr;   // [d, 3, Cp]
  // encoder workspace
  int E = 0;
  float* mel = nullptr;          // [E, nm, 3000]
  uint16_t* mel_t = nullptr;     // [E, 3002, Cp]
  uint32_t* segmax = nullptr;
  uint16_t* conv1_out = nullptr; // [E, 3002, d]
  float* resid = nullptr;        // [E*1500, d]
  uint16_t* lnb = nullptr;       // [E*1500, d]
  uint16_t *qb = nullptr, *kb = nullptr, *vtb = nullptr;  // [E*H, 1536, 64] / [E*H*64, 1536]
  uint16_t* attn_out = nullptr;  // [E*1500, d]
  uint16_t* fc1_out = nullptr;   // [E*1500, F]
  uint16_t* enc_out = nullptr;   // [E*1500, d]
  int32_t* slot_dev = nullptr;   // [E]
  int32_t* seg_len_dev = nullptr;  // [E] encoder positions per segment of the last encode
  int32_t* enc_len_dev = nullptr;  // [max_slots] encoder positions per slot (st.enc_len)
  int32_t* slot_host = nullptr;  // pinned [E]
  int last_n = 0;
  int last_rows = 1500;          // encoder positions per segment of the last encode
  int enc_stop = 1 << 30;        // debug: run only the first enc_stop layers
  bool enc_tap = false;          // debug: keep the fp32 encoder output (in resid)
  bool mel_tap = false;          // debug: also write the fp32 [n, n_mels, 3000] features
  // encoder GEMM grid cap (experiment knob, DM_ENC_MAX_CTAS): SMs left free
  // for the decode stream while a group encodes beside it
  int enc_max_ctas = std::getenv("DM_ENC_MAX_CTAS") ? std::atoi(std::getenv("DM_ENC_MAX_CTAS")) : 0;
  // decode
  DecodeState st{};
  int32_t* prompt_dev = nullptr;
  int32_t* active_dev = nullptr;
  int32_t* n_active_dev = nullptr;
  int32_t* page_table_dev = nullptr;
  std::vector<int32_t> page_table_host;
  std::vector<int> free_pages;
  std::vector<int> slot_pages;       // pages held per slot
  int32_t* staging = nullptr;        // pinned scratch for uploads
  std::vector<void*> allocs;
  cudaStream_t cap_stream = nullptr;
  cudaGraphExec_t step_exec = nullptr;
  cudaGraph_t step_graph = nullptr;
  int gemv_counter_base = 0;
  std::vector<TcGemvMaps> maps;   // [Ld * 6 + 1]: per layer qkv,o,xq,xo,fc1,fc2; LM head
  std::vector<GemvArgs> plans;    // same order: launch plan of each projection
  CUtensorMap xkv_map;            // cross-KV cache as [rows, 64] bf16 (box 64 x 64, 128B swizzle)
  // Independent decode groups (slot s belongs to group s % G): each has its own
  // row-space activations, active list, scratch, step graph and stream, so the
  // groups' latency-bound kernel chains overlap on the GPU.
  struct Group {
    DecodeState st{};
    std::vector<TcGemvMaps> maps;
    int32_t* active_dev = nullptr;
    int32_t* n_active_dev = nullptr;
    cudaStream_t stream = nullptr;
    cudaEvent_t done = nullptr;
    // one step graph per row bucket: per-row grids sized to the bucket, so a
    // step with few active rows does not schedule thousands of empty CTAs
    // (every kernel computes the same values whatever the grid)
    cudaGraph_t graph[kRowBuckets] = {};
    cudaGraphExec_t exec[kRowBuckets] = {};
    size_t nodes[kRowBuckets] = {};  // kernels per step graph (launch telemetry)
    int n_active_host = 0;
    // K-split partial sums of the linear projections (consumer-reduced)
    float *p_qkv = nullptr, *p_o = nullptr, *p_xq = nullptr, *p_xo = nullptr, *p_fc2 = nullptr;
    float* p_fc1 = nullptr;        // fc1 K-split partials when fc1 is split (fc1_split)
    float* p_lm = nullptr;         // LM-head K-split partials [splits][kRows][vocab]
    float* xpart = nullptr;        // cross-attention split results [kRows][H][8][68]
    int* xcnt = nullptr;           // [kRows * kMaxHeads] split arrival counters
  };
  std::vector<Group> groups;
  cudaEvent_t step_start = nullptr;
  // telemetry: kernels launched (graph nodes counted per replay)
  long long launches = 0, steps = 0, encodes = 0, segments = 0;
  bool fc1_split() const { return d / 64 > 8; }       // fc1's K does not fit one CTA
  // fc1's K split (fixed per engine): the GEMV writes partials and
  // gelu_hilo_kernel reduces them in split order, adds the bias, applies GELU
  int fc1_splits = std::getenv("DM_FC1_SPLITS") ? std::atoi(std::getenv("DM_FC1_SPLITS")) : 4;
  // fc1 split merge + GELU in the GEMV's last CTA per tile up to this many
  // rows, else gelu_hilo_kernel: the kernel measured faster at every row
  // count (1 row 1.37 -> 1.34 ms per step), so 0 (DM_FC1_TAIL_ROWS: experiments)
  int fc1_tail_rows = std::getenv("DM_FC1_TAIL_ROWS") ? std::atoi(std::getenv("DM_FC1_TAIL_ROWS")) : 0;
  // cross-attention split merge in the last CTA up to this many rows, else
  // xattn_merge_kernel (DM_XA_TAIL_MERGE_ROWS: experiments)
  int xa_tail_merge_rows = std::getenv("DM_XA_TAIL_MERGE_ROWS")
                               ? std::atoi(std::getenv("DM_XA_TAIL_MERGE_ROWS"))
                               : kXaTailMergeRows;
  // steps of <= gv_fuse_rows rows (at most 16) skip the split-merge and GELU
  // kernels: the cross-o and fc2 GEMVs build their operands from the raw
  // results (DM_GV_FUSE_ROWS: experiments; 0 disables)
  bool lm_argmax_epi = std::getenv("DM_LM_ARGMAX_EPI") != nullptr;   // (A/B: last-CTA merge)
  int gv_fuse_rows = std::min(16, std::getenv("DM_GV_FUSE_ROWS") ? std::atoi(std::getenv("DM_GV_FUSE_ROWS"))
                                                                 : kGvFuseRows);
  int encode_kernels() const { return 2 + 1 + 2 + 7 * L + 1 + 1; }

  // debug (DM_GUARD=1 at create): every allocation gets a 64 KB 0xA5 tail
  // guard; dm_whisper_debug(13) reports the allocations whose guard changed
  static constexpr size_t kGuard = 64 * 1024;
  bool guard = std::getenv("DM_GUARD") != nullptr;
  std::vector<size_t> alloc_bytes;
  int alloc(void** p, size_t bytes, bool zero = true) {
    DM_CHECK_CUDA(cudaMalloc(p, bytes + (guard ? kGuard : 0)));
    allocs.push_back(*p);
    alloc_bytes.push_back(bytes);
    if (zero) DM_CHECK_CUDA(cudaMemset(*p, 0, bytes));
    if (guard) DM_CHECK_CUDA(cudaMemset(static_cast<uint8_t*>(*p) + bytes, 0xA5, kGuard));
    return 0;
  }
  template <class T>
  int alloc_t(T** p, size_t count, bool zero = true) {
    return alloc(reinterpret_cast<void**>(p), count * sizeof(T), zero);
  }

  ~WhisperEngine() {
    for (auto& g : groups) {
      for (int b = 0; b < kRowBuckets; ++b) {
        if (g.exec[b]) cudaGraphExecDestroy(g.exec[b]);
        if (g.graph[b]) cudaGraphDestroy(g.graph[b]);
      }
      if (g.stream) cudaStreamDestroy(g.stream);
      if (g.done) cudaEventDestroy(g.done);
    }
    if (step_start) cudaEventDestroy(step_start);

    if (cap_stream) cudaStreamDestroy(cap_stream);
    for (void* p : allocs) cudaFree(p);
    if (slot_host) cudaFreeHost(slot_host);
    if (staging) cudaFreeHost(staging);
  }
};

__global__ void repack_conv1_kernel(const uint16_t* __restrict__ w, uint16_t* __restrict__ out,
                                    int d, int nm, int Cp) {
  // w [d, 3, nm] -> out [d, 3, Cp] (zero channels >= nm)
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= d * 3 * Cp) return;
  const int c = i % Cp, tap = (i / Cp) % 3, o = i / (3 * Cp);
  out[i] = c < nm ? w[(size_t(o) * 3 + tap) * nm + c] : uint16_t(0);
}

static int engine_init(WhisperEngine* e) {
  const dm_whisper_config& c = e->cfg;
  e->d = c.d_model; e->H = c.heads; e->L = c.enc_layers; e->Ld = c.dec_layers;
  e->F = c.ffn; e->nm = c.n_mels; e->Cp = c.n_mels <= 64 ? 64 : 128;
  DM_REQUIRE(e->d % 128 == 0 && e->d / e->H == 64, "d must be a multiple of 128 with head_dim 64");
  DM_REQUIRE(c.n_mels == 80 || c.n_mels == 128, "n_mels must be 80 or 128");
  DM_REQUIRE(c.max_slots >= 1 && c.max_slots <= 64, "max_slots must be in [1, 64]");
  DM_REQUIRE(c.max_encode_batch >= 1, "max_encode_batch >= 1");
  DM_REQUIRE(c.prompt_len >= 1 && c.prompt_len <= 8, "prompt_len in [1, 8]");
  DM_REQUIRE(c.num_pages >= c.max_slots, "num_pages >= max_slots");
  DM_REQUIRE(c.persistent_decode == 0 && c.fuse_ln == 0, "persistent_decode / fuse_ln are reserved (0)");
  const int d = e->d, E = c.max_encode_batch, S = c.max_slots;
  e->E = E;
  const size_t rows = size_t(E) * 1500;
  if (e->alloc_t(&e->conv1_w_pad, size_t(d) * 3 * e->Cp)) return 2;
  {
    const int n = d * 3 * e->Cp;
    repack_conv1_kernel<<<ceil_div(n, 256), 256>>>(e->W(0), e->conv1_w_pad, d, e->nm, e->Cp);
    DM_CHECK_LAUNCH();
  }
  if (e->alloc_t(&e->mel, size_t(E) * e->nm * 3000, false)) return 2;
  if (e->alloc_t(&e->mel_t, size_t(E) * 3002 * e->Cp)) return 2;
  if (e->alloc_t(&e->segmax, E)) return 2;
  if (e->alloc_t(&e->conv1_out, size_t(E) * 3002 * d)) return 2;
  if (e->alloc_t(&e->resid, rows * d, false)) return 2;
  if (e->alloc_t(&e->lnb, rows * d, false)) return 2;
  if (e->alloc_t(&e->qb, size_t(E) * e->H * 1536 * 64)) return 2;
  if (e->alloc_t(&e->kb, size_t(E) * e->H * 1536 * 64)) return 2;
  if (e->alloc_t(&e->vtb, size_t(E) * e->H * 64 * 1536)) return 2;
  if (e->alloc_t(&e->attn_out, rows * d, false)) return 2;
  if (e->alloc_t(&e->fc1_out, rows * e->F, false)) return 2;
  if (e->alloc_t(&e->enc_out, rows * d, false)) return 2;
  if (e->alloc_t(&e->slot_dev, E)) return 2;
  if (e->alloc_t(&e->seg_len_dev, E)) return 2;
  DM_CHECK_CUDA(cudaMallocHost(&e->slot_host, sizeof(int32_t) * E));
  if (int rc = e->ring.init()) return rc;
  if (e->alloc_t(&e->admit_args_dev, size_t(2) * S)) return 2;
  DM_CHECK_CUDA(cudaMallocHost(&e->staging, sizeof(int32_t) * (64 * 65 + 4096 + 256)));

  // decode state
  DecodeState& st = e->st;
  st.max_slots = S; st.d = d; st.heads = e->H; st.layers = e->Ld; st.ffn = e->F;
  st.vocab = c.vocab; st.page_tokens = 64; st.pages_per_slot = 7; st.eot = c.eot;
  st.prompt_len = c.prompt_len;
  st.grid_rows = kRows;            // debug / timing probes; step graphs use their bucket
  if (e->alloc_t(&e->prompt_dev, kMaxPrompt)) return 2;
  DM_CHECK_CUDA(cudaMemcpy(e->prompt_dev, c.prompt, sizeof(int32_t) * c.prompt_len,
                           cudaMemcpyHostToDevice));
  st.prompt = e->prompt_dev;
  if (e->alloc_t(&e->active_dev, S)) return 2;
  if (e->alloc_t(&e->n_active_dev, 1)) return 2;
  st.active = e->active_dev; st.n_active = e->n_active_dev;
  if (e->alloc_t(&st.pos, S)) return 2;
  if (e->alloc_t(&st.cur_tok, S)) return 2;
  if (e->alloc_t(&st.n_gen, S)) return 2;
  if (e->alloc_t(&st.cap, S)) return 2;
  if (e->alloc_t(&st.done, S)) return 2;
  {
    std::vector<int32_t> ones(S, 1);
    DM_CHECK_CUDA(cudaMemcpy(st.done, ones.data(), sizeof(int32_t) * S, cudaMemcpyHostToDevice));
  }
  if (e->alloc_t(&st.out_tokens, size_t(S) * 448)) return 2;
  if (e->alloc_t(&e->page_table_dev, size_t(S) * 7)) return 2;
  st.page_table = e->page_table_dev;
  e->page_table_host.assign(size_t(S) * 7, 0);
  e->slot_pages.assign(S, 0);
  for (int p = c.num_pages - 1; p >= 0; --p) e->free_pages.push_back(p);
  const size_t page_elems = size_t(e->Ld) * 2 * e->H * 64 * 64;
  if (e->alloc_t(&st.kv_pool, page_elems * c.num_pages)) return 2;
  uint16_t* xkv = nullptr;
  if (e->alloc_t(&xkv, size_t(e->Ld) * S * 2 * e->H * 1500 * 64)) return 2;
  st.xkv = xkv;
  if (e->alloc_t(&e->enc_len_dev, S)) return 2;
  {
    std::vector<int32_t> full(S, 1500);
    DM_CHECK_CUDA(cudaMemcpy(e->enc_len_dev, full.data(), sizeof(int32_t) * S, cudaMemcpyHostToDevice));
  }
  st.enc_len = e->enc_len_dev;
  const int G = std::max(1, std::min(c.decode_groups > 0 ? c.decode_groups : 1, S));
  e->groups.resize(G);
  const int tiles = ceil_div(c.vocab, 128);
  for (int gi = 0; gi < G; ++gi) {
    WhisperEngine::Group& gr = e->groups[gi];
    DecodeState& gs = gr.st;
    gs = st;                                   // shared slot-indexed state
    if (e->alloc_t(&gr.active_dev, kRows)) return 2;
    if (e->alloc_t(&gr.n_active_dev, 1)) return 2;
    gs.active = gr.active_dev; gs.n_active = gr.n_active_dev;
    if (e->alloc_t(&gs.x, size_t(kRows) * d)) return 2;
    if (e->alloc_t(&gs.xh, size_t(kRows) * d)) return 2;
    if (e->alloc_t(&gs.xl, size_t(kRows) * d)) return 2;
    if (e->alloc_t(&gs.ah, size_t(kRows) * d)) return 2;
    if (e->alloc_t(&gs.al, size_t(kRows) * d)) return 2;
    if (e->alloc_t(&gs.hh, size_t(kRows) * e->F)) return 2;
    if (e->alloc_t(&gs.hl, size_t(kRows) * e->F)) return 2;
    // launch plans (depend only on the projection shape) and their scratch
    e->plans.clear();
    for (int l = 0; l < e->Ld; ++l) {
      // consumers: attention kernels reduce <= kAttnSplits partials, LayerNorms <= kMaxHeads
      e->plans.push_back(gemv_plan(3 * d, d, GV_PARTIAL, 5));             // qkv (measured: <= 5)
      e->plans.push_back(gemv_plan(d, d, GV_PARTIAL, kMaxHeads));         // o
      e->plans.push_back(gemv_plan(d, d, GV_PARTIAL, kAttnSplits));       // xq
      e->plans.push_back(gemv_plan(d, d, GV_PARTIAL, kMaxHeads));         // xo
      // fc1: GELU in the GEMV epilogue when one CTA holds the whole K, else
      // K-split partials + gelu_hilo_kernel
      e->plans.push_back(e->fc1_split() ? gemv_plan(e->F, d, GV_PARTIAL, e->fc1_splits)
                                        : gemv_plan(e->F, d, GV_GELU_HILO));          // fc1
      e->plans.push_back(gemv_plan(d, e->F, GV_PARTIAL, kMaxHeads));      // fc2
    }
    {
      // LM head: the K split of the last-CTA ARGMAX plan (<= 8 k-blocks per
      // CTA); partials + lm_argmax_kernel unless DM_LM_ARGMAX_EPI=1
      GemvArgs lm = gemv_plan(c.vocab, d, GV_ARGMAX);
      if (!e->lm_argmax_epi) lm.epi = GV_PARTIAL;
      e->plans.push_back(lm);
    }
    if (e->alloc_t(&gr.p_qkv, gemv_part_floats(3 * d, d, GV_PARTIAL, 5))) return 2;
    if (e->alloc_t(&gr.p_o, gemv_part_floats(d, d, GV_PARTIAL, kMaxHeads))) return 2;
    if (e->alloc_t(&gr.p_xq, gemv_part_floats(d, d, GV_PARTIAL, kAttnSplits))) return 2;
    if (e->alloc_t(&gr.p_xo, gemv_part_floats(d, d, GV_PARTIAL, kMaxHeads))) return 2;
    if (e->alloc_t(&gr.p_fc2, gemv_part_floats(d, e->F, GV_PARTIAL, kMaxHeads))) return 2;
    if (e->fc1_split() &&
        e->alloc_t(&gr.p_fc1, gemv_part_floats(e->F, d, GV_PARTIAL, kMaxHeads))) return 2;
    size_t part = std::max<size_t>(1, std::max(gemv_part_floats(e->F, d, GV_GELU_HILO),
                                               gemv_part_floats(c.vocab, d, GV_ARGMAX)));
    if (e->fc1_split())     // the fused split-GELU epilogue of few-row steps: fc1's own split
      part = std::max(part, gemv_part_floats(e->F, d, GV_PARTIAL, e->fc1_splits) / kRows * 128 /
                                ceil_div(e->F, 128) * ceil_div(e->F, 128));
    if (e->alloc_t(&gs.part, part)) return 2;
    if (!e->lm_argmax_epi &&
        e->alloc_t(&gr.p_lm, size_t(e->plans.back().splits) * kRows * c.vocab)) return 2;
    if (e->alloc_t(&gs.counters, 4096)) return 2;
    if (e->alloc_t(&gr.xpart, size_t(kRows) * e->H * kXSplits * 68)) return 2;
    if (e->alloc_t(&gr.xcnt, size_t(kRows) * kMaxHeads)) return 2;
    if (e->alloc_t(&gs.amax_val, size_t(tiles) * kRows)) return 2;
    if (e->alloc_t(&gs.amax_idx, size_t(tiles) * kRows)) return 2;
    gs.logits_dbg = nullptr;
    // TMA maps of every decoder projection (weights [N, K] + this group's hi/lo inputs,
    // activation boxes of 16 rows so loads scale with the active rows)
    auto mk = [&](TcGemvMaps& m, int wi, int N, int K, const uint16_t* xh, const uint16_t* xl) {
      if (make_tmap_2d(&m.w, e->W(wi), K, N, uint64_t(K) * 2, 64, 128)) return 2;
      if (make_tmap_2d(&m.xh, xh, K, kRows, uint64_t(K) * 2, 64, kGvXBox)) return 2;
      if (make_tmap_2d(&m.xl, xl, K, kRows, uint64_t(K) * 2, 64, kGvXBox)) return 2;
      return 0;
    };
    gr.maps.resize(size_t(e->Ld) * 6 + 1);
    for (int l = 0; l < e->Ld; ++l) {
      const int b0 = e->dec_layer_base(l);
      TcGemvMaps* m = &gr.maps[size_t(l) * 6];
      if (mk(m[0], b0 + 2, 3 * d, d, gs.xh, gs.xl)) return 2;        // qkv
      if (mk(m[1], b0 + 4, d, d, gs.ah, gs.al)) return 2;            // o
      if (mk(m[2], b0 + 8, d, d, gs.xh, gs.xl)) return 2;            // xq
      if (mk(m[3], b0 + 10, d, d, gs.ah, gs.al)) return 2;           // xo
      if (mk(m[4], b0 + 14, e->F, d, gs.xh, gs.xl)) return 2;        // fc1
      if (mk(m[5], b0 + 16, d, e->F, gs.hh, gs.hl)) return 2;        // fc2
    }
    if (mk(gr.maps.back(), e->after_enc() + 2, c.vocab, d, gs.xh, gs.xl)) return 2;  // LM head
    DM_CHECK_CUDA(cudaStreamCreateWithFlags(&gr.stream, cudaStreamNonBlocking));
    DM_CHECK_CUDA(cudaEventCreateWithFlags(&gr.done, cudaEventDisableTiming));
  }
  DM_CHECK_CUDA(cudaEventCreateWithFlags(&e->step_start, cudaEventDisableTiming));
  e->gemv_counter_base = 0;
  {
    // group 0 doubles as the engine's default state (debug / timing probes)
    DecodeState shared = st;
    st = e->groups[0].st;
    e->maps = e->groups[0].maps;
    (void)shared;
  }
  if (make_tmap_2d(&e->xkv_map, st.xkv, 64, uint64_t(e->Ld) * S * 2 * e->H * 1500, 128, 64, 64))
    return 2;
  DM_CHECK_CUDA(cudaStreamCreateWithFlags(&e->cap_stream, cudaStreamNonBlocking));
  DM_CHECK_CUDA(cudaDeviceSynchronize());
  return 0;
}

// Per encode: encoder positions per segment (1500, or ceil(n / 320) for a
// length-aware encode), the slots' enc_len, the conv1 input's zero frame right
// after each segment's window (length-aware), and the conv1 output's two zero
// pad rows (its row stride follows the window).
__global__ void encode_prep_kernel(const int32_t* __restrict__ lengths, int n, int length_aware,
                                   const int32_t* __restrict__ slot_ids, int32_t* __restrict__ seg_len,
                                   int32_t* __restrict__ enc_len, uint16_t* __restrict__ mel_t, int ldt,
                                   uint16_t* __restrict__ conv1_out, int c1_rows, int d) {
  const int b = blockIdx.x;
  if (b >= n) return;
  int len = 1500;
  if (length_aware) {
    const int ns = min(max(lengths[b], 0), 480000);
    len = max(1, min(1500, (ns + 319) / 320));
  }
  if (threadIdx.x == 0) {
    seg_len[b] = len;
    enc_len[slot_ids[b]] = len;
  }
  if (length_aware)          // frame 2 len (row 2 len + 1) of the conv1 input: zero padding
    for (int c = threadIdx.x; c < ldt; c += blockDim.x)
      mel_t[(size_t(b) * 3002 + 2 * len + 1) * ldt + c] = 0;
  uint16_t* c1 = conv1_out + size_t(b) * c1_rows * d;
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    c1[c] = 0;
    c1[size_t(c1_rows - 1) * d + c] = 0;
  }
}

// rows: encoder positions computed per segment (1500, or the batch's longest
// length-aware window); length_aware: mask each segment to its own window.
static int encoder_forward(WhisperEngine* e, const int16_t* pcm, const int64_t* offsets,
                           const int32_t* lengths, int n, cudaStream_t s, int rows,
                           bool length_aware) {
  const int d = e->d, H = e->H;
  const int frames = 2 * rows, t_pad = ceil_div(rows, 128) * 128;
  const LogmelTables* tab = nullptr;
  if (int rc = get_logmel_tables(e->nm, &tab)) return rc;
  // the fp32 feature contract is written only for the debug tap (dm_whisper_debug 15)
  if (int rc = launch_logmel(pcm, offsets, lengths, n, e->nm, tab, e->mel_tap ? e->mel : nullptr,
                             e->mel_t, e->segmax, s, e->mel_tap ? 3000 : frames))
    return rc;
  encode_prep_kernel<<<n, 128, 0, s>>>(lengths, n, length_aware ? 1 : 0, e->slot_dev,
                                       e->seg_len_dev, e->enc_len_dev, e->mel_t, e->Cp,
                                       e->conv1_out, frames + 2, d);
  DM_CHECK_LAUNCH();
  // conv1 (implicit GEMM over the padded time-major mel), GELU
  {
    GemmArgs g;
    g.max_ctas = e->enc_max_ctas;
    g.A = e->mel_t; g.a_mode = A_CONV_S1; g.C = e->Cp; g.K = 3 * e->Cp; g.T = frames; g.Bt = n;
    g.a_rows = 3002;
    g.W = e->conv1_w_pad; g.N = d;
    g.epi.mode = EPI_CONV1; g.epi.bias = e->W(1); g.epi.out = e->conv1_out; g.epi.ldo = d;
    if (int rc = launch_gemm(g, s)) return rc;
  }
  // conv2 (stride 2), GELU, + sinusoid positions -> fp32 residual stream
  {
    GemmArgs g;
    g.max_ctas = e->enc_max_ctas;
    g.A = e->conv1_out; g.a_mode = A_CONV_S2; g.C = d; g.K = 3 * d; g.T = rows; g.Bt = n;
    g.W = e->W(2); g.N = d;
    g.epi.mode = EPI_CONV2_POS; g.epi.bias = e->W(3); g.epi.out = e->resid; g.epi.ldo = d;
    g.epi.pos = e->W(4);
    if (int rc = launch_gemm(g, s)) return rc;
  }
  const int M = n * rows;
  auto flat = [&](const uint16_t* A, int K, const uint16_t* Wt, int N) {
    GemmArgs g;
    g.max_ctas = e->enc_max_ctas;
    g.A = A; g.a_mode = A_FLAT; g.K = K; g.T = M; g.Bt = 1; g.lda = K; g.a_bstride = 0;
    g.W = Wt; g.N = N;
    return g;
  };
  for (int l = 0; l < e->L && l < e->enc_stop; ++l) {
    const int b0 = e->enc_layer_base(l);
    if (int rc = launch_layernorm_bf16(e->resid, e->W(b0 + 0), e->W(b0 + 1), e->lnb, M, d, s))
      return rc;
    {
      GemmArgs g = flat(e->lnb, d, e->W(b0 + 2), 3 * d);
      g.epi.mode = EPI_QKV; g.epi.bias = e->W(b0 + 3);
      g.epi.q = e->qb; g.epi.k = e->kb; g.epi.vt = e->vtb; g.epi.heads = H; g.epi.t_pad = t_pad;
      g.epi.seg_rows = rows;
      g.epi.q_scale = 0.125f;
      if (int rc = launch_gemm(g, s)) return rc;
    }
    if (int rc = launch_attention(e->qb, e->kb, e->vtb, n, H, rows, t_pad, e->attn_out, d, s,
                                  length_aware ? e->seg_len_dev : nullptr))
      return rc;
    {
      GemmArgs g = flat(e->attn_out, d, e->W(b0 + 4), d);
      g.epi.mode = EPI_RESID_F32; g.epi.bias = e->W(b0 + 5); g.epi.out = e->resid; g.epi.ldo = d;
      if (int rc = launch_gemm(g, s)) return rc;
    }
    if (int rc = launch_layernorm_bf16(e->resid, e->W(b0 + 6), e->W(b0 + 7), e->lnb, M, d, s))
      return rc;
    {
      GemmArgs g = flat(e->lnb, d, e->W(b0 + 8), e->F);
      g.epi.mode = EPI_GELU_BF16; g.epi.bias = e->W(b0 + 9); g.epi.out = e->fc1_out;
      g.epi.ldo = e->F;
      if (int rc = launch_gemm(g, s)) return rc;
    }
    {
      GemmArgs g = flat(e->fc1_out, e->F, e->W(b0 + 10), d);
      g.epi.mode = EPI_RESID_F32; g.epi.bias = e->W(b0 + 11); g.epi.out = e->resid; g.epi.ldo = d;
      if (int rc = launch_gemm(g, s)) return rc;
    }
  }
  const int a = e->after_enc();
  if (int rc = launch_layernorm_bf16(e->resid, e->W(a), e->W(a + 1), e->enc_out, M, d, s,
                                     e->enc_tap ? e->resid : nullptr))
    return rc;    // (debug tap: fp32 encoder output written in place over the residual)
  // cross-KV precompute for every decoder layer, scattered into the slots
  {
    const int x = e->after_dec();
    GemmArgs g = flat(e->enc_out, d, e->W(x), 2 * d * e->Ld);
    g.epi.mode = EPI_XKV; g.epi.bias = e->W(x + 1); g.epi.out = const_cast<uint16_t*>(e->st.xkv);
    g.epi.slot_ids = e->slot_dev; g.epi.n_slots = e->cfg.max_slots; g.epi.layers = e->Ld;
    g.epi.heads = H; g.epi.seg_rows = rows;
    if (int rc = launch_gemm(g, s)) return rc;
  }
  return 0;
}

__global__ void pdl_floor_kernel() {
  pdl_wait();
  pdl_trigger();
}
static int launch_pdl_floor(cudaStream_t s) {
  DM_CHECK_CUDA(launch_pdl(pdl_floor_kernel, dim3(1), dim3(32), 0, s));
  return 0;
}

#define DM_STEP(call)                 \
  do {                                \
    if (int rc = (call)) return rc;   \
    ++st.trace_id;                    \
  } while (0)

static int record_step(WhisperEngine* e, WhisperEngine::Group& grp, cudaStream_t s, int rows) {
  DecodeState st = grp.st;        // local copy: trace_id numbers the step's kernels
  st.trace_id = 0;
  st.grid_rows = rows;
  const int d = e->d;
  const int a = e->after_enc();
  auto gv = [&](int idx, float* part, uint16_t* yh, uint16_t* yl, const uint16_t* bias) {
    GemvArgs g = gemv_plan_for_rows(e->plans[idx], rows);
    g.bias = bias; g.part = part; g.yh = yh; g.yl = yl; g.counter_base = e->gemv_counter_base;
    return launch_gemv(st, grp.maps[idx], g, s);
  };
  auto ln = [&](int mode, int gi, const Partials& res) {
    LnArgs la{};
    la.mode = mode; la.g = e->W(gi); la.b = e->W(gi + 1);
    la.embed = e->W(a + 2); la.pos_emb = e->W(a + 3); la.res = res;
    return launch_ln(st, la, s);
  };
  Partials prev{};                 // residual partials feeding the next LayerNorm
  for (int l = 0; l < e->Ld; ++l) {
    const int b0 = e->dec_layer_base(l);
    const int pi = l * 6;
    const int gq = e->plans[pi].splits, go = e->plans[pi + 1].splits, gx = e->plans[pi + 2].splits;
    const int gf = e->plans[pi + 5].splits;
    // ln1 (+ embedding for layer 0, + previous fc2 residual otherwise)
    DM_STEP(ln(l == 0 ? 1 : 2, b0 + 0, prev));
    DM_STEP(gv(pi + 0, grp.p_qkv, nullptr, nullptr, nullptr));
    DM_STEP(launch_self_attn(st, l, Partials{grp.p_qkv, gq, 3 * d, e->W(b0 + 3)}, 0.125f, s));
    DM_STEP(gv(pi + 1, grp.p_o, nullptr, nullptr, nullptr));
    DM_STEP(ln(2, b0 + 6, Partials{grp.p_o, go, d, e->W(b0 + 5)}));
    DM_STEP(gv(pi + 2, grp.p_xq, nullptr, nullptr, nullptr));
    // cross-attention (o -> ah/al) -> cross-o projection (partials) -> ln3
    // the 8 split results of the cross-attention are merged by the last split
    // (<= xa_tail_merge_rows rows), by the cross-o GEMV while it builds its
    // operand (<= gv_fuse_rows), or by xattn_merge_kernel
    const bool tail_merge = rows <= e->xa_tail_merge_rows;
    const bool fuse = rows <= e->gv_fuse_rows;
    DM_STEP(launch_cross_attn(st, e->xkv_map, l, Partials{grp.p_xq, gx, d, e->W(b0 + 9)}, 0.125f,
                              grp.xpart, grp.xcnt, s, 0, tail_merge));
    if (!tail_merge && !fuse) DM_STEP(launch_xattn_merge(st, grp.xpart, s));
    {
      GemvArgs g = gemv_plan_for_rows(e->plans[pi + 3], rows);
      g.part = grp.p_xo; g.counter_base = e->gemv_counter_base;
      if (!tail_merge && fuse) { g.xsrc = GV_X_XMERGE; g.xp = grp.xpart; }
      DM_STEP(launch_gemv(st, grp.maps[pi + 3], g, s));
    }
    DM_STEP(ln(2, b0 + 12, Partials{grp.p_xo, e->plans[pi + 3].splits, d, e->W(b0 + 11)}));
    bool fc2_builds = false;     // fc2 computes GELU(fc1 partials) into its own operand
    if (e->fc1_split() && rows > e->fc1_tail_rows) {
      DM_STEP(gv(pi + 4, grp.p_fc1, nullptr, nullptr, nullptr));
      if (fuse)
        fc2_builds = true;
      else
        DM_STEP(launch_gelu_hilo(st, Partials{grp.p_fc1, e->plans[pi + 4].splits, e->F, e->W(b0 + 15)},
                                 st.hh, st.hl, s));
    } else if (e->fc1_split()) {
      GemvArgs g = e->plans[pi + 4];
      g.epi = GV_GELU_HILO;
      g = gemv_plan_for_rows(g, rows);
      g.bias = e->W(b0 + 15); g.part = nullptr; g.yh = st.hh; g.yl = st.hl;
      g.counter_base = e->gemv_counter_base;
      DM_STEP(launch_gemv(st, grp.maps[pi + 4], g, s));
    } else {
      DM_STEP(gv(pi + 4, nullptr, st.hh, st.hl, e->W(b0 + 15)));
    }
    {
      GemvArgs g = gemv_plan_for_rows(e->plans[pi + 5], rows);
      g.part = grp.p_fc2; g.counter_base = e->gemv_counter_base;
      if (fc2_builds) {
        g.xsrc = GV_X_GELU; g.xp = grp.p_fc1; g.xs_splits = e->plans[pi + 4].splits;
        g.xbias = e->W(b0 + 15);
      }
      DM_STEP(launch_gemv(st, grp.maps[pi + 5], g, s));
    }
    prev = Partials{grp.p_fc2, gf, d, e->W(b0 + 17)};
  }
  const int x = e->after_dec();
  DM_STEP(ln(2, x + 2, prev));                                   // final LayerNorm
  if (e->lm_argmax_epi) {
    DM_STEP(gv(e->Ld * 6, nullptr, nullptr, nullptr, nullptr));  // tied LM head + tile argmax
  } else {
    DM_STEP(gv(e->Ld * 6, grp.p_lm, nullptr, nullptr, nullptr));  // tied LM head partials
    DM_STEP(launch_lm_argmax(st, Partials{grp.p_lm, e->plans[e->Ld * 6].splits, e->cfg.vocab, nullptr}, s));
  }
  DM_STEP(launch_finalize(st, s));
  return 0;
}
#undef DM_STEP

static int build_step_graph(WhisperEngine* e) {
  for (auto& grp : e->groups) {
    for (int b = 0; b < kRowBuckets; ++b) {
      if (grp.exec[b]) {
        cudaGraphExecDestroy(grp.exec[b]);
        grp.exec[b] = nullptr;
      }
      if (grp.graph[b]) {
        cudaGraphDestroy(grp.graph[b]);
        grp.graph[b] = nullptr;
      }
      DM_CHECK_CUDA(cudaStreamBeginCapture(e->cap_stream, cudaStreamCaptureModeThreadLocal));
      int rc = record_step(e, grp, e->cap_stream, kRowBucket[b]);
      cudaGraph_t g = nullptr;
      cudaError_t ce = cudaStreamEndCapture(e->cap_stream, &g);
      if (rc) {
        if (g) cudaGraphDestroy(g);
        return rc;
      }
      DM_CHECK_CUDA(ce);
      grp.graph[b] = g;
      DM_CHECK_CUDA(cudaGraphGetNodes(g, nullptr, &grp.nodes[b]));
      DM_CHECK_CUDA(cudaGraphInstantiate(&grp.exec[b], g, 0));
    }
  }
  e->step_exec = e->groups[0].exec[kRowBuckets - 1];     // marks "built"
  return 0;
}

}  // namespace dm

using namespace dm;

// ================================================================ C ABI
extern "C" {

const char* dm_last_error(void) { return dm::last_error(); }
int dm_version(void) { return 1; }

int dm_fill_normal_bf16(uint16_t* dst, uint64_t numel, uint64_t key, float scale, float mean,
                        void* stream) {
  DM_REQUIRE(dst != nullptr || numel == 0, "null destination");
  if (numel == 0) return 0;
  uint64_t blocks = (numel + 255) / 256;
  if (blocks > 148ull * 64) blocks = 148ull * 64;
  fill_normal_kernel<<<unsigned(blocks), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      dst, numel, key, scale, mean);
  DM_CHECK_LAUNCH();
  return 0;
}

int dm_logmel(const int16_t* pcm, const int64_t* offsets, const int32_t* lengths, int n,
              int n_mels, float* out, void* stream) {
  DM_REQUIRE(n >= 0, "n < 0");
  DM_REQUIRE(n_mels == 80 || n_mels == 128, "n_mels must be 80 or 128");
  if (n == 0) return 0;
  DM_REQUIRE(pcm && offsets && lengths && out, "null pointer");
  const LogmelTables* tab = nullptr;
  if (int rc = get_logmel_tables(n_mels, &tab)) return rc;
  // per-segment max scratch: grown once, reused (no per-call allocation on the stream)
  // (one buffer per device: the caller's current device owns the stream)
  static std::map<int, std::pair<uint32_t*, int>> scratch;
  static std::mutex mu;
  int dev = 0;
  DM_CHECK_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  auto& sc = scratch[dev];
  if (sc.second < n) {
    DM_CHECK_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
    if (sc.first) cudaFree(sc.first);
    sc = {nullptr, 0};
    DM_CHECK_CUDA(cudaMalloc(reinterpret_cast<void**>(&sc.first), sizeof(uint32_t) * n));
    sc.second = n;
  }
  uint32_t* segmax = sc.first;
  return launch_logmel(pcm, offsets, lengths, n, n_mels, tab, out, nullptr, segmax,
                       static_cast<cudaStream_t>(stream));
}

int dm_logmel_operand(const int16_t* pcm, const int64_t* offsets, const int32_t* lengths, int n,
                      int n_mels, uint16_t* out, uint32_t* segmax, void* stream) {
  DM_REQUIRE(n >= 0, "n < 0");
  DM_REQUIRE(n_mels == 80 || n_mels == 128, "n_mels must be 80 or 128");
  if (n == 0) return 0;
  DM_REQUIRE(pcm && offsets && lengths && out && segmax, "null pointer");
  const LogmelTables* tab = nullptr;
  if (int rc = get_logmel_tables(n_mels, &tab)) return rc;
  return launch_logmel(pcm, offsets, lengths, n, n_mels, tab, nullptr, out, segmax,
                       static_cast<cudaStream_t>(stream));
}

int dm_gemm_bf16_f32(const uint16_t* A, const uint16_t* Wt, const uint16_t* bias, float* out,
                     int M, int N, int K, void* stream) {
  GemmArgs g;
  g.A = A; g.a_mode = A_FLAT; g.K = K; g.T = M; g.Bt = 1; g.lda = K; g.W = Wt; g.N = N;
  g.epi.mode = EPI_STORE_F32; g.epi.bias = bias; g.epi.out = out; g.epi.ldo = N;
  return launch_gemm(g, static_cast<cudaStream_t>(stream));
}

int dm_whisper_create(const dm_whisper_config* cfg, const uint16_t* weights,
                      const int64_t* offsets, int n_offsets, void** handle) {
  DM_REQUIRE(cfg && weights && offsets && handle, "null argument");
  const int expect = 5 + 12 * cfg->enc_layers + 4 + 18 * cfg->dec_layers + 4;
  DM_REQUIRE(n_offsets == expect, "offset table has " + std::to_string(n_offsets) +
                                      " entries, expected " + std::to_string(expect));
  auto* e = new WhisperEngine();
  if (cudaGetDevice(&e->device) != cudaSuccess) {
    delete e;
    DM_CHECK_CUDA(cudaGetLastError());
  }
  e->cfg = *cfg;
  e->w = weights;
  e->off.assign(offsets, offsets + n_offsets);
  for (int64_t o : e->off)
    if (o % 8 != 0) {
      delete e;
      DM_REQUIRE(false, "weight offsets must be 16-byte aligned");
    }
  if (int rc = engine_init(e)) {
    delete e;
    return rc;
  }
  *handle = e;
  return 0;
}

int dm_whisper_destroy(void* handle) {
  if (!handle) return 0;
  DM_ON_DEVICE(static_cast<WhisperEngine*>(handle)->device);
  delete static_cast<WhisperEngine*>(handle);
  return 0;
}

int dm_whisper_encode_lengths(void* handle, const int16_t* pcm, const int64_t* offsets,
                              const int32_t* lengths, const int32_t* host_lengths, int n,
                              const int32_t* slot_ids, void* stream) {
  auto* e = static_cast<WhisperEngine*>(handle);
  DM_REQUIRE(e != nullptr, "null handle");
  DM_ON_DEVICE(e->device);
  DM_REQUIRE(n >= 1 && n <= e->E, "n must be in [1, max_encode_batch]");
  for (int i = 0; i < n; ++i)
    DM_REQUIRE(slot_ids[i] >= 0 && slot_ids[i] < e->cfg.max_slots, "slot id out of range");
  int rows = 1500;
  if (host_lengths) {            // length-aware: the longest window of the batch
    rows = 1;
    for (int i = 0; i < n; ++i) {
      const int ns = std::min(std::max(host_lengths[i], 0), 480000);
      rows = std::max(rows, std::min(1500, (ns + 319) / 320));
    }
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (int rc = e->ring.upload(e->slot_dev, slot_ids, sizeof(int32_t) * n, s)) return rc;
  e->last_n = n;
  e->last_rows = rows;
  e->encodes += 1;
  e->segments += n;
  e->launches += e->encode_kernels();
  return encoder_forward(e, pcm, offsets, lengths, n, s, rows, host_lengths != nullptr);
}

int dm_whisper_encode(void* handle, const int16_t* pcm, const int64_t* offsets,
                      const int32_t* lengths, int n, const int32_t* slot_ids, void* stream) {
  return dm_whisper_encode_lengths(handle, pcm, offsets, lengths, nullptr, n, slot_ids, stream);
}

__global__ void admit_kernel(DecodeState st, const int32_t* args, int n) {
  // args: [slot, cap] * n
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int slot = args[2 * i], cap = args[2 * i + 1];
  st.pos[slot] = 0;
  st.cur_tok[slot] = st.prompt[0];
  st.n_gen[slot] = 0;
  st.cap[slot] = cap;
  st.done[slot] = 0;
}

int dm_whisper_admit(void* handle, const int32_t* slot_ids, const int32_t* caps, int n,
                     void* stream) {
  auto* e = static_cast<WhisperEngine*>(handle);
  DM_REQUIRE(e != nullptr, "null handle");
  DM_ON_DEVICE(e->device);
  DM_REQUIRE(n >= 0 && n <= e->cfg.max_slots, "bad n");
  if (n == 0) return 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // allocate pages (host side), then upload table rows + slot resets
  int need = 0;
  for (int i = 0; i < n; ++i) {
    DM_REQUIRE(slot_ids[i] >= 0 && slot_ids[i] < e->cfg.max_slots, "slot id out of range");
    DM_REQUIRE(caps[i] >= 1 && caps[i] <= 448 - e->cfg.prompt_len, "cap out of range");
    DM_REQUIRE(e->slot_pages[slot_ids[i]] == 0, "slot already holds pages (release it first)");
    need += ceil_div(e->cfg.prompt_len + caps[i], 64);
  }
  if (need > int(e->free_pages.size())) {
    set_error("self-KV page pool exhausted");
    return 3;
  }
  std::vector<int32_t> args(size_t(2) * n);
  for (int i = 0; i < n; ++i) {
    const int slot = slot_ids[i];
    const int np = ceil_div(e->cfg.prompt_len + caps[i], 64);
    for (int p = 0; p < 7; ++p) {
      int page = 0;
      if (p < np) {
        page = e->free_pages.back();
        e->free_pages.pop_back();
      }
      e->page_table_host[size_t(slot) * 7 + p] = page;
    }
    e->slot_pages[slot] = np;
    args[2 * i] = slot;
    args[2 * i + 1] = caps[i];
  }
  if (int rc = e->ring.upload(e->page_table_dev, e->page_table_host.data(),
                              sizeof(int32_t) * e->page_table_host.size(), s))
    return rc;
  if (int rc = e->ring.upload(e->admit_args_dev, args.data(), sizeof(int32_t) * 2 * n, s)) return rc;
  admit_kernel<<<ceil_div(n, 64), 64, 0, s>>>(e->st, e->admit_args_dev, n);
  DM_CHECK_LAUNCH();
  e->launches += 1;
  return 0;
}

int dm_whisper_release(void* handle, const int32_t* slot_ids, int n) {
  auto* e = static_cast<WhisperEngine*>(handle);
  DM_REQUIRE(e != nullptr, "null handle");
  DM_ON_DEVICE(e->device);
  for (int i = 0; i < n; ++i) {
    const int slot = slot_ids[i];
    DM_REQUIRE(slot >= 0 && slot < e->cfg.max_slots, "slot id out of range");
    for (int p = 0; p < e->slot_pages[slot]; ++p)
      e->free_pages.push_back(e->page_table_host[size_t(slot) * 7 + p]);
    e->slot_pages[slot] = 0;
  }
  return 0;
}

int dm_whisper_set_prompt(void* handle, const int32_t* tokens, int n, void* stream) {
  auto* e = static_cast<WhisperEngine*>(handle);
  DM_REQUIRE(e != nullptr && tokens != nullptr, "null argument");
  DM_ON_DEVICE(e->device);
  DM_REQUIRE(n >= 1 && n <= kMaxPrompt, "prompt length in [1, 224]");
  for (int s = 0; s < e->cfg.max_slots; ++s)
    DM_REQUIRE(e->slot_pages[s] == 0, "set the prompt while no slot is admitted");
  for (int i = 0; i < n; ++i)
    DM_REQUIRE(tokens[i] >= 0 && tokens[i] < e->cfg.vocab, "prompt token out of the vocabulary");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  DM_CHECK_CUDA(cudaStreamSynchronize(s));
  DM_CHECK_CUDA(cudaMemcpy(e->prompt_dev, tokens, sizeof(int32_t) * n, cudaMemcpyHostToDevice));
  e->cfg.prompt_len = n;
  e->st.prompt_len = n;
  for (auto& g : e->groups) g.st.prompt_len = n;
  e->step_exec = nullptr;              // step graphs bake the prompt length in: re-capture
  return 0;
}

int dm_whisper_set_active(void* handle, const int32_t* slot_ids, int n, void* stream) {
  auto* e = static_cast<WhisperEngine*>(handle);
  DM_REQUIRE(e != nullptr, "null handle");
  DM_ON_DEVICE(e->device);
  DM_REQUIRE(n >= 0 && n <= e->cfg.max_slots, "bad n");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int G = int(e->groups.size());
  // per group: [count, slots...]; uploads are stream-ordered after any step
  // graph already queued, which still sees the previous active list
  std::vector<int32_t> rows(size_t(G) * (kRows + 1), 0);
  for (int i = 0; i < n; ++i) {
    DM_REQUIRE(slot_ids[i] >= 0 && slot_ids[i] < e->cfg.max_slots, "slot id out of range");
    const int g = slot_ids[i] % G;
    int32_t* row = rows.data() + g * (kRows + 1);
    DM_REQUIRE(row[0] < kRows, "too many active slots in one decode group");
    row[1 + row[0]++] = slot_ids[i];
  }
  for (int g = 0; g < G; ++g) {
    int32_t* row = rows.data() + g * (kRows + 1);
    e->groups[g].n_active_host = row[0];
    if (int rc = e->ring.upload(e->groups[g].n_active_dev, row, sizeof(int32_t), s)) return rc;
    if (row[0])
      if (int rc = e->ring.upload(e->groups[g].active_dev, row + 1, sizeof(int32_t) * row[0], s))
        return rc;
  }
  return 0;
}

int dm_whisper_step(void* handle, int n_steps, void* stream) {
  auto* e = static_cast<WhisperEngine*>(handle);
  DM_REQUIRE(e != nullptr, "null handle");
  DM_ON_DEVICE(e->device);
  if (!e->step_exec)
    if (int rc = build_step_graph(e)) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  auto bucket_of = [](const WhisperEngine::Group& grp) {
    int b = 0;
    while (b < kRowBuckets - 1 && kRowBucket[b] < grp.n_active_host) ++b;
    return b;
  };
  if (e->groups.size() == 1) {
    const int b = bucket_of(e->groups[0]);
    for (int i = 0; i < n_steps; ++i) DM_CHECK_CUDA(cudaGraphLaunch(e->groups[0].exec[b], s));
    e->launches += (long long)n_steps * e->groups[0].nodes[b];
  } else {
    DM_CHECK_CUDA(cudaEventRecord(e->step_start, s));
    for (auto& grp : e->groups) {
      DM_CHECK_CUDA(cudaStreamWaitEvent(grp.stream, e->step_start, 0));
      const int b = bucket_of(grp);
      for (int i = 0; i < n_steps; ++i) DM_CHECK_CUDA(cudaGraphLaunch(grp.exec[b], grp.stream));
      e->launches += (long long)n_steps * grp.nodes[b];
      DM_CHECK_CUDA(cudaEventRecord(grp.done, grp.stream));
    }
    for (auto& grp : e->groups) DM_CHECK_CUDA(cudaStreamWaitEvent(s, grp.done, 0));
  }
  e->steps += n_steps;
  return 0;
}

int dm_whisper_stats(void* handle, int64_t* out, int n) {
  auto* e = static_cast<WhisperEngine*>(handle);
  DM_REQUIRE(e != nullptr && out != nullptr && n >= 4, "need 4 outputs");
  DM_ON_DEVICE(e->device);
  out[0] = e->launches; out[1] = e->steps; out[2] = e->encodes; out[3] = e->segments;
  return 0;
}

int dm_whisper_time_kernel(void* handle, int which, int layer, int iters, float* avg_ms,
                           void* stream) {
  auto* e = static_cast<WhisperEngine*>(handle);
  DM_REQUIRE(e != nullptr && avg_ms != nullptr && iters >= 1, "bad arguments");
  DM_ON_DEVICE(e->device);
  // layer < 0: launch i runs decoder layer i % Ld (every launch streams another
  // layer's weights / cross-KV, as inside a step); else every launch runs `layer`
  DM_REQUIRE(layer < e->Ld, "layer out of range");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // capture `iters` back-to-back launches in a graph so the timing sees the
  // GPU-side launch/complete latency, not host submission
  // probes run on decode group 0's state at its current active rows
  WhisperEngine::Group& grp = e->groups[0];
  DecodeState pst = grp.st;    // per-row grids sized like the step graph's bucket
  {
    int b = 0;
    while (b < kRowBuckets - 1 && kRowBucket[b] < grp.n_active_host) ++b;
    pst.grid_rows = kRowBucket[b];
  }
  const int d = e->d;
  auto gv = [&](int idx, float* part, uint16_t* yh, uint16_t* yl, const uint16_t* bias,
                cudaStream_t cs) {
    GemvArgs g = gemv_plan_for_rows(e->plans[idx], pst.grid_rows);
    g.bias = bias; g.part = part; g.yh = yh; g.yl = yl; g.counter_base = e->gemv_counter_base;
    return launch_gemv(pst, grp.maps[idx], g, cs);
  };
  auto launch_one = [&](int layer, cudaStream_t cs) -> int {
    const int b0 = e->dec_layer_base(layer), pi = layer * 6;
    switch (which) {
      case 0: {      // as in the step: split merge in the tail or its own kernel
        const bool tail = pst.grid_rows <= e->xa_tail_merge_rows;
        if (int rc = launch_cross_attn(pst, e->xkv_map, layer,
                                       Partials{grp.p_xq, e->plans[pi + 2].splits, d, e->W(b0 + 9)},
                                       0.125f, grp.xpart, grp.xcnt, cs, 0, tail))
          return rc;
        return tail ? 0 : launch_xattn_merge(pst, grp.xpart, cs);
      }
      case 1:
        return launch_self_attn(pst, layer,
                                Partials{grp.p_qkv, e->plans[pi].splits, 3 * d, e->W(b0 + 3)},
                                0.125f, cs);
      case 2:        // LM head (+ its argmax kernel, as in the step)
        if (e->lm_argmax_epi) return gv(e->Ld * 6, nullptr, nullptr, nullptr, nullptr, cs);
        if (int rc = gv(e->Ld * 6, grp.p_lm, nullptr, nullptr, nullptr, cs)) return rc;
        return launch_lm_argmax(pst, Partials{grp.p_lm, e->plans[e->Ld * 6].splits, e->cfg.vocab, nullptr}, cs);
      case 3: {
        LnArgs la{};
        la.mode = 2; la.g = e->W(b0 + 6); la.b = e->W(b0 + 7);
        la.res = Partials{grp.p_o, e->plans[pi + 1].splits, d, e->W(b0 + 5)};
        return launch_ln(pst, la, cs);
      }
      case 4: return gv(pi + 2, grp.p_xq, nullptr, nullptr, nullptr, cs);
      case 5: return gv(pi + 5, grp.p_fc2, nullptr, nullptr, nullptr, cs);
      case 6: return launch_pdl_floor(cs);
      case 7:
        if (e->fc1_split()) return gv(pi + 4, grp.p_fc1, nullptr, nullptr, nullptr, cs);
        return gv(pi + 4, nullptr, pst.hh, pst.hl, e->W(b0 + 15), cs);
      case 8: return gv(pi + 0, grp.p_qkv, nullptr, nullptr, nullptr, cs);
      case 9:        // the cross-attention reduced to its K/V stream (roofline probe)
        return launch_cross_attn(pst, e->xkv_map, layer,
                                 Partials{grp.p_xq, e->plans[pi + 2].splits, d, e->W(b0 + 9)},
                                 0.125f, grp.xpart, grp.xcnt, cs, 1);
      case 10: return gv(pi + 3, grp.p_xo, nullptr, nullptr, nullptr, cs);
      case 11:       // the cross-attention without its split merge (timing probe)
        return launch_cross_attn(pst, e->xkv_map, layer,
                                 Partials{grp.p_xq, e->plans[pi + 2].splits, d, e->W(b0 + 9)},
                                 0.125f, grp.xpart, grp.xcnt, cs, 2);
      default: set_error("unknown kernel id"); return 1;
    }
  };
  DM_CHECK_CUDA(cudaStreamBeginCapture(e->cap_stream, cudaStreamCaptureModeThreadLocal));
  int rc = 0;
  for (int i = 0; i < iters && rc == 0; ++i)
    rc = launch_one(layer < 0 ? i % e->Ld : layer, e->cap_stream);
  cudaGraph_t g = nullptr;
  cudaError_t ce = cudaStreamEndCapture(e->cap_stream, &g);
  if (rc) {
    if (g) cudaGraphDestroy(g);
    return rc;
  }
  DM_CHECK_CUDA(ce);
  cudaGraphExec_t ge = nullptr;
  DM_CHECK_CUDA(cudaGraphInstantiate(&ge, g, 0));
  DM_CHECK_CUDA(cudaGraphLaunch(ge, s));           // warm-up
  cudaEvent_t a, b;
  DM_CHECK_CUDA(cudaEventCreate(&a));
  DM_CHECK_CUDA(cudaEventCreate(&b));
  DM_CHECK_CUDA(cudaEventRecord(a, s));
  DM_CHECK_CUDA(cudaGraphLaunch(ge, s));
  DM_CHECK_CUDA(cudaEventRecord(b, s));
  DM_CHECK_CUDA(cudaEventSynchronize(b));
  float ms = 0.f;
  DM_CHECK_CUDA(cudaEventElapsedTime(&ms, a, b));
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  *avg_ms = ms / iters;
  e->launches += 2LL * iters;
  return 0;
}

int dm_whisper_read_async(void* handle, int32_t* done, int32_t* n_gen, int32_t* tokens,
                          void* stream) {
  auto* e = static_cast<WhisperEngine*>(handle);
  DM_REQUIRE(e != nullptr, "null handle");
  DM_ON_DEVICE(e->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int S = e->cfg.max_slots;
  if (done) DM_CHECK_CUDA(cudaMemcpyAsync(done, e->st.done, sizeof(int32_t) * S, cudaMemcpyDeviceToHost, s));
  if (n_gen) DM_CHECK_CUDA(cudaMemcpyAsync(n_gen, e->st.n_gen, sizeof(int32_t) * S, cudaMemcpyDeviceToHost, s));
  if (tokens)
    DM_CHECK_CUDA(cudaMemcpyAsync(tokens, e->st.out_tokens, sizeof(int32_t) * S * 448,
                                  cudaMemcpyDeviceToHost, s));
  return 0;
}

int dm_whisper_read(void* handle, int32_t* done, int32_t* n_gen, int32_t* tokens, void* stream) {
  if (int rc = dm_whisper_read_async(handle, done, n_gen, tokens, stream)) return rc;
  DM_CHECK_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
  return 0;
}

int dm_whisper_debug(void* handle, int which, void* host_dst, size_t bytes, void* stream) {
  auto* e = static_cast<WhisperEngine*>(handle);
  DM_REQUIRE(e != nullptr, "null handle");
  DM_ON_DEVICE(e->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const void* src = nullptr;
  size_t avail = 0;
  switch (which) {
    case 0: src = e->enc_out; avail = size_t(e->last_n) * e->last_rows * e->d * 2; break;
    case 1:
      DM_REQUIRE(e->mel_tap, "log-mel tap not enabled (dm_whisper_debug 15 before the encode)");
      src = e->mel; avail = size_t(e->last_n) * e->nm * 3000 * 4;
      break;
    case 15: e->mel_tap = bytes != 0; return 0;
    case 2:
      DM_REQUIRE(e->st.logits_dbg != nullptr, "logits tap not enabled");
      src = e->st.logits_dbg; avail = size_t(kRows) * e->cfg.vocab * 4;
      break;
    case 3: {
      if (!e->st.logits_dbg) {
        if (e->alloc_t(&e->st.logits_dbg, size_t(kRows) * e->cfg.vocab)) return 2;
        e->groups[0].st.logits_dbg = e->st.logits_dbg;    // tap: decode group 0 rows
        if (int rc = build_step_graph(e)) return rc;      // re-capture with the tap
      }
      return 0;
    }
    case 4: e->enc_stop = int(bytes); return 0;
    case 7: e->enc_tap = bytes != 0; return 0;
    case 10: {       // step timeline tap on (graph re-captured with per-kernel globaltimer marks)
      if (!e->groups[0].st.trace) {
        unsigned long long* t = nullptr;
        if (e->alloc_t(&t, kTraceSlots * 8)) return 2;
        e->groups[0].st.trace = t;
        if (int rc = build_step_graph(e)) return rc;
      }
      return 0;
    }
    case 11: {       // reset the timeline (entry/release minima to +inf, maxima to 0)
      DM_REQUIRE(e->groups[0].st.trace != nullptr, "timeline tap not enabled");
      std::vector<unsigned long long> init(kTraceSlots * 8, 0ull);
      for (int k = 0; k < kTraceSlots; ++k) init[k * 8] = init[k * 8 + 1] = ~0ull;
      DM_CHECK_CUDA(cudaMemcpyAsync(e->groups[0].st.trace, init.data(), init.size() * 8,
                                    cudaMemcpyHostToDevice, s));
      DM_CHECK_CUDA(cudaStreamSynchronize(s));
      return 0;
    }
    case 12:
      DM_REQUIRE(e->groups[0].st.trace != nullptr, "timeline tap not enabled");
      src = e->groups[0].st.trace; avail = size_t(kTraceSlots) * 8 * 8;
      break;
    case 13: {       // guard check: host_dst int32[bytes/4] = {n_bad, (index, first bad offset, KB)...}
      DM_REQUIRE(e->guard, "engine created without DM_GUARD=1");
      DM_CHECK_CUDA(cudaStreamSynchronize(s));
      std::vector<uint8_t> g(WhisperEngine::kGuard);
      auto* out = static_cast<int32_t*>(host_dst);
      const int cap = int(bytes / 4);
      int nbad = 0;
      for (size_t i = 0; i < e->allocs.size(); ++i) {
        DM_CHECK_CUDA(cudaMemcpy(g.data(), static_cast<uint8_t*>(e->allocs[i]) + e->alloc_bytes[i],
                                 g.size(), cudaMemcpyDeviceToHost));
        for (size_t k = 0; k < g.size(); ++k)
          if (g[k] != 0xA5) {
            if (3 + 3 * nbad < cap) {
              out[1 + 3 * nbad] = int(i);
              out[2 + 3 * nbad] = int(k);
              out[3 + 3 * nbad] = int(e->alloc_bytes[i] / 1024);
            }
            ++nbad;
            break;
          }
      }
      if (cap > 0) out[0] = nbad;
      return 0;
    }
    case 5: src = e->resid; avail = size_t(e->last_n) * e->last_rows * e->d * 4; break;
    case 6: src = e->attn_out; avail = size_t(e->last_n) * e->last_rows * e->d * 2; break;
    default: DM_REQUIRE(false, "unknown debug tap");
  }
  DM_REQUIRE(bytes <= avail, "debug copy larger than the tapped buffer");
  DM_CHECK_CUDA(cudaMemcpyAsync(host_dst, src, bytes, cudaMemcpyDeviceToHost, s));
  DM_CHECK_CUDA(cudaStreamSynchronize(s));
  return 0;
}

}  // extern "C"
