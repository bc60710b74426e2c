/*
 * dictamux_b200 — C ABI of the B200-native segment-transcription hot path.
 *
 * The reference (arxiv 2507.01021 "dictamux", /root/reference/pkg) reaches
 * its ASR engine only through a Python duck-typed contract and an HTTP wire
 * format; it binds no native library. Each entry point below replaces one
 * step of that path; the Python host side (paper_2507_01021_b200/_native.py)
 * binds them with ctypes and exposes the reference's own
 * `transcribe_batch(batch) -> list[TranscriptResult]` on top.
 *
 *   reference interface (file:line)                              replaced by
 *   -----------------------------------------------------------  -----------------------------
 *   pad_or_trim            pkg/src/dictamux/backend.py:87-99      dm_logmel (fused zero-fill)
 *   feature_extractor      PAPER.md:51                            dm_logmel
 *   model.encode           PAPER.md:56                            dm_whisper_encode
 *   model.model.generate   PAPER.md:57-59 (prompt + no_ts)        dm_whisper_admit / _step / _read
 *   SimBackend/RemoteBackend.transcribe_batch
 *                          pkg/src/dictamux/backend.py:162-178,221-237
 *                                                                 the sequence encode -> step* -> read
 *   "one batch in flight per device" SPEC.md:252, backend.py:160-168
 *                                                                 one dm_whisper handle per GPU
 *
 * Conventions: every function returns 0 on success, 1 on an invalid
 * argument, 2 on a CUDA/driver failure, 3 on resource exhaustion; the
 * message is in dm_last_error() (thread-local). No error is swallowed.
 * Device pointers are plain addresses; `stream` is a cudaStream_t (NULL =
 * legacy default stream). All work is stream-ordered; functions that return
 * host data synchronise the stream first.
 */
#ifndef DICTAMUX_B200_H_
#define DICTAMUX_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define DM_API __attribute__((visibility("default")))
#else
#define DM_API
#endif

#define DM_OK 0
#define DM_ERR_INVALID 1
#define DM_ERR_CUDA 2
#define DM_ERR_RESOURCE 3

DM_API const char* dm_last_error(void);
DM_API int dm_version(void);

/* Seeded weight fill (paper_2507_01021_b200/weights.py documents the rule):
 * dst[i] = bf16(fp32(sum16x4(splitmix64(key + i)) - 131070) * scale + mean). */
DM_API int dm_fill_normal_bf16(uint16_t* dst, uint64_t numel, uint64_t key, float scale, float mean,
                        void* stream);

/* K1: pad_or_trim + log-mel. pcm: concatenated int16 segments (device),
 * offsets[n] (int64, elements) and lengths[n] (int32) on the device. Samples
 * past 480,000 are trimmed, missing ones read as zero (backend.py:87-99).
 * out: [n, n_mels, 3000] fp32 = Whisper input_features. n_mels in {80,128}. */
DM_API int dm_logmel(const int16_t* pcm, const int64_t* offsets, const int32_t* lengths, int n,
              int n_mels, float* out, void* stream);
/* The same features as the encoder consumes them (the engine's product path):
 * out: [n, 3002, ldt] bf16 time-major (ldt = 64 if n_mels <= 64 else 128),
 * rows 1..3000 = bf16((max(x, max_seg - 8) + 4) / 4), bit for bit the
 * rounding of dm_logmel's values; rows 0 and 3001 and channels >= n_mels are
 * not written (the caller zeroes them once). segmax: [n] uint32 scratch. */
DM_API int dm_logmel_operand(const int16_t* pcm, const int64_t* offsets, const int32_t* lengths,
                             int n, int n_mels, uint16_t* out, uint32_t* segmax, void* stream);

/* Test hook for the tcgen05 GEMM: out[M, N] fp32 = A[M, K] . W[N, K]^T (+ bias). */
DM_API int dm_gemm_bf16_f32(const uint16_t* A, const uint16_t* W, const uint16_t* bias, float* out,
                     int M, int N, int K, void* stream);

/* ------------------------------------------------------------ Whisper engine */
typedef struct dm_whisper_config {
  int d_model, enc_layers, dec_layers, heads, ffn, n_mels, vocab;
  int eot;
  int prompt[8];
  int prompt_len;
  int max_slots;          /* concurrent decode slots (<= 64) */
  int max_encode_batch;   /* segments per dm_whisper_encode call */
  int num_pages;          /* self-KV pages of 64 tokens in the pool */
  int decode_groups;      /* independent decode groups (slot s -> group s % G), each with its
                             own step graph and stream; <= 0 means 1 */
  int persistent_decode;  /* reserved, must be 0 */
  int fuse_ln;            /* reserved, must be 0 */
} dm_whisper_config;

/* Weight offsets (elements into the bf16 blob), in this order:
 *  enc.conv1.w, enc.conv1.b, enc.conv2.w, enc.conv2.b, enc.pos,
 *  per encoder layer: ln1.g ln1.b qkv.w qkv.b o.w o.b ln2.g ln2.b fc1.w fc1.b fc2.w fc2.b,
 *  enc.ln.g, enc.ln.b, dec.embed, dec.pos,
 *  per decoder layer: ln1.g ln1.b qkv.w qkv.b o.w o.b ln2.g ln2.b xq.w xq.b xo.w xo.b
 *                     ln3.g ln3.b fc1.w fc1.b fc2.w fc2.b,
 *  dec.xkv.w, dec.xkv.b, dec.ln.g, dec.ln.b
 * (paper_2507_01021_b200/engine.py:whisper_offsets builds it from the manifest). */
DM_API int dm_whisper_create(const dm_whisper_config* cfg, const uint16_t* weights,
                      const int64_t* offsets, int n_offsets, void** handle);
DM_API int dm_whisper_destroy(void* handle);

/* log-mel -> encoder -> cross-KV for n (<= max_encode_batch) segments, written
 * into the decode slots slot_ids[n] (host array). pcm/offsets/lengths as in
 * dm_logmel (device). */
DM_API int dm_whisper_encode(void* handle, const int16_t* pcm, const int64_t* offsets,
                      const int32_t* lengths, int n, const int32_t* slot_ids, void* stream);
/* Length-aware encode (opt-in): as dm_whisper_encode, but
 * each segment's encoder runs on its own window of ceil(n / 320) positions
 * (<= 1500) instead of the 30 s pad_or_trim window: the log-mel frames past
 * the window are the conv's zero padding, attention is masked to the window,
 * and decode cross-attends only to it (fewer FLOPs and cross-KV bytes; the
 * result differs from the padded path). host_lengths: the same lengths as
 * `lengths`, on the host (they size the batch's window). */
DM_API int dm_whisper_encode_lengths(void* handle, const int16_t* pcm, const int64_t* offsets,
                                     const int32_t* lengths, const int32_t* host_lengths, int n,
                                     const int32_t* slot_ids, void* stream);
/* Reset n slots for a new segment: greedy cap per slot (tokens, <= 444);
 * allocates the slot's self-KV pages. Returns DM_ERR_RESOURCE if the page
 * pool is exhausted. */
DM_API int dm_whisper_admit(void* handle, const int32_t* slot_ids, const int32_t* caps, int n,
                     void* stream);
/* Free the pages of n slots (after their result was read). */
DM_API int dm_whisper_release(void* handle, const int32_t* slot_ids, int n);
/* The decoder prompt of later admissions (Listing 1's `prompt_tokens +
 * [no_timestamps]`; the reference carries it as
 * decode_options.prompt, backend.py:181-199): n <= 224 token ids, e.g.
 * [<|startofprev|>, previous-text ids..., <|sot|>, lang, task, <|notimestamps|>].
 * Only while no slot is admitted; the step graphs are re-captured. */
DM_API int dm_whisper_set_prompt(void* handle, const int32_t* tokens, int n, void* stream);
/* Decode slots set: slots[0..n) take part in subsequent steps. */
DM_API int dm_whisper_set_active(void* handle, const int32_t* slot_ids, int n, void* stream);
/* Run n_steps greedy decode steps for the active slots (CUDA graph). */
DM_API int dm_whisper_step(void* handle, int n_steps, void* stream);
/* Copy per-slot state to host: done[max_slots], n_gen[max_slots] and (if
 * tokens != NULL) tokens[max_slots * 448]. Synchronises the stream. */
DM_API int dm_whisper_read(void* handle, int32_t* done, int32_t* n_gen, int32_t* tokens, void* stream);
/* Same copies, stream-ordered and without synchronising (destinations should
 * be pinned host memory; the caller waits on an event it records after). */
DM_API int dm_whisper_read_async(void* handle, int32_t* done, int32_t* n_gen, int32_t* tokens,
                                 void* stream);
/* Debug/parity taps (synchronous copies to host):
 *  which = 0: encoder output of the last encode, [n, 1500, d] bf16 bits
 *  which = 1: log-mel of the last encode, [n, n_mels, 3000] fp32
 *  which = 2: logits of the last step, [64 rows of decode group 0, vocab] fp32 (enable first)
 *  which = 3: enable the logits tap (bytes ignored)
 *  which = 4: run only the first `bytes` encoder layers in later encodes
 *  which = 5: fp32 residual stream before the final LN, [n, 1500, d]
 *  which = 6: attention output of the last encoder layer run, [n, 1500, d] bf16
 *  which = 7: (bytes != 0) keep the fp32 encoder output; read it with which = 5
 *  which = 15: (bytes != 0) also write the fp32 features of later encodes (read with which = 1)
 */
DM_API int dm_whisper_debug(void* handle, int which, void* host_dst, size_t bytes, void* stream);

/* ------------------------------------------------------------ CTC engine (cfg5)
 * wav2vec2-base-shaped encoder-only CTC ("CTC models"; the
 * reference's segment-independence contract SPEC.md:13,103,515).
 * Weight offsets, in order: fe.conv0..6.w, fe.gn.g, fe.gn.b, fp.ln.g, fp.ln.b,
 * fp.proj.w, fp.proj.b, pos.w, pos.b, enc.ln.g, enc.ln.b, per layer
 * (qkv.w qkv.b o.w o.b ln1.g ln1.b fc1.w fc1.b fc2.w fc2.b ln2.g ln2.b), head.w, head.b. */
typedef struct dm_ctc_config {
  int hidden, layers, heads, ffn, vocab;
  int max_batch;          /* segments per dm_ctc_transcribe call */
  int max_samples;        /* longest segment (16 kHz samples) */
} dm_ctc_config;

DM_API int dm_ctc_create(const dm_ctc_config* cfg, const uint16_t* weights, const int64_t* offsets,
                         int n_offsets, void** handle);
DM_API int dm_ctc_destroy(void* handle);
/* Greedy CTC for n segments: pcm on the device, offsets/lengths on the HOST
 * (frame bookkeeping is host-side). Results stay on the device until read. */
DM_API int dm_ctc_transcribe(void* handle, const int16_t* pcm, const int64_t* offsets,
                             const int32_t* lengths, int n, void* stream);
/* tokens: [n, rows_per_segment] collapsed ids (first counts[i] valid per row). */
DM_API int dm_ctc_read(void* handle, int32_t* tokens, int32_t* counts, int32_t* rows_per_segment,
                       void* stream);
/* which = 0: per-frame argmax ids [n * rows] int32; 1: final hidden [n * rows, 768] fp32 */
DM_API int dm_ctc_debug(void* handle, int which, void* host_dst, size_t bytes, void* stream);

/* Telemetry: out[0..3] = kernels launched, decode steps, encode calls, segments. */
DM_API int dm_whisper_stats(void* handle, int64_t* out, int n);
/* Time one decode kernel over the current active slots with CUDA events on
 * `stream` (a probe: it may overwrite row-space activations): which =
 * 0 cross-attention(layer) (+ its split-merge kernel above kXaTailMergeRows
 * rows, as in the step), 1 self-attention(layer), 2 LM head, 3 decoder LN
 * (+ residual partials), 4 cross-q projection, 5 fc2 projection,
 * 6 empty PDL kernel (launch floor), 7 fc1 projection (+GELU), 8 qkv projection,
 * 9 the cross-attention's K/V stream alone (roofline probe), 10 cross-o projection,
 * 11 the cross-attention without its split merge (timing probe).
 * avg_ms = mean over iters back-to-back launches. layer < 0: launch i runs
 * decoder layer i % dec_layers (each launch streams a different layer's
 * cross-KV / weights, as inside a decode step). */
DM_API int dm_whisper_time_kernel(void* handle, int which, int layer, int iters, float* avg_ms,
                                  void* stream);

/* Batched VAD front: the reference's classify_frame
 * (pkg/src/dictamux/vad.py:123-133) for n_frames frames of any sessions:
 * out[f] = 1 (SPEECH) iff mean(pcm[offsets[f] .. + lengths[f]]^2) >=
 * threshold_rms_sq, with the mean exact (int64 sum, one double division), so
 * labels are bit-identical to the reference's float64 numpy. Device pointers. */
DM_API int dm_vad_classify(const int16_t* pcm, const int64_t* offsets, const int32_t* lengths,
                           int n_frames, double threshold_rms_sq, uint8_t* out, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* DICTAMUX_B200_H_ */
