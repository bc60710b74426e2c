// Batched GPU VAD front: the reference's per-frame energy
// classifier `classify_frame` (pkg/src/dictamux/vad.py:123-133) for the frames
// of many sessions in one launch.
//
// The reference computes mean_sq = float64 mean of the squared int16 samples
// and labels the frame SPEECH iff mean_sq >= threshold_rms^2. The sum of
// squares of <= 2^22 int16 samples is an integer below 2^53, so numpy's
// float64 sum is exact in any order; here it is an exact int64 sum, divided
// by the sample count in double (one correctly rounded division, as numpy's
// mean), compared with the same double threshold: bit-identical labels.
//
// One warp per frame; lanes stride over the samples (64-byte coalesced
// reads per warp iteration), xor-tree reduction of the int64 partials.

#include "../../include/dictamux_b200.h"
#include "common.cuh"

namespace dm {

__global__ void __launch_bounds__(256)
vad_classify_kernel(const int16_t* __restrict__ pcm, const int64_t* __restrict__ offsets,
                    const int32_t* __restrict__ lengths, int n_frames, double thr_sq,
                    uint8_t* __restrict__ out) {
  const int f = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (f >= n_frames) return;
  const int16_t* x = pcm + offsets[f];
  const int n = lengths[f];
  long long s = 0;
  for (int i = lane; i < n; i += 32) {
    const long long v = x[i];
    s += v * v;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) out[f] = (double(s) / double(n)) >= thr_sq ? 1 : 0;
}

}  // namespace dm

extern "C" {

int dm_vad_classify(const int16_t* pcm, const int64_t* offsets, const int32_t* lengths,
                    int n_frames, double threshold_rms_sq, uint8_t* out, void* stream) {
  DM_REQUIRE(n_frames >= 0, "n_frames < 0");
  if (n_frames == 0) return 0;
  DM_REQUIRE(pcm && offsets && lengths && out, "null pointer");
  const int per_block = 8;
  dm::vad_classify_kernel<<<dm::ceil_div(n_frames, per_block), 32 * per_block, 0,
                            static_cast<cudaStream_t>(stream)>>>(pcm, offsets, lengths, n_frames,
                                                                  threshold_rms_sq, out);
  DM_CHECK_LAUNCH();
  return 0;
}

}  // extern "C"
