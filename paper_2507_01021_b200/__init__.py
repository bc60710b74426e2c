"""B200-native rebuild of the batched segment-transcription hot path of
arxiv 2507.01021 ("dictamux"): pad_or_trim -> log-mel -> Whisper encode ->
greedy generate(prompt + <|notimestamps|>), behind the reference's own
`transcribe_batch(batch) -> list[TranscriptResult]` / SegmentQueue API.

Compute runs in hand-written sm_100a CUDA (csrc/, C ABI in
include/dictamux_b200.h); the Python here is the host side only.
"""

__version__ = "0.1.0"
