"""CPU oracle for the segment-transcription hot path — TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import anything under `oracle/`, and only as the
checker or the timed CPU baseline, never as the product path.

What it restates (the reference ships no ASR arithmetic):
  * `pad_or_trim` in the sample domain      — pkg/src/dictamux/backend.py:87-99
  * feature_extractor (log-mel)             — PAPER.md:51; restated from
    transformers 5.5.0 `models/whisper/feature_extraction_whisper.py:95-164`
    and `audio_utils.py:263-375,453-545` (third-party, pinned 5.5.0)
  * model.encode                            — PAPER.md:56; restated from
    `models/whisper/modeling_whisper.py:55-64,241-414,541-648`
  * model.model.generate(prompt+no_ts)      — PAPER.md:57-59; a hand-written
    greedy loop over `modeling_whisper.py:417-506,650-797,964-1081`
  * wav2vec2 CTC (cfg5)                     — `models/wav2vec2/modeling_wav2vec2.py`

Pinning: faster-whisper / CTranslate2 (the paper's library, unpinned — the
reference's pyproject.toml:10-16 does not list it) are absent and offline.
The oracle is pinned against transformers 5.5.0's own WhisperFeatureExtractor
and WhisperModel run on the same bf16-rounded weights (tests/test_oracle_vs_hf.py
when transformers imports; committed fixtures under tests/golden/ made by
scripts/make_golden.py otherwise). The reference's own tests pin only the
boundary (pad_or_trim, result order/shape, silence -> "", identical audio ->
identical text), mirrored in tests/test_backend_contract.py.
"""
