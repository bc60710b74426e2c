"""The drop-in backend: `B200Backend.transcribe_batch(batch)` satisfies the
reference's SupportsTranscribe contract (pkg/src/dictamux/scheduler.py:212-213)
exactly like SimBackend / RemoteBackend (pkg/src/dictamux/backend.py:148-277),
but runs Listing 1 on the B200:

  pad_or_trim -> log-mel -> Whisper encode -> greedy generate(prompt + no_ts)

Contract points honoured (file:line of the reference):
  * exactly one result per entry, in entry order, ids copied;
  * one `backend_time_ms` for the whole call on every row (test_backend.py:89-99);
  * empty batch / mixed sample rates -> ValueError (backend.py:142-145,163-165);
  * failures raise, and DispatchLoop turns them into per-entry error rows
    (scheduler.py:258-275) — partial results never happen (backend.py:3-4);
  * one batch in flight per device (backend.py:160,167);
  * pure-silence segments transcribe to "" (backend.py:130-135);
  * identical audio -> identical text regardless of batch mates (batch-invariant
    kernels; test_backend.py:118-131, test_server.py:334-342).
"""

from __future__ import annotations

import math
import threading
import time
from dataclasses import dataclass, field

import numpy as np

from .engine import SegmentJob, WhisperGPU
from .models import SAMPLE_RATE, byte_tokens, default_token_cap, get_model
from .types import TranscriptResult

_SYLLABLES = ("ka", "ri", "to", "ve", "na", "su", "mel", "or",
              "da", "pi", "lu", "sha", "en", "gro", "mi", "tan")


def pad_or_trim(samples: np.ndarray, window_s: float, sample_rate_hz: int) -> np.ndarray:
    """Sample-domain pad_or_trim with the reference's semantics
    (backend.py:87-99): truncate or zero-pad at the end to round(window_s*rate)
    samples; the input object itself when it already fits. (The GPU path never
    materialises the padded copy: dm_logmel reads past-the-end samples as 0.)"""
    target = int(round(window_s * sample_rate_hz))
    n = len(samples)
    if n == target:
        return samples
    if n > target:
        return samples[:target]
    out = np.zeros(target, dtype=samples.dtype if n else np.int16)
    out[:n] = samples
    return out


def _render(t: int) -> str:
    syl = [_SYLLABLES[(t >> (4 * k)) & 15] for k in range(4) if (t >> (4 * k)) or k == 0]
    return "".join(syl)


_WORDS: list[str] = []


def detokenize(ids: list[int]) -> str:
    """Deterministic rendering of token ids (no tokenizer files offline, and
    random-init weights make BPE text meaningless): one pseudo-word per id
    (table-driven; ids outside the Whisper vocabularies render on the fly)."""
    global _WORDS
    if not _WORDS:
        _WORDS = [_render(t) for t in range(51866)]
    words = _WORDS
    n = len(words)
    return " ".join(words[t] if 0 <= t < n else _render(int(t)) for t in ids)


def _is_silent(samples: np.ndarray) -> bool:
    """All-zero PCM (the reference's silence rule, backend.py:130-135). Speech
    almost always has a non-zero sample near the start: check a prefix first."""
    if len(samples) == 0:
        return True
    if samples[:256].any():
        return False
    return not samples.any()


@dataclass
class B200BackendConfig:
    model: str = "whisper-base"
    seed: int = 0
    init_std: float = 0.02
    device: int = 0
    max_slots: int = 64
    max_encode_batch: int = 32
    cap_tokens: int | None = None      # fixed greedy cap; None -> per-duration cap
    window_s: float = 30.0
    silence_is_empty: bool = True
    steps_per_poll: int = 8
    overlap_encode: bool = True         # next encode group on a second stream while others decode
    first_encode_batch: int = 8         # first group of an idle engine (longest caps first)
    # previous-text conditioning (the reference's decode_options.prompt,
    # backend.py:181-199): token ids, or a text turned into byte-level ids
    # (no tokenizer files offline); the decoder prompt becomes
    # <|startofprev|> + context + [SOT, lang, task, <|notimestamps|>]
    prompt_tokens: tuple[int, ...] | None = None
    prompt_text: str | None = None
    # opt-in length-aware encoder: skips the 30 s window's
    # zero padding; changes results vs the pad_or_trim contract
    length_aware: bool = False

    def __post_init__(self) -> None:
        get_model(self.model)
        if self.cap_tokens is not None and not 1 <= self.cap_tokens <= 444:
            raise ValueError("cap_tokens must be in [1, 444]")
        if self.window_s != 30.0:
            raise ValueError("Whisper's window is fixed at 30 s (480,000 samples)")


class B200Backend:
    """Batch-synchronous SupportsTranscribe on one B200."""

    def __init__(self, cfg: B200BackendConfig | None = None, engine: WhisperGPU | None = None):
        self.cfg = cfg or B200BackendConfig()
        dims = get_model(self.cfg.model)
        self.engine = engine or WhisperGPU(
            dims, seed=self.cfg.seed, init_std=self.cfg.init_std, device=self.cfg.device,
            max_slots=self.cfg.max_slots, max_encode_batch=self.cfg.max_encode_batch,
            steps_per_poll=self.cfg.steps_per_poll, overlap_encode=self.cfg.overlap_encode,
            first_encode_batch=self.cfg.first_encode_batch, length_aware=self.cfg.length_aware)
        self._device_lock = threading.Lock()
        ctx = list(self.cfg.prompt_tokens or ())
        if self.cfg.prompt_text:
            ctx += byte_tokens(self.cfg.prompt_text)
        if ctx:
            self.engine.set_prompt(dims.prompt_with_context(ctx))
        self._max_cap = 448 - len(getattr(self.engine, "prompt", dims.prompt))

    def cap_for(self, duration_s: float) -> int:
        cap = self.cfg.cap_tokens if self.cfg.cap_tokens is not None else default_token_cap(duration_s)
        return min(cap, self._max_cap)

    def transcribe_batch(self, batch) -> list[TranscriptResult]:
        entries = batch.entries
        if not entries:
            raise ValueError("a batch holds at least one segment")
        rates = {e.segment.sample_rate_hz for e in entries}
        if len(rates) > 1:
            raise ValueError(f"batch mixes sample rates {sorted(rates)}")
        if rates != {SAMPLE_RATE}:
            raise ValueError(f"the Whisper front end needs {SAMPLE_RATE} Hz audio, got {rates}")
        started = time.monotonic()
        texts: dict[int, str] = {}
        jobs = []
        for i, e in enumerate(entries):
            seg = e.segment
            samples = np.asarray(seg.samples)
            if samples.dtype != np.int16:
                samples = samples.astype(np.int16)
            if self.cfg.silence_is_empty and _is_silent(samples):
                texts[i] = ""
                continue
            jobs.append(SegmentJob(i, samples, self.cap_for(seg.duration_s)))
        with self._device_lock:
            try:
                ids = self.engine.run_jobs(jobs) if jobs else {}
            except BaseException:
                # free every slot's pages and drain both streams so the next
                # batch starts clean; the caller turns the raise into per-entry
                # error rows (scheduler.py:258-275, server.py:187-199)
                try:
                    self.engine.reset()
                finally:
                    raise
        for i, toks in ids.items():
            texts[i] = detokenize(toks)
        elapsed_ms = (time.monotonic() - started) * 1000.0
        return [TranscriptResult(segment_id=e.segment.segment_id,
                                 session_id=e.segment.session_id,
                                 text=texts[i], backend_time_ms=elapsed_ms)
                for i, e in enumerate(entries)]

    def close(self) -> None:
        self.engine.close()
