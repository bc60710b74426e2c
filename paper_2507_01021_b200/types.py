"""Data types of the reference's hot-path boundary, mirrored field for field
so this package runs standalone (the GPU box has no /root/reference) and stays
duck-type compatible with the reference's own objects:

  * SpeechSegment    — pkg/src/dictamux/vad.py:90-110 (the atom of multiplexing)
  * QueueEntry/Batch — pkg/src/dictamux/scheduler.py:64-79
  * TranscriptResult — pkg/src/dictamux/backend.py:29-49

B200Backend only reads `batch.entries[i].segment.{segment_id, session_id,
samples, sample_rate_hz, duration_s}` and returns TranscriptResult-shaped
objects, so the reference's Batch/SpeechSegment work unchanged.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class SpeechSegment:
    segment_id: str
    session_id: str
    samples: np.ndarray            # int16 PCM incl. VAD padding
    sample_rate_hz: int
    speech_start: float
    endpoint_time: float
    duration_s: float
    forced_split: bool = False
    final_flush: bool = False
    content_start_index: int = 0
    content_end_index: int = 0


@dataclass
class QueueEntry:
    segment: SpeechSegment
    enqueue_time: float

    @property
    def priority_key(self) -> tuple[float, str]:
        return (self.enqueue_time, self.segment.segment_id)


@dataclass
class Batch:
    batch_id: str
    entries: list[QueueEntry]
    formed_at: float
    total_audio_s: float


@dataclass
class TranscriptResult:
    segment_id: str
    session_id: str
    text: str
    backend_time_ms: float = 0.0
    queue_wait_ms: float = 0.0
    e2e_latency_ms: float = 0.0
    status: str = "ok"
    message: str = ""

    @property
    def is_error(self) -> bool:
        return self.status != "ok"


def make_segment(segment_id: str, samples: np.ndarray, *, session_id: str = "s",
                 rate: int = 16000, endpoint_time: float = 0.0) -> SpeechSegment:
    dur = len(samples) / float(rate)
    return SpeechSegment(segment_id=segment_id, session_id=session_id,
                         samples=np.asarray(samples, dtype=np.int16), sample_rate_hz=rate,
                         speech_start=endpoint_time - dur * 1000.0,
                         endpoint_time=endpoint_time, duration_s=dur)


def batch_of(segments, formed_at: float = 0.0, batch_id: str = "b0") -> Batch:
    entries = [QueueEntry(segment=s, enqueue_time=s.endpoint_time) for s in segments]
    return Batch(batch_id=batch_id, entries=entries, formed_at=formed_at,
                 total_audio_s=sum(s.duration_s for s in segments))
