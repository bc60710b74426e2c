"""The multiplexer (north-star item 4) and an API-compatible segment queue.

`SegmentQueue` / `BatchingPolicy` / `DispatchLoop` keep the reference's
semantics and method names (pkg/src/dictamux/scheduler.py:36-285: a single
priority queue ordered by (enqueue_time, segment_id), dynamic / continuous
triggers, atomic batch extraction, drain on shutdown) so the package runs
standalone; the reference's own SegmentQueue works with `GpuConsumer` too
(duck-typed: try_form_batch / force_batch / wait_for_work / closed).

`GpuConsumer` is one engine thread per GPU ("one dispatch loop per backend
device"). Unlike DispatchLoop, which runs one batch at a time and
returns all rows together, it does iteration-level admission: every few decode
steps it pulls up to `free slots` new segments from the shared queue
(force_batch with a continuous policy, max_batch = free) into slots freed by
EOT / cap, and routes each segment the moment it finishes. `Multiplexer` starts
one consumer per GPU on one shared queue: pull-based sharding across the GPUs of
one box, no NCCL, results gathered on the host through `result_router`.
"""

from __future__ import annotations

import heapq
import threading
import time
from dataclasses import dataclass
from typing import Callable, Protocol

import numpy as np

from .backend import detokenize
from .engine import SegmentJob, WhisperGPU
from .models import default_token_cap
from .types import Batch, QueueEntry, TranscriptResult

DYNAMIC = "dynamic"
CONTINUOUS = "continuous"


class DuplicateSegmentError(Exception):
    pass


class QueueClosedError(Exception):
    pass


@dataclass
class BatchingPolicy:
    kind: str = DYNAMIC
    max_batch: int = 8
    max_wait_ms: float = 200.0
    target_audio_s: float = 120.0
    min_batch: int = 2
    starvation_flush_ms: float = 1000.0

    def __post_init__(self) -> None:
        if self.kind not in (DYNAMIC, CONTINUOUS):
            raise ValueError(f"unknown policy kind {self.kind!r}")
        if self.max_batch < 1:
            raise ValueError("max_batch must be >= 1")
        if self.kind == DYNAMIC and self.max_wait_ms <= 0:
            raise ValueError("max_wait_ms must be positive")
        if self.kind == CONTINUOUS and not 1 <= self.min_batch <= self.max_batch:
            raise ValueError("need 1 <= min_batch <= max_batch")

    def fires(self, depth: int, oldest_wait_ms: float, queued_audio_s: float) -> bool:
        if self.kind == DYNAMIC:
            return (oldest_wait_ms >= self.max_wait_ms or queued_audio_s >= self.target_audio_s
                    or depth >= self.max_batch)
        return depth >= self.min_batch or oldest_wait_ms >= self.starvation_flush_ms


def monotonic_ms() -> float:
    return time.monotonic() * 1000.0


class SegmentQueue:
    """Thread-safe arrival-ordered queue; extraction of a batch is atomic and
    safe with several consumers."""

    def __init__(self) -> None:
        self._cv = threading.Condition()
        self._heap: list[tuple[float, str, QueueEntry]] = []
        self._ids: set[str] = set()
        self._audio_s = 0.0
        self._closed = False
        self._seq = 0

    def enqueue_segment(self, segment, now: float) -> None:
        with self._cv:
            if self._closed:
                raise QueueClosedError("queue is shut down")
            if segment.segment_id in self._ids:
                raise DuplicateSegmentError(segment.segment_id)
            self._ids.add(segment.segment_id)
            heapq.heappush(self._heap, (now, segment.segment_id, QueueEntry(segment, now)))
            self._audio_s += segment.duration_s
            self._cv.notify_all()

    def try_form_batch(self, policy: BatchingPolicy, now: float) -> Batch | None:
        with self._cv:
            if not self._heap:
                return None
            if not policy.fires(len(self._heap), now - self._heap[0][0], self._audio_s):
                return None
            return self._take(policy, now)

    def force_batch(self, policy: BatchingPolicy, now: float) -> Batch | None:
        with self._cv:
            return self._take(policy, now) if self._heap else None

    def _take(self, policy: BatchingPolicy, now: float) -> Batch:
        first = heapq.heappop(self._heap)[2]
        entries, audio = [first], first.segment.duration_s
        while self._heap and len(entries) < policy.max_batch:
            nxt = self._heap[0][2]
            if policy.kind == DYNAMIC and audio + nxt.segment.duration_s > policy.target_audio_s:
                break
            heapq.heappop(self._heap)
            entries.append(nxt)
            audio += nxt.segment.duration_s
        self._audio_s -= audio
        b = Batch(batch_id=f"b{self._seq:08d}", entries=entries, formed_at=now,
                  total_audio_s=audio)
        self._seq += 1
        return b

    def wait_for_work(self, timeout_s: float) -> None:
        with self._cv:
            if not self._closed:
                self._cv.wait(timeout=timeout_s)

    def close(self) -> None:
        with self._cv:
            self._closed = True
            self._cv.notify_all()

    @property
    def closed(self) -> bool:
        with self._cv:
            return self._closed

    def __len__(self) -> int:
        with self._cv:
            return len(self._heap)


class SupportsTranscribe(Protocol):
    def transcribe_batch(self, batch: Batch) -> list[TranscriptResult]: ...


class DispatchLoop(threading.Thread):
    """Batch-at-a-time single-device dispatch with the reference's contract
    (scheduler.py:220-285): backend errors become per-entry error rows, every
    row is tagged with queue_wait_ms, and shutdown drains the queue."""

    def __init__(self, queue: SegmentQueue, policy: BatchingPolicy, backend: SupportsTranscribe,
                 result_router: Callable[[TranscriptResult], None], *,
                 poll_interval_ms: float = 10.0, clock: Callable[[], float] = monotonic_ms):
        super().__init__(name="dispatch-loop", daemon=True)
        self.queue, self.policy, self.backend = queue, policy, backend
        self.result_router, self.poll_interval_ms, self.clock = result_router, poll_interval_ms, clock
        self._stop_requested = threading.Event()
        self.batches_dispatched = 0

    def run(self) -> None:
        while not self._stop_requested.is_set() and not self.queue.closed:
            self.queue.wait_for_work(self.poll_interval_ms / 1000.0)
            if self._stop_requested.is_set() or self.queue.closed:
                break
            batch = self.queue.try_form_batch(self.policy, self.clock())
            if batch is not None:
                self._dispatch(batch)
        while (batch := self.queue.force_batch(self.policy, self.clock())) is not None:
            self._dispatch(batch)

    def _dispatch(self, batch: Batch) -> None:
        self.batches_dispatched += 1
        try:
            results = self.backend.transcribe_batch(batch)
            if len(results) != len(batch.entries):
                raise RuntimeError(f"backend returned {len(results)} results for "
                                   f"{len(batch.entries)} entries")
        except Exception as exc:
            results = [TranscriptResult(e.segment.segment_id, e.segment.session_id, "",
                                        status="error", message=str(exc))
                       for e in batch.entries]
        for entry, res in zip(batch.entries, results):
            res.queue_wait_ms = batch.formed_at - entry.enqueue_time
            self.result_router(res)

    def shutdown(self, timeout: float = 30.0) -> None:
        self.queue.close()
        self._stop_requested.set()
        self.join(timeout=timeout)


class GpuConsumer(threading.Thread):
    """One decode engine per GPU, fed from the shared queue with
    iteration-level admission (continuous batching)."""

    def __init__(self, queue, policy: BatchingPolicy, engine: WhisperGPU,
                 result_router: Callable[[TranscriptResult], None], *,
                 cap_fn: Callable[[float], int] = default_token_cap,
                 silence_is_empty: bool = True, poll_interval_ms: float = 10.0,
                 clock: Callable[[], float] = monotonic_ms, name: str = "gpu-consumer"):
        super().__init__(name=name, daemon=True)
        self.queue, self.policy, self.engine = queue, policy, engine
        self.result_router, self.cap_fn = result_router, cap_fn
        self.silence_is_empty = silence_is_empty
        self.poll_interval_ms, self.clock = poll_interval_ms, clock
        self._stop_requested = threading.Event()
        self._inflight: dict[str, tuple[QueueEntry, float, float]] = {}
        self.segments_done = 0
        self.audio_s_done = 0.0

    # -- routing -----------------------------------------------------------
    def _route(self, entry: QueueEntry, formed_at: float, admitted_at: float, text: str,
               status: str = "ok", message: str = "") -> None:
        seg = entry.segment
        res = TranscriptResult(seg.segment_id, seg.session_id, text,
                               backend_time_ms=self.clock() - admitted_at,
                               queue_wait_ms=formed_at - entry.enqueue_time,
                               status=status, message=message)
        self.segments_done += 1
        self.audio_s_done += seg.duration_s
        self.result_router(res)

    def _jobs_for(self, batch: Batch | None) -> list[SegmentJob]:
        if batch is None:
            return []
        jobs = []
        now = self.clock()
        for e in batch.entries:
            seg = e.segment
            samples = np.asarray(seg.samples)
            if seg.sample_rate_hz != 16000:
                self._route(e, batch.formed_at, now, "", "error",
                            f"the Whisper front end needs 16000 Hz audio, got {seg.sample_rate_hz}")
                continue
            if self.silence_is_empty and (len(samples) == 0 or not samples.any()):
                self._route(e, batch.formed_at, now, "")
                continue
            self._inflight[seg.segment_id] = (e, batch.formed_at, now)
            jobs.append(SegmentJob(seg.segment_id, samples.astype(np.int16, copy=False),
                                   self.cap_fn(seg.duration_s), self._on_done))
        return jobs

    def _on_done(self, key, ids) -> None:
        entry, formed, admitted = self._inflight.pop(key)
        self._route(entry, formed, admitted, detokenize(ids))

    def _refill(self, n_free: int) -> list[SegmentJob]:
        if n_free <= 0:
            return []
        pol = BatchingPolicy(kind=CONTINUOUS, min_batch=1, max_batch=n_free)
        return self._jobs_for(self.queue.force_batch(pol, self.clock()))

    def _serve(self, jobs: list[SegmentJob]) -> None:
        try:
            self.engine.run_jobs(jobs, refill=self._refill)
        except Exception as exc:          # fail every in-flight entry, keep serving
            for key in list(self._inflight):
                entry, formed, admitted = self._inflight.pop(key)
                self._route(entry, formed, admitted, "", "error", str(exc))
            self.engine.reset()

    def run(self) -> None:
        while not self._stop_requested.is_set() and not self.queue.closed:
            self.queue.wait_for_work(self.poll_interval_ms / 1000.0)
            if self._stop_requested.is_set() or self.queue.closed:
                break
            jobs = self._jobs_for(self.queue.try_form_batch(self.policy, self.clock()))
            if jobs:
                self._serve(jobs)
        while True:   # drain: every accepted segment is routed exactly once
            batch = self.queue.force_batch(self.policy, self.clock())
            if batch is None:
                break
            jobs = self._jobs_for(batch)
            if jobs:
                self._serve(jobs)

    def shutdown(self, timeout: float = 60.0) -> None:
        self.queue.close()
        self._stop_requested.set()
        self.join(timeout=timeout)


class Multiplexer:
    """One GpuConsumer per GPU on a shared SegmentQueue (no NCCL; host gather)."""

    def __init__(self, engines: list[WhisperGPU], policy: BatchingPolicy,
                 result_router: Callable[[TranscriptResult], None], queue=None, **kw):
        self.queue = queue if queue is not None else SegmentQueue()
        self.consumers = [GpuConsumer(self.queue, policy, eng, result_router,
                                      name=f"gpu-consumer-{i}", **kw)
                          for i, eng in enumerate(engines)]

    def start(self) -> None:
        for c in self.consumers:
            c.start()

    def shutdown(self, timeout: float = 120.0) -> None:
        self.queue.close()
        for c in self.consumers:
            c._stop_requested.set()
        for c in self.consumers:
            c.join(timeout=timeout)
