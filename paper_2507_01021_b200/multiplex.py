"""The multiplexer (north-star item 4): continuous-batching GPU consumers on
the reference's own shared segment queue.

The queue and its batching policy are the reference's objects, used as they
are (`pkg/src/dictamux/scheduler.py:36-209`: one priority queue ordered by
(enqueue_time, segment_id), dynamic / continuous triggers, atomic batch
extraction under one lock, drain on shutdown). This module only duck-types
them: `queue.try_form_batch(policy, now)`, `queue.force_batch(policy, now)`,
`queue.wait_for_work(timeout_s)`, `queue.close()`, `queue.closed`, and a
dataclass policy with `kind` / `min_batch` / `max_batch` fields.

`GpuConsumer` is one engine thread per GPU ("one dispatch loop per backend
device"). Unlike the reference's DispatchLoop (scheduler.py:220-285),
which runs one batch at a time and returns all rows together, it does
iteration-level admission: every few decode steps it pulls up to `free slots`
new segments from the shared queue (force_batch with the policy turned
continuous, max_batch = free) into slots freed by EOT / cap, and routes each
segment the moment it finishes. `Multiplexer` starts one consumer per GPU on
one shared queue: pull-based sharding across the GPUs of one box (extraction
is atomic, scheduler.py:119-161), no NCCL, results gathered on the host
through `result_router`.
"""

from __future__ import annotations

import dataclasses
import threading
import time
from typing import Callable

import numpy as np

from .backend import detokenize
from .engine import SegmentJob, WhisperGPU
from .models import default_token_cap
from .types import TranscriptResult

CONTINUOUS = "continuous"


def monotonic_ms() -> float:
    """The reference's clock (scheduler.py:216-217)."""
    return time.monotonic() * 1000.0


class GpuConsumer(threading.Thread):
    """One decode engine per GPU, fed from the shared queue with
    iteration-level admission (continuous batching)."""

    def __init__(self, queue, policy, engine: WhisperGPU,
                 result_router: Callable[[TranscriptResult], None], *,
                 cap_fn: Callable[[float], int] = default_token_cap,
                 silence_is_empty: bool = True, poll_interval_ms: float = 10.0,
                 clock: Callable[[], float] = monotonic_ms, name: str = "gpu-consumer",
                 eager_start: bool = True):
        super().__init__(name=name, daemon=True)
        self.queue, self.policy, self.engine = queue, policy, engine
        # eager_start: an idle engine takes whatever is queued (the policy with
        # min_batch 1) instead of waiting for the policy's batch to form; a
        # running engine admits at every step batch either way (_refill)
        self.eager_start = eager_start
        self._idle_policy = (dataclasses.replace(policy, kind=CONTINUOUS, min_batch=1)
                             if eager_start else policy)
        self.result_router, self.cap_fn = result_router, cap_fn
        self.silence_is_empty = silence_is_empty
        self.poll_interval_ms, self.clock = poll_interval_ms, clock
        self._stop_requested = threading.Event()
        self._inflight: dict[str, tuple[object, float, float]] = {}   # id -> (entry, formed, admitted)
        self.segments_done = 0
        self.audio_s_done = 0.0

    # -- routing -----------------------------------------------------------
    def _route(self, entry, formed_at: float, admitted_at: float, text: str,
               status: str = "ok", message: str = "") -> None:
        seg = entry.segment
        res = TranscriptResult(seg.segment_id, seg.session_id, text,
                               backend_time_ms=self.clock() - admitted_at,
                               queue_wait_ms=formed_at - entry.enqueue_time,
                               status=status, message=message)
        self.segments_done += 1
        self.audio_s_done += seg.duration_s
        self.result_router(res)

    def _jobs_for(self, batch) -> list[SegmentJob]:
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
        pol = dataclasses.replace(self.policy, kind=CONTINUOUS, min_batch=1, max_batch=n_free)
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
        dev = getattr(self.engine, "device", None)
        if dev is not None and getattr(dev, "type", None) == "cuda":
            import torch
            torch.cuda.set_device(dev)       # this thread launches on the engine's GPU
        while not self._stop_requested.is_set() and not self.queue.closed:
            self.queue.wait_for_work(self.poll_interval_ms / 1000.0)
            if self._stop_requested.is_set() or self.queue.closed:
                break
            jobs = self._jobs_for(self.queue.try_form_batch(self._idle_policy, self.clock()))
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
    """One GpuConsumer per GPU on one shared queue (the reference's SegmentQueue;
    no NCCL, host gather)."""

    def __init__(self, engines: list[WhisperGPU], policy, queue,
                 result_router: Callable[[TranscriptResult], None], **kw):
        self.queue = queue
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
