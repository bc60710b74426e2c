"""Batched GPU VAD front.

The reference segments every session serially: `ingest_frame`
(`pkg/src/dictamux/vad.py:383-438`) labels each 30 ms frame with
`classify_frame` (`vad.py:123-133`: float64 mean of the squared samples
against the squared RMS threshold) and advances that session's state
machine. `GpuFrameClassifier.classify` labels the frames of any number of
sessions in one `dm_vad_classify` launch (bit-identical labels: the sum of
squares is exact), and `ingest_frames` then drives the reference's own
state machines with those labels, so the segments are exactly the
reference's. Worth it only when thousands of sessions stream at once.
"""

from __future__ import annotations

import contextlib
import ctypes as C
from typing import Sequence

import numpy as np
import torch

from . import _native

FULL_SCALE = 32768.0   # dBFS reference for signed 16-bit PCM (vad.py:22)


def threshold_sq(energy_threshold_db: float) -> float:
    """Squared linear RMS threshold, computed like VadConfig.energy_threshold_rms."""
    t = FULL_SCALE * 10.0 ** (energy_threshold_db / 20.0)
    return t * t


class GpuFrameClassifier:
    """One device (default cuda:0); buffers grow on demand."""

    def __init__(self, device: int = 0):
        if not torch.cuda.is_available():
            raise _native.DmError("no CUDA device: the GPU VAD front has no CPU fallback")
        self.device = torch.device("cuda", device)
        self.lib = _native.load()
        self.stream = torch.cuda.Stream(self.device)
        self._cap_samples = 0
        self._cap_frames = 0

    def _ensure(self, samples: int, frames: int) -> None:
        if samples > self._cap_samples:
            self._cap_samples = max(samples, 2 * self._cap_samples, 1 << 16)
            self._pcm_h = torch.empty(self._cap_samples, dtype=torch.int16, pin_memory=True)
            self._pcm_d = torch.empty(self._cap_samples, dtype=torch.int16, device=self.device)
        if frames > self._cap_frames:
            self._cap_frames = max(frames, 2 * self._cap_frames, 1024)
            n = self._cap_frames
            self._meta_h = torch.empty(3 * n, dtype=torch.int64, pin_memory=True)
            self._meta_d = torch.empty(3 * n, dtype=torch.int64, device=self.device)
            self._out_d = torch.empty(n, dtype=torch.uint8, device=self.device)
            self._out_h = torch.empty(n, dtype=torch.uint8, pin_memory=True)

    def classify(self, frames: Sequence[np.ndarray], energy_threshold_db: float) -> np.ndarray:
        """uint8 labels (1 = SPEECH) of `frames` (int16 arrays, non-empty)."""
        n = len(frames)
        if n == 0:
            return np.zeros(0, np.uint8)
        lens = [len(f) for f in frames]
        if min(lens) == 0:
            raise ValueError("cannot classify an empty frame")
        total = int(sum(lens))
        self._ensure(total, n)
        flat = self._pcm_h.numpy()[:total]
        offs = np.zeros(n, np.int64)
        pos = 0
        for i, f in enumerate(frames):
            flat[pos:pos + lens[i]] = np.asarray(f, dtype=np.int16)
            offs[i] = pos
            pos += lens[i]
        meta = self._meta_h.numpy()
        meta[:n] = offs
        meta[n:].view(np.int32)[:n] = lens
        with torch.cuda.stream(self.stream):
            self._pcm_d[:total].copy_(self._pcm_h[:total], non_blocking=True)
            self._meta_d[:2 * n].copy_(self._meta_h[:2 * n], non_blocking=True)
            md = self._meta_d.data_ptr()
            _native.check(self.lib.dm_vad_classify(
                C.c_void_p(self._pcm_d.data_ptr()), C.c_void_p(md), C.c_void_p(md + 8 * n), n,
                threshold_sq(energy_threshold_db), C.c_void_p(self._out_d.data_ptr()),
                C.c_void_p(self.stream.cuda_stream)))
            self._out_h[:n].copy_(self._out_d[:n], non_blocking=True)
        self.stream.synchronize()
        return self._out_h.numpy()[:n].copy()


@contextlib.contextmanager
def _labels_for(vad_module, labels: dict[int, bool]):
    """Within the block the reference module's classify_frame returns the
    precomputed label of each frame object (by identity)."""
    original = vad_module.classify_frame
    speech, silence = vad_module.FrameClass.SPEECH, vad_module.FrameClass.SILENCE

    def classify(cfg, frame):
        return speech if labels[id(frame)] else silence
    vad_module.classify_frame = classify
    try:
        yield
    finally:
        vad_module.classify_frame = original


def ingest_frames(vad_module, classifier: GpuFrameClassifier, cfg,
                  work: Sequence[tuple[object, object]]) -> list[list]:
    """Advance many sessions by one frame each (or several frames per session,
    in order): `work` is [(state, frame)]; returns the segments each call to
    the reference's `ingest_frame` finalized, in `work` order. The frames'
    labels come from one GPU launch; the state machine is the reference's.
    (The reference module's classify_frame is rebound for the duration of
    the call: drive a module from one thread at a time.)"""
    frames = [f for _, f in work]
    lab = classifier.classify([f.samples for f in frames], cfg.energy_threshold_db)
    labels = {id(f): bool(v) for f, v in zip(frames, lab)}
    out = []
    with _labels_for(vad_module, labels):
        for state, frame in work:
            out.append(vad_module.ingest_frame(state, cfg, frame))
    return out
