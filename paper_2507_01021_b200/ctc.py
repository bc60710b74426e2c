"""CTC encoder-only path (BASELINE.json cfg5): host side of the wav2vec2-base
engine (csrc/ctc.cu) and a drop-in `CTCBackend.transcribe_batch` with the same
contract as B200Backend / the reference's backends (backend.py:3-4,148-277).

CTC segments are independent ("segment-independence
contract"); one engine per GPU; variable-length segments are batched without
changing any segment's result (per-segment masked reductions)."""

from __future__ import annotations

import ctypes as C
import threading
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from .engine import materialize_weights
from .models import SAMPLE_RATE, WAV2VEC2_BASE, Wav2Vec2Dims
from .types import TranscriptResult
from .weights import Manifest, wav2vec2_manifest

# facebook/wav2vec2-base-960h character vocabulary (blank = <pad> = 0, "|" = space)
CTC_VOCAB = ("<pad>", "<s>", "</s>", "<unk>", "|", "E", "T", "A", "O", "N", "I", "H", "S", "R",
             "D", "L", "U", "M", "W", "C", "F", "G", "Y", "P", "B", "V", "K", "'", "X", "J",
             "Q", "Z")


def ctc_offsets(man: Manifest, dims: Wav2Vec2Dims) -> list[int]:
    names = [f"fe.conv{i}.w" for i in range(len(dims.conv_dim))]
    names += ["fe.gn.g", "fe.gn.b", "fp.ln.g", "fp.ln.b", "fp.proj.w", "fp.proj.b",
              "pos.w", "pos.b", "enc.ln.g", "enc.ln.b"]
    for i in range(dims.layers):
        names += [f"l{i}.{s}" for s in ("qkv.w", "qkv.b", "o.w", "o.b", "ln1.g", "ln1.b",
                                        "fc1.w", "fc1.b", "fc2.w", "fc2.b", "ln2.g", "ln2.b")]
    names += ["head.w", "head.b"]
    return [man[n].offset for n in names]


def ctc_text(ids) -> str:
    chars = []
    for t in ids:
        s = CTC_VOCAB[int(t)] if 0 <= int(t) < len(CTC_VOCAB) else "?"
        if s in ("<pad>", "<s>", "</s>"):
            continue
        chars.append(" " if s == "|" else ("?" if s == "<unk>" else s))
    return "".join(chars).strip()


class Wav2Vec2GPU:
    def __init__(self, dims: Wav2Vec2Dims = WAV2VEC2_BASE, *, seed: int = 0,
                 init_std: float = 0.02, device: int = 0, max_batch: int = 32,
                 max_samples: int = 16000 * 30):
        if not torch.cuda.is_available():
            raise _native.DmError("no CUDA device: the B200 engine has no CPU fallback")
        self.dims = dims
        self.device = torch.device("cuda", device)
        self.lib = _native.load()
        self.max_batch, self.max_samples = max_batch, max_samples
        with torch.cuda.device(self.device):
            self.stream = torch.cuda.Stream(self.device)
            self.man = wav2vec2_manifest(dims, seed, init_std)
            self.blob = materialize_weights(self.man, self.device, self.stream)
            offs = ctc_offsets(self.man, dims)
            cfg = _native.CtcConfigC(dims.hidden, dims.layers, dims.heads, dims.ffn, dims.vocab,
                                     max_batch, max_samples)
            h = C.c_void_p()
            _native.check(self.lib.dm_ctc_create(C.byref(cfg), C.c_void_p(self.blob.data_ptr()),
                                                 (C.c_int64 * len(offs))(*offs), len(offs),
                                                 C.byref(h)))
            self.handle = h
            self._pcm_host = torch.empty(max_batch * max_samples, dtype=torch.int16, pin_memory=True)
            self._pcm_dev = torch.empty(max_batch * max_samples, dtype=torch.int16, device=self.device)
        self.h2d_bytes = 0
        self.d2h_bytes = 0

    def close(self):
        if getattr(self, "handle", None):
            _native.check(self.lib.dm_ctc_destroy(self.handle))
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def _s(self):
        return C.c_void_p(self.stream.cuda_stream)

    def run(self, segs, resident: tuple[torch.Tensor, list[int]] | None = None) -> None:
        """Launch the CTC forward for one batch (<= max_batch segments)."""
        n = len(segs)
        if resident is not None:
            pcm, offs = resident
            lens = [len(s) for s in segs]
            base = pcm.data_ptr()
        else:
            host = self._pcm_host.numpy()
            offs, lens, pos = [], [], 0
            for s in segs:
                s = np.asarray(s, dtype=np.int16)
                if len(s) > self.max_samples:
                    raise ValueError(f"segment of {len(s)} samples exceeds max_samples")
                host[pos:pos + len(s)] = s
                offs.append(pos)
                lens.append(len(s))
                pos += len(s)
            with torch.cuda.stream(self.stream):
                if pos:
                    self._pcm_dev[:pos].copy_(self._pcm_host[:pos], non_blocking=True)
            self.h2d_bytes += 2 * pos
            base = self._pcm_dev.data_ptr()
        _native.check(self.lib.dm_ctc_transcribe(self.handle, C.c_void_p(base),
                                                 (C.c_int64 * n)(*offs), (C.c_int32 * n)(*lens),
                                                 n, self._s))

    def read(self, n: int) -> list[list[int]]:
        rows = C.c_int32()
        _native.check(self.lib.dm_ctc_read(self.handle, None, None, C.byref(rows), self._s))
        toks = np.empty(n * rows.value, np.int32)
        cnt = np.empty(n, np.int32)
        _native.check(self.lib.dm_ctc_read(self.handle, toks.ctypes.data_as(C.c_void_p),
                                           cnt.ctypes.data_as(C.c_void_p), None, self._s))
        self.d2h_bytes += toks.nbytes + cnt.nbytes
        toks = toks.reshape(n, rows.value)
        return [toks[i, :cnt[i]].tolist() for i in range(n)]

    def frame_ids(self, n: int) -> tuple[np.ndarray, int]:
        rows = C.c_int32()
        _native.check(self.lib.dm_ctc_read(self.handle, None, None, C.byref(rows), self._s))
        ids = np.empty(n * rows.value, np.int32)
        _native.check(self.lib.dm_ctc_debug(self.handle, 0, ids.ctypes.data_as(C.c_void_p),
                                            ids.nbytes, self._s))
        return ids.reshape(n, rows.value), rows.value

    def hidden(self, n: int) -> np.ndarray:
        rows = C.c_int32()
        _native.check(self.lib.dm_ctc_read(self.handle, None, None, C.byref(rows), self._s))
        h = np.empty((n, rows.value, self.dims.hidden), np.float32)
        _native.check(self.lib.dm_ctc_debug(self.handle, 1, h.ctypes.data_as(C.c_void_p),
                                            h.nbytes, self._s))
        return h

    def transcribe_ids(self, segs) -> list[list[int]]:
        out = []
        for i in range(0, len(segs), self.max_batch):
            chunk = segs[i:i + self.max_batch]
            self.run(chunk)
            out.extend(self.read(len(chunk)))
        return out


@dataclass
class CTCBackendConfig:
    seed: int = 0
    init_std: float = 0.02
    device: int = 0
    max_batch: int = 32
    max_samples: int = 16000 * 30
    silence_is_empty: bool = True


class CTCBackend:
    """SupportsTranscribe for the CTC model (batch-synchronous)."""

    def __init__(self, cfg: CTCBackendConfig | None = None, engine: Wav2Vec2GPU | None = None):
        self.cfg = cfg or CTCBackendConfig()
        self.engine = engine or Wav2Vec2GPU(seed=self.cfg.seed, init_std=self.cfg.init_std,
                                            device=self.cfg.device, max_batch=self.cfg.max_batch,
                                            max_samples=self.cfg.max_samples)
        self._lock = threading.Lock()

    def transcribe_batch(self, batch) -> list[TranscriptResult]:
        entries = batch.entries
        if not entries:
            raise ValueError("a batch holds at least one segment")
        rates = {e.segment.sample_rate_hz for e in entries}
        if len(rates) > 1:
            raise ValueError(f"batch mixes sample rates {sorted(rates)}")
        if rates != {SAMPLE_RATE}:
            raise ValueError(f"the CTC front end needs {SAMPLE_RATE} Hz audio, got {rates}")
        t0 = time.monotonic()
        idx, segs, texts = [], [], {}
        for i, e in enumerate(entries):
            x = np.asarray(e.segment.samples, dtype=np.int16)
            if self.cfg.silence_is_empty and (len(x) < 400 or not x.any()):
                texts[i] = ""
                continue
            idx.append(i)
            segs.append(x)
        if segs:
            with self._lock:
                ids = self.engine.transcribe_ids(segs)
            for i, t in zip(idx, ids):
                texts[i] = ctc_text(t)
        ms = (time.monotonic() - t0) * 1000.0
        return [TranscriptResult(e.segment.segment_id, e.segment.session_id, texts[i],
                                 backend_time_ms=ms) for i, e in enumerate(entries)]

    def close(self):
        self.engine.close()
