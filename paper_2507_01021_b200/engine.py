"""Host side of the Whisper engine: weights on the device, the C-ABI handle,
and the continuous-batching slot loop (K7) that both the batch-synchronous
`transcribe_batch` contract and the per-GPU multiplexer consumers drive.

torch is used only for device memory, pinned host buffers and streams; all
arithmetic runs in the sm_100a library (`_native`). No CPU fallback exists.
"""

from __future__ import annotations

import ctypes as C
import math
import time
from collections import deque
from dataclasses import dataclass, field
from typing import Callable, Hashable, Iterable, Sequence

import numpy as np
import torch

from . import _native
from .models import N_SAMPLES, WhisperDims
from .weights import Manifest, host_tensor_values, normal_scale, tensor_key, whisper_manifest

PROMPT_MAX = 8
MAX_TOKENS = 448


def whisper_offsets(man: Manifest, dims: WhisperDims) -> list[int]:
    """Offset table in the order include/dictamux_b200.h documents."""
    names = ["enc.conv1.w", "enc.conv1.b", "enc.conv2.w", "enc.conv2.b", "enc.pos"]
    for i in range(dims.enc_layers):
        p = f"enc.l{i}"
        names += [f"{p}.{s}" for s in ("ln1.g", "ln1.b", "qkv.w", "qkv.b", "o.w", "o.b",
                                       "ln2.g", "ln2.b", "fc1.w", "fc1.b", "fc2.w", "fc2.b")]
    names += ["enc.ln.g", "enc.ln.b", "dec.embed", "dec.pos"]
    for i in range(dims.dec_layers):
        p = f"dec.l{i}"
        names += [f"{p}.{s}" for s in ("ln1.g", "ln1.b", "qkv.w", "qkv.b", "o.w", "o.b",
                                       "ln2.g", "ln2.b", "xq.w", "xq.b", "xo.w", "xo.b",
                                       "ln3.g", "ln3.b", "fc1.w", "fc1.b", "fc2.w", "fc2.b")]
    names += ["dec.xkv.w", "dec.xkv.b", "dec.ln.g", "dec.ln.b"]
    return [man[n].offset for n in names]


def materialize_weights(man: Manifest, device: torch.device,
                        stream: torch.cuda.Stream) -> torch.Tensor:
    """Fill the flat bf16 blob on the device with the seeded generator
    (csrc/engine.cu fill_normal_kernel; bit-identical to oracle/weights.py)."""
    blob = torch.zeros(man.total_elems, dtype=torch.int16, device=device)
    base = blob.data_ptr()
    with torch.cuda.stream(stream):
        for t in man.tensors:
            if t.init == "normal":
                _native.call("dm_fill_normal_bf16", C.c_void_p(base + 2 * t.offset),
                             t.numel, tensor_key(man.seed, t.tid), normal_scale(t.std),
                             float(t.mean), C.c_void_p(stream.cuda_stream))
            elif t.init == "host":
                vals = torch.from_numpy(host_tensor_values(man, t).view(np.int16).reshape(-1))
                blob[t.offset:t.offset + t.numel].copy_(vals, non_blocking=False)
            elif t.init == "ones":
                blob[t.offset:t.offset + t.numel].fill_(0x3F80)
            for a, b in t.zero_ranges:
                blob[t.offset + a:t.offset + b].zero_()
    stream.synchronize()
    return blob


@dataclass(frozen=True)
class ResidentPCM:
    """A segment whose int16 PCM already sits in the engine's resident device
    buffer (set_resident) at [offset, offset + length)."""
    offset: int
    length: int


@dataclass
class SegmentJob:
    key: Hashable
    samples: np.ndarray          # int16
    cap: int
    on_done: Callable[[Hashable, list[int]], None] | None = None


@dataclass
class EngineStats:
    encode_calls: int = 0
    segments_encoded: int = 0
    steps: int = 0
    slot_steps: int = 0
    busy_s: float = 0.0


class WhisperGPU:
    """One engine per GPU (`SPEC.md:176` "one dispatch loop per backend
    device"): weights, encoder workspace, decode slots and the CUDA-graph
    decode step, all behind the C ABI."""

    def __init__(self, dims: WhisperDims, *, seed: int = 0, init_std: float = 0.02,
                 device: int | str | torch.device = 0, max_slots: int = 64,
                 max_encode_batch: int = 32, num_pages: int | None = None,
                 eot: int | None = None, steps_per_poll: int = 8,
                 decode_groups: int | None = None, first_encode_batch: int = 8,
                 overlap_encode: bool = True, decode_priority: int = -1,
                 length_aware: bool = False):
        if not torch.cuda.is_available():
            raise _native.DmError("no CUDA device: the B200 engine has no CPU fallback")
        self.dims = dims
        self.device = torch.device("cuda", device) if isinstance(device, int) else torch.device(device)
        self.lib = _native.load()
        self.max_slots = max_slots
        self.max_encode_batch = max_encode_batch
        self.steps_per_poll = steps_per_poll
        self.first_encode_batch = first_encode_batch
        self.overlap_encode = overlap_encode
        # opt-in: each segment encodes its own ceil(n / 320)
        # positions instead of the 30 s window; results differ from pad_or_trim
        self.length_aware = length_aware
        self.eot = dims.eot if eot is None else eot
        with torch.cuda.device(self.device):
            # run_jobs(overlap_encode) encodes on enc_stream so a new group's
            # encode overlaps the decode of the groups already admitted
            self.stream = torch.cuda.Stream(self.device, priority=decode_priority)
            self.enc_stream = torch.cuda.Stream(self.device)
            self.man = whisper_manifest(dims, seed, init_std)
            self.blob = materialize_weights(self.man, self.device, self.stream)
            offs = whisper_offsets(self.man, dims)
            cfg = _native.WhisperConfigC()
            cfg.d_model, cfg.enc_layers, cfg.dec_layers = dims.d_model, dims.enc_layers, dims.dec_layers
            cfg.heads, cfg.ffn, cfg.n_mels, cfg.vocab = dims.heads, dims.ffn, dims.n_mels, dims.vocab
            cfg.eot = self.eot
            for i, t in enumerate(dims.prompt):
                cfg.prompt[i] = t
            cfg.prompt_len = len(dims.prompt)
            self.prompt: tuple[int, ...] = tuple(dims.prompt)
            cfg.max_slots, cfg.max_encode_batch = max_slots, max_encode_batch
            cfg.num_pages = num_pages if num_pages is not None else max_slots * 7
            if decode_groups is None:
                decode_groups = 1
            cfg.decode_groups = decode_groups
            self.decode_groups = decode_groups
            arr = (C.c_int64 * len(offs))(*offs)
            h = C.c_void_p()
            _native.check(self.lib.dm_whisper_create(C.byref(cfg), C.c_void_p(self.blob.data_ptr()),
                                                     arr, len(offs), C.byref(h)))
            self.handle = h
            # double-buffered pinned staging for PCM uploads + device buffers: the
            # host copy of encode batch k + 1 overlaps the GPU work of batch k
            self._pcm_host = [torch.empty(max_encode_batch * N_SAMPLES, dtype=torch.int16,
                                          pin_memory=True) for _ in range(2)]
            self._pcm_dev = [torch.empty(max_encode_batch * N_SAMPLES, dtype=torch.int16,
                                         device=self.device) for _ in range(2)]
            self._meta_host = [torch.empty(3 * max_encode_batch, dtype=torch.int64,
                                           pin_memory=True) for _ in range(2)]
            self._meta_dev = [torch.empty(3 * max_encode_batch, dtype=torch.int64,
                                          device=self.device) for _ in range(2)]
            self._up_done = [torch.cuda.Event() for _ in range(2)]
            self._up_used = [False, False]
            self._up_next = 0
            # H2D uploads run on their own stream so the next group's copy
            # overlaps the current group's encode; buffer b is rewritten only
            # after the encode that read it (_enc_done[b])
            self.copy_stream = torch.cuda.Stream(self.device)
            self._enc_done = [torch.cuda.Event() for _ in range(2)]
            self._enc_used = [False, False]
            self._last_buf = 0
            self._done = np.zeros(max_slots, np.int32)
            self._ngen = np.zeros(max_slots, np.int32)
            self._tokens = np.zeros(max_slots * MAX_TOKENS, np.int32)
            # pinned double-buffered snapshots for the pipelined slot loop
            self._snaps = [(torch.zeros(max_slots, dtype=torch.int32, pin_memory=True),
                            torch.zeros(max_slots, dtype=torch.int32, pin_memory=True),
                            torch.zeros(max_slots * MAX_TOKENS, dtype=torch.int32,
                                        pin_memory=True)) for _ in range(2)]
            self._snap_ev = [torch.cuda.Event() for _ in range(2)]
        self.stats = EngineStats()
        self._held: set[int] = set()       # slots holding self-KV pages
        self._resident: torch.Tensor | None = None
        self.h2d_bytes = 0
        self.d2h_bytes = 0

    def close(self):
        if getattr(self, "handle", None):
            _native.check(self.lib.dm_whisper_destroy(self.handle))
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ----------------------------------------------------------- primitives
    @property
    def _s(self):
        return C.c_void_p(self.stream.cuda_stream)

    def _i32(self, xs: Sequence[int]):
        return (C.c_int32 * max(1, len(xs)))(*xs)

    def set_resident(self, pcm_dev: torch.Tensor | None) -> None:
        """Register a device int16 buffer that ResidentPCM jobs index into."""
        self._resident = pcm_dev

    def _stage(self) -> int:
        """Next staging buffer; waits only for the copy that last read it."""
        b = self._up_next
        self._up_next ^= 1
        if self._up_used[b]:
            self._up_done[b].synchronize()
        return b

    def upload_segments(self, segs: Sequence[np.ndarray], stream=None):
        """Trim (pad_or_trim's truncation; padding is implicit in the kernel)
        and copy PCM to the device (stream-ordered, double-buffered). Returns
        (pcm, offsets, lengths) device pointers."""
        stream = self.stream if stream is None else stream
        n = len(segs)
        b = self._stage()
        self._last_buf = b
        mh, md = self._meta_host[b], self._meta_dev[b]
        if n and all(isinstance(s, ResidentPCM) for s in segs):
            meta = mh.numpy()
            meta[:n] = [s.offset for s in segs]
            meta[n:].view(np.int32)[:n] = [min(s.length, N_SAMPLES) for s in segs]
            with torch.cuda.stream(self.copy_stream):
                if self._enc_used[b]:
                    self.copy_stream.wait_event(self._enc_done[b])
                md.copy_(mh, non_blocking=True)
                self._up_done[b].record(self.copy_stream)
            stream.wait_event(self._up_done[b])
            self._up_used[b] = True
            return (C.c_void_p(self._resident.data_ptr()), C.c_void_p(md.data_ptr()),
                    C.c_void_p(md.data_ptr() + 8 * n))
        ph, pd = self._pcm_host[b], self._pcm_dev[b]
        offs, lens = [], []
        pos = 0
        for s in segs:
            s = np.asarray(s)
            if s.dtype != np.int16:
                raise TypeError("segment samples must be int16 PCM")
            k = min(len(s), N_SAMPLES)
            ph[pos:pos + k].copy_(torch.from_numpy(s[:k]))      # (multithreaded host copy)
            offs.append(pos)
            lens.append(k)
            pos += k
        meta = mh.numpy()
        meta[:n] = offs
        meta32 = meta[n:].view(np.int32)     # lengths packed after offsets
        meta32[:n] = lens
        with torch.cuda.stream(self.copy_stream):
            if self._enc_used[b]:
                self.copy_stream.wait_event(self._enc_done[b])
            if pos:
                pd[:pos].copy_(ph[:pos], non_blocking=True)
            md.copy_(mh, non_blocking=True)
            self._up_done[b].record(self.copy_stream)
        stream.wait_event(self._up_done[b])
        self._up_used[b] = True
        self.h2d_bytes += 2 * pos + 12 * n
        return C.c_void_p(pd.data_ptr()), C.c_void_p(md.data_ptr()), C.c_void_p(md.data_ptr() + 8 * n)

    def encode(self, segs: Sequence[np.ndarray], slots: Sequence[int], stream=None) -> None:
        """Encode into the slots' cross-KV cache on `stream` (default: the
        decode stream, so a following admit/step/debug is ordered after it)."""
        stream = self.stream if stream is None else stream
        pcm, offp, lenp = self.upload_segments(segs, stream)
        if self.length_aware:
            host_lens = self._i32([min(s.length if isinstance(s, ResidentPCM) else len(s), N_SAMPLES)
                                   for s in segs])
            _native.check(self.lib.dm_whisper_encode_lengths(
                self.handle, pcm, offp, lenp, host_lens, len(segs), self._i32(slots),
                C.c_void_p(stream.cuda_stream)))
        else:
            _native.check(self.lib.dm_whisper_encode(self.handle, pcm, offp, lenp, len(segs),
                                                     self._i32(slots),
                                                     C.c_void_p(stream.cuda_stream)))
        b = self._last_buf
        self._enc_done[b].record(stream)          # buffer b free for the upload after next
        self._enc_used[b] = True
        self.stats.encode_calls += 1
        self.stats.segments_encoded += len(segs)

    def set_prompt(self, tokens: Sequence[int]) -> None:
        """Decoder prompt of later admissions (<= 224 ids; Listing 1's
        `prompt_tokens + [no_timestamps]`), e.g. dims.prompt_with_context(ids).
        Only while no slot is admitted; caps shrink to 448 - len(prompt)."""
        tokens = [int(t) for t in tokens]
        arr = (C.c_int32 * len(tokens))(*tokens)
        _native.check(self.lib.dm_whisper_set_prompt(self.handle, arr, len(tokens), self._s))
        self.prompt = tuple(tokens)

    def admit(self, slots: Sequence[int], caps: Sequence[int]) -> None:
        _native.check(self.lib.dm_whisper_admit(self.handle, self._i32(slots), self._i32(caps),
                                                len(slots), self._s))
        self._held.update(slots)

    def release(self, slots: Sequence[int]) -> None:
        _native.check(self.lib.dm_whisper_release(self.handle, self._i32(slots), len(slots)))
        self._held.difference_update(slots)

    def reset(self) -> None:
        """Drop every slot (after a failed run): free pages, empty active set."""
        self.enc_stream.synchronize()
        self.stream.synchronize()
        if self._held:
            self.release(sorted(self._held))
        self.set_active([])

    def set_active(self, slots: Sequence[int]) -> None:
        _native.check(self.lib.dm_whisper_set_active(self.handle, self._i32(slots), len(slots),
                                                     self._s))

    def step(self, n: int) -> None:
        _native.check(self.lib.dm_whisper_step(self.handle, n, self._s))

    def read(self, tokens: bool = False):
        tp = self._tokens.ctypes.data_as(C.c_void_p) if tokens else None
        _native.check(self.lib.dm_whisper_read(self.handle,
                                               self._done.ctypes.data_as(C.c_void_p),
                                               self._ngen.ctypes.data_as(C.c_void_p), tp,
                                               self._s))
        self.d2h_bytes += 8 * self.max_slots + (4 * self.max_slots * MAX_TOKENS if tokens else 0)
        return self._done, self._ngen, self._tokens.reshape(self.max_slots, MAX_TOKENS)

    def debug(self, which: int, out: np.ndarray | None = None) -> np.ndarray | None:
        if which in (3, 8, 15):
            _native.check(self.lib.dm_whisper_debug(self.handle, which, None, 0, self._s))
            return None
        _native.check(self.lib.dm_whisper_debug(self.handle, which,
                                                out.ctypes.data_as(C.c_void_p), out.nbytes,
                                                self._s))
        return out

    def counters(self) -> dict:
        out = np.zeros(4, np.int64)
        _native.check(self.lib.dm_whisper_stats(self.handle, out.ctypes.data_as(C.c_void_p), 4))
        return dict(launches=int(out[0]), steps=int(out[1]), encodes=int(out[2]),
                    segments=int(out[3]))

    def time_kernel(self, which: int, layer: int = 0, iters: int = 20) -> float:
        ms = C.c_float()
        _native.check(self.lib.dm_whisper_time_kernel(self.handle, which, layer, iters,
                                                      C.byref(ms), self._s))
        return ms.value

    def encoder_output(self, n: int, rows: int = 1500) -> np.ndarray:
        """bf16 encoder output of the last encode, [n, rows, d] (rows: the
        batch's window after a length-aware encode)."""
        bits = np.empty((n, rows, self.dims.d_model), np.uint16)
        self.debug(0, bits)
        return (bits.astype(np.uint32) << 16).view(np.float32)

    def encoder_output_f32(self, segs, slots) -> np.ndarray:
        """Encode with the fp32 tap on and return the final-LN output before
        its bf16 rounding (the cross-KV GEMM consumes the bf16 copy)."""
        _native.check(self.lib.dm_whisper_debug(self.handle, 7, None, 1, self._s))
        try:
            self.encode(segs, slots)
            out = np.empty((len(segs), 1500, self.dims.d_model), np.float32)
            return self.debug(5, out)
        finally:
            _native.check(self.lib.dm_whisper_debug(self.handle, 7, None, 0, self._s))

    def enable_mel_tap(self, on: bool = True) -> None:
        """Later encodes also write the fp32 [n, n_mels, 3000] features
        (the product path writes only the bf16 encoder operand)."""
        _native.check(self.lib.dm_whisper_debug(self.handle, 15, None, int(on), self._s))

    def log_mel(self, n: int) -> np.ndarray:
        return self.debug(1, np.empty((n, self.dims.n_mels, 3000), np.float32))

    # ----------------------------------------------------------- slot loop
    def _snap(self, b: int) -> None:
        """Stream-ordered snapshot of done / n_gen / tokens into pinned buffer b."""
        d, g, t = self._snaps[b]
        _native.check(self.lib.dm_whisper_read_async(
            self.handle, C.c_void_p(d.data_ptr()), C.c_void_p(g.data_ptr()),
            C.c_void_p(t.data_ptr()), self._s))
        self._snap_ev[b].record(self.stream)
        self.d2h_bytes += 8 * self.max_slots + 4 * self.max_slots * MAX_TOKENS

    def run_jobs(self, jobs: Iterable[SegmentJob],
                 refill: Callable[[int], list[SegmentJob]] | None = None) -> dict:
        """Continuous batching: admit jobs into free decode slots (encoding
        them in groups of <= max_encode_batch), step the active slots, route a
        segment as soon as its slot hits EOT or its cap, refill freed slots
        from `pending` then from `refill(n_free)` (the multiplexer hook).

        The host never waits on the step it just issued: each batch of steps
        runs up to the next slot's cap (predicted exactly on the host:
        prompt_len - 1 + cap steps), so cap-terminated slots leave the active
        set and free their pages with no wasted step; a stream-ordered
        snapshot of (done, n_gen, tokens) is taken after each batch and read
        one batch later (tokens of finished slots never change, and slots
        that hit EOT early only linger one batch -- their attention is
        skipped). Returns {key: token ids}.

        With overlap_encode, encodes run on
        enc_stream and a group is admitted (decode stream waits on its encode
        event) once the host sees its event complete -- or at once when
        nothing is decoding -- so the groups already admitted decode while the
        next group encodes; the jobs of one call are then taken longest cap
        first. Outputs are batch-invariant bit for bit either way."""
        overlap = self.overlap_encode
        jobs = list(jobs)
        if overlap:
            jobs.sort(key=lambda j: -j.cap)
            self.enc_stream.wait_stream(self.stream)   # encodes after prior work
        pending = deque(jobs)
        encoding: deque = deque()              # (event, [(slot, job)]) in flight on enc_stream
        free = list(range(self.max_slots - 1, -1, -1))
        # Slots freed while the decode stream may still read their cross-KV
        # (capped slots leave the active set after their last batch is queued;
        # early-EOT slots are found one batch late): an encode on enc_stream
        # into such a slot must first wait for the decode work queued so far
        # (write-after-read on xkv[slot]). Clean slots are handed out first.
        unfenced: set[int] = set()
        active: dict[int, SegmentJob] = {}
        left: dict[int, int] = {}              # slot -> steps to its cap
        waiting: list[tuple[int, SegmentJob]] = []   # finished, result in the next snapshot
        results: dict = {}
        prompt_extra = len(self.prompt) - 1
        t0 = time.perf_counter()
        prev = None                            # (snapshot buffer, [(slot, job)], active slots)
        b = 0
        dirty = True

        def route(slot: int, job: SegmentJob, snap) -> None:
            _, ngen, toks = snap
            ids = toks[slot, :ngen[slot]].tolist()
            results[job.key] = ids
            if job.on_done is not None:
                job.on_done(job.key, ids)

        while True:
            if free and refill is not None and len(pending) < len(free):
                pending.extend(refill(len(free) - len(pending)))
            while free and pending:
                take = []
                # an idle engine starts with a small group: the GPU begins
                # while the host still stages the rest of the PCM
                lim = self.max_encode_batch if (active or waiting or prev or encoding) else min(
                    self.max_encode_batch, self.first_encode_batch)
                if unfenced:
                    free.sort(key=lambda s: (s not in unfenced, -s))   # pop() takes clean, low ids first
                while free and pending and len(take) < lim:
                    take.append((free.pop(), pending.popleft()))
                slots = [s for s, _ in take]
                if overlap:
                    if unfenced.intersection(slots):
                        fence = torch.cuda.Event()
                        fence.record(self.stream)         # after every batch issued so far
                        self.enc_stream.wait_event(fence)
                        unfenced.clear()
                    self.encode([j.samples for _, j in take], slots, self.enc_stream)
                    ev = torch.cuda.Event()
                    ev.record(self.enc_stream)
                    encoding.append((ev, take))
                    continue
                self.encode([j.samples for _, j in take], slots)
                self.admit(slots, [j.cap for _, j in take])
                for s, j in take:
                    active[s] = j
                    left[s] = prompt_extra + j.cap
                dirty = True
            while encoding and (not active or encoding[0][0].query()):
                ev, take = encoding.popleft()
                self.stream.wait_event(ev)
                self.admit([s for s, _ in take], [j.cap for _, j in take])
                for s, j in take:
                    active[s] = j
                    left[s] = prompt_extra + j.cap
                dirty = True
            cur = None
            if active:
                if dirty:
                    self.set_active(sorted(active))
                    dirty = False
                n = max(1, min(self.steps_per_poll, min(left[s] for s in active)))
                self.step(n)
                self.stats.steps += n
                self.stats.slot_steps += n * len(active)
                for s in active:
                    left[s] -= n
                self._snap(b)
                capped = [s for s in active if left[s] <= 0]
                for s in capped:
                    waiting.append((s, active.pop(s)))
                if capped:
                    self.release(capped)
                    free.extend(capped)
                    unfenced.update(capped)
                    dirty = True
                cur = (b, waiting, set(active))
                waiting = []
                b ^= 1
            if prev is not None:
                pb, finished, was_active = prev
                self._snap_ev[pb].synchronize()
                snap = tuple(x.numpy() for x in self._snaps[pb])
                snap = (snap[0], snap[1], snap[2].reshape(self.max_slots, MAX_TOKENS))
                for s, j in finished:
                    route(s, j, snap)
                # early EOT: done in the snapshot while still listed as active
                eot = [s for s in was_active if s in active and snap[0][s]]
                for s in eot:
                    route(s, active.pop(s), snap)
                if eot:
                    self.release(eot)
                    free.extend(eot)
                    unfenced.update(eot)
                    dirty = True
            prev = cur
            if prev is None and not active and not pending and not encoding:
                break
        self.stats.busy_s += time.perf_counter() - t0
        return results

    def transcribe_ids(self, segs: Sequence[np.ndarray], caps: Sequence[int]) -> list[list[int]]:
        jobs = [SegmentJob(i, s, int(c)) for i, (s, c) in enumerate(zip(segs, caps))]
        out = self.run_jobs(jobs)
        return [out[i] for i in range(len(segs))]
