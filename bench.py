#!/usr/bin/env python
"""Benchmark: audio-seconds transcribed per second (RTFx) on B200, with the
p50/p95 per-segment latency of 64 concurrent users in the same line.

Workload (BASELINE.json configs[2], cfg3 -- the largest configuration that
fits one GPU): whisper-large-v3 random-init bf16 (seed 0), 64 synthetic
segments per GPU with durations uniform in [3, 30] s (loadgen-style speech =
uniform int16 noise in [-8000, 8000), per-user PCG64 seeded by
blake2s(f"{seed}:u{id}"), loadgen.py:50-53,97-98), continuous batching
(the reference's continuous policy, min_batch 32, max_batch 64) over 64
decode slots, greedy cap ceil(3.75 * duration) tokens (the sim text rate).
One "step" = the whole hot path over those 64 segments: log-mel -> encoder
-> cross-KV -> greedy decode of every segment to EOT/cap.

  value   : inputs (int16 PCM) already resident in HBM when the timed region
            starts; CUDA events on the engine stream, max over ranks.
  e2e     : the public API a user calls -- the reference's own SegmentQueue
            (continuous policy) -> B200Backend.transcribe_batch(batch) with
            host numpy PCM: pinned staging + H2D, kernels, D2H token reads,
            detokenisation.
  latency : 64 live users speaking in real time into the reference's
            SegmentQueue, one GpuConsumer per GPU (iteration-level
            admission); p50/p95 endpoint -> delivery by nearest rank
            (report.py:17-26), next to one user alone through the
            reference's own SequentialJobRunner (server.py:142-206).
  stages  : log-mel (HBM), encoder (bf16 tensor), decode step at 64 rows
            (HBM), each as a fraction of MEASURED_PEAKS.json.
  roofline: the dominant kernel (decode cross-attention + cross-o tail).

N GPUs: `--gpus N` launches N ranks itself (torch.distributed.run) unless
already under torchrun; one process per GPU, each with its own 64 segments
(weak scaling, no data-path collective: segments are independent, SURVEY.md
§8(e)); torch.distributed only for the barrier and the max-over-ranks time.

`--impl reference` times the reference path's CPU restatement (oracle/,
faster-whisper/CTranslate2 are absent) on the host cores
with all threads, rank 0 only, on the same model and workload.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "audio-seconds transcribed/sec (RTFx)"
UNIT = "audio_s/s"
MODEL = "whisper-large-v3"
REF = ROOT / "baseline" / "_ref"
FP32_PEAK_TFLOPS = 74.4            # 148 SMs x 128 FP32 lanes x 2 (FMA) x 1.965 GHz


# ---------------------------------------------------------------- workload
def user_rng(seed: int, user_id: str) -> np.random.Generator:
    dig = hashlib.blake2s(f"{seed}:{user_id}".encode(), digest_size=8).digest()
    return np.random.Generator(np.random.PCG64(int.from_bytes(dig, "big")))


def make_workload(n: int, rank: int = 0, seed: int = 0, lo: float = 3.0, hi: float = 30.0):
    """n segments for this rank (weak scaling: rank r owns users r*n .. r*n+n-1)."""
    segs = []
    for i in range(n):
        uid = f"u{rank * n + i:04d}"
        rng = user_rng(seed, uid)
        dur = float(rng.uniform(lo, hi))
        k = int(round(dur * 16000))
        segs.append((uid, rng.integers(-8000, 8000, size=k, dtype=np.int16)))
    return segs


def token_cap(duration_s: float) -> int:
    return max(1, min(444, math.ceil(3.75 * duration_s)))


def reference_scheduler():
    """The reference's own scheduler module (unmodified, baseline/_ref), or None."""
    if not (REF / "dictamux").exists():
        return None
    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    import dictamux.scheduler as rs
    return rs


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows: list[list[str]] = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.gpu}",
                                      f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([c.strip() for c in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self) -> dict:
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 5 + i and r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ---------------------------------------------------------------- dist
def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def max_over_ranks(x: float, world: int, device=None) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    if dist.get_backend() != "nccl":
        device = None                 # gloo (--share-devices): reduce on the host
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world: int):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def relaunch_under_torchrun(n: int) -> int:
    """`bench.py --gpus N` outside torchrun: start N ranks on this node."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr=127.0.0.1", f"--master-port={_free_port()}",
           str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd)


def pick_device(local: int, world: int, share: bool) -> tuple[int, str]:
    """(CUDA device, process-group backend) of this rank. Fewer visible GPUs
    than ranks is an error unless --share-devices (a plumbing check of the
    N-rank path on a 1-GPU lease: ranks never wait on each other's kernels,
    and the barrier/max-over-ranks runs on gloo)."""
    import torch
    n = torch.cuda.device_count()
    if n == 0:
        raise SystemExit("bench.py: no CUDA device (the B200 path has no CPU fallback)")
    if world > n:
        if not share:
            raise SystemExit(f"bench.py: --gpus {world} but only {n} CUDA device(s) visible")
        return local % n, "gloo"
    return local, "nccl"


# ---------------------------------------------------------------- CPU oracle
def _oracle_for(dims, blob=None, man=None, threads=None):
    from oracle.weights import load_all_f32, load_all_f32_from_bits
    from oracle.whisper import WhisperOracle
    from paper_2507_01021_b200.weights import whisper_manifest
    man = man or whisper_manifest(dims, 0, 0.02)
    w = load_all_f32_from_bits(man, blob) if blob is not None else load_all_f32(man, threads)
    return WhisperOracle(dims, seed=0, weights=w)


def cpu_oracle_rtfx(orc, segs, threads: int, budget_s: float = 20.0) -> dict:
    """Time the CPU restatement (oracle/) of the full path on a bounded sample."""
    import torch
    from oracle.logmel import log_mel_batch
    torch.set_num_threads(threads)
    audio, wall, used = 0.0, 0.0, 0
    for uid, x in segs:
        t0 = time.perf_counter()
        mel = log_mel_batch([x], orc.dims.n_mels)
        enc = orc.encode(mel)
        orc.greedy(enc[0], token_cap(len(x) / 16000.0))
        wall += time.perf_counter() - t0
        audio += len(x) / 16000.0
        used += 1
        if wall >= budget_s:
            break
    return {"value": audio / wall, "audio_s": audio, "wall_s": wall, "segments": used}


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def workload_name(segments: int) -> str:
    cfg = "cfg3" if MODEL == "whisper-large-v3" else ("cfg2" if MODEL == "whisper-base" else "side run")
    return (f"{cfg}: {MODEL} random-init bf16 (seed 0), {segments} segments/GPU x U[3,30] s "
            f"synthetic speech, continuous batching (min_batch 32, max_batch 64) over 64 decode "
            f"slots, greedy cap ceil(3.75*dur)")


# ---------------------------------------------------------------- arms
def run_reference(args, rank: int, world: int) -> None:
    """The reference path's CPU implementation (the oracle port: the
    reference's faster-whisper/CTranslate2 path is absent) on this host's
    cores. Each timed step = one segment of the same workload (rotating),
    transcribed end to end; warm-up steps run the shortest segment with cap 4."""
    if rank != 0:
        return
    from paper_2507_01021_b200.models import get_model
    threads = len(os.sched_getaffinity(0))
    dims = get_model(MODEL)
    t0 = time.perf_counter()
    orc = _oracle_for(dims, threads=threads)
    init_s = time.perf_counter() - t0
    segs = make_workload(args.segments, 0)
    import torch
    torch.set_num_threads(threads)
    short = min(segs, key=lambda s: len(s[1]))
    for _ in range(args.warmup):
        from oracle.logmel import log_mel_batch
        orc.greedy(orc.encode(log_mel_batch([short[1]], dims.n_mels))[0], 4)
    times, audios = [], []
    for it in range(args.steps):
        r = cpu_oracle_rtfx(orc, [segs[(it * 7) % len(segs)]], threads, budget_s=1e9)
        times.append(r["wall_s"])
        audios.append(r["audio_s"])
    value = sum(audios) / sum(times)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * sum(times) / len(times), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": workload_name(args.segments), "model": MODEL,
                   "sample_per_step": "1 workload segment (rotating, stride 7) end to end",
                   "weights_init_s": round(init_s, 1)},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{args.steps} workload segments ({sum(audios):.1f} audio-s), "
                                   f"one per step, full path (log-mel + encode + greedy) in "
                                   f"oracle/ (torch fp32 CPU, {threads} threads) on {cpu_model()}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_b200(args, rank: int, world: int, device: int) -> None:
    import torch
    from paper_2507_01021_b200.backend import B200Backend, B200BackendConfig
    from paper_2507_01021_b200.engine import ResidentPCM, SegmentJob, WhisperGPU
    from paper_2507_01021_b200.models import get_model
    from paper_2507_01021_b200.types import batch_of, make_segment

    torch.cuda.set_device(device)
    dev = torch.device("cuda", device)
    dims = get_model(MODEL)
    segs = make_workload(args.segments, rank)
    audio_s = sum(len(x) for _, x in segs) / 16000.0
    eng = WhisperGPU(dims, seed=0, device=device, max_slots=min(64, args.segments),
                     max_encode_batch=args.encode_batch, steps_per_poll=args.steps_per_poll,
                     first_encode_batch=args.first_encode_batch,
                     overlap_encode=bool(args.overlap_encode), decode_priority=args.decode_priority)
    backend = B200Backend(B200BackendConfig(model=MODEL, device=device), engine=eng)

    # resident inputs for `value`
    flat = np.concatenate([x for _, x in segs])
    pcm_dev = torch.from_numpy(flat).to(dev)
    eng.set_resident(pcm_dev)
    offs = np.cumsum([0] + [len(x) for _, x in segs[:-1]])
    res_jobs = lambda: [SegmentJob(uid, ResidentPCM(int(o), len(x)), token_cap(len(x) / 16000.0))
                        for (uid, x), o in zip(segs, offs)]
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def timed(fn):
        flush.fill_(1.0)                       # L2 flush (256 MB > 126 MB L2)
        torch.cuda.synchronize(dev)
        barrier(world)
        start = torch.cuda.Event(enable_timing=True)
        end = torch.cuda.Event(enable_timing=True)
        start.record(eng.stream)
        out = fn()
        end.record(eng.stream)
        torch.cuda.synchronize(dev)
        barrier(world)
        return start.elapsed_time(end), out

    if args.profile:
        # single timed-path step, nothing else (for ncu launch lists)
        eng.run_jobs(res_jobs())
        torch.cuda.synchronize(dev)
        print(json.dumps({"profile_step_done": True, **eng.counters()}), flush=True)
        return
    for _ in range(args.warmup):
        timed(lambda: eng.run_jobs(res_jobs()))
    c0 = eng.counters()
    clocks = ClockSampler(device)
    with clocks:
        step_ms = [timed(lambda: eng.run_jobs(res_jobs()))[0] for _ in range(args.steps)]
    c1 = eng.counters()
    ms = statistics.mean(step_ms)
    ms_max = max_over_ranks(ms, world, dev)
    value = world * audio_s / (ms_max / 1000.0)
    launches = c1["launches"] - c0["launches"]

    # e2e through the public API (host PCM -> results): the reference's own
    # SegmentQueue + continuous policy forms the batch (our mirror types when
    # the reference package is absent)
    rs = reference_scheduler()

    def e2e_once():
        if rs is not None:
            q = rs.SegmentQueue()
            for uid, x in segs:
                q.enqueue_segment(make_segment(uid, x, session_id=uid, endpoint_time=0.0), 0.0)
            pol = rs.BatchingPolicy(kind="continuous", min_batch=32, max_batch=len(segs))
            batch = q.try_form_batch(pol, 0.0)
        else:
            batch = batch_of([make_segment(uid, x, session_id=uid) for uid, x in segs])
        assert batch is not None and len(batch.entries) == len(segs)
        res = backend.transcribe_batch(batch)
        assert len(res) == len(segs) and not any(r.is_error for r in res)
        return res
    for _ in range(max(1, args.warmup // 2)):
        timed(e2e_once)
    h0, d0 = eng.h2d_bytes, eng.d2h_bytes
    e2e_ms = [timed(e2e_once)[0] for _ in range(args.steps)]
    h2d = (eng.h2d_bytes - h0) / args.steps
    d2h = (eng.d2h_bytes - d0) / args.steps
    e2e_ms_max = max_over_ranks(statistics.mean(e2e_ms), world, dev)
    e2e_value = world * audio_s / (e2e_ms_max / 1000.0)

    # opt-in length-aware encoder on the same engine and
    # workload: a separate number, never the headline (it changes results vs
    # the pad_or_trim contract; its parity is in tests/test_gpu_length_aware.py)
    length_aware = None
    if not args.no_stages:
        eng.length_aware = True
        for _ in range(args.warmup):
            timed(lambda: eng.run_jobs(res_jobs()))
        la_ms = [timed(lambda: eng.run_jobs(res_jobs()))[0] for _ in range(args.steps)]
        eng.length_aware = False
        la_ms = max_over_ranks(statistics.mean(la_ms), world, dev)
        length_aware = {"value": world * audio_s / (la_ms / 1000.0), "unit": UNIT,
                        "ms_per_step": la_ms,
                        "note": "opt-in: each segment encodes its own ceil(n/320) positions and "
                                "decode cross-attends only to them (results differ from "
                                "pad_or_trim); not the headline"}
    stages = measure_stages(eng, dims, segs, offs, pcm_dev) if not args.no_stages else None
    roof = measure_roofline(eng, dims) if not args.no_stages else None

    latency = None
    if args.latency_users > 0 and world == 1:
        latency = measure_latency(eng, dims, args, rs)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = len(os.sched_getaffinity(0))
        orc = _oracle_for(dims, blob=eng.blob.cpu().numpy().view(np.uint16), man=eng.man)
        r = cpu_oracle_rtfx(orc, segs, threads, budget_s=args.cpu_budget_s)
        cpu = {"value": r["value"], "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"first {r['segments']} of the {args.segments} workload segments "
                         f"({r['audio_s']:.1f} audio-s, {r['wall_s']:.1f} s wall), full path "
                         f"(log-mel+encode+greedy) in oracle/ torch fp32 on {cpu_model()}"}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "bf16", "data": "synthetic",
            "config": {"workload": workload_name(args.segments),
                       "model": MODEL, "segments_per_gpu": args.segments,
                       "audio_s_per_gpu": round(audio_s, 3),
                       "parallelism": f"replicas x{world} (no collective)",
                       "l2": "flushed between timed steps (256 MB write)",
                       "encode_batch": args.encode_batch, "first_encode_batch": args.first_encode_batch,
                       "overlap_encode": bool(args.overlap_encode),
                       "decode_priority": args.decode_priority,
                       "steps_per_poll": args.steps_per_poll},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h),
                    "path": ("reference SegmentQueue(continuous, min_batch 32) -> "
                             if rs is not None else "Batch -> ")
                            + "B200Backend.transcribe_batch (host int16)"},
            "latency": latency, "roofline": roof, "stages": stages, "cpu_baseline": cpu,
            "length_aware_opt_in": length_aware,
            "clocks": clocks.summary(), "gpu_launches": launches // args.steps,
            "gpu_launches_note": "kernels per timed step (C-ABI counter; graph nodes per replay)",
        }
        print(json.dumps(line), flush=True)


def _peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    return json.loads(p.read_text()) if p.exists() else {}


def measure_stages(eng, dims, segs, offs, pcm_dev) -> dict:
    """Per-stage throughput as a fraction of its roofline (north star: log-mel
    and decode on HBM GB/s, encoder on dense bf16 TFLOP/s), each timed live
    with CUDA events on the engine stream, L2 flushed before every timed call.

      log-mel : dm_logmel over the first E workload segments; algorithmic bytes
                = true int16 PCM (2 n) + the [n_mels, 3000] features written
                (SURVEY.md §8(d)).
      encoder : dm_whisper_encode of the same E segments (log-mel -> conv stem
                -> layers -> cross-KV); algorithmic FLOPs = E x (encoder +
                cross-KV) per segment, SURVEY.md §8(d).
      decode  : one greedy step with all 64 slots active (the E segments
                replicated); algorithmic bytes = decoder weights + every active
                slot's cross-KV + its self-KV up to the fed position."""
    import ctypes as C
    import torch
    from paper_2507_01021_b200 import _native
    from paper_2507_01021_b200.engine import ResidentPCM
    peaks = _peaks()
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    tc = float(peaks.get("bf16_tflops", 2250.0))
    tc_sus = float(peaks.get("bf16_tflops_sustained", tc))
    dev = pcm_dev.device
    E = eng.max_encode_batch
    sub = [(uid, x, int(o)) for (uid, x), o in zip(segs[:E], offs[:E])]
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def ev_ms(fn, reps=5):
        out = []
        for _ in range(reps):
            flush.fill_(1.0)
            torch.cuda.synchronize(dev)
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(eng.stream)
            fn()
            b.record(eng.stream)
            torch.cuda.synchronize(dev)
            out.append(a.elapsed_time(b))
        return statistics.median(out)

    # log-mel (K1) as the encoder consumes it: the bf16 time-major operand
    nm = dims.n_mels
    offs_d = torch.tensor([o for _, _, o in sub], dtype=torch.int64, device=dev)
    lens_d = torch.tensor([len(x) for _, x, _ in sub], dtype=torch.int32, device=dev)
    ldt = 64 if nm <= 64 else 128
    mel = torch.zeros(E, 3002, ldt, dtype=torch.int16, device=dev)
    segmax = torch.empty(E, dtype=torch.int32, device=dev)
    lm = lambda: _native.check(eng.lib.dm_logmel_operand(
        C.c_void_p(pcm_dev.data_ptr()), C.c_void_p(offs_d.data_ptr()),
        C.c_void_p(lens_d.data_ptr()), E, nm, C.c_void_p(mel.data_ptr()),
        C.c_void_p(segmax.data_ptr()), eng._s))
    lm()
    lm_ms = ev_ms(lm)
    lm_bytes = sum(2 * min(len(x), 480000) for _, x, _ in sub) + E * nm * 3000 * 2
    # FP32 work of the frames that are not wholly padding: the 200-point complex
    # FFT (8 x 25: 25 8-point + 8 25-point DFTs, 400 twiddle products), window,
    # real-FFT post-processing + power, the sparse mel dot products, log10
    live_frames = sum(min(3000, (min(len(x), 480000) + 200 + 159) // 160) for _, x, _ in sub)
    lm_flop = live_frames * 18_000
    # encoder (K2-K5)
    d, L, Ld, F = dims.d_model, dims.enc_layers, dims.dec_layers, dims.ffn
    enc_flop = (2 * nm * 3 * d * 3000 + 2 * 3 * d * d * 1500
                + L * (8 * d * d * 1500 + 4 * 1500 * 1500 * d + 4 * d * F * 1500)
                + 4 * Ld * d * d * 1500)
    jobs = [ResidentPCM(o, len(x)) for _, x, o in sub]
    slots = list(range(E))
    en = lambda: eng.encode(jobs, slots)
    en()
    en_ms = ev_ms(en, reps=3)
    # decode step at 64 rows (K6)
    S = eng.max_slots
    for i in range(E, S, E):
        eng.encode(jobs[:min(E, S - i)], list(range(i, min(S, i + E))))
    allslots = list(range(S))
    eng.admit(allslots, [400] * S)
    eng.set_active(allslots)
    eng.step(8)                       # past the prompt: positions 7..
    torch.cuda.synchronize(dev)
    # 8 back-to-back step graphs per timed call (as in the bench step; one
    # step streams ~17 GB, far more than L2), median of 5 calls: positions
    # 8..47, mean self-KV length ~28
    st_ms = ev_ms(lambda: eng.step(8), reps=5) / 8
    pos = 28
    eng.release(allslots)
    eng.set_active([])
    torch.cuda.synchronize(dev)
    w_bytes = 2 * (Ld * (4 * d * d + 2 * d * d + 2 * d * F) + dims.vocab * d)
    x_bytes = S * Ld * 2 * 1500 * d * 2
    kv_bytes = S * Ld * 2 * d * 2 * (pos + 1)   # keys 0..pos per slot and layer
    st_bytes = w_bytes + x_bytes + kv_bytes
    return {
        "logmel": {"bound": "hbm", "achieved": lm_bytes / (lm_ms / 1e3) / 1e9, "peak": hbm,
                   "unit": "GB/s", "frac": lm_bytes / (lm_ms / 1e3) / 1e9 / hbm,
                   "ms": lm_ms, "bytes": lm_bytes, "segments": E,
                   "bytes_note": "2 n int16 PCM read + the bf16 [3000, n_mels] encoder operand "
                                 "written (dm_logmel_operand, the product path)",
                   "fp32_tflops": lm_flop / (lm_ms / 1e3) / 1e12,
                   "fp32_frac": lm_flop / (lm_ms / 1e3) / 1e12 / FP32_PEAK_TFLOPS,
                   "fp32_note": f"~18 kFLOP per non-padding frame ({live_frames} frames) vs "
                                f"{FP32_PEAK_TFLOPS} TFLOP/s FP32 FMA peak (148 SMs x 128 x 2 x 1.965 GHz)"},
        "encoder": {"bound": "tensor", "achieved": E * enc_flop / (en_ms / 1e3) / 1e12, "peak": tc,
                    "unit": "TFLOP/s", "frac": E * enc_flop / (en_ms / 1e3) / 1e12 / tc,
                    "ms": en_ms, "flop": E * enc_flop, "segments": E,
                    "peak_sustained": tc_sus,
                    "frac_vs_sustained": E * enc_flop / (en_ms / 1e3) / 1e12 / tc_sus,
                    "note": "whole dm_whisper_encode (log-mel + conv stem + layers + LN + cross-KV); "
                            "frac vs the burst bf16 peak (one 8192^3 matmul), frac_vs_sustained vs "
                            "MEASURED_PEAKS' sustained figure (back-to-back matmuls: the power-capped "
                            "clocks a ~37 ms multi-kernel encode runs at)"},
        "decode_step": {"bound": "hbm", "achieved": st_bytes / (st_ms / 1e3) / 1e9, "peak": hbm,
                        "unit": "GB/s", "frac": st_bytes / (st_ms / 1e3) / 1e9 / hbm,
                        "ms": st_ms, "bytes": st_bytes, "rows": S,
                        "note": "CUDA-graph step (8 back to back per timed call, median of 5): weights + cross-KV + self-KV, 64 active slots"},
        "peak_source": "MEASURED_PEAKS.json (hbm_gbs burst copy, bf16_tflops burst)" if peaks else "fallback",
    }


def measure_roofline(eng, dims) -> dict:
    """Cross-attention (decode, K6) is the dominant kernel: per launch it
    streams every active slot's K and V of one layer, n_active * 2 * 1500 * d
    bf16 (L*2*1500*d*2 B per segment per step; 491.5 MB per
    launch at 64 rows on large-v3). Timed with CUDA events around a graph of
    one launch per decoder layer (launch i runs layer i % L, so every launch
    reads a different layer's cross-KV from HBM, PDL-chained as inside the
    step graph) at 64 active rows."""
    import torch
    peaks = _peaks()
    peak = float(peaks.get("hbm_gbs", 6650.0))
    S = eng.max_slots
    seg = np.random.default_rng(0).integers(-8000, 8000, size=160000, dtype=np.int16)
    slots = list(range(S))
    for i in range(0, S, eng.max_encode_batch):
        chunk = slots[i:i + eng.max_encode_batch]
        eng.encode([seg] * len(chunk), chunk)
    eng.admit(slots, [8] * S)
    eng.set_active(slots)
    eng.step(1)                      # q for the cross-attention
    L = dims.dec_layers
    runs = [eng.time_kernel(0, layer=-1, iters=2 * L) for _ in range(5)]
    ms = statistics.median(runs)
    # the same launches reduced to their K/V stream (what the CTA structure can
    # move with no compute): the gap to `ms` is the kernel's own overhead
    stream_ms = statistics.median(eng.time_kernel(9, layer=-1, iters=2 * L) for _ in range(5))
    eng.release(slots)
    eng.set_active([])
    torch.cuda.synchronize(eng.device)
    bytes_per_launch = S * 2 * 1500 * dims.d_model * 2
    achieved = bytes_per_launch / (ms / 1000.0) / 1e9
    traffic = None
    tf = ROOT / "profiles" / "r02_xattn_traffic_large_v3_v11.json"
    if tf.exists():     # dram read+write of one ncu --set full capture, scaled to rows
        t = json.loads(tf.read_text())
        traffic = (t["dram_bytes_read"] + t["dram_bytes_write"]) * S / t["rows"]
    return {"kernel": "cross_attn_kernel + xattn_merge_kernel (decode K6 cross-attention)",
            "bound": "hbm",
            "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": traffic,
            "traffic_unit": f"bytes per launch (ncu dram__bytes_read+write, {tf.name})",
            "timing": f"CUDA events on the engine stream around a graph of {2 * L} launches "
                      f"(each the cross-attention + its split-merge kernel, as in the step), "
                      f"launch i = decoder layer i % {L}, 64 active rows (median of 5)",
            "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst copy)" if peaks else "fallback",
            "bytes_per_launch": bytes_per_launch, "avg_launch_ms": ms,
            "kv_stream_only_ms": stream_ms,
            "kv_stream_only_frac": bytes_per_launch / (stream_ms / 1000.0) / 1e9 / peak,
            "per_unit": "2*1500*d*2 B per active slot per layer"}


def measure_latency(eng, dims, args, rs) -> dict | None:
    """p50/p95 per-segment latency of `latency_users` live users (cfg3) on
    this GPU vs one user alone through the reference's SequentialJobRunner."""
    if rs is None:
        return {"unavailable": "reference package not installed in baseline/_ref"}
    sys.path.insert(0, str(ROOT / "scripts"))
    import latency_bench as lb
    users = {f"u{i:03d}": lb.user_session(args.seed, f"u{i:03d}", args.latency_session_s)
             for i in range(args.latency_users)}
    policy = rs.BatchingPolicy(kind="continuous", min_batch=32, max_batch=64,
                               starvation_flush_ms=args.starvation_ms)
    mux = lb.run_multiplexed([eng], users, policy, rs, eager_start=bool(args.latency_eager))
    seq = lb.run_sequential_reference([eng], users["u000"], 64, MODEL)
    return {"users": args.latency_users, "session_s": args.latency_session_s,
            "policy": {"kind": "continuous", "min_batch": 32, "max_batch": 64,
                       "starvation_flush_ms": args.starvation_ms},
            "eager_start": bool(args.latency_eager),
            "multiplexed": mux, "sequential_single_user": seq,
            "p95_below_sequential": mux["p95_ms"] < seq["p95_ms"],
            "percentile": "nearest rank (report.py:17-26)"}


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--model", default=None,
                    help="side runs on another model (e.g. whisper-base for cfg2); default large-v3 (cfg3)")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--segments", type=int, default=64)
    ap.add_argument("--encode-batch", type=int, default=12,
                    help="segments per encoder launch (measured at large-v3 with overlap, RTFx: "
                         "8 -> 1748, 12 -> 1771, 16 -> 1735, 32 -> 1721, 64 -> 1630)")
    ap.add_argument("--steps-per-poll", type=int, default=8)
    ap.add_argument("--cpu-budget-s", type=float, default=20.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-stages", action="store_true")
    ap.add_argument("--overlap-encode", type=int, default=1,
                    help="1: encode the next group on a second stream while admitted groups decode")
    ap.add_argument("--decode-priority", type=int, default=-1,
                    help="CUDA stream priority of the decode stream (-1 high, 0 normal)")
    ap.add_argument("--first-encode-batch", type=int, default=12,
                    help="segments (longest caps first) in the first encode group of an idle engine; "
                         "the rest encode in --encode-batch groups on a second stream while the "
                         "admitted ones decode (no overlap, one 64-segment encode: 1693-1721)")
    ap.add_argument("--latency-users", type=int, default=64,
                    help="live users for the latency block (0: skip)")
    ap.add_argument("--latency-session-s", type=float, default=30.0)
    ap.add_argument("--latency-eager", type=int, default=1,
                    help="1 (GpuConsumer default): an idle consumer starts on whatever is queued; "
                         "0: it waits for the policy's batch (min_batch / starvation flush)")
    ap.add_argument("--starvation-ms", type=float, default=100.0)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--share-devices", action="store_true",
                    help="allow more ranks than visible GPUs (plumbing check; gloo barrier)")
    ap.add_argument("--profile", action="store_true",
                    help="run exactly one resident-input step and exit (ncu)")
    args = ap.parse_args()
    global MODEL
    if args.model:                       # side runs only; the headline is cfg3 (large-v3)
        MODEL = args.model
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_under_torchrun(args.gpus))
    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        run_reference(args, rank, world)    # rank 0 alone; no process group needed
        return
    device, backend = pick_device(local, world, args.share_devices)
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(device)
        dist.init_process_group(backend)
    run_b200(args, rank, world, device)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
