#!/usr/bin/env python
"""Benchmark: audio-seconds transcribed per second (RTFx) on B200.

Workload (BASELINE.json configs[1], the config the metric is quoted on that
fits one GPU): whisper-base random-init (seed 0), 64 synthetic segments per
GPU with durations uniform in [3, 30] s (loadgen-style speech = uniform int16
noise in [-8000, 8000), per-user PCG64 seeded by blake2s(f"{seed}:u{id}")),
dynamic batching (max_batch 64, target_audio_s 64*30 -> one batch), greedy
cap ceil(3.75 * duration) tokens (the sim text rate), continuous-batching
decode slots. One "step" = the whole hot path over that batch: log-mel ->
encoder -> cross-KV -> greedy decode of every segment to EOT/cap.

  value : inputs (int16 PCM) already resident in HBM when the timed region
          starts; CUDA events on the engine stream, max over ranks.
  e2e   : the public API a user calls — SegmentQueue (dynamic policy) ->
          B200Backend.transcribe_batch(batch) with host numpy PCM: pinned
          staging + H2D, kernels, D2H token reads, detokenisation.

N GPUs (torchrun): one process per GPU, each with its own 64 segments (weak
scaling, no data-path collective: segments are independent);
torch.distributed (nccl) only for the barrier and the max-over-ranks time.

`--impl reference` times the CPU oracle (the reference path has no compiled
implementation: faster-whisper/CTranslate2 are absent) on
the host cores with all threads, rank 0 only.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import math
import os
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
MODEL = "whisper-base"


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
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world: int):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


# ---------------------------------------------------------------- CPU oracle
def cpu_oracle_rtfx(segs, dims_name: str, threads: int, budget_s: float = 20.0) -> dict:
    """Time the CPU restatement (oracle/) of the full path on a bounded sample."""
    import torch
    from oracle.logmel import log_mel_batch
    from oracle.whisper import WhisperOracle
    from paper_2507_01021_b200.models import get_model
    torch.set_num_threads(threads)
    dims = get_model(dims_name)
    orc = WhisperOracle(dims, seed=0)
    audio, wall, used = 0.0, 0.0, 0
    for uid, x in segs:
        t0 = time.perf_counter()
        mel = log_mel_batch([x], dims.n_mels)
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


# ---------------------------------------------------------------- arms
def run_reference(args, rank: int, world: int) -> None:
    if rank != 0:
        return
    threads = len(os.sched_getaffinity(0))
    segs = make_workload(args.segments, 0)
    per_step = max(1, args.ref_segments_per_step)
    times, audios = [], []
    idx = 0
    for it in range(args.warmup + args.steps):
        sample = [segs[(idx + j) % len(segs)] for j in range(per_step)]
        idx += per_step
        r = cpu_oracle_rtfx(sample, MODEL, threads, budget_s=1e9)
        if it >= args.warmup:
            times.append(r["wall_s"])
            audios.append(r["audio_s"])
    value = sum(audios) / sum(times)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * sum(times) / len(times), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"cfg2: {MODEL} random-init, {args.segments} x U[3,30] s "
                               f"synthetic segments, greedy cap ceil(3.75*dur)",
                   "model": MODEL, "sample_per_step": f"{per_step} segments (rotating)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{per_step} segments per step x {args.steps} steps, "
                                   f"oracle/ (torch fp32 CPU) on {cpu_model()}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_b200(args, rank: int, world: int, local: int) -> None:
    import torch
    from paper_2507_01021_b200.backend import B200Backend, B200BackendConfig
    from paper_2507_01021_b200.engine import ResidentPCM, SegmentJob, WhisperGPU
    from paper_2507_01021_b200.models import get_model
    from paper_2507_01021_b200.multiplex import BatchingPolicy, SegmentQueue
    from paper_2507_01021_b200.types import make_segment

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dims = get_model(MODEL)
    segs = make_workload(args.segments, rank)
    audio_s = sum(len(x) for _, x in segs) / 16000.0
    eng = WhisperGPU(dims, seed=0, device=local, max_slots=min(64, args.segments),
                     max_encode_batch=args.encode_batch, steps_per_poll=args.steps_per_poll,
                     decode_groups=args.decode_groups, first_encode_batch=args.first_encode_batch,
                     overlap_encode=bool(args.overlap_encode), decode_priority=args.decode_priority)
    backend = B200Backend(B200BackendConfig(model=MODEL, device=local), engine=eng)

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
    clocks = ClockSampler(local)
    with clocks:
        step_ms = [timed(lambda: eng.run_jobs(res_jobs()))[0] for _ in range(args.steps)]
    c1 = eng.counters()
    ms = statistics.mean(step_ms)
    ms_max = max_over_ranks(ms, world, dev)
    value = world * audio_s / (ms_max / 1000.0)
    launches = c1["launches"] - c0["launches"]

    # dominant decode kernel: cross-attention over a full slot set, CUDA events
    roof = measure_roofline(eng, dims, args)
    stages = measure_stages(eng, dims, segs, offs, pcm_dev)

    # e2e through the public API (host PCM -> results)
    def e2e_once():
        q = SegmentQueue()
        for i, (uid, x) in enumerate(segs):
            q.enqueue_segment(make_segment(uid, x, session_id=uid, endpoint_time=0.0), 0.0)
        pol = BatchingPolicy(kind="dynamic", max_batch=len(segs), max_wait_ms=200.0,
                             target_audio_s=len(segs) * 30.0)
        batch = q.try_form_batch(pol, 0.0)
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

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = len(os.sched_getaffinity(0))
        r = cpu_oracle_rtfx(segs, MODEL, threads, budget_s=args.cpu_budget_s)
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
            "config": {"workload": f"cfg2: {MODEL} random-init (seed 0), {args.segments} "
                                   f"segments/GPU x U[3,30] s synthetic speech, dynamic batching "
                                   f"(one batch), greedy cap ceil(3.75*dur), 64 decode slots",
                       "model": MODEL, "segments_per_gpu": args.segments,
                       "audio_s_per_gpu": round(audio_s, 3),
                       "parallelism": f"replicas x{world} (no collective)",
                       "l2": "flushed between timed steps (256 MB write)",
                       "encode_batch": args.encode_batch, "first_encode_batch": args.first_encode_batch,
                       "overlap_encode": bool(args.overlap_encode),
                       "decode_priority": args.decode_priority,
                       "steps_per_poll": args.steps_per_poll,
                       "decode_groups": eng.decode_groups},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h),
                    "path": "SegmentQueue(dynamic) -> B200Backend.transcribe_batch (host int16)"},
            "roofline": roof, "stages": stages, "cpu_baseline": cpu, "clocks": clocks.summary(),
            "gpu_launches": launches // args.steps,
            "gpu_launches_note": "kernels per timed step (C-ABI counter; graph nodes per replay)",
        }
        print(json.dumps(line), flush=True)


def measure_stages(eng, dims, segs, offs, pcm_dev) -> dict:
    """Per-stage throughput as a fraction of its roofline (north star: log-mel
    and decode on HBM GB/s, encoder on dense bf16 TFLOP/s), each timed live
    with CUDA events on the engine stream, L2 flushed before every timed call.

      log-mel : dm_logmel over the first E workload segments; algorithmic bytes
                = true int16 PCM (2 n) + the fp32 [n_mels, 3000] features
                (SURVEY.md §8(d)).
      encoder : dm_whisper_encode of the same E segments (log-mel -> conv stem
                -> layers -> cross-KV); algorithmic FLOPs = E x (encoder +
                cross-KV) per segment, SURVEY.md §8(d).
      decode  : one greedy step with all 64 slots active (same E segments
                replicated); algorithmic bytes = decoder weights + every active
                slot's cross-KV + its self-KV up to the fed position."""
    import ctypes as C
    import json as _j
    import torch
    from paper_2507_01021_b200.engine import ResidentPCM
    peaks = _j.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    tc = float(peaks.get("bf16_tflops", 2250.0))
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

    # log-mel (K1)
    nm = dims.n_mels
    offs_d = torch.tensor([o for _, _, o in sub], dtype=torch.int64, device=dev)
    lens_d = torch.tensor([len(x) for _, x, _ in sub], dtype=torch.int32, device=dev)
    mel = torch.empty(E, nm, 3000, dtype=torch.float32, device=dev)
    from paper_2507_01021_b200 import _native
    lm = lambda: _native.check(eng.lib.dm_logmel(C.c_void_p(pcm_dev.data_ptr()),
                                                C.c_void_p(offs_d.data_ptr()),
                                                C.c_void_p(lens_d.data_ptr()), E, nm,
                                                C.c_void_p(mel.data_ptr()), eng._s))
    lm()
    lm_ms = ev_ms(lm)
    lm_bytes = sum(2 * min(len(x), 480000) for _, x, _ in sub) + E * nm * 3000 * 4
    # encoder (K2-K5)
    d, L, Ld, F = dims.d_model, dims.enc_layers, dims.dec_layers, dims.ffn
    enc_flop = (2 * nm * 3 * d * 3000 + 2 * 3 * d * d * 1500
                + L * (8 * d * d * 1500 + 4 * 1500 * 1500 * d + 4 * d * F * 1500)
                + 4 * Ld * d * d * 1500)
    jobs = [ResidentPCM(o, len(x)) for _, x, o in sub]
    slots = list(range(E))
    en = lambda: eng.encode(jobs, slots)
    en()
    en_ms = ev_ms(en)
    # decode step at 64 rows (K6)
    S = eng.max_slots
    for i in range(E, S, E):
        eng.encode(jobs[:min(E, S - i)], list(range(i, min(S, i + E))))
    allslots = list(range(S))
    eng.admit(allslots, [400] * S)
    eng.set_active(allslots)
    eng.step(8)                       # past the prompt: positions 7..
    torch.cuda.synchronize(dev)
    pos = 8
    st_ms = ev_ms(lambda: eng.step(1), reps=9)
    eng.release(allslots)
    eng.set_active([])
    torch.cuda.synchronize(dev)
    w_bytes = 2 * (Ld * (4 * d * d + 2 * d * d + 2 * d * F) + dims.vocab * d)
    x_bytes = S * Ld * 2 * 1500 * d * 2
    kv_bytes = S * Ld * 2 * d * 2 * (pos + 5)
    st_bytes = w_bytes + x_bytes + kv_bytes
    return {
        "logmel": {"bound": "hbm", "achieved": lm_bytes / (lm_ms / 1e3) / 1e9, "peak": hbm,
                   "unit": "GB/s", "frac": lm_bytes / (lm_ms / 1e3) / 1e9 / hbm,
                   "ms": lm_ms, "bytes": lm_bytes, "segments": E,
                   "note": "FFT+mel is ~27 MFLOP/segment: the kernel sits at the FP32 ridge"},
        "encoder": {"bound": "tensor", "achieved": E * enc_flop / (en_ms / 1e3) / 1e12, "peak": tc,
                    "unit": "TFLOP/s", "frac": E * enc_flop / (en_ms / 1e3) / 1e12 / tc,
                    "ms": en_ms, "flop": E * enc_flop, "segments": E,
                    "note": "whole dm_whisper_encode (log-mel + conv stem + layers + LN + cross-KV)"},
        "decode_step": {"bound": "hbm", "achieved": st_bytes / (st_ms / 1e3) / 1e9, "peak": hbm,
                        "unit": "GB/s", "frac": st_bytes / (st_ms / 1e3) / 1e9 / hbm,
                        "ms": st_ms, "bytes": st_bytes, "rows": S,
                        "note": "one CUDA-graph step: weights + cross-KV + self-KV, 64 active slots"},
        "peak_source": "MEASURED_PEAKS.json (hbm_gbs burst copy, bf16_tflops burst)" if peaks else "fallback",
    }


def measure_roofline(eng, dims, args) -> dict:
    """Cross-attention (decode, K6; cross-o projection fused in its tail) is
    the dominant HBM stream: per launch it reads every active slot's K and V
    for one layer: n_active * 2 * 1500 * d bf16 (SURVEY.md §8(d):
    L*2*1500*d*2 B per segment per step). The 2*d*d B cross-o weight slices
    (L2-resident across the batch) are not counted."""
    import json as _j
    peaks = _j.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    peak = float(peaks.get("hbm_gbs", 6650.0))
    S = eng.max_slots
    # fill all slots with a resident segment so the kernel runs at full batch
    seg = np.random.default_rng(0).integers(-8000, 8000, size=160000, dtype=np.int16)
    slots = list(range(S))
    for i in range(0, S, eng.max_encode_batch):
        chunk = slots[i:i + eng.max_encode_batch]
        eng.encode([seg] * len(chunk), chunk)
    eng.admit(slots, [8] * S)
    eng.set_active(slots)
    eng.step(1)                      # q for the cross-attention
    ms = statistics.mean(eng.time_kernel(0, layer=l, iters=20) for l in range(dims.dec_layers))
    eng.release(slots)
    eng.set_active([])
    rows = sum(1 for s in slots if s % eng.decode_groups == 0)     # decode group 0's rows
    bytes_per_launch = rows * 2 * 1500 * dims.d_model * 2
    achieved = bytes_per_launch / (ms / 1000.0) / 1e9
    traffic = None
    tf = ROOT / "profiles" / "r01_xattn_traffic_v10.json"
    if tf.exists():     # dram read+write of one ncu --set full capture (64 rows), scaled to rows
        t = _j.loads(tf.read_text())
        traffic = (t["dram_bytes_read"] + t["dram_bytes_write"]) * rows / t["rows"]
    return {"kernel": "cross_attn_kernel (decode K6, + cross-o tail)", "bound": "hbm", "achieved": achieved,
            "peak": peak, "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
            "traffic_unit": "bytes per launch (ncu dram__bytes_read+write, profiles/r01_xattn_traffic_v10.json)",
            "timing": "CUDA events on the engine stream around a graph of 20 back-to-back launches "
                      "per decoder layer at a full 64-row batch, after the timed region",
            "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst copy)" if peaks else "fallback",
            "bytes_per_launch": bytes_per_launch, "avg_launch_ms": ms,
            "per_unit": "2*1500*d*2 B per active slot per layer"}


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--segments", type=int, default=64)
    ap.add_argument("--encode-batch", type=int, default=64,
                    help="segments per encoder launch (64: the whole cfg2 batch in one encode)")
    ap.add_argument("--steps-per-poll", type=int, default=8)
    ap.add_argument("--cpu-budget-s", type=float, default=20.0)
    ap.add_argument("--ref-segments-per-step", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--decode-groups", type=int, default=None)
    ap.add_argument("--overlap-encode", type=int, default=1,
                    help="1: encode the next group on a second stream while admitted groups decode")
    ap.add_argument("--decode-priority", type=int, default=-1,
                    help="CUDA stream priority of the decode stream (-1 high, 0 normal)")
    ap.add_argument("--first-encode-batch", type=int, default=24,
                    help="segments (longest caps first) in the first encode group of an idle "
                         "engine; the rest encode on a second stream while it decodes "
                         "(measured, overlap on: 20 -> e2e 18.5k, 24 -> 18.7k, 32 -> 18.3k RTFx; "
                         "overlap off, 16: 18.1k)")
    ap.add_argument("--profile", action="store_true",
                    help="run exactly one resident-input step and exit (ncu)")
    args = ap.parse_args()
    rank, world, local = dist_env()
    if world > 1:
        import torch
        import torch.distributed as dist
        if args.impl == "b200":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl")
        else:
            dist.init_process_group("gloo")
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_b200(args, rank, world, local)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
