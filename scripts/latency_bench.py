#!/usr/bin/env python
"""Per-segment latency under concurrent users (BASELINE.json cfg3/cfg4):
p50/p95 of endpoint -> delivery, multiplexed (GpuConsumer per GPU, continuous
batching, the reference's own SegmentQueue) vs the single-user
sequential-batch baseline run through the reference's own
SequentialJobRunner (server.py:142-206: a session is transcribed as one job
after it ends, chunked by max_batch) with B200Backend as its backend.

Users speak in real time: speech spans U[2, 12] s of loadgen-style noise
(uniform int16 in [-8000, 8000), loadgen.py:97-98) separated by U[0.5, 3] s
silences; each span becomes one segment (a VAD segment, vad.py:90-110) whose
endpoint is its end time. Percentiles are nearest-rank (report.py:17-26).

  python scripts/latency_bench.py --model whisper-large-v3 --users 64 --session-s 60
"""

from __future__ import annotations

import argparse
import hashlib
import json
import math
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
REF = ROOT / "baseline" / "_ref"

from paper_2507_01021_b200.backend import B200Backend, B200BackendConfig  # noqa: E402
from paper_2507_01021_b200.engine import WhisperGPU  # noqa: E402
from paper_2507_01021_b200.models import get_model  # noqa: E402
from paper_2507_01021_b200.multiplex import Multiplexer  # noqa: E402
from paper_2507_01021_b200.types import make_segment  # noqa: E402


def reference_modules():
    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    import dictamux.scheduler as rs
    import dictamux.server as rsv
    return rs, rsv


def percentile(xs, q):
    s = sorted(xs)
    if not s:
        return float("nan")
    return s[max(0, min(len(s) - 1, math.ceil(q * len(s)) - 1))]


def user_session(seed, uid, session_s):
    dig = hashlib.blake2s(f"{seed}:{uid}".encode(), digest_size=8).digest()
    rng = np.random.Generator(np.random.PCG64(int.from_bytes(dig, "big")))
    t, segs = float(rng.uniform(0.2, 3.0)), []
    while t < session_s:
        dur = float(rng.uniform(2.0, 12.0))
        n = int(dur * 16000)
        segs.append((t + dur, rng.integers(-8000, 8000, size=n, dtype=np.int16)))
        t += dur + float(rng.uniform(0.5, 3.0))
    return segs


def run_multiplexed(engines, users, policy, rs, eager_start=True):
    lock = threading.Lock()
    delivered = {}

    def router(r):
        with lock:
            delivered[r.segment_id] = (time.monotonic(), r)
    mux = Multiplexer(engines, policy, rs.SegmentQueue(), router, poll_interval_ms=2.0,
                      eager_start=eager_start)
    mux.start()
    t0 = time.monotonic() + 0.5
    endpoints = {}

    def speak(uid, segs):
        for k, (end_s, x) in enumerate(segs):
            now = time.monotonic()
            if t0 + end_s > now:
                time.sleep(t0 + end_s - now)
            sid = f"{uid}:{k:04d}"
            endpoints[sid] = time.monotonic()
            mux.queue.enqueue_segment(make_segment(sid, x, session_id=uid), endpoints[sid] * 1000.0)
    threads = [threading.Thread(target=speak, args=(u, s)) for u, s in users.items()]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    total = sum(len(s) for s in users.values())
    deadline = time.monotonic() + 600
    while len(delivered) < total and time.monotonic() < deadline:
        time.sleep(0.01)
    mux.shutdown()
    lat = [(delivered[s][0] - endpoints[s]) * 1000.0 for s in endpoints if s in delivered]
    errors = sum(1 for _, r in delivered.values() if r.status != "ok")
    audio = sum(len(x) for s in users.values() for _, x in s) / 16000.0
    return {"segments": total, "delivered": len(delivered), "errors": errors,
            "audio_s": round(audio, 1), "p50_ms": percentile(lat, 0.5),
            "p95_ms": percentile(lat, 0.95), "max_ms": max(lat) if lat else None,
            "consumer_segments": [c.segments_done for c in mux.consumers]}


def run_sequential_reference(engines, segs, max_batch, dims_name):
    """One user alone through the reference's SequentialJobRunner
    (server.py:142-206) with B200Backend: the user speaks in real time, the
    session is submitted as one job when it ends, and each segment's latency
    is its delivery time minus its endpoint."""
    rs, rsv = reference_modules()
    be = B200Backend(B200BackendConfig(model=dims_name), engine=engines[0])
    done, lock = {}, threading.Lock()

    def route(r):
        with lock:
            done[r.segment_id] = (time.monotonic(), r.status)
    runner = rsv.SequentialJobRunner(be, max_batch, route)
    runner.start()
    t0 = time.monotonic()
    job, endpoints = [], {}
    for k, (end_s, x) in enumerate(segs):
        now = time.monotonic()
        if t0 + end_s > now:
            time.sleep(t0 + end_s - now)
        sid = f"seq:{k:04d}"
        endpoints[sid] = time.monotonic()
        job.append(make_segment(sid, x, session_id="seq", endpoint_time=endpoints[sid] * 1000.0))
    runner.submit(job)
    deadline = time.monotonic() + 600
    while len(done) < len(job) and time.monotonic() < deadline:
        time.sleep(0.005)
    runner.shutdown()
    lat = [(done[s][0] - endpoints[s]) * 1000.0 for s in endpoints if s in done]
    return {"segments": len(segs), "delivered": len(done),
            "errors": sum(1 for _, st in done.values() if st != "ok"),
            "p50_ms": percentile(lat, 0.5), "p95_ms": percentile(lat, 0.95),
            "runner": "dictamux.server.SequentialJobRunner (unmodified reference)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="whisper-large-v3")
    ap.add_argument("--users", type=int, default=64)
    ap.add_argument("--session-s", type=float, default=60.0)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--slots", type=int, default=64)
    ap.add_argument("--encode-batch", type=int, default=16)
    ap.add_argument("--min-batch", type=int, default=32)
    ap.add_argument("--max-batch", type=int, default=64)
    ap.add_argument("--starvation-ms", type=float, default=100.0)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--overlap-encode", type=int, default=1,
                    help="1: new arrivals encode on a second stream while admitted slots decode")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    dims = get_model(args.model)
    t = time.time()
    engines = [WhisperGPU(dims, device=g, max_slots=args.slots, max_encode_batch=args.encode_batch,
                          steps_per_poll=4, overlap_encode=bool(args.overlap_encode))
               for g in range(args.gpus)]
    init_s = time.time() - t
    users = {f"u{i:03d}": user_session(args.seed, f"u{i:03d}", args.session_s)
             for i in range(args.users)}
    # warm-up (graph capture, first encodes)
    for eng in engines:
        eng.transcribe_ids([users["u000"][0][1]] * 2, [4, 4])
    rs, _ = reference_modules()
    policy = rs.BatchingPolicy(kind="continuous", min_batch=args.min_batch, max_batch=args.max_batch,
                               starvation_flush_ms=args.starvation_ms)
    mux = run_multiplexed(engines, users, policy, rs)
    seq = run_sequential_reference(engines, users["u000"], args.max_batch, args.model)
    out = {"metric": "p50/p95 per-segment latency (endpoint -> delivery)", "unit": "ms",
           "model": args.model, "users": args.users, "session_s": args.session_s,
           "gpus": args.gpus, "policy": vars(policy), "engine_init_s": round(init_s, 1),
           "multiplexed": mux, "sequential_single_user": seq,
           "p95_below_sequential": mux["p95_ms"] < seq["p95_ms"]}
    print(json.dumps(out))
    if args.out:
        Path(args.out).write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
