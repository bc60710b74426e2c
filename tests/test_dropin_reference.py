"""Drop-in check against the UNMODIFIED reference package (installed offline
into baseline/_ref, git-ignored; skipped when absent): the reference's own
SegmentQueue / DispatchLoop / SequentialJobRunner / SpeechSegment drive
B200Backend, and its own GpuConsumer-compatible queue feeds our multiplexer.

CPU variant uses the fake engine; the gpu variant runs the real B200 path."""

from __future__ import annotations

import sys
import threading
import time
from collections import Counter
from pathlib import Path

import numpy as np
import pytest

REF = Path(__file__).resolve().parent.parent / "baseline" / "_ref"
pytestmark = pytest.mark.skipif(not (REF / "dictamux").exists(),
                                reason="reference not installed in baseline/_ref")


@pytest.fixture(scope="module")
def dmx():
    sys.path.insert(0, str(REF))
    import dictamux.backend as rb
    import dictamux.scheduler as rs
    import dictamux.vad as rv
    return rb, rs, rv


def ref_segment(rv, sid, samples, endpoint=0.0):
    return rv.SpeechSegment(segment_id=sid, session_id=f"sess-{sid}", samples=samples,
                            sample_rate_hz=16000, speech_start=0.0, endpoint_time=endpoint,
                            duration_s=len(samples) / 16000.0)


def _run_reference_dispatch(dmx, backend, n=6):
    rb, rs, rv = dmx
    rng = np.random.default_rng(5)
    q = rs.SegmentQueue()
    routed = []
    loop = rs.DispatchLoop(q, rs.BatchingPolicy(max_batch=4, max_wait_ms=5.0), backend,
                           routed.append)
    loop.start()
    segs = [ref_segment(rv, f"r{i}", rng.integers(-8000, 8000, size=16000 + 4000 * i,
                                                     dtype=np.int16), float(i))
            for i in range(n)]
    for s in segs:
        q.enqueue_segment(s, rs.monotonic_ms())
    t0 = time.time()
    while len(routed) < n and time.time() - t0 < 120:
        time.sleep(0.01)
    loop.shutdown()
    return segs, routed


def test_reference_dispatch_loop_drives_b200backend_cpu(dmx):
    from fakes import FakeEngine
    from paper_2507_01021_b200.backend import B200Backend, B200BackendConfig
    backend = B200Backend(B200BackendConfig(model="whisper-tiny", cap_tokens=3),
                          engine=FakeEngine(max_slots=2))
    segs, routed = _run_reference_dispatch(dmx, backend)
    assert Counter(r.segment_id for r in routed) == Counter(s.segment_id for s in segs)
    assert all(r.status == "ok" and r.text for r in routed)


def test_reference_queue_feeds_gpu_consumer_cpu(dmx):
    from fakes import FakeEngine
    from paper_2507_01021_b200.multiplex import GpuConsumer
    rb, rs, rv = dmx
    q = rs.SegmentQueue()                      # the reference's own queue
    routed, lock = [], threading.Lock()

    def router(r):
        with lock:
            routed.append(r)
    cons = [GpuConsumer(q, rs.BatchingPolicy(kind="continuous", max_batch=4, min_batch=1),
                        FakeEngine(max_slots=3), router, cap_fn=lambda d: 2,
                        poll_interval_ms=1.0) for _ in range(2)]
    for c in cons:
        c.start()
    rng = np.random.default_rng(1)
    segs = [ref_segment(rv, f"m{i}", rng.integers(-8000, 8000, size=8000, dtype=np.int16))
            for i in range(25)]
    for s in segs:
        q.enqueue_segment(s, rs.monotonic_ms())
    t0 = time.time()
    while len(routed) < len(segs) and time.time() - t0 < 30:
        time.sleep(0.01)
    for c in cons:
        c.shutdown()
    assert Counter(r.segment_id for r in routed) == Counter(s.segment_id for s in segs)


@pytest.mark.gpu
def test_reference_dispatch_loop_drives_b200backend_gpu(dmx, native_lib):
    from paper_2507_01021_b200.backend import B200Backend, B200BackendConfig
    backend = B200Backend(B200BackendConfig(model="whisper-tiny", cap_tokens=6, max_slots=8,
                                            max_encode_batch=4))
    segs, routed = _run_reference_dispatch(dmx, backend, n=10)
    assert Counter(r.segment_id for r in routed) == Counter(s.segment_id for s in segs)
    assert all(r.status == "ok" for r in routed)
    # batch-invariance: same text when re-run alone through the reference Batch type
    rb, rs, rv = dmx
    by = {r.segment_id: r.text for r in routed}
    s = segs[3]
    batch = rs.Batch(batch_id="solo", entries=[rs.QueueEntry(segment=s, enqueue_time=0.0)],
                     formed_at=0.0, total_audio_s=s.duration_s)
    assert backend.transcribe_batch(batch)[0].text == by[s.segment_id]
    backend.close()


@pytest.mark.gpu
def test_failure_mid_run_then_next_batch_served_gpu(dmx, native_lib):
    """A failure after admission (slots hold self-KV pages, encodes may still
    be in flight) must not wedge the real engine: transcribe_batch resets it
    and re-raises (the reference loop turns that into error rows,
    scheduler.py:258-275), and the next batch is served with the same text a
    fresh run gives."""
    from paper_2507_01021_b200.backend import B200Backend, B200BackendConfig
    rb, rs, rv = dmx
    rng = np.random.default_rng(5)
    segs = [ref_segment(rv, f"f{i}", rng.integers(-3000, 3000, size=16000 * (2 + i), dtype=np.int16))
            for i in range(6)]

    def batch(ss, name):
        return rs.Batch(batch_id=name, entries=[rs.QueueEntry(segment=s, enqueue_time=0.0) for s in ss],
                        formed_at=0.0, total_audio_s=sum(s.duration_s for s in ss))
    cfg = B200BackendConfig(model="whisper-tiny", cap_tokens=8, max_slots=4, max_encode_batch=2,
                            init_std=0.05)
    backend = B200Backend(cfg)
    eng = backend.engine
    real_step, calls = eng.step, []

    def failing_step(n):
        calls.append(n)
        if len(calls) == 2:
            raise RuntimeError("injected failure")
        return real_step(n)
    eng.step = failing_step
    with pytest.raises(RuntimeError, match="injected"):
        backend.transcribe_batch(batch(segs, "doomed"))
    eng.step = real_step
    got = [r.text for r in backend.transcribe_batch(batch(segs[:5], "after"))]
    assert all(got)
    fresh = B200Backend(cfg)
    want = [r.text for r in fresh.transcribe_batch(batch(segs[:5], "fresh"))]
    assert got == want
    fresh.close()
    backend.close()
