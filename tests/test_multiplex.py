"""Queue semantics mirrored from the reference (pkg/tests/test_scheduler.py)
and the per-GPU continuous-batching consumers (conservation, iteration-level
admission, failure isolation) with fake engines on the host."""

from __future__ import annotations

import random
import threading
import time
from collections import Counter

import numpy as np
import pytest

from fakes import FakeEngine
from paper_2507_01021_b200.multiplex import (CONTINUOUS, DYNAMIC, BatchingPolicy,
                                             DuplicateSegmentError, GpuConsumer, Multiplexer,
                                             QueueClosedError, SegmentQueue)
from paper_2507_01021_b200.types import make_segment


def seg(sid, dur=1.0, session="s", val=None):
    n = int(dur * 16000)
    rng = np.random.default_rng(abs(hash(sid)) % (2 ** 32))
    x = rng.integers(-8000, 8000, size=n, dtype=np.int16) if val is None else np.full(n, val, np.int16)
    return make_segment(sid, x, session_id=session)


def test_fifo_tiebreak_duplicates_closed():
    q = SegmentQueue()
    q.enqueue_segment(seg("b"), 5.0)
    q.enqueue_segment(seg("a"), 5.0)
    q.enqueue_segment(seg("c"), 1.0)
    b = q.force_batch(BatchingPolicy(max_batch=8, target_audio_s=1e9), 10.0)
    assert [e.segment.segment_id for e in b.entries] == ["c", "a", "b"]
    with pytest.raises(DuplicateSegmentError):
        q.enqueue_segment(seg("a"), 11.0)
    q.close()
    with pytest.raises(QueueClosedError):
        q.enqueue_segment(seg("z"), 12.0)


def test_dynamic_and_continuous_triggers():
    q = SegmentQueue()
    dyn = BatchingPolicy(kind=DYNAMIC, max_batch=3, max_wait_ms=100.0, target_audio_s=10.0)
    q.enqueue_segment(seg("a", 2.0), 0.0)
    assert q.try_form_batch(dyn, 50.0) is None
    assert q.try_form_batch(dyn, 100.0) is not None           # wait trigger
    for i in range(3):
        q.enqueue_segment(seg(f"d{i}", 1.0), 200.0)
    b = q.try_form_batch(dyn, 200.0)                          # depth trigger
    assert b is not None and len(b.entries) == 3
    cont = BatchingPolicy(kind=CONTINUOUS, max_batch=4, min_batch=2, starvation_flush_ms=500.0)
    q.enqueue_segment(seg("x"), 300.0)
    assert q.try_form_batch(cont, 301.0) is None
    assert q.try_form_batch(cont, 800.0) is not None           # starvation flush
    # dynamic cut at target audio
    for i in range(4):
        q.enqueue_segment(seg(f"t{i}", 4.0), 900.0)
    b = q.force_batch(BatchingPolicy(kind=DYNAMIC, max_batch=8, target_audio_s=10.0), 901.0)
    assert len(b.entries) == 2


def run_mux(n_gpus, segs, engines_kw=None, policy=None):
    routed = []
    lock = threading.Lock()

    def router(r):
        with lock:
            routed.append(r)
    engines = [FakeEngine(**(engines_kw or {})) for _ in range(n_gpus)]
    mux = Multiplexer(engines, policy or BatchingPolicy(kind=CONTINUOUS, max_batch=4, min_batch=1),
                      router, cap_fn=lambda d: max(1, int(d * 3)), poll_interval_ms=1.0)
    mux.start()
    for i, s in enumerate(segs):
        mux.queue.enqueue_segment(s, time.monotonic() * 1000.0)
        if i % 7 == 0:
            time.sleep(0.001)
    t0 = time.time()
    while len(routed) < len(segs) and time.time() - t0 < 20:
        time.sleep(0.01)
    mux.shutdown()
    return routed, engines, mux


@pytest.mark.parametrize("n_gpus", [1, 2, 4])
def test_conservation_every_segment_routed_once(n_gpus):
    segs = [seg(f"g{i}", random.Random(i).uniform(0.2, 2.0), session=f"u{i % 5}") for i in range(60)]
    routed, engines, mux = run_mux(n_gpus, segs, {"max_slots": 3})
    assert Counter(r.segment_id for r in routed) == Counter(s.segment_id for s in segs)
    assert all(r.status == "ok" for r in routed)
    assert all(e.max_active <= 3 for e in engines)
    if n_gpus > 1:   # pull-based sharding spreads work
        assert sum(1 for c in mux.consumers if c.segments_done) >= 2


def test_identical_audio_identical_text_across_gpus():
    base = seg("orig", 1.0)
    twins = [make_segment(f"twin{i}", base.samples.copy(), session_id="t") for i in range(8)]
    routed, _, _ = run_mux(2, twins, {"max_slots": 2})
    assert len({r.text for r in routed}) == 1


def test_failure_isolated_and_consumer_keeps_serving():
    segs = [seg(f"f{i}", 0.5) for i in range(12)]
    routed, engines, _ = run_mux(1, segs, {"max_slots": 2, "fail_on": {"f3"}})
    assert Counter(r.segment_id for r in routed) == Counter(s.segment_id for s in segs)
    assert any(r.status == "error" for r in routed)
    assert any(r.status == "ok" for r in routed)
    assert engines[0].resets >= 1


def test_silence_and_bad_rate_routed_without_engine():
    s0 = seg("quiet", 1.0, val=0)
    s1 = seg("loud", 1.0)
    s2 = seg("rate", 1.0)
    s2.sample_rate_hz = 8000
    routed, engines, _ = run_mux(1, [s0, s1, s2])
    by = {r.segment_id: r for r in routed}
    assert by["quiet"].text == "" and by["quiet"].status == "ok"
    assert by["rate"].status == "error"
    assert by["loud"].text
    assert engines[0].admitted == ["loud"]


def test_iteration_level_admission_refills_free_slots():
    # long segment + many short ones: shorts must be admitted while the long one runs
    segs = [seg("long", 3.0)] + [seg(f"s{i}", 0.2) for i in range(10)]
    routed, engines, _ = run_mux(1, segs, {"max_slots": 2, "step_s": 0.01})
    order = [r.segment_id for r in routed]
    assert engines[0].admitted[0] == "long"
    assert order.index("long") >= 3          # shorts entered freed slots while it decoded
    assert engines[0].max_active == 2
