"""The per-GPU continuous-batching consumers (conservation, iteration-level
admission, failure isolation, multi-engine sharding) on the reference's OWN
SegmentQueue / BatchingPolicy (pkg/src/dictamux/scheduler.py, installed in
baseline/_ref), with fake engines on the host."""

from __future__ import annotations

import random
import threading
import time
from collections import Counter

import numpy as np
import pytest

import refdmx
from fakes import FakeEngine
from paper_2507_01021_b200.multiplex import GpuConsumer, Multiplexer

pytestmark = pytest.mark.skipif(not refdmx.AVAILABLE, reason="reference not installed in baseline/_ref")


@pytest.fixture(scope="module", autouse=True)
def _ref():
    global rb, rs, rv
    rb, rs, rv = refdmx.load()


def seg(sid, dur=1.0, session="s", val=None):
    n = int(dur * 16000)
    rng = np.random.default_rng(abs(hash(sid)) % (2 ** 32))
    x = rng.integers(-8000, 8000, size=n, dtype=np.int16) if val is None else np.full(n, val, np.int16)
    return refdmx.ref_segment(rv, sid, x, session=session)


def run_mux(n_gpus, segs, engines_kw=None, policy=None):
    routed = []
    lock = threading.Lock()

    def router(r):
        with lock:
            routed.append(r)
    engines = [FakeEngine(**(engines_kw or {})) for _ in range(n_gpus)]
    mux = Multiplexer(engines, policy or rs.BatchingPolicy(kind="continuous", max_batch=4, min_batch=1),
                      rs.SegmentQueue(), router, cap_fn=lambda d: max(1, int(d * 3)), poll_interval_ms=1.0)
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
    twins = [refdmx.ref_segment(rv, f"twin{i}", base.samples.copy(), session="t") for i in range(8)]
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


def test_failed_run_resets_engine_before_next_batch():
    """A failure mid-run leaves slots holding pages; the consumer resets the
    engine, so the NEXT batch is served (not wedged into error rows)."""
    routed, lock = [], threading.Lock()

    def router(r):
        with lock:
            routed.append(r)
    eng = FakeEngine(max_slots=2, fail_on={"bad"})
    q = rs.SegmentQueue()
    c = GpuConsumer(q, rs.BatchingPolicy(kind="continuous", max_batch=2, min_batch=1), eng,
                    router, cap_fn=lambda d: 2, poll_interval_ms=1.0)
    c.start()
    q.enqueue_segment(seg("ok0", 0.5), 0.0)
    q.enqueue_segment(seg("bad", 0.5), 0.0)
    t0 = time.time()
    while len(routed) < 2 and time.time() - t0 < 10:
        time.sleep(0.005)
    for i in range(3):
        q.enqueue_segment(seg(f"w{i}", 0.5), 1.0)
    while len(routed) < 5 and time.time() - t0 < 10:
        time.sleep(0.005)
    c.shutdown()
    by = {r.segment_id: r.status for r in routed}
    assert by["bad"] == "error"
    assert [by[f"w{i}"] for i in range(3)] == ["ok"] * 3
    assert eng.resets >= 1 and not eng.held


def test_refill_policy_keeps_reference_policy_fields():
    """The refill policy is the reference's own dataclass turned continuous
    (min_batch 1, max_batch = free slots), other fields preserved."""
    q = rs.SegmentQueue()
    pol = rs.BatchingPolicy(kind="dynamic", max_batch=8, max_wait_ms=50.0, target_audio_s=3.0)
    c = GpuConsumer(q, pol, FakeEngine(), lambda r: None, cap_fn=lambda d: 1)
    for i in range(5):
        q.enqueue_segment(seg(f"p{i}", 2.0), 0.0)
    jobs = c._refill(4)         # continuous: no target_audio cut at 3 s
    assert len(jobs) == 4


@pytest.mark.parametrize("eager", [True, False])
def test_idle_consumer_eager_start(eager):
    """An idle consumer with eager_start (the default) serves a lone segment at
    once; with eager_start=False it honours the policy (min_batch 8, long
    starvation flush) and keeps waiting."""
    q = rs.SegmentQueue()
    routed = []
    pol = rs.BatchingPolicy(kind="continuous", max_batch=8, min_batch=8, starvation_flush_ms=60000.0)
    c = GpuConsumer(q, pol, FakeEngine(), routed.append, cap_fn=lambda d: 1, poll_interval_ms=1.0,
                    eager_start=eager)
    c.start()
    q.enqueue_segment(seg("lone", 0.5), time.monotonic() * 1000.0)
    t0 = time.time()
    while not routed and time.time() - t0 < 1.0:
        time.sleep(0.01)
    got = [r.segment_id for r in routed]
    c.shutdown()                    # the drain serves it in any case
    assert got == (["lone"] if eager else [])
    assert [r.segment_id for r in routed] == ["lone"]
