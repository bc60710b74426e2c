"""B200Backend honours the reference's transcribe_batch contract
(pkg/src/dictamux/backend.py:3-4,130-178; pkg/tests/test_backend.py:40-137),
checked on the host with a fake engine; and DispatchLoop turns backend
failures into per-entry error rows (scheduler.py:258-275)."""

from __future__ import annotations

import numpy as np
import pytest

from fakes import FakeEngine
from paper_2507_01021_b200.backend import (B200Backend, B200BackendConfig, detokenize,
                                           pad_or_trim)
import refdmx
from paper_2507_01021_b200.types import batch_of, make_segment


def backend(**kw):
    return B200Backend(B200BackendConfig(model="whisper-tiny", cap_tokens=4), engine=FakeEngine(**kw))


def seg(i, n=16000, rate=16000, val=None, session=None):
    rng = np.random.default_rng(i)
    x = rng.integers(-8000, 8000, size=n, dtype=np.int16) if val is None else np.full(n, val, np.int16)
    s = make_segment(f"s{i}", x, session_id=session or f"u{i}")
    s.sample_rate_hz = rate
    return s


def test_pad_or_trim_kats():
    assert len(pad_or_trim(np.zeros(0, np.int16), 30.0, 16000)) == 480_000
    x = np.arange(480_000, dtype=np.int16)
    assert pad_or_trim(x, 30.0, 16000) is x
    y = np.arange(500_000).astype(np.int16)
    assert np.array_equal(pad_or_trim(y, 30.0, 16000), y[:480_000])
    for n in (0, 1, 1999, 4000):
        assert len(pad_or_trim(np.ones(n, np.int16), 0.25, 8000)) == 2000


def test_results_in_entry_order_with_shared_time():
    b = backend()
    res = b.transcribe_batch(batch_of([seg(i) for i in range(5)]))
    assert [r.segment_id for r in res] == [f"s{i}" for i in range(5)]
    assert [r.session_id for r in res] == [f"u{i}" for i in range(5)]
    assert len({r.backend_time_ms for r in res}) == 1
    assert all(r.status == "ok" and r.text for r in res)


def test_silence_transcribes_empty():
    b = backend()
    res = b.transcribe_batch(batch_of([seg(0, val=0), seg(1), seg(2, n=0)]))
    assert res[0].text == "" and res[2].text == "" and res[1].text != ""
    assert b.engine.admitted == [1]


def test_identical_audio_identical_text_across_ids_and_batches():
    b = backend()
    a = seg(3)
    twin = make_segment("other-id", a.samples.copy(), session_id="x")
    r1 = b.transcribe_batch(batch_of([a]))[0].text
    r2 = b.transcribe_batch(batch_of([seg(9), twin, seg(4)]))[1].text
    assert r1 == r2 != ""


def test_rejects_empty_and_mixed_rates():
    b = backend()
    with pytest.raises(ValueError):
        b.transcribe_batch(batch_of([]))
    with pytest.raises(ValueError):
        b.transcribe_batch(batch_of([seg(0, rate=8000), seg(1)]))
    with pytest.raises(ValueError):
        b.transcribe_batch(batch_of([seg(0, rate=8000)]))


def test_more_entries_than_slots_all_served():
    b = backend(max_slots=3)
    res = b.transcribe_batch(batch_of([seg(i) for i in range(11)]))
    assert len(res) == 11 and all(r.text for r in res)
    assert b.engine.max_active <= 3


def test_detokenize_deterministic():
    assert detokenize([1, 2, 50257]) == detokenize([1, 2, 50257])
    assert detokenize([]) == ""
    assert detokenize([5]) != detokenize([6])


@pytest.mark.skipif(not refdmx.AVAILABLE, reason="reference not installed in baseline/_ref")
def test_dispatch_loop_converts_failures_to_error_rows():
    _, rs, _ = refdmx.load()
    eng = FakeEngine(fail_on={1})
    b = B200Backend(B200BackendConfig(model="whisper-tiny", cap_tokens=2), engine=eng)
    q = rs.SegmentQueue()
    routed = []
    loop = rs.DispatchLoop(q, rs.BatchingPolicy(max_batch=2, max_wait_ms=1.0), b, routed.append)
    loop.start()
    for i in range(4):
        q.enqueue_segment(seg(10 + i), float(i))
    import time
    time.sleep(0.3)
    loop.shutdown()
    ids = sorted(r.segment_id for r in routed)
    assert ids == [f"s{10 + i}" for i in range(4)]
    # the FakeEngine fails on job key 1 (second entry of a batch)
    assert any(r.status == "error" for r in routed)
    assert all(r.queue_wait_ms >= 0 for r in routed)


def test_failure_resets_engine_so_next_batch_is_served():
    """transcribe_batch resets the engine when a run fails (slots would keep
    their self-KV pages and every later admit would be refused)."""
    eng = FakeEngine(max_slots=2, fail_on={1})
    b = B200Backend(B200BackendConfig(model="whisper-tiny", cap_tokens=2), engine=eng)
    with pytest.raises(RuntimeError):
        b.transcribe_batch(batch_of([seg(20), seg(21)]))
    assert eng.resets == 1 and not eng.held
    out = b.transcribe_batch(batch_of([seg(22)]))
    assert out[0].status == "ok" and out[0].text
