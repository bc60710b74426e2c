"""Batched GPU VAD front against the reference's own
classify_frame / ingest_frame (pkg/src/dictamux/vad.py:123-133,383-438):
bit-identical frame labels (random, silent, near-threshold and odd-length
frames) and identical segments for many interleaved sessions driven by the
reference's state machine with GPU labels."""

from __future__ import annotations

import numpy as np
import pytest

import refdmx

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not refdmx.AVAILABLE, reason="reference not installed")]


@pytest.fixture(scope="module")
def ref(native_lib):
    refdmx.load()
    import dictamux.loadgen as lg
    import dictamux.vad as rv
    from paper_2507_01021_b200.vad import GpuFrameClassifier
    return rv, lg, GpuFrameClassifier(0)


def test_labels_bit_identical(ref):
    rv, _, clf = ref
    cfg = rv.VadConfig()
    rng = np.random.default_rng(0)
    thr = cfg.energy_threshold_rms
    frames = []
    for i in range(4000):
        n = 480 if i % 7 else int(rng.integers(1, 960))
        kind = i % 4
        if kind == 0:
            f = rng.integers(-8000, 8000, size=n, dtype=np.int16)
        elif kind == 1:
            f = np.zeros(n, np.int16)
        else:     # constant amplitude near the threshold: mean_sq = a^2
            a = int(round(thr)) + int(rng.integers(-2, 3))
            f = np.full(n, a if kind == 2 else -a, np.int16)
        frames.append(f)
    got = clf.classify(frames, cfg.energy_threshold_db)
    want = np.array([rv.classify_frame(cfg, rv.AudioFrame("s", f)) is rv.FrameClass.SPEECH
                     for f in frames], np.uint8)
    assert np.array_equal(got, want)
    assert 0 < want.sum() < len(want)
    for db in (-60.0, -20.0):
        got = clf.classify(frames[:500], db)
        cfg2 = rv.VadConfig(energy_threshold_db=db)
        want = np.array([rv.classify_frame(cfg2, rv.AudioFrame("s", f)) is rv.FrameClass.SPEECH
                         for f in frames[:500]], np.uint8)
        assert np.array_equal(got, want)


def test_sessions_segment_like_the_reference(ref):
    """64 loadgen users streamed frame by frame, all sessions' frames of a
    tick labelled in one launch: the same segments as the reference."""
    rv, lg, clf = ref
    from paper_2507_01021_b200.vad import ingest_frames
    cfg = rv.VadConfig()
    users = [lg.generate_user_audio(0, f"u{i:03d}", (20.0, 45.0), 0.6) for i in range(64)]
    n = 480
    ticks = max(len(u.samples) // n for u in users)
    st_gpu = [rv.make_state(u.user_id) for u in users]
    st_ref = [rv.make_state(u.user_id) for u in users]
    segs_gpu = {u.user_id: [] for u in users}
    segs_ref = {u.user_id: [] for u in users}
    for k in range(ticks):
        work, owners = [], []
        for u, sg, sr in zip(users, st_gpu, st_ref):
            x = u.samples[k * n:(k + 1) * n]
            if len(x) < n:
                continue
            cap = (k + 1) * 30.0
            work.append((sg, rv.AudioFrame(u.user_id, x, 16000, cap)))
            owners.append(u.user_id)
            segs_ref[u.user_id] += rv.ingest_frame(sr, cfg, rv.AudioFrame(u.user_id, x, 16000, cap))
        for uid, out in zip(owners, ingest_frames(rv, clf, cfg, work)):
            segs_gpu[uid] += out
    for u, sg, sr in zip(users, st_gpu, st_ref):
        segs_gpu[u.user_id] += rv.finalize_stream(sg, cfg)
        segs_ref[u.user_id] += rv.finalize_stream(sr, cfg)
    total = 0
    for uid in segs_ref:
        a, b = segs_gpu[uid], segs_ref[uid]
        assert [s.segment_id for s in a] == [s.segment_id for s in b]
        for x, y in zip(a, b):
            assert np.array_equal(x.samples, y.samples)
            assert (x.speech_start, x.endpoint_time, x.duration_s) == \
                (y.speech_start, y.endpoint_time, y.duration_s)
        total += len(b)
    assert total > 64
    assert rv.classify_frame.__name__ == "classify_frame"       # rebinding undone
