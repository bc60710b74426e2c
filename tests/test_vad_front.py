"""Host logic of the batched VAD front (paper_2507_01021_b200.vad) on CPU:
ingest_frames drives the reference's state machine with externally computed
labels (here the reference's own classify_frame stands in for the GPU) and
restores the module afterwards."""

from __future__ import annotations

import numpy as np
import pytest

import refdmx

pytestmark = pytest.mark.skipif(not refdmx.AVAILABLE, reason="reference not installed")


class RefClassifier:
    def __init__(self, rv):
        self.rv = rv

    def classify(self, frames, db):
        cfg = self.rv.VadConfig(energy_threshold_db=db)
        return np.array([self.rv.classify_frame(cfg, self.rv.AudioFrame("s", f))
                         is self.rv.FrameClass.SPEECH for f in frames], np.uint8)


def test_ingest_frames_matches_serial_reference():
    refdmx.load()
    import dictamux.loadgen as lg
    import dictamux.vad as rv
    from paper_2507_01021_b200.vad import ingest_frames, threshold_sq
    cfg = rv.VadConfig()
    assert threshold_sq(cfg.energy_threshold_db) == cfg.energy_threshold_rms ** 2
    users = [lg.generate_user_audio(1, f"v{i}", (15.0, 25.0), 0.6) for i in range(6)]
    clf = RefClassifier(rv)
    original = rv.classify_frame
    a = [rv.make_state(u.user_id) for u in users]
    b = [rv.make_state(u.user_id) for u in users]
    got, want = [], []
    for k in range(min(len(u.samples) for u in users) // 480):
        work = [(s, rv.AudioFrame(u.user_id, u.samples[k * 480:(k + 1) * 480], 16000, 30.0 * k))
                for u, s in zip(users, a)]
        for out in ingest_frames(rv, clf, cfg, work):
            got += [x.segment_id for x in out]
        for u, s in zip(users, b):
            want += [x.segment_id for x in rv.ingest_frame(
                s, cfg, rv.AudioFrame(u.user_id, u.samples[k * 480:(k + 1) * 480], 16000, 30.0 * k))]
    assert got == want and got
    assert rv.classify_frame is original
