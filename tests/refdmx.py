"""Import the UNMODIFIED reference package (`dictamux`, installed offline into
baseline/_ref, git-ignored) for tests that drive our code through the
reference's own queue / dispatch loop / server objects."""

from __future__ import annotations

import sys
from pathlib import Path

REF = Path(__file__).resolve().parent.parent / "baseline" / "_ref"
AVAILABLE = (REF / "dictamux").exists()


def load():
    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    import dictamux.backend as rb
    import dictamux.scheduler as rs
    import dictamux.vad as rv
    return rb, rs, rv


def ref_segment(rv, sid, samples, endpoint=0.0, session=None):
    return rv.SpeechSegment(segment_id=sid, session_id=session or f"sess-{sid}", samples=samples,
                            sample_rate_hz=16000, speech_start=0.0, endpoint_time=endpoint,
                            duration_s=len(samples) / 16000.0)
