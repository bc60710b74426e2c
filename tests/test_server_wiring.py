"""The reference's own DictationServer (websocket protocol, VAD, sessions,
result ordering -- pkg/src/dictamux/server.py) serving through the B200 path
via `paper_2507_01021_b200.server.dictation_server`.
Mirrors the reference's live-server tests (pkg/tests/test_server.py:328-342:
sequential round trip, mode equivalence on transcript text) with B200Backend
as the backend: a fake engine on CPU, the real engine (whisper-tiny) on GPU."""

from __future__ import annotations

import json
import threading
import time

import numpy as np
import pytest

import refdmx

pytestmark = pytest.mark.skipif(not refdmx.AVAILABLE, reason="reference not installed in baseline/_ref")
RATE = 16000


def _ref():
    refdmx.load()
    import dictamux.server as rsv
    from dictamux.backend import SimBackendConfig
    from dictamux.scheduler import BatchingPolicy
    return rsv, SimBackendConfig, BatchingPolicy


class Live:
    """A dictation server + uvicorn on an ephemeral port (like the reference's
    tests/conftest.py LiveServer), here around `dictation_server(...)`."""

    def __init__(self, dictation):
        import uvicorn
        rsv, _, _ = _ref()
        self.dictation = dictation
        self.dictation.start()
        self._uv = uvicorn.Server(uvicorn.Config(rsv.create_app(dictation), host="127.0.0.1",
                                                 port=0, log_level="error"))
        self._t = threading.Thread(target=self._uv.run, daemon=True)
        self._t.start()
        deadline = time.time() + 15
        while not self._uv.started:
            assert time.time() < deadline, "server did not start"
            time.sleep(0.01)
        self.port = self._uv.servers[0].sockets[0].getsockname()[1]
        self.url = f"ws://127.0.0.1:{self.port}/ws"

    def stop(self):
        self._uv.should_exit = True
        self._t.join(timeout=10)
        self.dictation.stop()


def speech(seconds, amp, seed=None):
    n = int(seconds * RATE)
    if seed is None:
        return np.full(n, amp, dtype="<i2").tobytes()
    rng = np.random.default_rng(seed)
    return rng.integers(-amp, amp, size=n, dtype=np.int16).astype("<i2").tobytes()


def dictate(url, stream, session_id="client", chunk=3200, timeout=60.0):
    from websockets.sync.client import connect
    events = []
    with connect(url) as ws:
        ws.send(json.dumps({"type": "start", "session_id": session_id, "sample_rate_hz": RATE}))
        for i in range(0, len(stream), chunk):
            ws.send(stream[i:i + chunk])
        ws.send(json.dumps({"type": "end"}))
        deadline = time.time() + timeout
        while time.time() < deadline:
            m = json.loads(ws.recv(timeout=timeout))
            events.append(m)
            if m["type"] in ("closed", "error"):
                break
    return events


def config(mode):
    rsv, SimBackendConfig, BatchingPolicy = _ref()
    return rsv.ServerConfig(mode=mode, policy=BatchingPolicy(kind="dynamic", max_wait_ms=40.0),
                            sim_backend=SimBackendConfig(fixed_overhead_ms=1.0, per_row_ms=1.0),
                            max_sessions=20)


STREAM = (speech(4.0, 1200, seed=1) + speech(1.0, 0) + speech(3.5, 1500, seed=2)
          + speech(1.0, 0) + speech(6.0, 900, seed=3) + speech(1.0, 0))


def _run_modes(make_backend, **kw):
    from paper_2507_01021_b200.server import dictation_server
    texts = {}
    for mode, iteration_level in (("multiplexed", True), ("multiplexed", False), ("sequential", True)):
        live = Live(dictation_server(config(mode), make_backend(), iteration_level=iteration_level, **kw))
        try:
            ev = dictate(live.url, STREAM)
        finally:
            live.stop()
        assert ev[-1]["type"] == "closed", ev[-3:]
        texts[(mode, iteration_level)] = [e["text"] for e in ev if e["type"] == "transcript"]
    return texts


def test_reference_server_modes_agree_cpu():
    from fakes import FakeEngine
    from paper_2507_01021_b200.backend import B200Backend, B200BackendConfig
    make = lambda: B200Backend(B200BackendConfig(model="whisper-tiny", cap_tokens=3),
                               engine=FakeEngine(max_slots=2))
    texts = _run_modes(make)
    first = texts[("multiplexed", True)]
    assert len(first) == 3 and all(first)
    assert all(t == first for t in texts.values()), texts


@pytest.mark.gpu
def test_reference_server_modes_agree_gpu(native_lib):
    """Sequential vs multiplexed (GpuConsumer and the reference DispatchLoop)
    through the real engine: identical transcript texts (batch invariance)."""
    from paper_2507_01021_b200.backend import B200Backend, B200BackendConfig
    make = lambda: B200Backend(B200BackendConfig(model="whisper-tiny", init_std=0.05, max_slots=8,
                                                 max_encode_batch=4))
    texts = _run_modes(make)
    first = texts[("multiplexed", True)]
    assert len(first) == 3 and all(first)
    assert all(t == first for t in texts.values()), texts
    assert len(set(first)) == 3          # audio-dependent text at std 0.05
