"""In-process wiring of the B200 path into the reference's own server
(§8(b) "What calls it", option (ii)).

The reference's `DictationServer` picks its backend from
`backend_kind in {"sim", "remote"}` (`pkg/src/dictamux/server.py:214-217`,
validated at `:73-76`); "remote" ships base64 PCM16 in JSON over HTTP
(`backend.py:181-199`), ~3.6 ms of host time per segment. `dictation_server()`
returns the UNMODIFIED reference server class extended in-process instead:

  * sequential mode: the reference's `SequentialJobRunner` (`server.py:142-206`)
    drives `B200Backend.transcribe_batch` exactly as it drives SimBackend;
  * multiplexed mode: by default one `GpuConsumer` per engine pulls from the
    server's own `SegmentQueue` with iteration-level admission (continuous
    batching into free decode slots, results routed through the server's
    `route_result` the moment each segment finishes); with
    `iteration_level=False` the reference's `DispatchLoop` (`scheduler.py:220-285`)
    drives `B200Backend.transcribe_batch` one batch at a time.

Nothing in the reference changes: sessions, VAD, the websocket protocol,
result ordering and stats are the reference's code. The reference package
(`dictamux`) must be importable; this module imports it lazily.
"""

from __future__ import annotations

from typing import Sequence

from .backend import B200Backend
from .engine import WhisperGPU
from .multiplex import GpuConsumer

_CLASS = None


def _server_class():
    global _CLASS
    if _CLASS is not None:
        return _CLASS
    from dictamux.server import MULTIPLEXED, DictationServer

    class B200DictationServer(DictationServer):
        """`DictationServer` whose backend is the B200 path."""

        def __init__(self, config, backend: B200Backend, *,
                     engines: Sequence[WhisperGPU] | None = None,
                     iteration_level: bool = True, poll_interval_ms: float = 2.0):
            super().__init__(config)          # builds the configured sim/remote backend ...
            close = getattr(self.backend, "close", None)
            if close:
                close()
            self.backend = backend            # ... which the B200 path replaces
            self.engines = list(engines) if engines else [backend.engine]
            self.iteration_level = iteration_level
            self.poll_interval_ms = poll_interval_ms
            self.consumers: list[GpuConsumer] = []

        def start(self) -> None:
            if self.config.mode == MULTIPLEXED and self.iteration_level:
                self.consumers = [
                    GpuConsumer(self.queue, self.config.policy, eng, self.route_result,
                                cap_fn=self.backend.cap_for,
                                silence_is_empty=self.backend.cfg.silence_is_empty,
                                poll_interval_ms=self.poll_interval_ms,
                                name=f"b200-consumer-{i}")
                    for i, eng in enumerate(self.engines)]
                for c in self.consumers:
                    c.start()
            else:
                super().start()

        def stop(self) -> None:
            if self.consumers:
                self.queue.close()            # drain: every accepted segment is routed once
                for c in self.consumers:
                    c._stop_requested.set()
                for c in self.consumers:
                    c.join(timeout=120.0)
                self.consumers = []
            super().stop()                    # closes the backend (and its engine)

    _CLASS = B200DictationServer
    return _CLASS


def dictation_server(config, backend: B200Backend, **kw):
    """A reference `DictationServer` (unstarted) serving through `backend`.

    `config` is the reference's `ServerConfig`; its `backend_kind` is ignored
    (leave the default "sim"). Keyword arguments: `engines` (one WhisperGPU
    per GPU for multiplexed mode; default the backend's engine),
    `iteration_level` (default True), `poll_interval_ms`."""
    return _server_class()(config, backend, **kw)
