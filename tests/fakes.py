"""Host-side test doubles (no GPU): a FakeEngine with WhisperGPU.run_jobs
semantics (slot-limited continuous batching, slots keep their pages after a
failure until reset(), a job finishes after `cap`
steps, tokens derived from the audio bytes so identical audio -> identical
ids regardless of batch mates)."""

from __future__ import annotations

import hashlib
import threading
from collections import deque

import numpy as np


class FakeEngine:
    def __init__(self, max_slots=4, max_encode_batch=2, fail_on=None, step_s=0.0):
        self.max_slots = max_slots
        self.max_encode_batch = max_encode_batch
        self.fail_on = fail_on or set()
        self.step_s = step_s
        self.admitted = []
        self.resets = 0
        self.held = set()          # slots holding self-KV pages, like WhisperGPU
        self.prompt = (50258, 50259, 50359, 50363)
        self.max_active = 0
        self.lock = threading.Lock()

    @staticmethod
    def ids_for(samples, cap):
        h = hashlib.blake2s(np.asarray(samples, np.int16).tobytes(), digest_size=16).digest()
        return [h[i % 16] * 100 + i for i in range(cap)]

    def run_jobs(self, jobs, refill=None):
        import time
        if self.held:      # the real engine refuses to admit into a slot that kept its pages
            raise RuntimeError("slot already holds pages (release it first)")
        pending = deque(jobs)
        active = {}
        results = {}
        while True:
            free = self.max_slots - len(active)
            if free and refill is not None and len(pending) < free:
                pending.extend(refill(free - len(pending)))
            while pending and len(active) < self.max_slots:
                j = pending.popleft()
                if j.key in self.fail_on:
                    raise RuntimeError(f"injected failure on {j.key}")
                active[j.key] = [j, 0]
                self.held.add(j.key)
                self.admitted.append(j.key)
            self.max_active = max(self.max_active, len(active))
            if not active:
                break
            if self.step_s:
                time.sleep(self.step_s)
            for key in list(active):
                active[key][1] += 1
                j, n = active[key]
                if n >= j.cap:
                    del active[key]
                    self.held.discard(key)
                    ids = self.ids_for(j.samples, j.cap)
                    results[key] = ids
                    if j.on_done:
                        j.on_done(key, ids)
        return results

    def set_prompt(self, tokens):
        self.prompt = tuple(tokens)

    def reset(self):
        self.resets += 1
        self.held.clear()

    def close(self):
        pass
