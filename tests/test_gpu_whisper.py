"""End-to-end parity of the Whisper engine (encoder output, decoder logits,
greedy tokens) against the fp32 CPU oracle on identical seeded weights."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from paper_2507_01021_b200.models import WHISPER_BASE, WHISPER_TINY

pytestmark = pytest.mark.gpu


def _segments(n, durs, seed=0):
    rng = np.random.default_rng(seed)
    return [rng.integers(-8000, 8000, size=int(round(d * 16000)), dtype=np.int16)
            for d in durs[:n]]


@pytest.fixture(scope="module")
def tiny_pair(native_lib):
    from oracle.whisper import WhisperOracle
    from paper_2507_01021_b200.engine import WhisperGPU
    orc = WhisperOracle(WHISPER_TINY, seed=0)
    gpu = WhisperGPU(WHISPER_TINY, seed=0, max_slots=16, max_encode_batch=8, decode_groups=2)
    return orc, gpu


def test_encoder_output_within_bf16_tolerance(tiny_pair):
    from oracle.logmel import log_mel_batch
    orc, gpu = tiny_pair
    segs = _segments(3, [10.0, 3.0, 30.0], seed=1)
    gpu.enable_mel_tap()
    gpu.encode(segs, [0, 1, 2])
    mel = gpu.log_mel(3)
    gpu.enable_mel_tap(False)
    want_mel = log_mel_batch(segs, 80)
    assert np.abs(mel - want_mel).max() <= 1e-4 * max(1.0, np.abs(want_mel).max())
    got = gpu.encoder_output(3)
    want = orc.encode(want_mel).numpy()
    err = np.abs(got - want).max()
    assert err <= 2e-2, err


def test_greedy_tokens_match_oracle(tiny_pair):
    orc, gpu = tiny_pair
    from oracle.logmel import log_mel_batch
    durs = [10.0] * 8
    segs = _segments(8, durs, seed=2)
    caps = [32] * 8
    got = gpu.transcribe_ids(segs, caps)
    enc = orc.encode(log_mel_batch(segs, 80))
    want = [orc.greedy(enc[b], 32) for b in range(8)]
    same = sum(g == w for g, w in zip(got, want))
    assert same >= 8 * 0.99, (got, want)


def test_batch_invariance_bitwise(tiny_pair):
    """A segment decodes to identical tokens alone and inside a mixed batch
    (the reference pins text equality across batchings:
    pkg/tests/test_server.py:334-342, test_bench.py:163-168)."""
    _, gpu = tiny_pair
    segs = _segments(6, [4.0, 12.0, 7.5, 30.0, 3.0, 20.0], seed=3)
    caps = [5, 20, 9, 31, 3, 25]
    together = gpu.transcribe_ids(segs, caps)
    alone = [gpu.transcribe_ids([s], [c])[0] for s, c in zip(segs, caps)]
    assert together == alone
    assert [len(t) for t in together] == caps


def test_batch_invariance_across_mma_widths(native_lib):
    """The decode projections size their MMA N to the active rows (16-row
    granules); a segment's tokens must not depend on that width: 40 segments
    decoded together (N = 48) equal each segment decoded alone (N = 16)."""
    from paper_2507_01021_b200.engine import WhisperGPU
    gpu = WhisperGPU(WHISPER_TINY, seed=0, init_std=0.05, max_slots=64, max_encode_batch=16)
    rng = np.random.default_rng(11)
    durs = rng.uniform(3.0, 30.0, size=40)
    segs = _segments(40, list(durs), seed=12)
    caps = [int(c) for c in rng.integers(2, 9, size=40)]
    together = gpu.transcribe_ids(segs, caps)
    alone = [gpu.transcribe_ids([s], [c])[0] for s, c in zip(segs[:12], caps[:12])]
    assert together[:12] == alone
    pairs = gpu.transcribe_ids(segs[12:], caps[12:])       # 28 rows: N = 32
    assert pairs == together[12:]
    gpu.close()


def test_decoder_logits_match_oracle(tiny_pair):
    orc, gpu = tiny_pair
    from oracle.logmel import log_mel_batch
    segs = _segments(2, [6.0, 15.0], seed=4)
    gpu.debug(3)                                  # enable the logits tap (decode group 0)
    slots = [0, gpu.decode_groups]                # two slots of decode group 0 -> rows 0, 1
    gpu.encode(segs, slots)
    gpu.admit(slots, [8, 8])
    gpu.set_active(slots)
    enc = orc.encode(log_mel_batch(segs, 80))
    logits = np.empty((gpu.max_slots, WHISPER_TINY.vocab), np.float32)
    prompt = list(WHISPER_TINY.prompt)
    for step in range(6):
        gpu.step(1)
        gpu.debug(2, logits)
        _, ngen, toks = gpu.read(tokens=True)
        for b in range(2):
            fed = prompt[:min(step + 1, 4)] + toks[slots[b], :max(0, step - 3)].tolist()
            ref = orc.decoder_logits(torch.tensor([fed]), enc[b:b + 1])[0, -1].numpy()
            err = np.abs(logits[b] - ref).max()
            assert err <= 2e-2, (step, b, err)
    gpu.release(slots)
    gpu.set_active([])


def test_eot_releases_slot(native_lib):
    """Pick the EOT id the model actually emits so the EOT path runs."""
    from oracle.logmel import log_mel_batch
    from oracle.whisper import WhisperOracle
    from paper_2507_01021_b200.engine import WhisperGPU
    segs = _segments(2, [5.0, 9.0], seed=5)
    orc = WhisperOracle(WHISPER_TINY, seed=0)
    enc = orc.encode(log_mel_batch(segs, 80))
    free_run = orc.greedy(enc[0], 12)
    eot = free_run[0]
    gpu = WhisperGPU(WHISPER_TINY, seed=0, max_slots=4, max_encode_batch=2, eot=eot)
    got = gpu.transcribe_ids(segs, [12, 12])
    want = [orc.greedy(enc[b], 12, eot=eot) for b in range(2)]
    assert got == want
    assert got[0] == []
    gpu.close()


def test_overlapped_encode_matches_serial(native_lib):
    """run_jobs with the next encode group on a second stream (overlap_encode,
    longest caps first) returns the same tokens as the serial order, over
    several groups joining a running decode batch."""
    from paper_2507_01021_b200.engine import SegmentJob, WhisperGPU
    gpu = WhisperGPU(WHISPER_TINY, seed=0, init_std=0.05, max_slots=24, max_encode_batch=6,
                     first_encode_batch=4)
    durs = [3.0, 28.0, 9.0, 15.0, 4.5, 30.0, 12.0, 6.0, 21.0, 7.0, 18.0, 25.0,
            3.5, 11.0, 27.0, 5.0, 16.0, 8.0, 29.0, 10.0]
    segs = _segments(len(durs), durs, seed=7)
    caps = [max(1, int(np.ceil(d * 1.5))) for d in durs]
    jobs = lambda: [SegmentJob(i, s, c) for i, (s, c) in enumerate(zip(segs, caps))]
    gpu.overlap_encode = False
    serial = gpu.run_jobs(jobs())
    gpu.overlap_encode = True
    for _ in range(3):
        assert gpu.run_jobs(jobs()) == serial
    assert [len(serial[i]) for i in range(len(durs))] == caps


def test_decode_under_concurrent_stream_load(native_lib):
    """Decode steps sharing the SMs with another stream's kernels give the same
    tokens (regression: the LayerNorm kernel polled an mbarrier before thread 0
    had initialised it, which faulted once another stream's CTAs shared the SM)."""
    from paper_2507_01021_b200.engine import WhisperGPU
    gpu = WhisperGPU(WHISPER_TINY, seed=0, init_std=0.05, max_slots=16, max_encode_batch=8)
    segs = _segments(16, [5.0 + i for i in range(16)], seed=8)
    caps = [40] * 16
    alone = gpu.transcribe_ids(segs, caps)
    side = torch.cuda.Stream()
    a = torch.randn(4096, 4096, device="cuda", dtype=torch.bfloat16)
    for _ in range(3):
        with torch.cuda.stream(side):
            for _ in range(100):
                a = torch.tanh(a @ a * 1e-3)
        assert gpu.transcribe_ids(segs, caps) == alone
    torch.cuda.synchronize()


def test_gpu_consumer_refill_on_real_engine(native_lib):
    """GpuConsumer on the real engine with iteration-level admission: more
    segments than decode slots arrive on the reference's SegmentQueue while the
    engine decodes; every segment is routed once and its text equals the
    batch-synchronous B200Backend's (batch invariance through refills). Two
    engines on cuda:0 share the queue (the multi-GPU consumer path with the
    device of each engine made current in its thread)."""
    import threading
    import time
    from collections import Counter
    import refdmx
    if not refdmx.AVAILABLE:
        pytest.skip("reference not installed in baseline/_ref")
    _, rs, rv = refdmx.load()
    from paper_2507_01021_b200.backend import B200Backend, B200BackendConfig
    from paper_2507_01021_b200.engine import WhisperGPU
    from paper_2507_01021_b200.multiplex import Multiplexer
    from paper_2507_01021_b200.types import batch_of, make_segment
    engines = [WhisperGPU(WHISPER_TINY, seed=0, init_std=0.05, device=0, max_slots=4,
                          max_encode_batch=2, steps_per_poll=2) for _ in range(2)]
    rng = np.random.default_rng(31)
    durs = rng.uniform(1.0, 8.0, size=18)
    segs = _segments(18, list(durs), seed=32)
    routed, lock = [], threading.Lock()

    def router(r):
        with lock:
            routed.append(r)
    mux = Multiplexer(engines, rs.BatchingPolicy(kind="continuous", min_batch=1, max_batch=4),
                      rs.SegmentQueue(), router, poll_interval_ms=1.0)
    mux.start()
    for i, x in enumerate(segs):
        mux.queue.enqueue_segment(refdmx.ref_segment(rv, f"c{i}", x), rs.monotonic_ms())
        time.sleep(0.01)
    t0 = time.time()
    while len(routed) < len(segs) and time.time() - t0 < 120:
        time.sleep(0.01)
    mux.shutdown()
    assert Counter(r.segment_id for r in routed) == Counter(f"c{i}" for i in range(len(segs)))
    assert all(r.status == "ok" for r in routed)
    assert all(c.segments_done for c in mux.consumers)          # both engines served
    backend = B200Backend(B200BackendConfig(model="whisper-tiny", init_std=0.05), engine=engines[0])
    want = backend.transcribe_batch(batch_of([make_segment(f"c{i}", x) for i, x in enumerate(segs)]))
    by = {r.segment_id: r.text for r in routed}
    assert [by[w.segment_id] for w in want] == [w.text for w in want]
    for e in engines:
        e.close()
