"""Opt-in length-aware encoder against its oracle
definition (oracle/whisper.py `encode_length_aware`: the feature extractor's
frames cut to the segment's own ceil(n / 320)-position window, zero padding
after it; decode cross-attends only to that window). It changes results vs
the pad_or_trim contract, so it has its own parity report here."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from paper_2507_01021_b200.models import WHISPER_BASE, WHISPER_TINY

pytestmark = pytest.mark.gpu


def _segs(durs, seed):
    rng = np.random.default_rng(seed)
    return [rng.integers(-8000, 8000, size=int(round(d * 16000)), dtype=np.int16) for d in durs]


def _window(n):
    return max(1, min(1500, (min(n, 480000) + 319) // 320))


@pytest.mark.parametrize("dims", [WHISPER_TINY, WHISPER_BASE], ids=["tiny", "base"])
def test_encoder_rows_match_oracle(native_lib, dims):
    from oracle.logmel import log_mel_batch
    from oracle.whisper import WhisperOracle
    from paper_2507_01021_b200.engine import WhisperGPU
    segs = _segs([3.0, 10.2, 27.0, 31.0, 0.5], seed=201)
    gpu = WhisperGPU(dims, seed=0, max_slots=8, max_encode_batch=8, length_aware=True)
    gpu.encode(segs, list(range(len(segs))))
    rows = max(_window(len(x)) for x in segs)
    got = gpu.encoder_output(len(segs), rows=rows)
    orc = WhisperOracle(dims, seed=0)
    mel = log_mel_batch(segs, dims.n_mels)
    for i, x in enumerate(segs):
        ln = _window(len(x))
        want = orc.encode_length_aware(mel[i], len(x)).numpy()
        assert want.shape[0] == ln
        err = np.abs(got[i, :ln] - want)
        assert (err <= 2e-2 + np.abs(want) * 2.0 ** -9).all(), (i, float(err.max()))
    gpu.close()


def test_tokens_and_batch_invariance(native_lib):
    """Decode parity from the GPU's own window (oracle greedy over the same
    encoder rows; near-tie audit), and a short segment decodes identically
    alone (a short batch window) and beside a 30 s one (a 1500-row window)."""
    from oracle.whisper import WhisperOracle
    from paper_2507_01021_b200.engine import WhisperGPU
    from test_gpu_parity import TIE_TOL_DECODE, audit
    std = 0.05
    segs = _segs([4.0, 12.0, 30.0, 7.5], seed=202)
    caps = [40, 60, 90, 30]
    gpu = WhisperGPU(WHISPER_TINY, seed=0, init_std=std, max_slots=8, max_encode_batch=4,
                     length_aware=True)
    got = gpu.transcribe_ids(segs, caps)
    gpu.encode(segs, list(range(4)))
    enc = torch.from_numpy(gpu.encoder_output(4, rows=1500).copy())
    orc = WhisperOracle(WHISPER_TINY, seed=0, init_std=std)
    wins = [_window(len(x)) for x in segs]
    want = [orc.greedy(enc[i, :wins[i]], caps[i]) for i in range(4)]
    same, divs = audit(orc, [enc[i, :wins[i]] for i in range(4)], got, want, WHISPER_TINY.eot,
                       TIE_TOL_DECODE, "tiny length-aware decode only")
    assert all(d["near_tie"] for d in divs), divs
    alone = [gpu.transcribe_ids([s], [c])[0] for s, c in zip(segs, caps)]
    assert alone == got
    # the padded path differs: the window changes the result
    gpu.length_aware = False
    padded = gpu.transcribe_ids(segs[:1], caps[:1])[0]
    assert padded != got[0]
    gpu.close()
