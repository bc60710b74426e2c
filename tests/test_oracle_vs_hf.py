"""Live cross-check of the oracle against transformers' Whisper (when it
imports): feature extractor, encoder, teacher-forced decoder logits."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from hf_bridge import build_hf_whisper, hf_available, hf_log_mel
from oracle.logmel import log_mel_batch, mel_filters, pad_or_trim
from oracle.weights import load_all_f32
from oracle.whisper import WhisperOracle
from paper_2507_01021_b200.models import WHISPER_TINY
from paper_2507_01021_b200.weights import whisper_manifest

pytestmark = pytest.mark.skipif(not hf_available(), reason="transformers not importable")


@pytest.mark.parametrize("n_mels", [80, 128])
def test_mel_filter_bank_matches_transformers(n_mels):
    from transformers.audio_utils import mel_filter_bank
    ref = mel_filter_bank(201, n_mels, 0.0, 8000.0, 16000, norm="slaney", mel_scale="slaney")
    assert np.allclose(mel_filters(n_mels), ref, rtol=1e-12, atol=1e-15)


def test_logmel_matches_feature_extractor():
    rng = np.random.default_rng(7)
    segs = [rng.integers(-8000, 8000, size=n, dtype=np.int16) for n in (16_000, 100_000, 0)]
    assert np.abs(log_mel_batch(segs, 80) - hf_log_mel(segs, 80)).max() <= 2e-5


def test_encoder_and_logits_match_transformers():
    man = whisper_manifest(WHISPER_TINY, seed=1)
    w = load_all_f32(man)
    orc = WhisperOracle(WHISPER_TINY, weights=w)
    hf = build_hf_whisper(WHISPER_TINY, w)
    rng = np.random.default_rng(1)
    mel = log_mel_batch([rng.integers(-8000, 8000, size=80_000, dtype=np.int16)], 80)
    with torch.no_grad():
        eo = orc.encode(mel)
        eh = hf.model.encoder(torch.from_numpy(mel)).last_hidden_state
        assert (eo - eh).abs().max().item() <= 1e-4
        toks = torch.tensor([list(WHISPER_TINY.prompt) + [11, 222, 3333]])
        lo = orc.decoder_logits(toks, eo)
        lh = hf(encoder_outputs=(eo,), decoder_input_ids=toks).logits
        assert (lo - lh).abs().max().item() <= 1e-4
        # incremental greedy == full-recompute greedy
        ids = orc.greedy(eo[0], 6)
        full = list(WHISPER_TINY.prompt)
        for t in ids:
            nxt = int(torch.argmax(orc.decoder_logits(torch.tensor([full]), eo)[0, -1]))
            assert nxt == t
            full.append(t)


def test_pad_or_trim_reference_semantics():
    # pkg/tests/test_backend.py:40-62 restated
    out = pad_or_trim(np.zeros(0, np.int16))
    assert len(out) == 480_000 and not out.any()
    x = np.arange(480_000, dtype=np.int16)
    assert pad_or_trim(x) is x
    y = np.arange(500_000).astype(np.int16)
    assert np.array_equal(pad_or_trim(y), y[:480_000])
