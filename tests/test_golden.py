"""The CPU oracle pinned against committed fixtures produced by transformers
5.5.0 (scripts/make_golden.py): log-mel values, encoder outputs, greedy
tokens on the seeded tiny model. Runs on CPU only."""

from __future__ import annotations

import hashlib
import json
from pathlib import Path

import numpy as np
import pytest
import torch

from oracle.logmel import log_mel_batch
from oracle.weights import load_all_f32
from oracle.whisper import WhisperOracle
from paper_2507_01021_b200.models import WHISPER_TINY
from paper_2507_01021_b200.weights import whisper_manifest

G = Path(__file__).resolve().parent / "golden"
FIX = json.loads((G / "golden.json").read_text())


def _segments():
    z = np.load(G / "audio.npz")
    return [z[f"arr_{i}"] for i in range(len(z.files))]


@pytest.fixture(scope="module")
def mel():
    return log_mel_batch(_segments(), 80)


def test_logmel_matches_transformers_fixture(mel):
    ref = np.load(G / "mel_hf.npz")
    frames = FIX["mel_frames"]
    assert np.abs(mel[:, :, frames] - ref["mel_slices"]).max() <= 2e-5
    assert np.allclose(mel.sum(axis=(1, 2)), ref["mel_sum"], rtol=1e-6, atol=1e-2)
    assert np.allclose((mel.astype(np.float64) ** 2).sum(axis=(1, 2)), ref["mel_sumsq"], rtol=1e-6)


@pytest.mark.parametrize("std", ["0.02", "0.05"])
def test_encoder_and_tokens_match_transformers_fixture(mel, std):
    fx = FIX["tiny"][std]
    man = whisper_manifest(WHISPER_TINY, seed=0, init_std=float(std))
    w = load_all_f32(man)
    sha = hashlib.sha256(b"".join(np.ascontiguousarray(w[t.name]).tobytes()
                                  for t in man.tensors)).hexdigest()
    assert sha == fx["weights_sha256"], "seeded weight generator drifted"
    orc = WhisperOracle(WHISPER_TINY, weights=w)
    enc = orc.encode(mel)
    rows = np.load(G / f"enc_hf_std{std}.npz")["enc_rows"]
    assert np.abs(enc[:, [0, 1, 700, 1499], :].numpy() - rows).max() <= 1e-4
    assert np.allclose(enc.sum(dim=(1, 2)).numpy(), fx["enc_sum"], rtol=1e-4, atol=1e-2)
    toks = [orc.greedy(enc[b], 12) for b in range(len(mel))]
    assert toks == fx["tokens"]
