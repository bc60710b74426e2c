"""Seeded weight manifest + generator (host logic, CPU)."""

from __future__ import annotations

import numpy as np

from oracle.weights import blob_bits, tensor_bits, tensor_f32
from paper_2507_01021_b200.engine import whisper_offsets
from paper_2507_01021_b200.models import WHISPER_BASE, WHISPER_LARGE_V3, WHISPER_TINY
from paper_2507_01021_b200.weights import (ALIGN_ELEMS, splitmix64, whisper_manifest,
                                           wav2vec2_manifest)
from paper_2507_01021_b200.models import WAV2VEC2_BASE


def test_splitmix64_known_answers():
    # reference values of the published splitmix64 finaliser (seed 0 stream)
    assert splitmix64(0) == 0xE220A8397B1DCDAF
    assert splitmix64(0x9E3779B97F4A7C15) == 0x6E789E6AA1B965F4


def test_manifest_alignment_and_counts():
    for dims in (WHISPER_TINY, WHISPER_BASE, WHISPER_LARGE_V3):
        man = whisper_manifest(dims)
        offs = [t.offset for t in man.tensors]
        assert all(o % ALIGN_ELEMS == 0 for o in offs)
        assert offs == sorted(offs)
        n = sum(t.numel for t in man.tensors)
        assert man.total_elems >= n
        assert len(whisper_offsets(man, dims)) == 5 + 12 * dims.enc_layers + 4 + 18 * dims.dec_layers + 4
    # large-v3 parameter count ~1.55 B (Whisper large-v3 has 1.55 B)
    n = sum(t.numel for t in whisper_manifest(WHISPER_LARGE_V3).tensors)
    assert 1.50e9 < n < 1.60e9
    assert wav2vec2_manifest(WAV2VEC2_BASE).total_elems > 9e7


def test_generator_statistics_and_zero_ranges():
    man = whisper_manifest(WHISPER_TINY, seed=0)
    w = tensor_f32(man, "enc.l0.fc1.w")
    assert abs(float(w.mean())) < 1e-3
    assert abs(float(w.std()) - 0.02) < 1e-3
    g = tensor_f32(man, "enc.l0.ln1.g")
    assert abs(float(g.mean()) - 1.0) < 0.01
    b = tensor_f32(man, "enc.l0.qkv.b")
    d = WHISPER_TINY.d_model
    assert not b[d:2 * d].any() and b[:d].any() and b[2 * d:].any()
    xb = tensor_f32(man, "dec.xkv.b")
    for l in range(WHISPER_TINY.dec_layers):
        assert not xb[l * 2 * d:l * 2 * d + d].any()


def test_generator_deterministic_and_seeded():
    m0, m1 = whisper_manifest(WHISPER_TINY, seed=0), whisper_manifest(WHISPER_TINY, seed=1)
    a = tensor_bits(m0, m0["dec.l0.fc1.w"])
    assert np.array_equal(a, tensor_bits(m0, m0["dec.l0.fc1.w"]))
    assert not np.array_equal(a, tensor_bits(m1, m1["dec.l0.fc1.w"]))
    blob = blob_bits(m0)
    t = m0["enc.pos"]
    assert blob[t.offset:t.offset + t.numel].any()
