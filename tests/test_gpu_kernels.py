"""GPU parity of the individual sm_100a kernels against the CPU oracle and
plain fp32 references (run on a B200 via `pytest -m gpu`)."""

from __future__ import annotations

import ctypes as C

import numpy as np
import pytest
import torch

from paper_2507_01021_b200 import _native
from paper_2507_01021_b200.models import WHISPER_TINY
from paper_2507_01021_b200.weights import whisper_manifest

pytestmark = pytest.mark.gpu


def _ptr(t: torch.Tensor):
    return C.c_void_p(t.data_ptr())


def test_weight_fill_bit_exact(native_lib):
    """Device weight generator == numpy restatement, bit for bit."""
    from oracle.weights import blob_bits
    from paper_2507_01021_b200.engine import materialize_weights
    man = whisper_manifest(WHISPER_TINY, seed=3)
    s = torch.cuda.Stream()
    blob = materialize_weights(man, torch.device("cuda", 0), s)
    got = blob.cpu().numpy().view(np.uint16)
    want = blob_bits(man)
    assert got.shape == want.shape
    assert np.array_equal(got, want)


@pytest.mark.parametrize("lengths", [
    (160_000, 48_000, 0, 480_000, 500_000, 77),
    (30_000,),
])
@pytest.mark.parametrize("n_mels", [80, 128])
def test_logmel_matches_oracle(native_lib, lengths, n_mels):
    from oracle.logmel import log_mel_batch
    rng = np.random.default_rng(sum(lengths) + n_mels)
    segs = [rng.integers(-8000, 8000, size=n, dtype=np.int16) for n in lengths]
    if len(segs) > 1:   # a structured (non-white) segment too
        t = np.arange(len(segs[0])) / 16000.0
        segs[0] = (3000 * np.sin(2 * np.pi * 440 * t) * (1 + np.sin(2 * np.pi * 3 * t))
                   ).astype(np.int16)
    flat = np.concatenate(segs) if sum(lengths) else np.zeros(1, np.int16)
    offs = np.cumsum([0] + [len(s) for s in segs[:-1]]).astype(np.int64)
    pcm = torch.from_numpy(flat).cuda()
    off = torch.from_numpy(offs).cuda()
    ln = torch.tensor(lengths, dtype=torch.int32).cuda()
    out = torch.empty(len(segs), n_mels, 3000, device="cuda")
    _native.call("dm_logmel", _ptr(pcm), _ptr(off), _ptr(ln), len(segs), n_mels, _ptr(out), None)
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    want = log_mel_batch(segs, n_mels)
    err = np.abs(got - want)
    # north-star tolerance: 1e-4 relative (values are O(1); use |ref| + 1 floor)
    rel = err / np.maximum(np.abs(want), 1.0)
    assert rel.max() <= 1e-4, (rel.max(), np.unravel_index(rel.argmax(), rel.shape))


@pytest.mark.parametrize("M,N,K", [(128, 128, 64), (300, 384, 384), (1500, 1536, 512),
                                   (777, 2048, 1280), (2048, 512, 2048)])
def test_tcgen05_gemm_matches_fp32(native_lib, M, N, K):
    g = torch.Generator().manual_seed(M * 7 + N + K)
    A = torch.randn(M, K, generator=g).bfloat16()
    W = torch.randn(N, K, generator=g).bfloat16()
    b = torch.randn(N, generator=g).bfloat16()
    ref = A.float() @ W.float().T + b.float()
    Ad, Wd, bd = A.cuda(), W.cuda(), b.cuda()
    out = torch.empty(M, N, device="cuda")
    _native.call("dm_gemm_bf16_f32", _ptr(Ad), _ptr(Wd), _ptr(bd), _ptr(out), M, N, K, None)
    torch.cuda.synchronize()
    err = (out.cpu() - ref).abs().max().item()
    assert err <= 1e-3 * (K ** 0.5), err


_PAIR_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_2507_01021_b200 import _native
_native.load()
g = torch.Generator().manual_seed(5)
M, N, K = 1000, 512, 2048
A = torch.randn(M, K, generator=g).bfloat16().cuda()
W = torch.randn(N, K, generator=g).bfloat16().cuda()
b = torch.randn(N, generator=g).bfloat16().cuda()
out = torch.empty(M, N, device="cuda")
_native.call("dm_gemm_bf16_f32", A.data_ptr(), W.data_ptr(), b.data_ptr(), out.data_ptr(), M, N, K, None)
torch.cuda.synchronize()
np.save(sys.argv[2], out.cpu().numpy())
"""


def test_cta_pair_gemm_bitwise_equals_single_sm(native_lib, tmp_path):
    """Long-K GEMMs run on CTA pairs (tcgen05 cta_group::2, M = 256); the
    single-SM kernel (DM_GEMM_NO_PAIR=1) issues the same per-element MMA
    sequence, so the two must agree bit for bit (batch invariance does not
    depend on which kernel a shape selects)."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = str(Path(__file__).resolve().parent.parent)
    outs = []
    for env_extra, name in (({}, "pair.npy"), ({"DM_GEMM_NO_PAIR": "1"}, "single.npy")):
        env = dict(os.environ, **env_extra)
        path = tmp_path / name
        subprocess.run([sys.executable, "-c", _PAIR_SCRIPT, root, str(path)], env=env, check=True,
                       timeout=300)
        outs.append(np.load(path))
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("n_mels", [80, 128])
def test_logmel_operand_is_bf16_of_features(native_lib, n_mels):
    """The product path's bf16 operand (pass 1 writes bf16((x+4)/4) unclamped,
    pass 2 clamps in place) is bit for bit the bf16 rounding of the fp32
    feature contract (clamp to max-8, then normalise)."""
    import ctypes as C
    from paper_2507_01021_b200 import _native
    lib = _native.load()
    rng = np.random.default_rng(7 + n_mels)
    segs = [rng.integers(-8000, 8000, size=n, dtype=np.int16) for n in (160_000, 48_000, 480_000, 1000)]
    t = np.arange(200_000) / 16000.0
    segs.append((3000 * np.sin(2 * np.pi * 440 * t)).astype(np.int16))
    dev = torch.device("cuda", 0)
    flat = torch.from_numpy(np.concatenate(segs)).to(dev)
    offs = torch.tensor(np.cumsum([0] + [len(x) for x in segs[:-1]]), dtype=torch.int64, device=dev)
    lens = torch.tensor([len(x) for x in segs], dtype=torch.int32, device=dev)
    n = len(segs)
    out = torch.empty(n, n_mels, 3000, dtype=torch.float32, device=dev)
    ldt = 64 if n_mels <= 64 else 128
    op = torch.zeros(n, 3002, ldt, dtype=torch.int16, device=dev)
    segmax = torch.empty(n, dtype=torch.int32, device=dev)
    P = lambda x: C.c_void_p(x.data_ptr())
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    _native.check(lib.dm_logmel(P(flat), P(offs), P(lens), n, n_mels, P(out), s))
    _native.check(lib.dm_logmel_operand(P(flat), P(offs), P(lens), n, n_mels, P(op), P(segmax), s))
    torch.cuda.synchronize()
    want = out.to(torch.bfloat16).view(torch.int16).transpose(1, 2).cpu().numpy()
    got = op.cpu().numpy()
    assert np.array_equal(got[:, 1:3001, :n_mels], want)
    assert not got[:, 0].any() and not got[:, 3001].any() and not got[:, :, n_mels:].any()
