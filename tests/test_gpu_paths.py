"""The decode step's alternative kernel paths compute the same bits.

Several stages have two implementations chosen by active-row count or an
experiment knob: the cross-attention split merge (merge kernel,
inside the cross-o GEMV's operand builder, or the last-arriving split), fc1's
split-K merge + GELU (GELU kernel, fc2's operand builder, or the GEMV's last
CTA), and the LM head's argmax (partials + argmax kernel, or the GEMV's last
CTA). Each claims the same arithmetic in the same order; these tests decode
the same segments with every alternative forced and require identical tokens
and identical logits, alone (few-row buckets) and batched."""

from __future__ import annotations

import os

import numpy as np
import pytest

from paper_2507_01021_b200.models import WHISPER_LARGE_V3, WHISPER_TINY

pytestmark = pytest.mark.gpu

ALT = {"DM_XA_TAIL_MERGE_ROWS": "64",     # every step merges in the last split
       "DM_GV_FUSE_ROWS": "0",            # no operand builders: merge + GELU kernels
       "DM_LM_ARGMAX_EPI": "1",           # LM head argmax in the GEMV's last CTA
       "DM_FC1_TAIL_ROWS": "16"}          # fc1 split merged in the GEMV's last CTA (<= 16 rows)


def _decode(dims, segs, caps, env):
    import torch
    from paper_2507_01021_b200.engine import WhisperGPU
    saved = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        gpu = WhisperGPU(dims, seed=0, init_std=0.05, max_slots=32, max_encode_batch=8)
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    together = gpu.transcribe_ids(segs, caps)
    cnt = gpu.counters()
    per_step = cnt["launches"] / max(1, cnt["steps"])   # kernels per step (graph nodes)
    alone = [gpu.transcribe_ids([s], [c])[0] for s, c in zip(segs[:2], caps[:2])]
    gpu.debug(3)                                  # logits tap (decode group 0 rows)
    gpu.transcribe_ids(segs[:1], caps[:1])
    logits = gpu.debug(2, np.zeros((64, dims.vocab), np.float32))[0].copy()
    gpu.close()
    del gpu
    torch.cuda.empty_cache()
    return together, alone, logits, per_step


@pytest.mark.parametrize("dims", [WHISPER_TINY, WHISPER_LARGE_V3], ids=["tiny", "large-v3"])
def test_alternative_paths_same_bits(native_lib, dims):
    rng = np.random.default_rng(91)
    segs = [rng.integers(-8000, 8000, size=int(rng.uniform(3, 20) * 16000), dtype=np.int16)
            for _ in range(20)]
    caps = [12] * len(segs)
    base = _decode(dims, segs, caps, {})
    alt = _decode(dims, segs, caps, ALT)
    assert base[0] == alt[0]                     # 20 segments decoded together
    assert base[1] == alt[1] == base[0][:2]      # alone (1-row steps) == batched
    np.testing.assert_array_equal(base[2], alt[2])
    assert base[3] != alt[3]                     # the knobs did switch kernels
