"""CTC path (cfg5, wav2vec2-base shape) on the B200 vs the CPU oracle:
final hidden states (bf16 tolerance), per-frame argmax, collapsed tokens,
and batch invariance across variable-length batches."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctc_pair(native_lib):
    from oracle.wav2vec2 import Wav2Vec2Oracle
    from paper_2507_01021_b200.ctc import Wav2Vec2GPU
    return Wav2Vec2Oracle(seed=0), Wav2Vec2GPU(seed=0, max_batch=8, max_samples=16000 * 10)


def _segs(seed, lens):
    rng = np.random.default_rng(seed)
    out = [rng.integers(-8000, 8000, size=n, dtype=np.int16) for n in lens]
    t = np.arange(lens[0]) / 16000.0
    out[0] = (5000 * np.sin(2 * np.pi * 220 * t) * (1 + np.sin(2 * np.pi * 3 * t))).astype(np.int16)
    return out


def _edit(a, b):
    d = list(range(len(b) + 1))
    for i, x in enumerate(a, 1):
        prev, d[0] = d[0], i
        for j, y in enumerate(b, 1):
            cur = min(d[j] + 1, d[j - 1] + 1, prev + (x != y))
            prev, d[j] = d[j], cur
    return d[len(b)]


def test_ctc_matches_oracle(ctc_pair):
    """Hidden states within bf16 tolerance; per-frame argmax identical except
    at near-ties (oracle top1-top2 margin below the logit error bound); token
    sequences identical up to those near-tie frames."""
    from oracle.wav2vec2 import frames_for
    orc, gpu = ctc_pair
    segs = _segs(1, [16000, 37000, 8000, 64000, 123457, 400])
    gpu.run(segs)
    toks = gpu.read(len(segs))
    ids, rows = gpu.frame_ids(len(segs))
    hid = gpu.hidden(len(segs))
    head_w = orc.w["head.w"].numpy()
    agree = total = same = 0
    for b, x in enumerate(segs):
        T = frames_for(len(x))
        h_ref = orc.hidden(x).numpy()
        err = float(np.abs(hid[b, :T] - h_ref).max())
        # 12 post-LN encoder layers on bf16 GEMM inputs: measured max-abs
        # 0.019-0.022 on these segments (the 1-layer-deeper analogue of the
        # Whisper encoder's 2e-2); asserted with a 25% margin
        assert err <= 2.5e-2, (b, err)
        lg = h_ref @ head_w.T + orc.w["head.b"].numpy()
        ref_ids = lg.argmax(-1)
        top2 = np.sort(lg, axis=-1)[:, -2:]
        margin = top2[:, 1] - top2[:, 0]
        # logit error bound from the hidden-state error: |dh| * ||w_row||_1
        bound = 2 * err * np.abs(head_w).sum(axis=1).max()
        bad = np.nonzero(ids[b, :T] != ref_ids)[0]
        assert (margin[bad] <= bound).all(), (b, margin[bad], bound)
        agree += T - len(bad)
        total += T
        want = orc.transcribe_ids(x)
        same += toks[b] == want
        # the GPU's collapse (repeats merged, blanks dropped) of its own frame
        # argmax is exact; vs the oracle, only flipped near-tie frames may differ
        assert toks[b] == _collapse(ids[b, :T]), b
        dist = _edit(toks[b], want)
        assert dist <= 2 * len(bad), (b, dist, len(bad))
        if not len(bad):
            assert toks[b] == want, b
        print(f"seg {b}: T={T} hidden max|err|={err:.3g} frame flips={len(bad)} "
              f"(near-tie margins <= {bound:.3g}) token edit distance={dist}")
    assert agree >= 0.99 * total, (agree, total)


def _collapse(frame_ids, blank=0):
    out, prev = [], None
    for t in frame_ids.tolist():
        if t != prev and t != blank:
            out.append(t)
        prev = t
    return out


def test_ctc_batch_invariance(ctc_pair):
    _, gpu = ctc_pair
    segs = _segs(2, [48000, 16000, 70000, 9000, 160000])
    together = gpu.transcribe_ids(segs)
    alone = [gpu.transcribe_ids([s])[0] for s in segs]
    assert together == alone
