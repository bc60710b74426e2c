"""Greedy-token parity where the model actually listens to the audio.

At init std 0.02 random-init Whisper emits one token for every segment, so
token equality there proves little. These tests use init std 0.05, where the
greedy stream depends on the audio (tests/golden/golden.json shows distinct
streams per segment), and compare the B200 path with the fp32 CPU oracle
(oracle/whisper.py, itself pinned to transformers by tests/test_golden.py):

  * full path (GPU log-mel -> bf16 encoder -> decode) vs the oracle's fp32
    encoder + decode: identical sequences, every divergence a near-tie;
  * decode only (the oracle decodes from the GPU's own bf16 encoder output):
    isolates the decode step and its paged self-KV / cross-KV cache;
  * long decodes (cap 130 and 444) so self-KV pages 1..6 and the
    global-memory branch of the self-attention kernel (positions >= 128,
    decode.cu) are compared, not just the smem-staged first two pages.

Near-tie rule (north star: "any divergence traced to argmax near-ties"):
at the first step k where the GPU's token differs, the oracle is run
teacher-forced on the GPU's own prefix; the divergence is a near-tie when the
oracle's top-1 logit exceeds its logit for the GPU's token by at most
TIE_TOL (full path; the bf16 encoder output moves decoder logits by up to
~1e-1 at std 0.05) or TIE_TOL_DECODE (decode only: same encoder input, so
only the decode arithmetic differs). Every comparison's numbers are printed.
"""

from __future__ import annotations

import json
import os
from pathlib import Path

import numpy as np
import pytest
import torch

from paper_2507_01021_b200.models import WHISPER_BASE, WHISPER_LARGE_V3, WHISPER_TINY

pytestmark = pytest.mark.gpu

STD = 0.05
TIE_TOL = 0.25            # logit units, full path (bf16 encoder vs fp32 oracle encoder)
TIE_TOL_DECODE = 0.05     # logit units, decode only (identical encoder input)
ENC_TOL_LV3_STD05 = 4e-2  # large-v3 encoder output max-abs at std 0.05 (see the test)
REPORT = Path(os.environ.get("GRAFT_REPO_ROOT", Path(__file__).resolve().parent.parent)) / \
    "gpurun_out" / "parity_report.jsonl"


def _segments(durs, seed):
    rng = np.random.default_rng(seed)
    return [rng.integers(-8000, 8000, size=int(round(d * 16000)), dtype=np.int16) for d in durs]


def first_divergence(a, b):
    for k in range(min(len(a), len(b))):
        if a[k] != b[k]:
            return k
    return None if len(a) == len(b) else min(len(a), len(b))


def audit(orc, enc, got, want, eot, tol, label, prompt=None):
    """Classify each segment: identical, or diverging at step k with the
    oracle's teacher-forced gap (top-1 logit minus the logit of the GPU's
    token) at that step. Returns (n_identical, divergences)."""
    prompt = list(orc.dims.prompt if prompt is None else prompt)
    same, divs = 0, []
    for b, (g, w) in enumerate(zip(got, want)):
        k = first_divergence(g, w)
        if k is None:
            same += 1
            continue
        fed = torch.tensor([prompt + list(g[:k])])
        eb = enc[b]                                # [T, d] (a batch row or a list item)
        logits = orc.decoder_logits(fed, eb.reshape(1, -1, eb.shape[-1]))[0, -1]
        tok = g[k] if k < len(g) else eot
        gap = float(logits.max() - logits[tok])
        top2 = torch.topk(logits, 2).values
        divs.append({"segment": b, "step": k, "gpu_token": int(tok),
                     "oracle_token": int(torch.argmax(logits)), "gap": gap,
                     "oracle_margin": float(top2[0] - top2[1]), "near_tie": gap <= tol})
    rec = {"label": label, "segments": len(got), "identical": same,
           "identical_frac": same / max(1, len(got)), "tie_tol": tol,
           "tokens_compared": int(sum(len(w) for w in want)), "divergences": divs}
    print(json.dumps(rec))
    try:
        REPORT.parent.mkdir(exist_ok=True)
        with REPORT.open("a") as f:
            f.write(json.dumps(rec) + "\n")
    except OSError:
        pass
    return same, divs


def oracle_from_engine(dims, gpu):
    """Oracle weights sliced from the engine's device blob (bit-identical to
    the host generator: test_weight_fill_bit_exact*), to skip regenerating
    1.6 B values on the host for large-v3."""
    from oracle.weights import load_all_f32_from_bits
    from oracle.whisper import WhisperOracle
    bits = gpu.blob.cpu().numpy().view(np.uint16)
    return WhisperOracle(dims, seed=0, init_std=STD, weights=load_all_f32_from_bits(gpu.man, bits))


def gpu_encoder_out(gpu, segs):
    """The bf16 encoder output the decoder consumes, widened to fp32."""
    gpu.encode(segs, list(range(len(segs))))
    return torch.from_numpy(gpu.encoder_output(len(segs)).copy())


@pytest.fixture(scope="module")
def tiny(native_lib):
    from oracle.whisper import WhisperOracle
    from paper_2507_01021_b200.engine import WhisperGPU
    gpu = WhisperGPU(WHISPER_TINY, seed=0, init_std=STD, max_slots=16, max_encode_batch=8)
    orc = WhisperOracle(WHISPER_TINY, seed=0, init_std=STD)
    yield orc, gpu
    gpu.close()


def test_cfg1_tiny_full_path(tiny):
    """cfg1: whisper-tiny, 8 x 10 s segments, batch 8, greedy cap 32."""
    from oracle.logmel import log_mel_batch
    orc, gpu = tiny
    segs = _segments([10.0] * 8, seed=101)
    got = gpu.transcribe_ids(segs, [32] * 8)
    enc = orc.encode(log_mel_batch(segs, 80))
    want = [orc.greedy(enc[b], 32) for b in range(8)]
    assert len({tuple(w) for w in want}) > 1, "oracle streams do not depend on the audio"
    same, divs = audit(orc, enc, got, want, WHISPER_TINY.eot, TIE_TOL, "cfg1 tiny full path")
    assert all(d["near_tie"] for d in divs), divs


def test_cfg1_tiny_decode_only_long_caps(tiny):
    """Decode from the GPU's own encoder output with caps 130 and 444: self-KV
    pages 0..6 and positions >= 128 (the global-memory branch of
    self_attn_kernel) against the oracle's KV-cached greedy loop."""
    orc, gpu = tiny
    segs = _segments([12.0, 30.0, 4.0, 21.0], seed=102)
    caps = [444, 130, 200, 444]
    enc = gpu_encoder_out(gpu, segs)
    got = gpu.transcribe_ids(segs, caps)
    want = [orc.greedy(enc[b], caps[b]) for b in range(len(segs))]
    assert max(len(g) for g in got) > 400
    same, divs = audit(orc, enc, got, want, WHISPER_TINY.eot, TIE_TOL_DECODE,
                       "tiny decode-only caps 130-444")
    assert all(d["near_tie"] for d in divs), divs


def test_cfg2_base_bench_settings(native_lib):
    """whisper-base with the bench's engine settings (64 slots, encode batch
    64, first encode group 24, overlapped encode on a second stream) over the
    whole 64-segment cfg2 workload; 8 of the segments (the longest and
    shortest caps included) are compared with the oracle: full path and
    decode only."""
    import bench
    from oracle.logmel import log_mel_batch
    from paper_2507_01021_b200.engine import SegmentJob, WhisperGPU
    gpu = WhisperGPU(WHISPER_BASE, seed=0, init_std=STD, max_slots=64, max_encode_batch=64,
                     first_encode_batch=24, overlap_encode=True)
    segs = bench.make_workload(64, 0)
    caps = [bench.token_cap(len(x) / 16000.0) for _, x in segs]
    out = gpu.run_jobs([SegmentJob(i, x, c) for i, ((_, x), c) in enumerate(zip(segs, caps))])
    order = sorted(range(64), key=lambda i: caps[i])
    pick = sorted(set(order[:3] + order[-3:] + [10, 40]))
    sub = [segs[i][1] for i in pick]
    got = [out[i] for i in pick]
    assert [len(g) for g in got] == [caps[i] for i in pick]      # no EOT at std 0.05 here
    orc = oracle_from_engine(WHISPER_BASE, gpu)
    enc = orc.encode(log_mel_batch(sub, 80))
    want = [orc.greedy(enc[j], caps[i]) for j, i in enumerate(pick)]
    same, divs = audit(orc, enc, got, want, WHISPER_BASE.eot, TIE_TOL, "cfg2 base full path")
    assert all(d["near_tie"] for d in divs), divs
    enc_g = gpu_encoder_out(gpu, sub)
    want_d = [orc.greedy(enc_g[j], caps[i]) for j, i in enumerate(pick)]
    same_d, divs_d = audit(orc, enc_g, got, want_d, WHISPER_BASE.eot, TIE_TOL_DECODE,
                           "cfg2 base decode only")
    assert all(d["near_tie"] for d in divs_d), divs_d
    gpu.close()


@pytest.mark.slow
def test_cfg3_large_v3_bench_settings_and_encoder_bound(native_lib):
    """whisper-large-v3 (the bench model, cfg3) with the bench's engine
    settings (64 slots, encode batch 64, first group 24, overlapped encode)
    over the whole 64-segment bench workload; three segments (shortest,
    median and longest cap, up to 113 tokens) compared with the oracle:
    full path and decode only. The bf16 encoder output the decoder consumes
    is within ENC_TOL_LV3_STD05 + its own storage rounding (half a bf16 ulp,
    <= 2^-9 |x|) of the fp32 oracle. At std 0.05 the 32 bf16-input layers
    accumulate more error than at the product's std 0.02 (where
    tests/test_gpu_large_v3.py holds the north-star 2e-2): measured max-abs
    0.031 here vs 0.021 there."""
    import bench
    from oracle.logmel import log_mel_batch
    from paper_2507_01021_b200.engine import SegmentJob, WhisperGPU
    gpu = WhisperGPU(WHISPER_LARGE_V3, seed=0, init_std=STD, max_slots=64, max_encode_batch=64,
                     first_encode_batch=24, overlap_encode=True)
    segs = bench.make_workload(64, 0)
    caps = [bench.token_cap(len(x) / 16000.0) for _, x in segs]
    out = gpu.run_jobs([SegmentJob(i, x, c) for i, ((_, x), c) in enumerate(zip(segs, caps))])
    order = sorted(range(64), key=lambda i: caps[i])
    pick = [order[0], order[32], order[-1]]
    sub = [segs[i][1] for i in pick]
    got = [out[i] for i in pick]
    enc_g = gpu_encoder_out(gpu, sub)
    orc = oracle_from_engine(WHISPER_LARGE_V3, gpu)
    gpu.close()
    del gpu
    torch.cuda.empty_cache()
    enc = orc.encode(log_mel_batch(sub, 128))
    err = (enc_g - enc).abs()
    bound = ENC_TOL_LV3_STD05 + enc.abs() * 2.0 ** -9
    print(f"large-v3 std 0.05 bf16 encoder output: max|err| {float(err.max()):.4g}, "
          f"mean {float(err.mean()):.3g}, max(err - bound) {float((err - bound).max()):.4g}")
    want = [orc.greedy(enc[j], caps[i]) for j, i in enumerate(pick)]
    same, divs = audit(orc, enc, got, want, WHISPER_LARGE_V3.eot, TIE_TOL, "cfg3 large-v3 full path")
    assert all(d["near_tie"] for d in divs), divs
    want_d = [orc.greedy(enc_g[j], caps[i]) for j, i in enumerate(pick)]
    same_d, divs_d = audit(orc, enc_g, got, want_d, WHISPER_LARGE_V3.eot, TIE_TOL_DECODE,
                           "cfg3 large-v3 decode only")
    assert all(d["near_tie"] for d in divs_d), divs_d
    assert bool((err <= bound).all()), float((err - bound).max())


def test_slot_reuse_under_overlapped_encode(native_lib):
    """More jobs than slots with overlapped encode: freed slots are re-encoded
    on the encode stream while the decode stream may still read their cross-KV
    (the write-after-read fence in run_jobs). Tokens equal the serial order
    and the oracle's (decode only, per segment) for a sample."""
    from paper_2507_01021_b200.engine import SegmentJob, WhisperGPU
    from oracle.whisper import WhisperOracle
    gpu = WhisperGPU(WHISPER_TINY, seed=0, init_std=STD, max_slots=8, max_encode_batch=4,
                     first_encode_batch=4, steps_per_poll=2)
    rng = np.random.default_rng(104)
    durs = list(rng.uniform(3.0, 30.0, size=40))
    segs = _segments(durs, seed=105)
    caps = [int(c) for c in rng.integers(3, 40, size=40)]
    jobs = lambda: [SegmentJob(i, s, c) for i, (s, c) in enumerate(zip(segs, caps))]
    gpu.overlap_encode = False
    serial = gpu.run_jobs(jobs())
    gpu.overlap_encode = True
    for _ in range(3):
        assert gpu.run_jobs(jobs()) == serial
    orc = WhisperOracle(WHISPER_TINY, seed=0, init_std=STD)
    pick = [0, 13, 27, 39]
    enc = gpu_encoder_out(gpu, [segs[i] for i in pick])
    want = [orc.greedy(enc[j], caps[i]) for j, i in enumerate(pick)]
    same, divs = audit(orc, enc, [serial[i] for i in pick], want, WHISPER_TINY.eot,
                       TIE_TOL_DECODE, "tiny slot reuse (40 jobs, 8 slots)")
    assert all(d["near_tie"] for d in divs), divs
    gpu.close()


def test_weight_fill_bit_exact_large_v3(native_lib):
    """The device generator at large-v3 shapes (std 0.05) equals the numpy
    restatement bit for bit on a sample of tensors (every kind of init)."""
    from oracle.weights import tensor_bits
    from paper_2507_01021_b200.engine import materialize_weights
    from paper_2507_01021_b200.weights import whisper_manifest
    man = whisper_manifest(WHISPER_LARGE_V3, seed=0, init_std=STD)
    blob = materialize_weights(man, torch.device("cuda", 0), torch.cuda.Stream())
    bits = blob.cpu().numpy().view(np.uint16)
    names = ["enc.conv1.w", "enc.pos", "enc.l0.qkv.w", "enc.l0.qkv.b", "enc.l0.ln1.g",
             "enc.l31.fc2.w", "dec.embed", "dec.l31.xo.w", "dec.xkv.w", "dec.ln.b"]
    for n in names:
        t = man[n]
        assert np.array_equal(bits[t.offset:t.offset + t.numel], tensor_bits(man, t)), n


def test_prompt_tokens_with_context(tiny):
    """Listing 1's `prompt_tokens + [no_timestamps]` with previous-text
    context: <|startofprev|> + context ids + [SOT, en, transcribe,
    notimestamps] (the reference's decode_options.prompt as byte-level ids);
    decode-only parity with the oracle's greedy loop on the same prompt, and
    the backend's prompt_text wiring produces that prompt."""
    from paper_2507_01021_b200.backend import B200Backend, B200BackendConfig
    from paper_2507_01021_b200.models import byte_tokens
    orc, gpu = tiny
    prompt = WHISPER_TINY.prompt_with_context(byte_tokens("courtroom dictation"))
    assert len(prompt) == 1 + 19 + 4
    segs = _segments([9.0, 22.0, 4.0], seed=106)
    caps = [40, 60, 25]
    gpu.set_prompt(prompt)
    try:
        enc = gpu_encoder_out(gpu, segs)
        got = gpu.transcribe_ids(segs, caps)
        want = [orc.greedy(enc[b], caps[b], prompt=prompt) for b in range(3)]
        same, divs = audit(orc, enc, got, want, WHISPER_TINY.eot, TIE_TOL_DECODE,
                           "tiny prompt with context", prompt=prompt)
        assert all(d["near_tie"] for d in divs), divs
        plain = [orc.greedy(enc[b], caps[b]) for b in range(3)]
        assert want != plain                          # the context changes the decode
    finally:
        gpu.set_prompt(WHISPER_TINY.prompt)
    be = B200Backend(B200BackendConfig(model="whisper-tiny", init_std=STD, max_slots=8,
                                       max_encode_batch=4, prompt_text="courtroom dictation"))
    assert be.engine.prompt == prompt
    be.close()
