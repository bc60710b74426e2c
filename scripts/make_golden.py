"""Generate the committed golden fixtures under tests/golden/ by running
transformers 5.5.0 (the installed third-party Whisper; faster-whisper and
CTranslate2 — the paper's library — are absent offline) on the shared seeded
weights and synthetic audio. The oracle is checked against these fixtures in
tests/test_golden.py, so the pin survives on machines without transformers.

  python scripts/make_golden.py
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from hf_bridge import build_hf_whisper, hf_log_mel  # noqa: E402
from oracle.weights import load_all_f32  # noqa: E402
from paper_2507_01021_b200.models import WHISPER_TINY  # noqa: E402
from paper_2507_01021_b200.weights import whisper_manifest  # noqa: E402

OUT = ROOT / "tests" / "golden"


def segments():
    rng = np.random.default_rng(2507)
    lens = [48_000, 0, 160_000, 500_000]
    segs = [rng.integers(-8000, 8000, size=n, dtype=np.int16) for n in lens]
    t = np.arange(64_000) / 16000.0
    segs.append((6000 * np.sin(2 * np.pi * 300 * t) * np.sin(2 * np.pi * 2 * t)).astype(np.int16))
    return segs


def greedy_hf(model, enc, prompt, cap, eot):
    ids = list(prompt)
    out = []
    with torch.no_grad():
        while True:
            logits = model(encoder_outputs=(enc,), decoder_input_ids=torch.tensor([ids])).logits
            nxt = int(torch.argmax(logits[0, -1]))
            if nxt == eot:
                break
            out.append(nxt)
            if len(out) >= cap:
                break
            ids.append(nxt)
    return out


def main():
    OUT.mkdir(parents=True, exist_ok=True)
    segs = segments()
    np.savez_compressed(OUT / "audio.npz", *segs)
    mel = hf_log_mel(segs, 80).astype(np.float32)            # [5, 80, 3000]
    frames = np.array([0, 1, 2, 150, 299, 300, 301, 999, 1000, 2999])
    fixtures = {"generator": "transformers " + __import__("transformers").__version__,
                "mel_frames": frames.tolist()}
    np.savez_compressed(OUT / "mel_hf.npz", mel_slices=mel[:, :, frames],
                        mel_sum=mel.sum(axis=(1, 2)), mel_sumsq=(mel.astype(np.float64) ** 2).sum(axis=(1, 2)))
    results = {}
    for std in (0.02, 0.05):
        man = whisper_manifest(WHISPER_TINY, seed=0, init_std=std)
        w = load_all_f32(man)
        blob_sha = hashlib.sha256(b"".join(
            np.ascontiguousarray(w[t.name]).tobytes() for t in man.tensors)).hexdigest()
        model = build_hf_whisper(WHISPER_TINY, w)
        with torch.no_grad():
            enc = model.model.encoder(torch.from_numpy(mel)).last_hidden_state
        toks = [greedy_hf(model, enc[b:b + 1], WHISPER_TINY.prompt, 12, WHISPER_TINY.eot)
                for b in range(len(segs))]
        results[str(std)] = {"weights_sha256": blob_sha, "tokens": toks,
                             "enc_sum": enc.sum(dim=(1, 2)).tolist(),
                             "enc_abs_max": enc.abs().amax(dim=(1, 2)).tolist()}
        np.savez_compressed(OUT / f"enc_hf_std{std}.npz",
                            enc_rows=enc[:, [0, 1, 700, 1499], :].numpy())
    fixtures["tiny"] = results
    (OUT / "golden.json").write_text(json.dumps(fixtures, indent=1))
    print("wrote", sorted(p.name for p in OUT.iterdir()))


if __name__ == "__main__":
    main()
