"""CPU fp32 restatement of Whisper encode + greedy generate (test only).

Follows transformers 5.5.0 `models/whisper/modeling_whisper.py`:
  * encoder `:541-648`: conv1 (k3 p1) + GELU, conv2 (k3 s2 p1) + GELU,
    + sinusoid positions (`:55-64`, `:623-625`), pre-LN layers (`:380-414`),
    final LN (`:643`); GELU is exact erf (`activations.py:318`);
  * attention `:241-357`: q = (x Wq + bq) * head_dim^-0.5 (`:310`), k has no
    bias (`:279`), softmax in fp32;
  * decoder `:417-506,650-797`: token + learned position embedding, pre-LN
    self-attn (causal) / cross-attn / MLP, final LN; tied LM head
    (`:966,971,1081`).
The greedy loop is hand-written (not `generate()`), so no logits processor
applies: prompt [SOT, en, transcribe, notimestamps] (`PAPER.md:57-59`) or a
given one (e.g. <|startofprev|> + context + that), then argmax (lowest index on
ties) until EOT or the per-segment cap.

Weights: the bf16-rounded values from the shared manifest, widened to fp32.
All activations fp32 (the GPU path keeps bf16 GEMM inputs in the encoder and
fp32 activations in the decoder; SURVEY.md §7 "Design rule").
"""

from __future__ import annotations

import math

import numpy as np
import torch
import torch.nn.functional as F

from paper_2507_01021_b200.models import WhisperDims
from paper_2507_01021_b200.weights import whisper_manifest

from .weights import load_all_f32

LN_EPS = 1e-5


class WhisperOracle:
    def __init__(self, dims: WhisperDims, seed: int = 0,
                 weights: dict[str, np.ndarray] | None = None,
                 init_std: float = 0.02):
        self.dims = dims
        self.man = whisper_manifest(dims, seed, init_std)
        raw = weights if weights is not None else load_all_f32(self.man)
        self.w = {k: torch.from_numpy(np.ascontiguousarray(v))
                  for k, v in raw.items()}

    # ---------------------------------------------------------------- utils
    def _ln(self, x, name):
        return F.layer_norm(x, (x.shape[-1],), self.w[f"{name}.g"],
                            self.w[f"{name}.b"], LN_EPS)

    def _lin(self, x, name):
        return F.linear(x, self.w[f"{name}.w"], self.w.get(f"{name}.b"))

    @staticmethod
    def _attn(q, k, v, causal=False):
        # q [B, h, Tq, hd] pre-scaled; k, v [B, h, Tk, hd]
        s = q @ k.transpose(-1, -2)
        if causal:
            tq, tk = s.shape[-2:]
            mask = torch.ones(tq, tk, dtype=torch.bool).tril(tk - tq)
            s = s.masked_fill(~mask, float("-inf"))
        return torch.softmax(s, dim=-1) @ v

    def _split(self, x):
        B, T, _ = x.shape
        h = self.dims.heads
        return x.view(B, T, h, -1).transpose(1, 2)

    def _merge(self, x):
        B, h, T, hd = x.shape
        return x.transpose(1, 2).reshape(B, T, h * hd)

    # -------------------------------------------------------------- encoder
    @torch.no_grad()
    def encode(self, mel: np.ndarray | torch.Tensor) -> torch.Tensor:
        """mel [B, n_mels, 3000] -> [B, 1500, d] fp32."""
        d = self.dims.d_model
        x = torch.as_tensor(mel, dtype=torch.float32)
        w1 = self.w["enc.conv1.w"].permute(0, 2, 1)          # [d, in, 3]
        w2 = self.w["enc.conv2.w"].permute(0, 2, 1)
        x = F.gelu(F.conv1d(x, w1, self.w["enc.conv1.b"], padding=1))
        x = F.gelu(F.conv1d(x, w2, self.w["enc.conv2.b"], stride=2,
                            padding=1))
        x = x.permute(0, 2, 1)
        x = x + self.w["enc.pos"][:x.shape[1]]
        scale = self.dims.head_dim ** -0.5
        for i in range(self.dims.enc_layers):
            p = f"enc.l{i}"
            h = self._ln(x, f"{p}.ln1")
            qkv = self._lin(h, f"{p}.qkv")
            q, k, v = qkv[..., :d] * scale, qkv[..., d:2 * d], qkv[..., 2 * d:]
            a = self._attn(self._split(q), self._split(k), self._split(v))
            x = x + self._lin(self._merge(a), f"{p}.o")
            h = self._ln(x, f"{p}.ln2")
            x = x + self._lin(F.gelu(self._lin(h, f"{p}.fc1")), f"{p}.fc2")
        return self._ln(x, "enc.ln")

    @torch.no_grad()
    def encode_length_aware(self, mel: np.ndarray | torch.Tensor, n_samples: int) -> torch.Tensor:
        """The opt-in length-aware encoder's definition: the feature
        extractor's frames of the padded window (same values and clamp), cut to
        the segment's own window of ceil(n / 320) positions (2 frames each; the
        conv sees zero padding after it) -> [len, d]."""
        n = min(int(n_samples), 480000)
        ln = max(1, min(1500, (n + 319) // 320))
        m = torch.as_tensor(mel, dtype=torch.float32).reshape(1, self.dims.n_mels, -1)
        return self.encode(m[:, :, :2 * ln])[0]

    # -------------------------------------------------------------- decoder
    def cross_kv(self, enc: torch.Tensor):
        """Per layer (k, v), each [B, h, 1500, hd]."""
        d = self.dims.d_model
        kv = F.linear(enc, self.w["dec.xkv.w"], self.w["dec.xkv.b"])
        out = []
        for l in range(self.dims.dec_layers):
            k = kv[..., l * 2 * d:l * 2 * d + d]
            v = kv[..., l * 2 * d + d:(l + 1) * 2 * d]
            out.append((self._split(k), self._split(v)))
        return out

    @torch.no_grad()
    def decoder_logits(self, tokens: torch.Tensor, enc: torch.Tensor
                       ) -> torch.Tensor:
        """Full (non-incremental) teacher-forced forward: tokens [B, T] ->
        logits [B, T, V]."""
        d = self.dims.d_model
        B, T = tokens.shape
        xkv = self.cross_kv(enc)
        x = self.w["dec.embed"][tokens] + self.w["dec.pos"][:T]
        scale = self.dims.head_dim ** -0.5
        for l in range(self.dims.dec_layers):
            p = f"dec.l{l}"
            h = self._ln(x, f"{p}.ln1")
            qkv = self._lin(h, f"{p}.qkv")
            q, k, v = qkv[..., :d] * scale, qkv[..., d:2 * d], qkv[..., 2 * d:]
            a = self._attn(self._split(q), self._split(k), self._split(v),
                           causal=True)
            x = x + self._lin(self._merge(a), f"{p}.o")
            h = self._ln(x, f"{p}.ln2")
            q = self._split(self._lin(h, f"{p}.xq") * scale)
            a = self._attn(q, *xkv[l])
            x = x + self._lin(self._merge(a), f"{p}.xo")
            h = self._ln(x, f"{p}.ln3")
            x = x + self._lin(F.gelu(self._lin(h, f"{p}.fc1")), f"{p}.fc2")
        x = self._ln(x, "dec.ln")
        return x @ self.w["dec.embed"].T

    @torch.no_grad()
    def greedy(self, enc: torch.Tensor, cap: int, eot: int | None = None,
               return_margins: bool = False, prompt=None):
        """Greedy decode of ONE segment (enc [1500, d] or [1, 1500, d]) with a
        KV cache. Returns generated ids (EOT excluded) and optionally the
        top1-top2 logit margin of every step."""
        dims = self.dims
        d = dims.d_model
        eot = dims.eot if eot is None else eot
        enc = enc.reshape(1, -1, d)
        xkv = self.cross_kv(enc)
        scale = dims.head_dim ** -0.5
        cache = [[None, None] for _ in range(dims.dec_layers)]
        prompt = list(dims.prompt if prompt is None else prompt)
        out: list[int] = []
        margins: list[float] = []
        pos = 0
        feed = prompt
        while True:
            ids = torch.tensor([feed])
            T = len(feed)
            x = self.w["dec.embed"][ids] + self.w["dec.pos"][pos:pos + T]
            for l in range(dims.dec_layers):
                p = f"dec.l{l}"
                h = self._ln(x, f"{p}.ln1")
                qkv = self._lin(h, f"{p}.qkv")
                q = self._split(qkv[..., :d] * scale)
                k = self._split(qkv[..., d:2 * d])
                v = self._split(qkv[..., 2 * d:])
                if cache[l][0] is not None:
                    k = torch.cat([cache[l][0], k], dim=2)
                    v = torch.cat([cache[l][1], v], dim=2)
                cache[l] = [k, v]
                a = self._attn(q, k, v, causal=True)
                x = x + self._lin(self._merge(a), f"{p}.o")
                h = self._ln(x, f"{p}.ln2")
                q = self._split(self._lin(h, f"{p}.xq") * scale)
                a = self._attn(q, *xkv[l])
                x = x + self._lin(self._merge(a), f"{p}.xo")
                h = self._ln(x, f"{p}.ln3")
                x = x + self._lin(F.gelu(self._lin(h, f"{p}.fc1")),
                                  f"{p}.fc2")
            pos += T
            x = self._ln(x[:, -1], "dec.ln")
            logits = (x @ self.w["dec.embed"].T)[0]
            top2 = torch.topk(logits, 2)
            nxt = int(torch.argmax(logits))      # first max on ties
            margins.append(float(top2.values[0] - top2.values[1]))
            if nxt == eot:
                break
            out.append(nxt)
            if len(out) >= cap:
                break
            feed = [nxt]
        return (out, margins) if return_margins else out

    def transcribe_ids(self, mels: np.ndarray, caps, eot: int | None = None):
        enc = self.encode(mels)
        return [self.greedy(enc[b], int(c), eot) for b, c in
                enumerate(caps)]
