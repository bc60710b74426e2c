"""CPU fp32 restatement of the CTC encoder-only path (BASELINE.json cfg5) —
test infrastructure only.

Follows transformers 5.5.0 `models/wav2vec2/modeling_wav2vec2.py`
(wav2vec2-base: feat_extract_norm="group", do_stable_layer_norm=False):
  * input normalisation: zero mean / unit variance per segment
    (`feature_extraction_wav2vec2.py` zero_mean_unit_var_norm, eps 1e-7);
  * feature encoder `:254-324,382-420`: conv0 (1->512, k10 s5, no bias) ->
    GroupNorm(512 groups = per-channel over time, eps 1e-5) -> GELU; conv1-4
    (k3 s2), conv5-6 (k2 s2), each -> GELU;
  * feature projection `:423-436`: LayerNorm(512) -> Linear(512->768);
  * positional conv `:326-369`: Conv1d(768, 768, k128, pad 64, groups 16)
    (weight-norm folded), drop the last frame (SamePad), GELU, add;
  * encoder `:658-729`: LayerNorm, then 12 post-LN layers `:553-582`
    (attention q*head_dim^-0.5 + residual -> LN -> GELU MLP + residual -> LN);
  * ForCTC `:1605-1708`: lm_head 768->32, greedy: argmax per frame, collapse
    repeats, drop blank (id 0).
Segments are processed one at a time, unpadded (GroupNorm and the attention
span are per segment).
"""

from __future__ import annotations

import numpy as np
import torch
import torch.nn.functional as F

from paper_2507_01021_b200.models import WAV2VEC2_BASE, Wav2Vec2Dims
from paper_2507_01021_b200.weights import wav2vec2_manifest

from .weights import load_all_f32


def frames_for(n: int, dims: Wav2Vec2Dims = WAV2VEC2_BASE) -> int:
    L = n
    for k, s in zip(dims.conv_kernel, dims.conv_stride):
        if L < k:
            return 0
        L = (L - k) // s + 1
    return L


def normalize(samples_i16: np.ndarray) -> np.ndarray:
    x = np.asarray(samples_i16, np.float32) / 32768.0
    x64 = x.astype(np.float64)
    return ((x64 - x64.mean()) / np.sqrt(x64.var() + 1e-7)).astype(np.float32)


def ctc_collapse(ids, blank: int = 0) -> list[int]:
    out, prev = [], None
    for t in ids:
        t = int(t)
        if t != prev and t != blank:
            out.append(t)
        prev = t
    return out


class Wav2Vec2Oracle:
    def __init__(self, dims: Wav2Vec2Dims = WAV2VEC2_BASE, seed: int = 0,
                 weights: dict[str, np.ndarray] | None = None, init_std: float = 0.02):
        self.dims = dims
        self.man = wav2vec2_manifest(dims, seed, init_std)
        raw = weights if weights is not None else load_all_f32(self.man)
        self.w = {k: torch.from_numpy(np.ascontiguousarray(v)) for k, v in raw.items()}

    def _ln(self, x, name):
        return F.layer_norm(x, (x.shape[-1],), self.w[f"{name}.g"], self.w[f"{name}.b"],
                            self.dims.ln_eps)

    def _lin(self, x, name):
        return F.linear(x, self.w[f"{name}.w"], self.w.get(f"{name}.b"))

    @torch.no_grad()
    def features(self, samples_i16: np.ndarray) -> torch.Tensor:
        """Feature encoder output after the projection: [T', 768] (pre pos-conv)."""
        d = self.dims
        x = torch.from_numpy(normalize(samples_i16))[None, None]      # [1, 1, n]
        for i, (k, s) in enumerate(zip(d.conv_kernel, d.conv_stride)):
            w = self.w[f"fe.conv{i}.w"].permute(0, 2, 1)                # [out, in, k]
            x = F.conv1d(x, w, stride=s)
            if i == 0:
                x = F.group_norm(x, d.conv_dim[0], self.w["fe.gn.g"], self.w["fe.gn.b"], 1e-5)
            x = F.gelu(x)
        x = x[0].T                                                       # [T', 512]
        return self._lin(self._ln(x, "fp.ln"), "fp.proj")

    @torch.no_grad()
    def logits(self, samples_i16: np.ndarray) -> torch.Tensor:
        return self._lin(self.hidden(samples_i16), "head")

    @torch.no_grad()
    def hidden(self, samples_i16: np.ndarray) -> torch.Tensor:
        """Final encoder hidden states [T', 768] (input to the CTC head)."""
        d = self.dims
        h = self.features(samples_i16)                                   # [T', 768]
        g, cg = d.pos_conv_groups, d.hidden // d.pos_conv_groups
        w = self.w["pos.w"].reshape(d.hidden, d.pos_conv_kernel, cg).permute(0, 2, 1)
        pc = F.conv1d(h.T[None], w, self.w["pos.b"], padding=d.pos_conv_kernel // 2, groups=g)
        pc = F.gelu(pc[:, :, :-1])[0].T
        x = self._ln(h + pc, "enc.ln")
        H, hd = d.heads, d.head_dim
        for i in range(d.layers):
            p = f"l{i}"
            qkv = self._lin(x, f"{p}.qkv")
            q, k, v = qkv[:, :d.hidden] * hd ** -0.5, qkv[:, d.hidden:2 * d.hidden], qkv[:, 2 * d.hidden:]
            T = x.shape[0]
            q, k, v = (t.view(T, H, hd).transpose(0, 1) for t in (q, k, v))
            a = torch.softmax(q @ k.transpose(-1, -2), dim=-1) @ v
            a = a.transpose(0, 1).reshape(T, d.hidden)
            x = self._ln(x + self._lin(a, f"{p}.o"), f"{p}.ln1")
            x = self._ln(x + self._lin(F.gelu(self._lin(x, f"{p}.fc1")), f"{p}.fc2"), f"{p}.ln2")
        return x

    def transcribe_ids(self, samples_i16: np.ndarray) -> list[int]:
        if frames_for(len(samples_i16), self.dims) == 0:
            return []
        return ctc_collapse(torch.argmax(self.logits(samples_i16), dim=-1).tolist(), self.dims.blank)
