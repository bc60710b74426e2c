"""Seeded random-init weight manifest shared by the GPU engine and the oracle.

Weights are random-init (there is no network for checkpoints, SURVEY.md §5
"Checkpoint / resume"). Every tensor lives in ONE flat bf16 blob at a
256-byte aligned offset; the manifest below fixes names, shapes, layouts and
the init rule. The values come from a counter-based hash generator so the
device fill kernel (`csrc/weights.cu`) and the CPU oracle
(`oracle/weights.py`) produce bit-identical bytes without shipping a 3 GB
blob:

    key     = splitmix64((seed * 0x100000001B3 + tensor_id) mod 2^64)
    h_i     = splitmix64(key + i)                      (element i)
    s_i     = sum of the four 16-bit fields of h_i     (integer, exact)
    v_i     = bf16_rne( fp32(s_i - 131070) * fp32(std*sqrt(3)/65536) + mean )

(Irwin-Hall(4) approximation of N(mean, std); every fp32 op is a single
correctly-rounded multiply/add, so numpy and CUDA agree bit for bit.)

Layouts are chosen for the GPU and documented per tensor; the oracle permutes
where PyTorch's convention differs (conv taps).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .models import MAX_TARGET_POSITIONS, N_CTX, WhisperDims, Wav2Vec2Dims

ALIGN_ELEMS = 128              # 256 bytes of bf16
MASK64 = (1 << 64) - 1
INIT_STD = 0.02


def splitmix64(x: int) -> int:
    z = (x + 0x9E3779B97F4A7C15) & MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def tensor_key(seed: int, tensor_id: int) -> int:
    return splitmix64((seed * 0x100000001B3 + tensor_id) & MASK64)


def normal_scale(std: float) -> float:
    """fp32 multiplier applied to the centred integer Irwin-Hall sum."""
    return float(np.float32(std * math.sqrt(3.0) / 65536.0))


@dataclass
class TensorSpec:
    name: str
    shape: tuple[int, ...]
    init: str                          # "normal" | "zeros" | "ones" | "host"
    std: float = INIT_STD
    mean: float = 0.0
    zero_ranges: list[tuple[int, int]] = field(default_factory=list)
    layout: str = ""
    offset: int = 0                    # element offset in the blob
    tid: int = 0

    @property
    def numel(self) -> int:
        return int(np.prod(self.shape))


@dataclass
class Manifest:
    model: str
    seed: int
    tensors: list[TensorSpec]
    total_elems: int
    init_std: float = INIT_STD

    def __getitem__(self, name: str) -> TensorSpec:
        return self._index[name]

    def __post_init__(self):
        self._index = {t.name: t for t in self.tensors}

    @property
    def nbytes(self) -> int:
        return self.total_elems * 2


def _finalize(model: str, seed: int, specs: list[TensorSpec],
              init_std: float = INIT_STD) -> Manifest:
    off = 0
    for tid, t in enumerate(specs):
        if t.init == "normal":
            t.std = init_std
        t.tid = tid
        t.offset = off
        off += (t.numel + ALIGN_ELEMS - 1) // ALIGN_ELEMS * ALIGN_ELEMS
    return Manifest(model=model, seed=seed, tensors=specs, total_elems=off,
                    init_std=init_std)


def _lin(specs, name, n_out, n_in, bias=True, zero_bias=None):
    specs.append(TensorSpec(f"{name}.w", (n_out, n_in), "normal",
                            layout="[out, in] (K-major)"))
    if bias:
        specs.append(TensorSpec(f"{name}.b", (n_out,), "normal",
                                zero_ranges=list(zero_bias or [])))


def _ln(specs, name, d):
    specs.append(TensorSpec(f"{name}.g", (d,), "normal", mean=1.0))
    specs.append(TensorSpec(f"{name}.b", (d,), "normal"))


def whisper_manifest(dims: WhisperDims, seed: int = 0,
                     init_std: float = INIT_STD) -> Manifest:
    """Whisper encoder/decoder parameters (shapes per
    `transformers/models/whisper/modeling_whisper.py:241-506,541-797`).

    Fused layouts: self-attention q|k|v is one [3d, d] matrix whose k-bias
    slice is pinned to zero (k_proj has no bias, modeling_whisper.py:279);
    the decoder's cross-attention k|v for ALL layers is one [L*2*d, d] matrix
    so the cross-KV precompute is a single GEMM. Conv weights are tap-major
    [out, tap, in] so conv1d(k=3) is an implicit GEMM with K = 3*in.
    """
    d, f, L = dims.d_model, dims.ffn, dims.enc_layers
    s: list[TensorSpec] = []
    s.append(TensorSpec("enc.conv1.w", (d, 3, dims.n_mels), "normal",
                        layout="[out, tap, in]"))
    s.append(TensorSpec("enc.conv1.b", (d,), "normal"))
    s.append(TensorSpec("enc.conv2.w", (d, 3, d), "normal",
                        layout="[out, tap, in]"))
    s.append(TensorSpec("enc.conv2.b", (d,), "normal"))
    s.append(TensorSpec("enc.pos", (N_CTX, d), "host",
                        layout="sinusoids(1500, d), modeling_whisper.py:55-64"))
    for i in range(L):
        p = f"enc.l{i}"
        _ln(s, f"{p}.ln1", d)
        _lin(s, f"{p}.qkv", 3 * d, d, zero_bias=[(d, 2 * d)])
        _lin(s, f"{p}.o", d, d)
        _ln(s, f"{p}.ln2", d)
        _lin(s, f"{p}.fc1", f, d)
        _lin(s, f"{p}.fc2", d, f)
    _ln(s, "enc.ln", d)
    Ld = dims.dec_layers
    s.append(TensorSpec("dec.embed", (dims.vocab, d), "normal",
                        layout="[vocab, d]; tied LM head"))
    s.append(TensorSpec("dec.pos", (MAX_TARGET_POSITIONS, d), "normal"))
    for i in range(Ld):
        p = f"dec.l{i}"
        _ln(s, f"{p}.ln1", d)
        _lin(s, f"{p}.qkv", 3 * d, d, zero_bias=[(d, 2 * d)])
        _lin(s, f"{p}.o", d, d)
        _ln(s, f"{p}.ln2", d)
        _lin(s, f"{p}.xq", d, d)
        _lin(s, f"{p}.xo", d, d)
        _ln(s, f"{p}.ln3", d)
        _lin(s, f"{p}.fc1", f, d)
        _lin(s, f"{p}.fc2", d, f)
    # cross k|v for all layers: rows [l*2d, l*2d+d) = k_l, [l*2d+d, (l+1)*2d) = v_l
    s.append(TensorSpec("dec.xkv.w", (Ld * 2 * d, d), "normal",
                        layout="[L*2*d, d]: per layer k rows then v rows"))
    s.append(TensorSpec("dec.xkv.b", (Ld * 2 * d,), "normal",
                        zero_ranges=[(l * 2 * d, l * 2 * d + d)
                                     for l in range(Ld)]))
    _ln(s, "dec.ln", d)
    return _finalize(dims.name, seed, s, init_std)


def wav2vec2_manifest(dims: Wav2Vec2Dims, seed: int = 0,
                      init_std: float = INIT_STD) -> Manifest:
    """wav2vec2-base CTC parameters (shapes per
    `transformers/models/wav2vec2/modeling_wav2vec2.py:254-465,466-611,
    1605-1708`). conv_bias=False; GroupNorm(512, 512) on conv layer 0 only;
    the positional conv's weight-norm is folded into one plain weight
    (weight_norm is a reparametrisation; random-init draws the effective
    weight directly). Conv weights tap-major [out, tap, in]; the grouped
    positional conv is [groups, out_per_group, tap, in_per_group]."""
    s: list[TensorSpec] = []
    cin = 1
    for i, (c, k) in enumerate(zip(dims.conv_dim, dims.conv_kernel)):
        s.append(TensorSpec(f"fe.conv{i}.w", (c, k, cin), "normal",
                            layout="[out, tap, in]"))
        cin = c
    _ln(s, "fe.gn", dims.conv_dim[0])           # GroupNorm affine
    _ln(s, "fp.ln", dims.conv_dim[-1])
    _lin(s, "fp.proj", dims.hidden, dims.conv_dim[-1])
    g = dims.pos_conv_groups
    cg = dims.hidden // g
    s.append(TensorSpec("pos.w", (g, cg, dims.pos_conv_kernel, cg), "normal",
                        layout="[group, out/g, tap, in/g]"))
    s.append(TensorSpec("pos.b", (dims.hidden,), "normal"))
    _ln(s, "enc.ln", dims.hidden)
    for i in range(dims.layers):
        p = f"l{i}"
        _lin(s, f"{p}.qkv", 3 * dims.hidden, dims.hidden)
        _lin(s, f"{p}.o", dims.hidden, dims.hidden)
        _ln(s, f"{p}.ln1", dims.hidden)
        _lin(s, f"{p}.fc1", dims.ffn, dims.hidden)
        _lin(s, f"{p}.fc2", dims.hidden, dims.ffn)
        _ln(s, f"{p}.ln2", dims.hidden)
    _lin(s, "head", dims.vocab, dims.hidden)
    return _finalize(dims.name, seed, s, init_std)


def sinusoids(length: int, channels: int, max_timescale: float = 10000.0
              ) -> np.ndarray:
    """Whisper encoder positions (`modeling_whisper.py:55-64`), computed in
    float64 and returned as float32."""
    inc = math.log(max_timescale) / (channels // 2 - 1)
    inv = np.exp(-inc * np.arange(channels // 2, dtype=np.float64))
    t = np.arange(length, dtype=np.float64)[:, None] * inv[None, :]
    return np.concatenate([np.sin(t), np.cos(t)], axis=1).astype(np.float32)


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16 bit pattern (uint16)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    rounding = ((u >> 16) & 1) + np.uint32(0x7FFF)
    return ((u + rounding) >> 16).astype(np.uint16)


def host_tensor_values(man: Manifest, spec: TensorSpec) -> np.ndarray:
    """Values for init == "host" tensors, as bf16 bits."""
    if spec.name == "enc.pos":
        return f32_to_bf16_bits(sinusoids(*spec.shape))
    raise KeyError(spec.name)
