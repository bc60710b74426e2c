"""numpy restatement of the seeded weight generator (test infrastructure only).

Bit-exact twin of `paper_2507_01021_b200/csrc/weights.cu` per the rule
documented in `paper_2507_01021_b200/weights.py`. Used to build the oracle's
fp32 weights (bf16-rounded values widened to fp32) and to check the device
fill bit for bit.
"""

from __future__ import annotations

import numpy as np

from paper_2507_01021_b200.weights import (Manifest, TensorSpec,
                                           host_tensor_values, normal_scale,
                                           tensor_key)

_C1 = np.uint64(0x9E3779B97F4A7C15)
_C2 = np.uint64(0xBF58476D1CE4E5B9)
_C3 = np.uint64(0x94D049BB133111EB)


def _splitmix64_np(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = x + _C1
        z = (z ^ (z >> np.uint64(30))) * _C2
        z = (z ^ (z >> np.uint64(27))) * _C3
        return z ^ (z >> np.uint64(31))


def tensor_bits(man: Manifest, spec: TensorSpec,
                chunk: int = 1 << 22) -> np.ndarray:
    """bf16 bit patterns (uint16) of one tensor, flat."""
    n = spec.numel
    if spec.init == "host":
        out = host_tensor_values(man, spec).reshape(-1)
    elif spec.init == "zeros":
        out = np.zeros(n, np.uint16)
    elif spec.init == "ones":
        out = np.full(n, 0x3F80, np.uint16)
    else:
        key = np.uint64(tensor_key(man.seed, spec.tid))
        scale = np.float32(normal_scale(spec.std))
        mean = np.float32(spec.mean)
        out = np.empty(n, np.uint16)
        for s0 in range(0, n, chunk):
            idx = np.arange(s0, min(n, s0 + chunk), dtype=np.uint64)
            with np.errstate(over="ignore"):
                h = _splitmix64_np(idx + key)
            m = np.uint64(0xFFFF)
            s = ((h & m) + ((h >> np.uint64(16)) & m)
                 + ((h >> np.uint64(32)) & m) + (h >> np.uint64(48)))
            z = (s.astype(np.int64) - 131070).astype(np.float32)
            v = (z * scale) + mean                       # fp32, RNE each op
            u = v.view(np.uint32)
            rnd = ((u >> np.uint32(16)) & np.uint32(1)) + np.uint32(0x7FFF)
            out[s0:s0 + len(idx)] = ((u + rnd) >> np.uint32(16)).astype(np.uint16)
    for a, b in spec.zero_ranges:
        out[a:b] = 0
    return out


def bf16_bits_to_f32(bits: np.ndarray) -> np.ndarray:
    return (bits.astype(np.uint32) << np.uint32(16)).view(np.float32)


def tensor_f32(man: Manifest, name: str) -> np.ndarray:
    spec = man[name]
    return bf16_bits_to_f32(tensor_bits(man, spec)).reshape(spec.shape)


def blob_bits(man: Manifest) -> np.ndarray:
    """The whole flat blob (uint16), padding zero."""
    out = np.zeros(man.total_elems, np.uint16)
    for spec in man.tensors:
        out[spec.offset:spec.offset + spec.numel] = tensor_bits(man, spec)
    return out


def load_all_f32(man: Manifest, threads: int | None = None) -> dict[str, np.ndarray]:
    """Every tensor as fp32. Large normal-init tensors are generated in
    chunks on a thread pool (numpy's elementwise kernels release the GIL):
    large-v3 is 1.6 B values."""
    import os
    from concurrent.futures import ThreadPoolExecutor
    threads = threads or len(os.sched_getaffinity(0))
    out = {t.name: np.empty(t.numel, np.float32) for t in man.tensors}
    chunk = 1 << 22
    work = []
    for t in man.tensors:
        if t.init == "normal" and t.numel > chunk:
            work += [(t, s0) for s0 in range(0, t.numel, chunk)]
        else:
            work.append((t, None))

    def run(item):
        t, s0 = item
        if s0 is None:
            out[t.name][:] = bf16_bits_to_f32(tensor_bits(man, t))
            return
        n = min(chunk, t.numel - s0)
        part = TensorSpec(t.name, (n,), t.init, t.std, t.mean,
                          [(max(a - s0, 0), min(b - s0, n)) for a, b in t.zero_ranges
                           if b > s0 and a < s0 + n])
        part.tid = t.tid
        bits = tensor_bits_range(man, part, s0, n)
        out[t.name][s0:s0 + n] = bf16_bits_to_f32(bits)

    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(run, work))
    return {t.name: out[t.name].reshape(t.shape) for t in man.tensors}


def tensor_bits_range(man: Manifest, spec: TensorSpec, start: int, n: int) -> np.ndarray:
    """bf16 bits of elements [start, start + n) of a normal-init tensor
    (spec.zero_ranges relative to start)."""
    key = np.uint64(tensor_key(man.seed, spec.tid))
    scale = np.float32(normal_scale(spec.std))
    mean = np.float32(spec.mean)
    idx = np.arange(start, start + n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        h = _splitmix64_np(idx + key)
    m = np.uint64(0xFFFF)
    s = ((h & m) + ((h >> np.uint64(16)) & m)
         + ((h >> np.uint64(32)) & m) + (h >> np.uint64(48)))
    z = (s.astype(np.int64) - 131070).astype(np.float32)
    v = (z * scale) + mean
    u = v.view(np.uint32)
    rnd = ((u >> np.uint32(16)) & np.uint32(1)) + np.uint32(0x7FFF)
    out = ((u + rnd) >> np.uint32(16)).astype(np.uint16)
    for a, b in spec.zero_ranges:
        out[a:b] = 0
    return out


def load_all_f32_from_bits(man: Manifest, bits: np.ndarray) -> dict[str, np.ndarray]:
    """The same fp32 tensors sliced out of a flat bf16 blob (uint16) -- e.g.
    the device blob read back, whose bytes `tests/test_gpu_kernels.py`
    checks against `tensor_bits` -- to skip regenerating billions of values
    on the host for large-v3."""
    out = {}
    for t in man.tensors:
        out[t.name] = bf16_bits_to_f32(bits[t.offset:t.offset + t.numel]).reshape(t.shape)
    return out
