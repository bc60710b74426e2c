"""Stage-by-stage encoder comparison GPU vs oracle (debug aid)."""
import sys, numpy as np, torch, ctypes as C
sys.path.insert(0, '.')
import torch.nn.functional as F
from paper_2507_01021_b200.models import WHISPER_TINY
from paper_2507_01021_b200.engine import WhisperGPU
from paper_2507_01021_b200 import _native
from oracle.whisper import WhisperOracle
from oracle.logmel import log_mel_batch
orc = WhisperOracle(WHISPER_TINY)
gpu = WhisperGPU(WHISPER_TINY, max_slots=4, max_encode_batch=2)
rng = np.random.default_rng(1)
segs = [rng.integers(-8000, 8000, size=160000, dtype=np.int16), rng.integers(-8000, 8000, size=48000, dtype=np.int16)]
mel = log_mel_batch(segs, 80)
d = 384
def oracle_stem(mel):
    w = orc.w
    x = torch.as_tensor(mel)
    c1 = F.gelu(F.conv1d(x, w["enc.conv1.w"].permute(0,2,1), w["enc.conv1.b"], padding=1))
    c2 = F.gelu(F.conv1d(c1, w["enc.conv2.w"].permute(0,2,1), w["enc.conv2.b"], stride=2, padding=1))
    return c1, c2.permute(0,2,1) + w["enc.pos"]
c1, x0 = oracle_stem(mel)
for stop in range(0, 3):
    _native.check(gpu.lib.dm_whisper_debug(gpu.handle, 4, None, stop, gpu._s))
    gpu.encode(segs, [0, 1])
    res = np.empty((2, 1500, d), np.float32); gpu.debug(5, res)
    # oracle residual after `stop` layers
    x = x0.clone()
    for i in range(stop):
        p = f"enc.l{i}"
        h = orc._ln(x, f"{p}.ln1"); qkv = orc._lin(h, f"{p}.qkv")
        q, k, v = qkv[..., :d]*0.125, qkv[..., d:2*d], qkv[..., 2*d:]
        a = orc._attn(orc._split(q), orc._split(k), orc._split(v)); am = orc._merge(a)
        x = x + orc._lin(am, f"{p}.o")
        h = orc._ln(x, f"{p}.ln2"); x = x + orc._lin(F.gelu(orc._lin(h, f"{p}.fc1")), f"{p}.fc2")
    err = np.abs(res - x.numpy())
    print("stop", stop, "resid maxerr", err.max(), "at", np.unravel_index(err.argmax(), err.shape), "scale", np.abs(x.numpy()).max())
    if stop >= 1:
        at = np.empty((2, 1500, d), np.uint16); gpu.debug(6, at)
        at = (at.astype(np.uint32) << 16).view(np.float32)
        e2 = np.abs(at - am.numpy()); print("   attn maxerr", e2.max(), np.unravel_index(e2.argmax(), e2.shape), np.abs(am.numpy()).max())
        # per position error profile
        pe = e2.max(axis=(0,2)); print("   attn err by pos block", [round(float(pe[i:i+128].max()),3) for i in range(0,1500,128)])
