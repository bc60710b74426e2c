"""Encoder kernel durations (CUPTI via torch.profiler, not ncu) for encode
batches of E segments: python scripts/enc_kernels.py [model] [E...]"""
import collections, json, sys
sys.path.insert(0, '.')
import numpy as np, torch
from torch.profiler import profile, ProfilerActivity
from paper_2507_01021_b200.engine import WhisperGPU
from paper_2507_01021_b200.models import get_model

name = sys.argv[1] if len(sys.argv) > 1 else "whisper-large-v3"
Es = [int(x) for x in sys.argv[2:]] or [12, 64]
dims = get_model(name)
out = {}
rng = np.random.default_rng(0)
for E in Es:
    eng = WhisperGPU(dims, max_slots=E, max_encode_batch=E)
    segs = [rng.integers(-8000, 8000, size=480000, dtype=np.int16) for _ in range(E)]
    for _ in range(2):
        eng.encode(segs, list(range(E)))
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        eng.encode(segs, list(range(E)))
        torch.cuda.synchronize()
    fam = collections.defaultdict(list)
    for e in prof.events():
        if e.device_type.name == "CUDA" and e.device_time_total > 0:
            fam[e.name.split("(")[0].replace("void ", "")].append(e.device_time_total)
    out[E] = {k: {"n": len(v), "mean_us": round(sum(v) / len(v), 1), "total_ms": round(sum(v) / 1e3, 2)}
              for k, v in sorted(fam.items(), key=lambda kv: -sum(kv[1]))}
    tot = sum(sum(v) for v in fam.values()) / 1e3
    flop = E * (2 * dims.n_mels * 3 * dims.d_model * 3000 + 2 * 3 * dims.d_model ** 2 * 1500
                + dims.enc_layers * (8 * dims.d_model ** 2 * 1500 + 4 * 1500 ** 2 * dims.d_model
                                     + 4 * dims.d_model * dims.ffn * 1500)
                + 4 * dims.dec_layers * dims.d_model ** 2 * 1500)
    print(E, f"sum of kernel time {tot:.2f} ms -> {flop / tot / 1e9:.0f} TFLOP/s", json.dumps(out[E]))
    eng.close()
    del eng
    torch.cuda.empty_cache()
