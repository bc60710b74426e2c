"""Cross-attention kernels side by side per active-row count: the cluster
kernel (which 0) and the streaming kernel (which 9), each timed with CUDA
events around a graph of 2L launches cycling through the decoder layers.
Usage: python scripts/xattn_compare.py [model] [rows...]"""
import json, statistics, sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2507_01021_b200.engine import WhisperGPU
from paper_2507_01021_b200.models import get_model

name = sys.argv[1] if len(sys.argv) > 1 else "whisper-large-v3"
rows_list = [int(x) for x in sys.argv[2:]] or [64, 48, 32, 24, 16, 8, 4, 1]
dims = get_model(name)
import os
eng = WhisperGPU(dims, max_slots=64, max_encode_batch=32,
                 length_aware=bool(int(os.environ.get("LA", "0"))))
seg = np.random.default_rng(0).integers(-8000, 8000, size=160000, dtype=np.int16)
slots = list(range(64))
for i in range(0, 64, 32):
    eng.encode([seg] * 32, slots[i:i + 32])
eng.admit(slots, [200] * 64)
L = dims.dec_layers
out = {}
for rows in rows_list:
    eng.set_active(slots[:rows])
    eng.step(2)
    torch.cuda.synchronize()
    r = {}
    for which, label in ((0, "xattn"), (9, "kv_stream_only"), (11, "no_merge"), (10, "xo_gemv")):
        us = statistics.median(1000 * eng.time_kernel(which, layer=-1, iters=2 * L) for _ in range(5))
        gbs = rows * 2 * 1500 * dims.d_model * 2 / (us * 1e-6) / 1e9
        r[label] = {"us": round(us, 2), "GBps": round(gbs, 1)}
    out[rows] = r
    print(rows, r, flush=True)
print(json.dumps({"model": name, "per_rows": out}))
