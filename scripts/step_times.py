"""Decode step time per active-row count (CUDA events on the engine stream
around 20 back-to-back step-graph replays; no trace marks).
Usage: python scripts/step_times.py [model] [rows...]"""
import json, statistics, sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2507_01021_b200.engine import WhisperGPU
from paper_2507_01021_b200.models import get_model

name = sys.argv[1] if len(sys.argv) > 1 else "whisper-large-v3"
rows_list = [int(x) for x in sys.argv[2:]] or [64, 48, 32, 16, 8, 4, 2, 1]
dims = get_model(name)
S = 64
eng = WhisperGPU(dims, max_slots=S, max_encode_batch=32)
seg = np.random.default_rng(0).integers(-8000, 8000, size=160000, dtype=np.int16)
slots = list(range(S))
for i in range(0, S, 32):
    eng.encode([seg] * 32, slots[i:i + 32])
eng.admit(slots, [400] * S)
out = {}
for rows in rows_list:
    eng.set_active(slots[:rows])
    eng.step(4)
    ts = []
    for _ in range(5):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(eng.stream)
        eng.step(20)
        b.record(eng.stream)
        b.synchronize()
        ts.append(a.elapsed_time(b) / 20)
    out[rows] = round(1000 * statistics.median(ts), 1)
    print(rows, out[rows], "us per step", flush=True)
print(json.dumps({"model": name, "step_us": out}))
