"""Per-step time of back-to-back decode step graphs (CUDA events around
eng.step(n)) at several active-row counts: compare with the in-step span of
scripts/step_trace.py to see the cost of the graph-launch boundary."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2507_01021_b200.engine import WhisperGPU
from paper_2507_01021_b200.models import get_model

dims = get_model(sys.argv[1] if len(sys.argv) > 1 else "whisper-base")
eng = WhisperGPU(dims, max_slots=64, max_encode_batch=32)
seg = np.random.default_rng(0).integers(-8000, 8000, size=160000, dtype=np.int16)
slots = list(range(64))
for i in range(0, 64, 32):
    eng.encode([seg] * 32, slots[i:i + 32])
eng.admit(slots, [400] * 64)
for rows in (64, 8, 1):
    eng.set_active(slots[:rows])
    eng.step(4)
    torch.cuda.synchronize()
    res = {}
    for n in (1, 8, 32):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(eng.stream); eng.step(n); b.record(eng.stream); torch.cuda.synchronize()
        res[n] = round(1000 * a.elapsed_time(b) / n, 1)
    print(f"rows {rows}: us per step (n=1, 8, 32): {res}")
