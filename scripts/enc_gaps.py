"""Gaps between consecutive encoder kernels of one dm_whisper_encode (CUPTI
via torch.profiler): python scripts/enc_gaps.py [model] [E]"""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
from torch.profiler import profile, ProfilerActivity
from paper_2507_01021_b200.engine import WhisperGPU
from paper_2507_01021_b200.models import get_model

name = sys.argv[1] if len(sys.argv) > 1 else "whisper-large-v3"
E = int(sys.argv[2]) if len(sys.argv) > 2 else 12
eng = WhisperGPU(get_model(name), max_slots=E, max_encode_batch=E)
rng = np.random.default_rng(0)
segs = [rng.integers(-8000, 8000, size=480000, dtype=np.int16) for _ in range(E)]
for _ in range(2):
    eng.encode(segs, list(range(E)))
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    eng.encode(segs, list(range(E)))
    torch.cuda.synchronize()
ev = sorted([e for e in prof.events() if e.device_type.name == "CUDA" and e.device_time_total > 0],
            key=lambda e: e.time_range.start)
span = (ev[-1].time_range.end - ev[0].time_range.start) / 1e3
busy = sum(e.device_time_total for e in ev) / 1e3
gaps = [(ev[i + 1].time_range.start - ev[i].time_range.end, ev[i].name[:40], ev[i + 1].name[:40])
        for i in range(len(ev) - 1)]
print(f"{len(ev)} kernels/copies, span {span:.2f} ms, busy {busy:.2f} ms, gaps {span - busy:.2f} ms")
for g, a, b in sorted(gaps, reverse=True)[:12]:
    print(f"  gap {g:8.1f} us after {a} -> {b}")
