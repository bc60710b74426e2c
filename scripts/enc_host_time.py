import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2507_01021_b200.engine import WhisperGPU
from paper_2507_01021_b200.models import get_model
E = 12
eng = WhisperGPU(get_model("whisper-large-v3"), max_slots=E, max_encode_batch=E)
rng = np.random.default_rng(0)
segs = [rng.integers(-8000, 8000, size=480000, dtype=np.int16) for _ in range(E)]
for _ in range(3): eng.encode(segs, list(range(E)))
torch.cuda.synchronize()
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
for rep in range(3):
    flush.fill_(1.0); torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(eng.stream)
    t0 = time.perf_counter(); eng.encode(segs, list(range(E))); t1 = time.perf_counter()
    b.record(eng.stream); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"host issue {1e3*(t1-t0):.2f} ms, total {1e3*(t2-t0):.2f} ms, events {a.elapsed_time(b):.2f} ms")
for rep in range(3):
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(eng.stream); eng.encode(segs, list(range(E))); b.record(eng.stream); torch.cuda.synchronize()
    print(f"no flush: events {a.elapsed_time(b):.2f} ms")
import subprocess
print(subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_throttle_reasons.active", "--format=csv"], capture_output=True, text=True).stdout)
