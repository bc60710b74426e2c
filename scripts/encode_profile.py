"""One encode batch (for ncu captures of the encoder kernels)."""
import sys; sys.path.insert(0, '.')
import numpy as np, torch
from paper_2507_01021_b200.engine import WhisperGPU
from paper_2507_01021_b200.models import get_model
name = sys.argv[1] if len(sys.argv) > 1 else "whisper-base"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 32
eng = WhisperGPU(get_model(name), max_slots=n, max_encode_batch=n)
rng = np.random.default_rng(0)
segs = [rng.integers(-8000, 8000, size=480000, dtype=np.int16) for _ in range(n)]
for _ in range(2):
    eng.encode(segs, list(range(n)))
torch.cuda.synchronize()
print("ok")
